// main() of the reference test binaries built against the drop-in.
#include <gtest/gtest.h>

GD_GTEST_MAIN
