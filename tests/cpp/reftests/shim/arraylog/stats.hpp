// Reference header name -> the B200 drop-in (see ../dropin_all.hpp).
#pragma once
#include "../dropin_all.hpp"
