// dropin_all.hpp — compiles the reference's own gtest files UNMODIFIED
// against the B200 drop-in.
//
// The reference test files include "arraylog/<header>.hpp"; this directory
// comes first on the include path, and every header here includes this
// file.  It pulls in the reference headers (types, program, planner,
// parser, stats, accountant, EBM: host code the drop-in keeps) with the
// hot-path entry points renamed *_reference by macros, then re-exports the
// device implementations (include/arraylog_b200/arraylog_b200.hpp) under
// the reference names in namespace arraylog.  So `canonicalize`,
// `group_starts`, `range_lookup`, `join_count`, `join_materialize`,
// `select_project`, `merge_sorted`, `difference`, `permute_columns`,
// `read_facts`, `to_tsv`, `write_relation`, `file_is_all_integers` and
// `engine` in the test files are the sm_100a kernels of libgdlog_b200.so.
// `build_index` / `index_map` stay the reference's: the device index
// layout is free (SURVEY §8c "Unpinned"), and range_lookup on a
// reference-built container answers from the device index.
#pragma once

// Standard headers first, so the renaming macros below touch only the
// reference's own code.
#include <algorithm>
#include <array>
#include <atomic>
#include <bit>
#include <cctype>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <iterator>
#include <json.hpp>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <optional>
#include <random>
#include <set>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

#define canonicalize canonicalize_reference
#define group_starts group_starts_reference
#define range_lookup range_lookup_reference
#define join_count join_count_reference
#define join_materialize join_materialize_reference
#define select_project select_project_reference
#define merge_sorted merge_sorted_reference
#define difference difference_reference
#define permute_columns permute_columns_reference
#define read_facts read_facts_reference
#define to_tsv to_tsv_reference
#define write_relation write_relation_reference
#define file_is_all_integers file_is_all_integers_reference
#define engine engine_reference
#include ARRAYLOG_REF_UMBRELLA
#undef canonicalize
#undef group_starts
#undef range_lookup
#undef join_count
#undef join_materialize
#undef select_project
#undef merge_sorted
#undef difference
#undef permute_columns
#undef read_facts
#undef to_tsv
#undef write_relation
#undef file_is_all_integers
#undef engine

// the drop-in's dictionary (token-file) paths call the reference's host code
#define ARRAYLOG_B200_REF(name) ::arraylog::name##_reference
#include "arraylog_b200/arraylog_b200.hpp"

namespace arraylog {
using b200::canonicalize;
using b200::difference;
using b200::engine;
using b200::file_is_all_integers;
using b200::group_starts;
using b200::join_count;
using b200::join_materialize;
using b200::merge_sorted;
using b200::permute_columns;
using b200::range_lookup;
using b200::read_facts;
using b200::select_project;
using b200::to_tsv;
using b200::write_relation;
// to_tsv(run_stats) (stats.hpp:50-64) is host formatting: the reference's
inline std::string to_tsv(const run_stats& s) { return to_tsv_reference(s); }
}  // namespace arraylog
