// tsv.h — device fact ingestion / TSV output (tsv.cu), internal API.
#pragma once

#include <string>

#include "engine.h"
#include "ops.h"

namespace gd {

// read_facts (io.hpp:64-114) of numeric text: canonical rows into `rows`
// (device), returns the row count; load_error with the reference's message
// (`name` stands for the path) on the first bad line.
u64 parse_facts_device(Ctx& c, const char* h_text, u64 len, u32 arity, const std::string& name, DevBuf<u64>& rows);
// file_is_all_integers (io.hpp:145-170).
bool facts_all_integers_device(Ctx& c, const char* h_text, u64 len);
// to_tsv (io.hpp:118-133) of device rows into host memory; returns the byte
// length (h_out == nullptr: length only).
u64 rows_to_tsv_device(Ctx& c, const u64* d_rows, u64 n, u32 arity, char* h_out, u64 capacity);
// read_facts' message for a flagged line (host restatement of the checks).
std::string tsv_line_error(const char* text, u64 len, u64 line_idx, u32 arity, const std::string& name);

}  // namespace gd
