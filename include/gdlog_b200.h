/*
 * gdlog_b200.h — C-ABI of the B200-native GDlog semi-naive fixpoint hot path.
 *
 * This is the drop-in boundary.  The reference (`arraylog`,
 * /root/reference/proj/include/arraylog) has no FFI of its own: its boundary
 * is a header-only C++ API.  Every entry point below replaces one reference
 * function or method; the replaced interface is cited as  file:line  relative
 * to proj/include/arraylog/.  The C++ wrapper that restores the reference
 * signatures on top of this ABI is include/arraylog_b200/arraylog_b200.hpp,
 * the Python mirror is paper_2311_02206_b200/arraylog.py.
 *
 * Conventions
 *  - No exceptions cross the boundary.  Every call returns a gd_status; the
 *    message of the last failure is gd_last_error(ctx), and for
 *    GD_ERR_BUDGET the phase name ("index", "join", "dedup", "difference",
 *    "merge", "other") is gd_last_error_phase(ctx).  The status codes map
 *    1:1 to the reference's exception types (types.hpp:19-72).
 *  - Tuples cross the boundary as flat row-major uint64_t arrays
 *    (tuple_array::data, tuple_array.hpp:19-51) plus a row count and an
 *    arity; `canonical` flags mirror tuple_array::canonical.
 *  - "host" pointers are ordinary CPU memory (pinned or pageable); the
 *    `_device` variants take device pointers on the context's device.
 *  - All device work is ordered on the context's stream.  A context (and the
 *    engines created from it) is not thread-safe: one host thread per ctx,
 *    like the reference's single-threaded orchestration (engine.hpp:34-39).
 *  - `workers` / `stride_rows` knobs are accepted and ignored: results never
 *    depend on them (acceptance criterion 7).
 */
#ifndef GDLOG_B200_H
#define GDLOG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GD_ABI_VERSION 1

/* Fixed maxima of the plan blob (plan.hpp:18-58).  The built-in programs
 * (builtins.hpp:13-41) need arity 2, 2 steps, 3 variants, 1 filter. */
#define GD_MAX_ARITY 8
#define GD_MAX_FILTERS 8
#define GD_MAX_STEPS 6
#define GD_MAX_VARIANTS 8

typedef enum gd_status {
    GD_OK = 0,
    GD_ERR_LOGIC = 1,       /* std::logic_error: precondition / internal fault */
    GD_ERR_CONFIG = 2,      /* config_error   (types.hpp:19)  */
    GD_ERR_USAGE = 3,       /* usage_error    (types.hpp:24)  */
    GD_ERR_LOAD = 4,        /* load_error     (types.hpp:29)  */
    GD_ERR_PLAN = 5,        /* plan_error     (types.hpp:34)  */
    GD_ERR_BUDGET = 6,      /* budget_error   (types.hpp:40-72), phase via gd_last_error_phase */
    GD_ERR_CUDA = 7,        /* CUDA runtime failure (no reference equivalent) */
    GD_ERR_UNSUPPORTED = 8, /* shape the device encoding cannot hold */
    GD_ERR_INVALID_ARG = 9, /* null pointer / bad handle at the C boundary */
    GD_ERR_NCCL = 10        /* NCCL failure in the native partitioned driver */
} gd_status;

/* ------------------------------------------------------------------ */
/* Context                                                              */

typedef struct gd_ctx gd_ctx;

/* Creates a context on CUDA device `device`.  `stream` is a cudaStream_t
 * (0 = create a private non-blocking stream).  Fails with GD_ERR_CUDA when
 * no device is present: there is no CPU fallback. */
gd_status gd_ctx_create(int device, void* stream, gd_ctx** out);
gd_status gd_ctx_destroy(gd_ctx* ctx);
const char* gd_last_error(const gd_ctx* ctx);
const char* gd_last_error_phase(const gd_ctx* ctx);
int gd_abi_version(void);
/* Number of kernels this context has launched (for the bench's gpu_launches). */
uint64_t gd_ctx_kernel_launches(const gd_ctx* ctx);
gd_status gd_ctx_synchronize(gd_ctx* ctx);
/* Returns the context's cached free device blocks to the driver (after a
 * large run, before another context or library allocates). */
gd_status gd_ctx_trim(gd_ctx* ctx);

/* Live per-kernel timing with CUDA events on the context stream (used by
 * bench.py for the roofline).  Classes: 0 sort pass, 1 sort histogram,
 * 2 diff+merge, 3 join probe, 4 join materialize, 5 index build,
 * 6 compaction/select, 7 other, 8 difference, 9 fused join+insert of the
 * resident loop, 10 loop control (gate/end).  read() synchronizes and
 * reports, per class, total milliseconds, launches and algorithmic bytes. */
#define GD_KCLASS_COUNT 11
gd_status gd_ctx_set_profiling(gd_ctx* ctx, int enable);
gd_status gd_ctx_profile_read(gd_ctx* ctx, double* ms, uint64_t* launches,
                              uint64_t* bytes);
gd_status gd_ctx_profile_reset(gd_ctx* ctx);
/* Host-side counters since context creation: seconds spent inside the
 * stream-ordered allocator and in stream synchronizations, and their
 * counts (diagnostics for launch/sync-bound long tails). */
gd_status gd_ctx_host_counters(gd_ctx* ctx, double* alloc_seconds,
                               uint64_t* allocs, double* sync_seconds,
                               uint64_t* syncs);
/* Bytes copied host->device and device->host by this context since its
 * creation (the e2e bench reports the bytes that actually cross PCIe:
 * relation downloads move packed keys when the encoding allows). */
gd_status gd_ctx_transfer_bytes(gd_ctx* ctx, uint64_t* h2d, uint64_t* d2h);

/* Device configuration of a context (SURVEY §5 "Config / flags": the
 * reference's engine_config, engine.hpp:25-32, stays ABI-identical in
 * gd_engine_config; every device-only knob lives here).  The library reads
 * no environment variables: a context starts from gd_device_config_default
 * and every later call on it (and on engines created from it) uses the
 * configuration last set.  None of these knobs changes a result, only how
 * the device computes it (tests compare every mode with the reference). */
typedef enum gd_loop_mode {
    GD_LOOP_GRAPH = 0, /* whole fixpoint = one CUDA graph with a device-side while node */
    GD_LOOP_EAGER = 1, /* direct launches, one host check per iteration */
    GD_LOOP_BATCH = 2  /* a graph of one iteration launched loop_batch times per host check */
} gd_loop_mode;

typedef enum gd_partition_exchange {
    GD_EXCHANGE_PEER = 0, /* rows stored straight into the owners' inboxes over peer memory (CUDA IPC
                             mappings), device-side barriers: the partitioned fixpoint is one CUDA graph */
    GD_EXCHANGE_NCCL = 1  /* NCCL send/recv all-to-all-v, one host round trip per iteration */
} gd_partition_exchange;

typedef struct gd_device_config {
    uint32_t size;                  /* sizeof(gd_device_config) (version check) */
    int32_t resident_loop;          /* 1: resident device loop when eligible; 0: host-driven loop */
    int32_t loop_mode;              /* gd_loop_mode */
    uint32_t loop_batch;            /* iterations per host check in GD_LOOP_BATCH (16) */
    int32_t min_capacities;         /* tests: every loop capacity starts at its minimum, so the
                                       overflow -> rollback -> grow paths run on small inputs (0) */
    int32_t split_insert;           /* final steps materialize to a temp, then insert (0) */
    int32_t dense_inner;            /* dense offset array for static one-column inners (1) */
    uint32_t index_growth;          /* head-index growth: load 1/index_growth after a growth (8) */
    uint32_t insert_waves;          /* fused-insert grid in waves of resident CTAs (0 = auto) */
    int32_t rehash_cas_only;        /* index growth by CAS re-spread instead of the zone pass (0) */
    uint32_t zone_slots;            /* shared-memory slots per zone-pass CTA (4096, <= 8192) */
    int32_t partition_loop;         /* partitioned mode on the loop kernels when eligible (1) */
    int32_t hash_dedup;             /* host-driven loop: hash pre-dedup of duplicate-heavy join output (1) */
    uint64_t hash_dedup_min_rows;   /* ... for join outputs of at least this many rows (1 << 20) */
    uint64_t dedup_part_slots;      /* L2-resident hash-set part, power of two (8 << 20) */
    int32_t dedup_split;            /* split large dedup sets into L2-sized parts (1) */
    int32_t host_unpack;            /* downloads move packed keys, host threads unpack (1) */
    double download_direct_frac;    /* pinned destinations: share of rows unpacked on the device and DMA'd
                                       into the caller's rows (0: with delta-compressed keys the host's
                                       row writes, not PCIe, bound the download) */
    uint64_t download_chunk_rows;   /* staging chunk of packed downloads (1 << 20) */
    uint32_t sort_items;            /* onesweep keys per thread: 4, 8 or 16 (16) */
    uint32_t trace;                 /* stderr traces: bit 0 resident loop, bit 1 downloads, bit 2 sort (0) */
    int32_t warp_expand;            /* final steps over a dense inner: count + warp-expanded insert (1:
                                       C2 155.7 ms vs 162.4 for probe + scan + merge-path fused insert,
                                       with expand_keys_per_lane = 4) */
    uint32_t sort_digit_bits;       /* pipelined sort: widest digit, 8..10 (10) */
    uint64_t heavy_rows;            /* ... rows with more outputs are expanded as segments of this many (4096) */
    int32_t sort_pipeline;          /* u64 sorts: 0 classic onesweep; 1 pipelined (bulk-copy prefetch, wide
                                       digits, ballot multi-split, keys staged in place, static tile order, cooperative launch); 2 the same with a
                                       separate staging buffer; 3 in place with MATCH.ANY ranking;
                                       4 classic onesweep with ballot ranking (0) */
    uint32_t partition_exchange;    /* gd_engine_run_partitioned: gd_partition_exchange (GD_EXCHANGE_PEER) */
    uint64_t sort_pipeline_min_keys; /* ... for sorts of at least this many keys (1 << 20) */
    uint64_t temp_limit_rows;       /* resident loop: a chain temp above this many rows is materialized
                                       in windows of at most this many (0: half the free HBM) */
    uint32_t peer_timeout_ms;       /* peer exchange: a device barrier waiting longer fails the run with
                                       GD_ERR_NCCL instead of hanging the GPU (60000) */
    uint32_t insert_slots;          /* head-index insert: 0 CAS first; 1 home slot loaded, then CAS, collisions
                                       probed one key after another; 2 the same with every key's probe
                                       steps batched (1) */
    uint32_t insert_pipeline;       /* inserts of materialized keys (split final steps, partition inboxes):
                                       two batches in flight per thread, batched probing (0) */
    uint32_t insert_per_thread;     /* materialized-key inserts (insert_pipeline = 0): keys per thread,
                                       8 (4 CTAs/SM), 4 (6 CTAs/SM) or 2 (8 CTAs/SM) (8) */
    uint32_t sort_ballot;           /* classic sort of >= 16 x sort_pipeline_min_keys keys: a pass whose input
                                       holds at least this many distinct digits per 32 consecutive keys
                                       (sampled before the pass) ranks with ballots, else MATCH.ANY;
                                       0 = MATCH.ANY always (12) */
    uint32_t l2_fetch_bytes;        /* cudaLimitMaxL2FetchGranularity set for the device when the context
                                       is configured: 32 / 64 / 128 bytes, 0 = leave the driver's (0) */
    uint32_t sort_min_ctas;         /* classic onesweep: 4 = registers capped for 4 CTAs per SM, else the
                                       compiler's choice (3 per SM) (0) */
    uint32_t expand_keys_per_lane;  /* warp-expanded insert: keys per lane per insert round, 8 (3 CTAs/SM,
                                       4 inner loads per lane in flight) or 4 (5 CTAs/SM, one) (4) */
    uint32_t warp_append;           /* merge-path fused insert: log append with one atomic per warp instead
                                       of one per CTA tile (two CTA barriers fewer per tile) (0) */
    uint32_t precount;              /* a single self-recursive warp-expanded step (TC): the insert computes
                                       the next iteration's row ranges, so loop_count only gates (0:
                                       C2 158.8 vs 155.5 ms — the count kernel keeps its launch and gate,
                                       the insert grows by more than the count saves) */
    uint32_t count_ctas_per_sm;     /* loop_count grid = SMs x this (0: 4) */
    uint32_t download_delta;        /* host downloads of canonical u64 keys: 2 = 32-key blocks of byte-aligned
                                       offsets from the block's first key, rows rebuilt by host threads with
                                       vector adds; 1 = gaps of 64-key blocks bit-packed, keys rebuilt by a
                                       running sum; 0 = packed 8-byte keys (2) */
    uint32_t index_load_pct;        /* resident-loop head index: grows when its load would pass this percentage
                                       (0: 50) */
    uint32_t download_pipeline;     /* resident-loop heads of at least download_pipeline_min_rows rows: the
                                       final sort runs top digit first, then per top-digit segment, and each
                                       sorted segment is packed for the host download, which rebuilds
                                       segment s while the device sorts the later ones (0: C2 166.4 vs
                                       155.2 ms of device time, e2e only 6 ms shorter — 75% of C2's rows
                                       share one top digit, so the first segment is most of the sort) */
    uint64_t download_pipeline_min_rows;  /* (1 << 24) */
    uint32_t gate_in_insert;        /* a single warp-expanded step (TC): the capacity gate is evaluated by every
                                       CTA of the insert kernel instead of loop_count's last CTA (1) */
    uint32_t pdl;                   /* the warp-expanded insert is a programmatic dependent launch of loop_count
                                       (its CTAs take SM slots as the count's retire, then wait for it) (0) */
    uint32_t count_ahead;           /* a single self-recursive warp-expanded step over light inner groups (TC):
                                       the insert sums the next iteration's candidates as it appends its rows,
                                       so the graph iteration is the insert kernel alone (0: C2 152.7-152.9
                                       vs 152.1-152.4 ms; a near-empty iteration 22.5 -> 20.6 us) */
    uint64_t chain_chunk_rows;      /* host-driven loop: a final join step with more output rows than this runs
                                       in row ranges of about this many outputs, the sink hash-deduplicated
                                       between them (0: an eighth of the free HBM) */
    uint32_t log_growth;            /* resident loop: a full head log grows to this many times the rows it must
                                       hold, when free HBM allows (4: C2 149.6 vs 152.9-153.2 ms at 2x,
                                       3 rollbacks instead of 8; 0 means 2) */
    uint32_t download_overlap_pack;  /* byte-offset downloads: pack per 4 M-row chunk with an event behind each,
                                       the host rebuilding chunk 0 while the device packs the rest (needs
                                       8 B per row of scratch) (0) */
} gd_device_config;

void gd_device_config_default(gd_device_config* cfg);
/* GD_ERR_CONFIG on out-of-range fields or a size mismatch. */
gd_status gd_ctx_set_device_config(gd_ctx* ctx, const gd_device_config* cfg);
gd_status gd_ctx_get_device_config(const gd_ctx* ctx, gd_device_config* cfg);

/* ------------------------------------------------------------------ */
/* Join-spec and plan data (ra.hpp:18-66, plan.hpp:18-58)              */

typedef enum gd_operand_kind {
    GD_OUTER_COL = 0, /* operand::outer(c)    ra.hpp:25 */
    GD_INNER_COL = 1, /* operand::inner(c)    ra.hpp:28 */
    GD_CONSTANT = 2   /* operand::constant(v) ra.hpp:31 */
} gd_operand_kind;

typedef struct gd_operand {
    uint32_t kind;   /* gd_operand_kind */
    uint32_t column;
    uint64_t value;
} gd_operand;

/* row_filter (ra.hpp:48-54): (lhs == rhs) must equal require_equal. */
typedef struct gd_filter {
    gd_operand lhs;
    gd_operand rhs;
    uint32_t require_equal;
    uint32_t reserved;
} gd_filter;

/* join_step (plan.hpp:31-39). */
typedef struct gd_join_step {
    uint32_t inner_rel;                 /* relation id */
    uint32_t join_column_count;         /* 0 = Cartesian */
    uint32_t inner_perm[GD_MAX_ARITY];  /* first arity(inner_rel) entries used */
    uint32_t proj_arity;
    uint32_t nfilters;
    gd_operand proj[GD_MAX_ARITY];
    gd_filter filters[GD_MAX_FILTERS];
} gd_join_step;

typedef enum gd_version { GD_FULL = 0, GD_DELTA = 1 } gd_version; /* plan.hpp:18 */

/* rule_variant (plan.hpp:43-50). nsteps == 0: select/project off the source. */
typedef struct gd_variant {
    uint32_t src_rel;
    uint32_t src_version;               /* gd_version */
    uint32_t src_perm[GD_MAX_ARITY];
    uint32_t nsteps;
    uint32_t sel_arity;
    uint32_t nsel_filters;
    uint32_t reserved;
    gd_join_step steps[GD_MAX_STEPS];
    gd_operand sel_proj[GD_MAX_ARITY];
    gd_filter sel_filters[GD_MAX_FILTERS];
} gd_variant;

/* rule_plan (plan.hpp:52-58). */
typedef struct gd_rule_plan {
    uint32_t rule_index;
    uint32_t head_rel;
    uint32_t head_arity;
    uint32_t recursive;
    uint32_t nvariants;
    uint32_t reserved;
    gd_variant variants[GD_MAX_VARIANTS];
} gd_rule_plan;

/* ------------------------------------------------------------------ */
/* Kernel-level entry points (unit parity; host buffers in and out)     */
/* Each call uploads its inputs, runs the sm_100a kernels, downloads.   */

/* slot_key() of the first `ncols` columns of each row (hash.hpp:28-60),
 * bit-exact with the reference Murmur3 mix. out[n]. */
gd_status gd_prefix_hash(gd_ctx* ctx, const uint64_t* rows, uint64_t n,
                         uint32_t arity, uint32_t ncols, uint64_t* out);

/* canonicalize (tuple_array.hpp:73-133): sort + dedup.  out has room for
 * n*arity values; *out_n receives the distinct row count. */
gd_status gd_canonicalize(gd_ctx* ctx, const uint64_t* rows, uint64_t n,
                          uint32_t arity, uint64_t* out, uint64_t* out_n);

/* The sort inside canonicalize (tuple_array.hpp:73-133) on DEVICE keys:
 * LSD radix sort of n packed u64 keys, each < 2^nbits (stable),
 * d_tmp of n keys as scratch; *in_tmp = 1 when the sorted keys ended in
 * d_tmp, 0 when in d_keys.  Stream-ordered on the context stream. */
gd_status gd_sort_keys_device(gd_ctx* ctx, uint64_t* d_keys, uint64_t* d_tmp, uint64_t n,
                              uint32_t nbits, int* in_tmp);

/* permute_columns (ra.hpp:426-454). rel must be canonical. */
gd_status gd_permute_columns(gd_ctx* ctx, const uint64_t* rows, uint64_t n,
                             uint32_t arity, int canonical,
                             const uint32_t* perm, uint32_t perm_len,
                             uint64_t* out, uint64_t* out_n);

/* group_starts (index_map.hpp:46-66). out_starts has room for n entries. */
gd_status gd_group_starts(gd_ctx* ctx, const uint64_t* rows, uint64_t n,
                          uint32_t arity, int canonical, uint32_t prefix_len,
                          uint64_t* out_starts, uint64_t* out_count);

/* build_index (index_map.hpp:74-124) + range_lookup (container.hpp:52-89):
 * builds the device HISA index over the canonical rows, then answers one
 * lookup per key (keys: nkeys x prefix_len row-major).  Also reports the
 * index's slot_count() and occupied() (index_map.hpp:30-39). */
gd_status gd_index_lookup(gd_ctx* ctx, const uint64_t* rows, uint64_t n,
                          uint32_t arity, int canonical, uint32_t prefix_len,
                          double load_factor, const uint64_t* keys,
                          uint64_t nkeys, uint32_t key_len, uint64_t* out_start,
                          uint64_t* out_count, uint64_t* out_slot_count,
                          uint64_t* out_occupied);

/* One side of a join_spec (ra.hpp:60-66): a relation_container with an
 * optional index of prefix `index_prefix_len` (0 = no index). */
typedef struct gd_container_view {
    const uint64_t* rows;
    uint64_t n;
    uint32_t arity;
    uint32_t canonical;
    uint32_t index_prefix_len;
    uint32_t reserved;
    double load_factor;
} gd_container_view;

typedef struct gd_join_spec {
    uint32_t join_column_count;
    uint32_t proj_arity;
    uint32_t nfilters;
    uint32_t reserved;
    gd_operand proj[GD_MAX_ARITY];
    gd_filter filters[GD_MAX_FILTERS];
} gd_join_spec;

/* join_count (ra.hpp:141-182). */
gd_status gd_join_count(gd_ctx* ctx, const gd_container_view* outer,
                        const gd_container_view* inner,
                        const gd_join_spec* spec, uint64_t* out_total);

/* join_materialize (ra.hpp:189-263): out must hold exactly
 * out_capacity_rows * proj_arity values; a mismatch with the join size is
 * GD_ERR_LOGIC ("output capacity mismatch").  Row order equals the
 * reference: outer-row order, then inner-range order. */
gd_status gd_join_materialize(gd_ctx* ctx, const gd_container_view* outer,
                              const gd_container_view* inner,
                              const gd_join_spec* spec, uint64_t* out,
                              uint64_t out_capacity_rows);

/* select_project (ra.hpp:267-293). out room: n * proj_arity. */
gd_status gd_select_project(gd_ctx* ctx, const uint64_t* rows, uint64_t n,
                            uint32_t arity, const gd_operand* proj,
                            uint32_t proj_arity, const gd_filter* filters,
                            uint32_t nfilters, uint64_t* out, uint64_t* out_n);

/* merge_sorted (ra.hpp:299-381): disjoint canonical union.  buffer_rows is
 * the caller's merge-buffer capacity (too small -> GD_ERR_LOGIC); out holds
 * (nf + nd) * arity values.  Overlapping inputs -> GD_ERR_LOGIC. */
gd_status gd_merge_sorted(gd_ctx* ctx, const uint64_t* full, uint64_t nf,
                          int full_canonical, const uint64_t* delta,
                          uint64_t nd, int delta_canonical, uint32_t arity,
                          uint64_t buffer_rows, uint64_t* out);

/* difference (ra.hpp:386-422): rows of new_rel absent from full. */
gd_status gd_difference(gd_ctx* ctx, const uint64_t* new_rows, uint64_t nn,
                        int new_canonical, const uint64_t* full, uint64_t nf,
                        int full_canonical, uint32_t arity, uint64_t* out,
                        uint64_t* out_n);

/* ------------------------------------------------------------------ */
/* Engine (engine.hpp:25-277): the performance entry.                   */

/* engine_config (engine.hpp:25-32). memory_budget_bytes = UINT64_MAX is
 * "unlimited" (budget.hpp:19). */
typedef struct gd_engine_config {
    uint64_t memory_budget_bytes;
    uint32_t ebm_enabled;
    uint32_t alpha;
    double load_factor;
    uint32_t workers;     /* accepted, ignored */
    uint32_t reserved;
    uint64_t stride_rows; /* accepted, ignored */
} gd_engine_config;

/* run_stats (stats.hpp:21-46) plus device-only counters. phase_seconds is
 * indexed in kPhaseOrder: index, join, dedup, difference, merge, other. */
typedef struct gd_run_stats {
    double phase_seconds[6];
    double total_seconds;
    uint64_t iterations;
    uint64_t buffer_allocations;
    uint64_t charge_events;
    uint64_t peak_tracked_bytes;
    uint64_t peak_temp_bytes;
    /* device extras */
    uint64_t join_tuples;        /* sum over all join steps of output rows */
    uint64_t device_bytes_peak;  /* peak bytes held in the device arena */
    double kernel_seconds[6];    /* CUDA-event time per phase */
    uint64_t algo_bytes[6];      /* algorithmic HBM bytes per phase */
} gd_run_stats;

/* Per-iteration counters of one recursive relation:
 * delta_in = |Δ| consumed, join = J rows appended, new_unique = N,
 * delta_out = D, full_after = |F| after the merge. */
typedef struct gd_iter_record {
    uint64_t delta_in;
    uint64_t join;
    uint64_t new_unique;
    uint64_t delta_out;
    uint64_t full_after;
} gd_iter_record;

/* ---- fact ingestion and canonical TSV output ------
 * The text is parsed / produced on the device.  Numeric files only: the
 * reference's dictionary mode (io.hpp:19-41) interns tokens on the host
 * (arraylog.py) before the rows reach the device. */

/* read_facts(path, arity) (io.hpp:64-114): `text` holds the file bytes,
 * `name` (nullable) stands for the path in messages.  Writes the canonical
 * rows (sorted, duplicates collapsed) to out[count * arity]; GD_ERR_LOAD
 * with the reference's message on the first bad line ("<name>:<line>:
 * expected N columns, got M" / "'tok' is not an unsigned integer" / "value
 * is reserved"); GD_ERR_INVALID_ARG (count set) when capacity_rows is too
 * small. */
gd_status gd_parse_facts(gd_ctx* ctx, const char* name, const char* text, uint64_t len, uint32_t arity,
                         uint64_t* out, uint64_t capacity_rows, uint64_t* count);
/* file_is_all_integers (io.hpp:145-170): *result = 1 when every data token
 * is an unsigned decimal below the sentinel. */
gd_status gd_facts_all_integers(gd_ctx* ctx, const char* text, uint64_t len, int* result);
/* to_tsv(rel) (io.hpp:118-133) of n canonical rows: the bytes into
 * out[capacity] (out == NULL: *len only). */
gd_status gd_rows_to_tsv(gd_ctx* ctx, const uint64_t* rows, uint64_t n, uint32_t arity, char* out,
                         uint64_t capacity, uint64_t* len);

typedef struct gd_engine gd_engine;

/* engine(program, engine_config) (engine.hpp:66-88).  Relations are ids
 * 0..nrels-1 with their arities, an EDB flag (edb_decl, program.hpp:73) and
 * their names (nullable: "r<id>").  Names only order the per-iteration
 * copy refresh like the reference's name-keyed relation map
 * (engine.hpp:209-210) and label errors. */
gd_status gd_engine_create(gd_ctx* ctx, const gd_engine_config* cfg,
                           uint32_t nrels, const uint32_t* arities,
                           const uint32_t* is_edb, const char* const* names,
                           gd_engine** out);
gd_status gd_engine_destroy(gd_engine* eng);

/* set_plans / override_plans (engine.hpp:97-101, 300-310). */
gd_status gd_engine_set_plans(gd_engine* eng, const gd_rule_plan* plans,
                              uint32_t nplans);

/* load_edb (engine.hpp:107-128): rejects the kEmptySlot sentinel
 * (GD_ERR_LOAD), canonicalizes when canonical == 0. */
gd_status gd_engine_load_edb(gd_engine* eng, uint32_t rel,
                             const uint64_t* rows, uint64_t n, int canonical);
gd_status gd_engine_load_edb_device(gd_engine* eng, uint32_t rel,
                                    const uint64_t* d_rows, uint64_t n,
                                    int canonical);

/* seed / iterate_to_fixpoint / run (engine.hpp:130-257). */
/* load_edb(name, read_facts(path, arity)) with the text parsed on the
 * device straight into the relation (no host rows). */
gd_status gd_engine_load_edb_tsv(gd_engine* eng, uint32_t rel, const char* name, const char* text,
                                 uint64_t len);
/* write_relation / to_tsv of relation(rel) (io.hpp:118-143): the canonical
 * TSV bytes into out[capacity] (out == NULL: *len only). */
gd_status gd_engine_relation_tsv(gd_engine* eng, uint32_t rel, char* out, uint64_t capacity, uint64_t* len);
gd_status gd_engine_seed(gd_engine* eng);
gd_status gd_engine_iterate(gd_engine* eng);
gd_status gd_engine_run(gd_engine* eng);

/* relation(name) (engine.hpp:259-264): row count, then download into a
 * host (or device) buffer of count*arity values. */
gd_status gd_engine_relation_count(gd_engine* eng, uint32_t rel, uint64_t* n);
gd_status gd_engine_relation_download(gd_engine* eng, uint32_t rel,
                                      uint64_t* out, uint64_t capacity_rows);
gd_status gd_engine_relation_download_device(gd_engine* eng, uint32_t rel,
                                             uint64_t* d_out,
                                             uint64_t capacity_rows);
/* Order-independent 64-bit digest of a relation, computed on the device
 * (sum of fmix64(row hash)); used by the bench to check full-size runs
 * without a download. */
gd_status gd_engine_relation_digest(gd_engine* eng, uint32_t rel,
                                    uint64_t* digest);

/* stats() (engine.hpp:270-277). */
gd_status gd_engine_stats(gd_engine* eng, gd_run_stats* out);
/* accountant() (engine.hpp:103-105): the state of the engine's logical-byte
 * ledger (memory_accountant, budget.hpp:16-67) — current bytes per category
 * {container, temp, buffer}, peak, peak temp, charge events and the budget
 * (UINT64_MAX = unlimited).  Any pointer may be NULL. */
gd_status gd_engine_accountant(gd_engine* eng, uint64_t current[3], uint64_t* peak, uint64_t* peak_temp,
                               uint64_t* events, uint64_t* budget);
/* run_stats::delta_history entry of one recursive relation. */
gd_status gd_engine_delta_history(gd_engine* eng, uint32_t rel, uint64_t* out,
                                  uint64_t capacity, uint64_t* len);
gd_status gd_engine_iter_log(gd_engine* eng, uint32_t rel, gd_iter_record* out,
                             uint64_t capacity, uint64_t* len);
/* Encoding chosen at seed time: bits per column, key words, dictionary. */
gd_status gd_engine_encoding(gd_engine* eng, uint32_t* bits,
                             uint32_t* key_words, uint32_t* dictionary);

/* ------------------------------------------------------------------ */
/* Hash-partitioned multi-GPU mode.                     */
/* Every IDB tuple lives on rank owner(t) = fmix64(digest(t)) % nranks;  */
/* EDB relations are replicated.  One iteration is split in two halves   */
/* around the caller's all-to-all (NCCL via torch.distributed):           */
/*   begin: joins on the local Δ, route rows to owners, local dedup;      */
/*          send buffer = encoded keys grouped by destination rank.       */
/*   end:   merge received keys into the local full; new local Δ.         */

gd_status gd_engine_set_partition(gd_engine* eng, uint32_t rank,
                                  uint32_t nranks);
/* Number of 64-bit words per exchanged tuple (1 or 2). */
gd_status gd_engine_exchange_words(gd_engine* eng, uint32_t* words);
/* Runs the local half of one iteration.  send_counts[nranks] receives the
 * row count for each destination; *d_send points to the device send
 * buffer (valid until the next call). */
gd_status gd_engine_partition_begin(gd_engine* eng, uint64_t* send_counts,
                                    const void** d_send);
gd_status gd_engine_partition_end(gd_engine* eng, const void* d_recv,
                                  uint64_t recv_rows, uint64_t* local_delta);
/* Global termination is decided by the caller (all-reduce of local Δ). */
gd_status gd_engine_partition_finish(gd_engine* eng);

/* Native driver: the whole partitioned fixpoint of one rank with the
 * exchanges issued by the library itself on the context's stream (NCCL
 * send/recv over NVLink).  Per iteration: joins + owner counts on the
 * device, one all-to-all of (count, local |Δ|, overflow flag) per peer,
 * one readback, owner scatter, one all-to-all-v of the rows, insert and
 * end-of-iteration bookkeeping on the device — a single host
 * synchronisation.  Every rank calls it collectively after
 * gd_engine_set_partition + seeding; *iterations = global iterations. */
typedef struct gd_comm gd_comm;
gd_status gd_nccl_unique_id(uint8_t id[128]);
/* nranks / rank as in gd_engine_set_partition; the id is rank 0's
 * gd_nccl_unique_id, shared by the caller (e.g. a torch.distributed
 * broadcast). */
gd_status gd_nccl_comm_create(gd_ctx* ctx, const uint8_t id[128], uint32_t nranks, uint32_t rank,
                              gd_comm** out);
/* Destroys a communicator of either kind. */
gd_status gd_nccl_comm_destroy(gd_comm* comm);
/* Test transport for the same driver: nranks ranks as host threads of one
 * process, each with its own context and engine on one GPU; messages are
 * device-to-device copies between barriers.  Validates the driver's
 * multi-rank logic where only one GPU is available. */
typedef struct gd_loopback_hub gd_loopback_hub;
gd_status gd_loopback_hub_create(uint32_t nranks, gd_loopback_hub** out);
gd_status gd_loopback_hub_destroy(gd_loopback_hub* hub);
gd_status gd_loopback_comm_create(gd_loopback_hub* hub, uint32_t rank, gd_comm** out);
gd_status gd_engine_run_partitioned(gd_engine* eng, gd_comm* comm, uint64_t max_iters,
                                    uint64_t* iterations);

#ifdef __cplusplus
}
#endif

#endif /* GDLOG_B200_H */
