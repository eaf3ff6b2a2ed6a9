// loop.h — the resident device loop of the semi-naive fixpoint (engine.hpp:
// 181-257) for relations that are never a join inner (TC's Reach, SG's SG,
// …): the whole iteration runs on the device with every size read from
// device memory, so one iteration is a fixed kernel sequence that is
// captured once into a CUDA graph and repeated under a device-side `while`
// condition (termination = every Δ empty, detected on the device).
//
// Relation store of a loop head h:
//   log_h   append-only array of packed keys; log[0, dhi) is the full
//           relation, log[dlo, dhi) the current Δ (delta ⊆ full,
//           SPEC.md:306), new rows are appended at log_n;
//   tab_h   HISA index over the whole tuple (prefix_len = arity): open
//           addressing; membership of a join output in full is one slot
//           CAS, and a per-slot stamp (last iteration that produced the key)
//           gives the distinct count of the iteration's join output
//           (canonicalize's unique) in the same pass.
// Dedup + difference + append are fused into the join's materialize:
// the join output J is never written to HBM.  The canonical (sorted) full
// relation is produced once, by the onesweep radix sort, when the loop ends.
#pragma once

#include "ops.h"

namespace gd {

constexpr u32 kLoopMaxHeads = 8;
constexpr u32 kLoopMaxSteps = 32;  // variant-steps per iteration
constexpr u64 kLoopMatTile = 1024; // merge-path items (rows + outputs) per materialize tile

// Wide slot (keys of more than 56 bits): the key and the stamp of the last
// iteration that produced it.
struct HSlot {
    u64 key;    // kEmptySlot when free
    u32 stamp;  // iteration - epoch_base that last produced the key
    u32 pad;
};
// Packed slot (keys of at most 64 - sbits bits, sbits >= 8): one u64 word
// key << sbits | stamp, so insertion and the stamp update are one CAS.

// Where a step's outer rows come from (resolved on the device).
enum LoopOuterKind : u32 {
    LO_STATIC = 0,  // (ptr, n) fixed at capture
    LO_DELTA = 1,   // log of head `head`, [dlo, dhi)
    LO_FULL = 2,    // log of head `head`, [0, dhi)
    LO_TEMP = 3,    // ptr = temp buffer, n = ctl.step_total[src_step]
};

struct LoopOuter {
    u32 kind;
    u32 head;
    u32 src_step;
    u32 pad;
    const u64* ptr;
    u64 n;
};

struct LoopHeadState {
    u64 log_n;  // rows in the log (= |full| after the iteration)
    u64 dlo, dhi;
    u64 cand;   // candidate upper bound of this iteration's insertions
    u64 J, N, D;  // join rows (post-filter), distinct join rows, new rows
};

// Device control block of one engine's loop.
struct LoopCtl {
    u32 iter;      // completed iterations
    u32 done;      // every Δ empty
    u32 overflow;  // a capacity was exceeded: iteration rolled back, host grows
    u32 nheads;
    u64 hist_cap;
    u32 epoch_base;    // stamps are iter + 1 - epoch_base
    u32 need_restamp;  // stamp range exhausted: host rebuilds the tables
    u32 ctas_done;     // last-CTA detection of the fused gate / end epilogues
    u32 pad;
    LoopHeadState h[kLoopMaxHeads];
    u64 step_cand[kLoopMaxSteps];   // candidates (pre-filter) of each step
    u64 step_total[kLoopMaxSteps];  // rows produced (post-filter) of each step
    u64 step_n[kLoopMaxSteps];      // outer rows of each step
    // capacities the host must provide after an overflow
    u64 need_rows[kLoopMaxSteps];
    u64 need_splits[kLoopMaxSteps];
    u64 need_temp[kLoopMaxSteps];
    u64 need_log[kLoopMaxHeads];
    u64 need_tab[kLoopMaxHeads];
    u64 need_hist;
    u64 heavy_n[kLoopMaxSteps];    // (row, segment) items queued by loop_count
    u64 last_cand[kLoopMaxSteps];  // step_cand of the last completed iteration (profiler)
    // peer-memory partitioned loop (loop_peer_*)
    u64 part_epoch;    // barriers passed (identical on every rank)
    u64 part_recv;     // rows this rank received this iteration
    u64 part_join;     // join rows produced by this rank, all iterations
    u64 part_last_D;   // this rank's |Δ| of its last completed iteration
    u32 part_inbox_over;  // a routed row did not fit a peer's inbox (this rank saw it)
    u32 part_over;        // some rank overflowed: the iteration was rolled back on every rank
    u32 part_stall;       // this rank's insert did not fit its log / index: the host finishes it
    u32 part_stall_any;   // some rank stalled (the graph stopped on every rank)
    u32 part_timeout;     // a device barrier waited past its limit (the host raises GD_ERR_NCCL)
    u32 dbg_rank;         // ... the first rank missing, its flag and the epoch waited for
    u64 dbg_flag, dbg_epoch;
    // output window of a chain temp (host-driven windowed iteration, when a
    // step's temp exceeds gd_device_config.temp_limit_rows): step win_step
    // materializes only its outputs [win_lo, win_hi); win_hi = 0: no window
    u32 win_step;
    u32 pad2;
    u64 win_lo, win_hi;
    // precount (a single self-recursive warp-expanded step): the insert
    // computes the next iteration's row ranges, heavy items and candidate
    // count for the rows it appends; loop_count then only gates
    u32 pre_valid;    // this iteration's ranges / heavy items / step_cand came from the last insert
    u32 pre_sel;      // buffer set of this iteration (0: rc / row_start / row_off, 1: the *2 set)
    u32 pre_bad;      // the precount overflowed a buffer: the next iteration counts itself
    u32 pad4;
    u64 pre_cand, pre_heavy_n;
};

// ---- peer-memory partitioned loop --------------
// Every rank owns a mailbox and an inbox in its HBM, mapped into every other
// rank (CUDA IPC over NVLink / NVSwitch; plain pointers for the loopback
// ranks of one GPU).  A routing kernel appends each join row straight into
// its owner's inbox (one system-scope cursor atomic per warp round and
// destination, then coalesced peer stores); two device-side barriers per
// iteration carry the overflow flags and the |Δ| sum, so the whole
// partitioned fixpoint runs inside one CUDA graph with no host round trip.
constexpr u32 kPeerVals = 4;
struct PeerMail {
    unsigned long long flag[64];        // flag[s] = last barrier epoch rank s reached
    unsigned long long val[64][kPeerVals];  // rank s's payload of that barrier
    unsigned long long cursor;          // rows appended to this rank's inbox this iteration
    unsigned long long pad[7];
};
struct PeerTab {
    u64* inbox[64];      // rank q's inbox, mapped here
    u64 cap[64];         // its capacity (rows)
    PeerMail* mail[64];  // rank q's mailbox, mapped here
    u32 P, rank;
};

// Per-iteration history written by loop_end: rec[i * nheads + h] and the
// post-filter totals of every step, steps[i * nsteps + s].
struct LoopHist {
    gd_iter_record* rec;
    u64* steps;
    u32 nsteps;
};

// Storage of one head (captured into the graph).
struct LoopHeadBufs {
    u64* log;
    u64 log_cap;
    void* tab;      // u64[tab_cap] (packed, sbits > 0) or HSlot[tab_cap]
    u64 tab_cap;
    u64 tab_limit;  // max keys before the table must grow
    u32 sbits;      // stamp bits of packed slots; 0 = wide HSlot
    u32 warp_append;  // fused inserts append with one atomic per warp instead of per CTA tile
};
inline u64 loop_slot_bytes(u32 sbits) { return sbits ? 8 : sizeof(HSlot); }
// Stamp bits for keys of `key_bits` bits (0: wide slots).
inline u32 loop_stamp_bits(u32 key_bits) {
    const u32 spare = key_bits >= 64 ? 0 : 64 - key_bits;
    return spare >= 8 ? (spare > 24 ? 24 : spare) : 0;
}

// Dense form of a static inner's HISA index (join prefix of one column whose
// values span at most a few times the row count): off[p - lo] = first row
// with prefix p, off[span] = n.  A probe is one 8-byte L2-resident read
// instead of a random slot of the hash table; ranges equal range_lookup's.
struct LoopDense {
    const u32* off;  // nullptr: use the hash index
    u64 lo;
    u64 span;
};
// Builds the dense form when worthwhile (span <= 4n + 4096, n < 2^32);
// returns false otherwise.
bool loop_dense_build(Ctx& c, const u64* rows, u64 n, u32 arity, u32 bits, DevBuf<u32>& off, u64& lo,
                      u64& span);

// Per-step buffers: row_start / row_off hold rows_cap entries, splits the
// merge-path split of every materialize tile (splits_cap entries).
struct LoopStepBufs {
    u64* row_start;
    u64* row_off;
    u64 rows_cap;
    u64* splits;
    u64 splits_cap;
    u64* rc;  // warp-expanded steps: row r's inner range, start << 32 | count (loop_count writes it)
    // precounted steps (the next iteration's ranges written by this
    // iteration's insert): the second buffer set; LoopCtl.pre_sel picks
    // which set is the current iteration's
    u64* rc2;
    u64* row_start2;
    u64* row_off2;
};

// Candidate bound of the final steps -> overflow check of every head.
struct LoopGateDesc {
    u32 nfinal;
    u32 final_step[kLoopMaxSteps];
    u32 final_head[kLoopMaxSteps];
    u64 log_cap[kLoopMaxHeads];
    u64 tab_limit[kLoopMaxHeads];
    u32 stamp_max;  // largest stamp every head's slots can hold
};

struct LoopEndDesc {
    LoopHist hist;
    unsigned long long cond;  // cudaGraphConditionalHandle
    int use_cond;
    u32 pre_step;  // precounted step (its next-iteration counts become current), or ~0u
};

// ---- launchers (loop.cu); all stream-ordered on `s`, no host sync ----
int loop_grid(const Ctx& c);
// Kernel occupancies (called once before the first launch or capture).
void loop_prepare();
void loop_table_clear(Ctx& c, void* tab, u64 cap, u32 sbits);
// Streaming u64 fill / copy kernels (growth path).
void loop_fill_u64(Ctx& c, u64* p, u64 n, u64 v);
void loop_copy_u64(Ctx& c, u64* d, const u64* s, u64 n);
// Inserts keys (unique) into an empty table (stamp 0).
void loop_table_fill(Ctx& c, void* tab, u64 cap, u32 sbits, const u64* keys, u64 n);
// Moves every key (nkeys of them) of old_tab into the larger tab, stamps 0.
// tab is uninitialised on entry: every slot is written.
void loop_table_rehash(Ctx& c, const void* old_tab, u64 old_cap, void* tab, u64 cap, u32 sbits, u64 nkeys);
// Resets every stamp to 0 in place (new stamp epoch).
void loop_table_restamp(Ctx& c, void* tab, u64 cap, u32 sbits);

// One HISA probe per outer row: row_start, counts (into row_off), per-CTA sums.
void loop_probe(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const DevJoin& jd,
                const IndexView<u64>* ix, const LoopDense& dense, u64 inner_n, const LoopStepBufs& sb,
                u64* block_sums);
// Exclusive scan of the counts + the materialize splits; when `gate` is
// non-null the last CTA also runs the gate (it must be the iteration's last
// candidate-producing launch).
void loop_scan(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const LoopStepBufs& sb,
               const u64* block_sums, const LoopGateDesc* gate);
void loop_gate(Ctx& c, cudaStream_t s, LoopCtl* ctl, const LoopGateDesc& g);
void loop_materialize_temp(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o,
                           const u64* inner, const DevJoin& jd, const LoopStepBufs& sb, u64* temp, u64 temp_cap);
// Candidate bound of a select (nsteps == 0) final step = its outer rows.
void loop_select_cand(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o);
// Final steps; when `end` is non-null the last CTA records the iteration.
// Final step fused: expansion + insertion + append (the product path).
void loop_materialize_insert(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, u32 head, const LoopOuter& o,
                             const u64* inner, const DevJoin& jd, const LoopStepBufs& sb,
                             const LoopHeadBufs& hb, const LoopEndDesc* end);
// Inserts the step's materialized join rows (ctl.step_total of them) into
// the head's full-tuple index and appends the new ones to its log.
void loop_insert_keys(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, u32 head, const u64* keys,
                      const LoopHeadBufs& hb, const LoopEndDesc* end);
void loop_select_insert(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, u32 head, const LoopOuter& o,
                        const DevJoin& jd, const LoopHeadBufs& hb, const LoopEndDesc* end);
// ---- partitioned mode ----
constexpr u32 kLoopMaxRanks = 64;
// Per-destination counts of keys[0, *n_ptr) (owner = key_hash64(key) mod P).
void loop_owner_count(Ctx& c, const u64* keys, const u64* n_ptr, u64 cap, u32 P, unsigned long long* counts);
// Native partitioned driver: meta[3p..3p+2] = (rows for rank p, this
// rank's |Δ| (at least `min_delta`), overflow flag) for the counts exchange.
void loop_part_meta(Ctx& c, const unsigned long long* counts, const LoopCtl* ctl, u32 P, u64 min_delta, u64* meta);
// End of a partitioned iteration on the device: records
// {|Δ in|, recv_rows, N, D, log_n} at hist[iter], advances the Δ window
// and the iteration, clears the final step's row count.
void loop_part_advance(Ctx& c, LoopCtl* ctl, u32 final_step, u64 recv_rows, gd_iter_record* hist);
// Scatter into out grouped by destination (offsets: exclusive prefix of the
// counts; cursors zeroed).  Order inside a group is unspecified.
void loop_owner_scatter(Ctx& c, const u64* keys, const u64* n_ptr, u32 P, const unsigned long long* offsets,
                        unsigned long long* cursors, u64* out);

// ---- peer-memory partitioned loop ----
// Routes the step's materialized rows (ctl.step_total of them) to their
// owners' inboxes (owner = key_hash64(key) mod P).
void loop_route_keys(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const u64* keys, const PeerTab* tab);
// Warp-expanded final step over a dense inner, routed instead of inserted.
void loop_expand_route(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const u64* inner,
                       const DevJoin& jd, const LoopDense& dense, const LoopStepBufs& sb, u64 heavy_rows,
                       const PeerTab* tab);
struct PeerSyncDesc {
    const PeerTab* tab;
    u64 timeout_ns;  // a barrier that waits longer stops the graph (part_timeout)
    u32 final_step, nsteps;
    u64 log_cap, tab_limit;
    u32 stamp_max;
    gd_iter_record* hist;
    u64 hist_cap;
    unsigned long long cond;  // cudaGraphConditionalHandle
    int use_cond;
};
// Barrier 1 (after routing): overflow consensus (rollback on every rank),
// the received row count, the capacity gate of this rank's insert.
void loop_peer_sync1(Ctx& c, cudaStream_t s, LoopCtl* ctl, const PeerSyncDesc& d);
// Barrier 2 (after the insert): the iteration record, the Δ window, the
// |Δ| sum (termination) and stall consensus; sets the while condition.
void loop_peer_sync2(Ctx& c, cudaStream_t s, LoopCtl* ctl, const PeerSyncDesc& d);

// ---- warp-expanded final step over a dense inner ----
// loop_count: one read of the dense offsets per outer row, the candidate
// sum, rows with more than heavy_rows outputs queued as (row, segment)
// items in sb.row_start / sb.row_off; the gate in its last CTA when `gate`.
void loop_count(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const DevJoin& jd,
                const LoopDense& dense, const LoopStepBufs& sb, u64 heavy_rows, const LoopGateDesc* gate);
// Expansion fused with dedup + difference + append: every warp expands 32
// outer rows at a time into a shared buffer and inserts 256 keys at a
// time, then the heavy items; loop_end in the last CTA when `end`.
// gate: the iteration's capacity gate, evaluated by every CTA at its start
// (the step must be the iteration's only candidate producer, nothing
// inserted before it in the iteration).
void loop_expand_insert(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, u32 head, const LoopOuter& o,
                        const u64* inner, const DevJoin& jd, const LoopDense& dense, const LoopStepBufs& sb,
                        u64 heavy_rows, const LoopHeadBufs& hb, const LoopEndDesc* end,
                        const LoopGateDesc* gate = nullptr, bool count_ahead = false);
// Largest inner group of a dense index (max off[i + 1] - off[i]; one host sync).
u64 loop_dense_max_group(Ctx& c, const LoopDense& dv);

// The same expansion appended to the step's temp (split final step, then
// loop_insert_keys over the temp).
void loop_expand_temp(Ctx& c, cudaStream_t s, LoopCtl* ctl, u32 step, const LoopOuter& o, const u64* inner,
                      const DevJoin& jd, const LoopDense& dense, const LoopStepBufs& sb, u64 heavy_rows, u64* temp,
                      u64 temp_cap);

// Records the iteration (or rolls it back on overflow) and sets the graph's
// while-condition (cond ignored unless use_cond).
void loop_end(Ctx& c, cudaStream_t s, LoopCtl* ctl, const LoopEndDesc& end);

}  // namespace gd
