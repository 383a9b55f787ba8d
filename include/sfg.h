/*
 * sfg.h — C ABI of the B200 fuzzing inner loop (libsfg_b200.so).
 *
 * The reference (simt_forge, pure Python) has no FFI; its drop-in seams are
 * Python calls.  Each entry point below replaces one of them for a whole
 * batch ("round") of fuzz inputs, stream-ordered on the caller's CUDA stream:
 *
 *   sfg_plan + sfg_mutate + sfg_apply
 *       <- schedule_next        pkg/src/simt_forge/campaign.py:593-603
 *          mutate_testcase      pkg/src/simt_forge/mutation.py:499-518
 *          PhaseRunner._materialize (payload bytes) campaign.py:440-450
 *   sfg_execute
 *       <- PhaseRunner.run_phase(COMPUTE)  campaign.py:483-561
 *          executor.launch / _exec_one     executor.py:390-424, 210-377
 *          sanitizer.check_access          sanitizer.py:145-187
 *          CoverageMap.record_launch/edge  coverage.py:59-71
 *   sfg_triage_stop/absorb/admit + sfg_commit
 *       <- _absorb_iteration    campaign.py:825-846
 *          new_edges_since / merge_from    coverage.py:85-113
 *          FindingsLog.add      sanitizer.py:216-225
 *   sfg_compact + sfg_regen
 *       <- Corpus.admit         campaign.py:581-582
 *   sfg_scan_u32 / sfg_scan_u64   order-dependent bookkeeping (rotation counts,
 *          alloc ids, admission order) as exclusive prefix sums
 *
 * Conventions: every pointer argument except the host tables passed to
 * sfg_program_create is a DEVICE pointer owned by the caller; `stream` is a
 * cudaStream_t.  No call allocates or synchronizes.  Return 0 on success,
 * nonzero on error with a message from sfg_last_error().  Record layouts are
 * in paper_2603_05725_b200/csrc/sfg_types.h.
 */
#ifndef SFG_B200_H
#define SFG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sfg_program sfg_program;

typedef struct sfg_corpus_dev {  /* device corpus as of the round start */
  const void* meta;              /* sfg_entry[n]          */
  const void* vals;              /* sfg_val[n * n_args]   */
  const void* data;              /* payload arena         */
  int32_t n;
  int32_t n_seeds;
} sfg_corpus_dev;

int sfg_abi_version(void);
/* sizes/offsets of the record structs (layout self-check for host packers):
 * 0 ins 1 kernel 2 hostop 3 binding 4 rec 5 val 6 op 7 child 8 entry 9 verdict
 * 10 prog 11 offsetof(prog,kernels) 12 offsetof(prog,recent_weight) 13 offsetof(prog,copyout_arg) */
size_t sfg_layout_probe(int which);
const char* sfg_last_error(void);

/* Upload the lowered harness (host tables; sizes in records). */
int sfg_program_create(const void* prog, size_t prog_bytes, const void* ins, size_t n_ins,
                       const void* hostops, size_t n_hostops, const void* binds, size_t n_binds,
                       const void* base_recs, size_t n_recs, const void* const_blob,
                       size_t const_bytes, const void* base_blob_dev, sfg_program** out);
/* Replace the scalar header (campaign knobs: stop rule, budget, readback). */
int sfg_program_update(sfg_program* p, const void* prog, size_t prog_bytes);
void sfg_program_destroy(sfg_program* p);
size_t sfg_execute_smem_bytes(const sfg_program* p);
/* Generated CUDA source of the program's specialized execute kernel (0 if the
 * generic interpreter is used, i.e. SFG_JIT=0). Copies at most cap-1 bytes. */
size_t sfg_program_jit_source(const sfg_program* p, char* buf, size_t cap);
/* Generate + NVRTC-compile the specialized kernel for a lowered program without
 * loading it (no GPU needed).  out receives the source (and log on failure). */
int sfg_jit_check(const void* prog, size_t prog_bytes, const void* ins, uint64_t max_edge_events, char* out,
                  size_t cap, size_t* cubin_bytes);
/* Process-wide counts of NVRTC compiles and of programs loaded from the on-disk
 * cubin cache ($SFG_JIT_CACHE, default ~/.cache/sfg_b200_jit; "0" disables). */
void sfg_jit_stats(int* compiles, int* disk_hits);

int sfg_plan(const sfg_program* p, const sfg_corpus_dev* c, int64_t it0, int n, int32_t* parent,
             int8_t* picks, uint32_t* int_flags, void* stream);
/* Sequential stream discipline (the reference fuzz_loop itself, campaign.py:714-749:
 * one worker stream Stream(master_seed, 1000 + w), one MutationSchedule): one
 * thread generates children it0 .. it0+n-1 in order from the worker state *state
 * (device, sfg_stream_state_bytes() bytes), rotation counts from counts_base,
 * writing children / vals as sfg_mutate does, the int-arg picks per input
 * (int_flags[n][n_int_args]) and the stream state before every input and after
 * the last (states[n + 1]), so that a round can be cut after an admission and
 * resumed from there.  sfg_stream_state_init fills a host buffer with
 * Stream(seed, stream_id)'s initial state. */
size_t sfg_stream_state_bytes(void);
int sfg_stream_state_init(uint64_t seed, uint64_t stream_id, void* out_host);
int sfg_plan_seq(const sfg_program* p, const sfg_corpus_dev* c, int64_t it0, int n, const void* state,
                 const uint64_t* counts_base, void* children, void* vals, uint32_t* int_flags, void* states,
                 void* stream);
/* Sequential discipline in parallel (mutate.cu "seqgen"): the same outputs as
 * sfg_plan_seq (children, vals, int_flags, states[n + 1]) computed without a
 * one-thread walk: every candidate child boundary of the worker stream's next
 * `words` words draws one child, pointer doubling finds the boundaries reachable
 * from *state, and the children are generated in parallel from them.  Requires
 * it0 >= 2, saturated rotation counts (every mutable column of counts_base >= 3),
 * no fan-out and no corpus entry leaving the recent window inside the round.
 * stats[0] = children whose start was found (the round must be cut after
 * stats[0] - 1 when < n; states[stats[0]] is exact), stats[1] = words drawn by
 * them.  scratch: sfg_seq_scratch_ints(n, words) int32 of device memory. */
int64_t sfg_seq_scratch_ints(int n, int64_t words);
int sfg_plan_seq_par(const sfg_program* p, const sfg_corpus_dev* c, int64_t it0, int n, const void* state,
                     int64_t words, const uint64_t* counts_base, void* children, void* vals, uint32_t* int_flags,
                     void* states, int32_t* scratch, int64_t scratch_ints, uint64_t* stats, void* stream);
/* Children it0 .. it0+n-1 (batched contract).  Input i's rotation count of int
 * column c is counts_base[c] + counts_prefix[i][c]; counts_prefix may be NULL when
 * every mutable column of counts_base is >= 3 (the counts then no longer steer
 * generation, mutation.py:378-386, and no plan pass / pick scans are needed). */
int sfg_mutate(const sfg_program* p, const sfg_corpus_dev* c, int64_t it0, int n,
               const uint64_t* counts_prefix, const uint64_t* counts_base, void* children,
               void* vals, void* stream);
int sfg_apply(const sfg_program* p, const sfg_corpus_dev* c, int n, const void* children,
              const void* vals, const uint64_t* work_base, uint8_t* work, void* stream);
int sfg_regen(const sfg_program* p, const sfg_corpus_dev* c, int n_sel, const int32_t* sel,
              const void* children, const void* vals, const uint64_t* dst_off, uint8_t* dst,
              void* stream);
/* work_counter: 8 ints of device scratch private to this launch pair (the
 * persistent specialized kernels hand out inputs from it; [1] = number of
 * soft-cap deferrals, [3] = number of inputs to re-run thread-sequentially;
 * concurrent launches need their own).  deferred: 2n ints (the two lists).
 * Group-parallel mode (specialized kernel, programs whose launches have more
 * than one simulated thread): the simulated threads of a launch run on the
 * lanes of a group at once, with per-word conflict tags over the input's work
 * region in shared memory; a chunk of threads with a cross-thread conflict is
 * undone (work-region snapshot in shared memory) and re-run in place thread
 * after thread; an input whose work region exceeds the shared-memory tag
 * capacity is listed for a thread-sequential re-run.
 * max_work_bytes bounds every input's work region of this round.  deferred ==
 * NULL (inputs whose payloads cannot be re-materialized): thread-sequential.
 * soft_cap != 0 (specialized kernel only): an input one of whose simulated
 * threads would retire soft_cap instructions (cumulative over threads when
 * they run sequentially) is abandoned and listed; sfg_execute_deferred
 * re-materializes the listed inputs' payloads and runs them from scratch with
 * the real budget (soft-cap list group-parallel, spread one input per warp;
 * then the sequential list).  Results are identical to soft_cap 0 and to
 * sequential execution (executor.py:405-424).
 * n_live (with order): the schedule holds *n_live inputs (sfg_dedupe representatives).
 * c != NULL (the campaign's corpus as of the round start): the kernel builds every
 * input's arrays in its work region itself, from its parent's payload, before its
 * COMPUTE phase (sfg_apply fused into the execute pass); c == NULL: the work
 * regions were built by sfg_apply (or by the host, execute_testcases). */
int sfg_execute(const sfg_program* p, const sfg_corpus_dev* c, int n, const void* children, const void* vals,
                const uint64_t* work_base, uint8_t* work, void* verdicts, uint32_t* edge_counts,
                uint8_t* readouts, const uint64_t* readout_base, int* work_counter,
                uint64_t soft_cap, int32_t* deferred, int64_t max_work_bytes, const int32_t* order,
                const int32_t* n_live, void* stream);
int sfg_execute_deferred(const sfg_program* p, const sfg_corpus_dev* c, int n, const void* children,
                         const void* vals, const uint64_t* work_base, uint8_t* work, void* verdicts,
                         uint32_t* edge_counts, uint8_t* readouts, const uint64_t* readout_base,
                         int* work_counter, int32_t* deferred, int64_t max_work_bytes,
                         void* stream);
/* Trace mode (replaces the reference's ExecHooks / TraceHooks per event,
 * executor.py:108-135, cli.py:42-45): run the inputs through the generic
 * interpreter and record every on_mem_access / on_control_flow event of input i
 * into trace[i * trace_cap * 4 ...] (4 uint64 words per event; layout in
 * csrc/execute.cu); trace_count[i] = events produced (> trace_cap: truncated). */
int sfg_execute_trace(const sfg_program* p, int n, const void* children, const void* vals,
                      const uint64_t* work_base, uint8_t* work, void* verdicts, uint32_t* edge_counts,
                      uint8_t* readouts, const uint64_t* readout_base, uint64_t* trace,
                      uint32_t trace_cap, uint32_t* trace_count, void* stream);
/* A non-blocking CUDA stream (cudaStreamCreateWithPriority).  The Python host keeps
 * one process-wide ring of them, created back to back, so that each round in
 * flight owns a hardware work queue (CUDA_DEVICE_MAX_CONNECTIONS) for the life of
 * the process instead of drawing from torch's shared stream pool. */
int sfg_stream_create(int priority, void** out);
/* Lanes per input of the program's group-parallel mode (1 = thread-sequential). */
int sfg_program_group(const sfg_program* p);
/* Bulk-pass schedule: order[0..n) = a permutation of the round's inputs grouped by
 * a hash of their scalar arguments and array shapes (inputs likely to take the
 * same path share warps).  Pass it as sfg_execute's `order` (NULL = identity).
 * scratch: sfg_order_scratch_ints(n) ints of device memory. */
size_t sfg_order_scratch_ints(int n);
/* Bit a set: harness argument a can steer the simulated kernels' control flow
 * (taint analysis at program creation); sfg_order hashes only these. */
uint32_t sfg_program_order_mask(const sfg_program* p);
/* The same analysis on host tables, no device needed (tests, tooling). */
uint32_t sfg_control_mask(const void* prog, size_t prog_bytes, const void* ins, const void* hostops,
                          size_t n_hostops, const void* binds);
int sfg_order(const sfg_program* p, int n, const void* vals, int32_t* order, int32_t* scratch,
              const int32_t* rep, int32_t* n_live, void* stream);
/* Duplicate inputs (order.cu): rep[i] = the input whose execution stands for input i
 * (itself, or an earlier-inserted input with equal argument descriptors, the same
 * parent and the same data-level array op -- a COMPUTE phase is a pure function of
 * them).  table: `slots` uint64 words (a power of two >= 2n), cleared here.  Pass
 * rep to sfg_order (only representatives are scheduled, their count to *n_live) and
 * n_live to sfg_execute; after sfg_execute_deferred, sfg_dup_fill copies each
 * representative's verdict and edge-count row to its duplicates. */
int sfg_dedupe(const sfg_program* p, int n, const void* children, const void* vals, uint64_t* table, int slots,
               int32_t* rep, void* stream);
int sfg_dup_fill(const sfg_program* p, int n, const int32_t* rep, void* verdicts, uint32_t* edge_counts,
                 void* stream);
/* Grouped schedule (every input runs): full[0..n) = the representatives in `order`
 * (the first *n_live entries, sfg_order with rep), each directly followed by its
 * duplicates, so a warp of the bulk pass takes runs of equal inputs.  scratch:
 * sfg_group_scratch_ints(n) int32 of device memory.  Pass full as sfg_execute's
 * order with n_live = NULL. */
size_t sfg_group_scratch_ints(int n);
int sfg_group_schedule(const sfg_program* p, int n, const int32_t* rep, const int32_t* order, const int32_t* n_live,
                       int32_t* full, int32_t* scratch, void* stream);
/* Triage in three stream-ordered phases so that a multi-GPU campaign can merge
 * the per-rank partials between them: a rank owns the global
 * round indices [i_base, i_base + n).  All indices written are GLOBAL round
 * indices; "none" is INT32_MAX, so the merge is a signed MIN all-reduce.
 *   stop:   scalars[0] = min stop-rule finding, scalars[1] = min fatal     -> MIN
 *   absorb: first_hit[E], key_first[K]                                     -> MIN
 *           edge_delta[E], key_count[K], entered_cnt[n_kernels]            -> SUM
 *           allocs[n] (per input, 0 past the stop)   (local; exclusive-scanned)
 *   admit:  admit[n] = no finding, it != 1, first hitter of an edge unseen
 *           at the round start (ghit)                                       (local)
 * sfg_commit folds the merged delta into the campaign map (edge_total,
 * ghit, entered mask).  Callers fill scalars/first_hit/key_first with
 * INT32_MAX and zero the SUM buffers before the stop phase. */
int sfg_triage_stop(const sfg_program* p, int n, int i_base, const void* verdicts, int32_t* scalars,
                    void* stream);
int sfg_triage_absorb(const sfg_program* p, int n, int i_base, const void* verdicts,
                      const uint32_t* edge_counts, const int32_t* scalars, int32_t* first_hit,
                      uint64_t* edge_delta, int32_t* key_first, uint64_t* key_count,
                      uint64_t* entered_cnt, uint64_t* allocs, void* stream);
int sfg_triage_admit(const sfg_program* p, int n, int i_base, const void* verdicts,
                     const uint32_t* edge_counts, const void* children, const int32_t* scalars,
                     const int32_t* first_hit, const uint8_t* ghit, uint64_t* admit, void* stream);
int sfg_commit(const sfg_program* p, const uint64_t* edge_delta, const uint64_t* entered_cnt,
               uint64_t* edge_total, uint8_t* ghit, uint32_t* entered, void* stream);
/* Context-sensitive hashed coverage map (derived view; admission stays on exact
 * edges): every live input (round index <= scalars[0]) sets, per hit edge e, the
 * byte slot fmix64(edge_ctx[e] ^ bucket(count) * 0x9E3779B97F4A7C15) & (2^map_bits - 1)
 * of map (2^map_bits bytes, 4-byte aligned); new_slots[0] += slots turned on.
 * Byte flags: the cross-GPU merge is a MAX all-reduce of map. */
int sfg_ctxmap(int n, int n_edges, int i_base, const uint32_t* edge_counts, const int32_t* scalars,
               const uint64_t* edge_ctx, uint8_t* map, int map_bits, uint64_t* new_slots, void* stream);
/* admitted children (admit/pos from the admit phase + scan) -> contiguous staging
 * rows (sfg_child, n_args x sfg_val): the records ranks exchange on admission */
int sfg_select(const sfg_program* p, const void* children, const void* vals, const uint64_t* admit,
               const uint64_t* pos, int n, void* stage_children, void* stage_vals, void* stream);
/* admit == NULL: every row counts (staged rows); compact then appends rows 0..n-1 in order */
int sfg_child_bytes(const sfg_program* p, const void* vals, const uint64_t* admit, int n,
                    uint64_t* bytes, void* stream);
int sfg_compact(const sfg_program* p, const void* children, const void* vals, const uint64_t* admit,
                const uint64_t* pos, const uint64_t* boff, int n, int n_corpus, uint64_t corpus_bytes,
                void* cmeta, void* cvals, void* cchild, int32_t* sel, uint64_t* dst_off, void* stream);
/* exclusive prefix sum of in[i*stride + col] into out[i*out_stride + out_col]; tmp holds
 * ceil(n/2048) u64; *total (device) receives the sum when non-null */
int sfg_scan_u32(const uint32_t* in, int64_t n, int stride, int col, uint64_t* out, int out_stride,
                 int out_col, uint64_t* tmp, uint64_t* total, void* stream);
int sfg_scan_u64(const uint64_t* in, int64_t n, int stride, int col, uint64_t* out, int out_stride,
                 int out_col, uint64_t* tmp, uint64_t* total, void* stream);

#ifdef __cplusplus
}
#endif
#endif
