// C ABI (include/sfg.h): host-side launch wrappers around the sm_100a kernels.
// No torch types cross this boundary; the Python host passes raw device
// pointers (torch tensors' data_ptr) and torch's current stream.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/sfg.h"
#include "common.cuh"

struct sfg_program {
  sfg_prog P;
  cudaLibrary_t jit_lib = nullptr;    // specialized execute kernel (jit.cu), if built
  cudaKernel_t jit_kernel = nullptr;
  cudaKernel_t jit_tail = nullptr;    // tail pass over deferred long inputs (one-warp CTAs)
  int jit_grid = 0;                   // resident CTAs (occupancy x SMs)
  int tail_grid = 0;                  // resident one-warp tail CTAs
  int tail_k = 1;                     // long inputs per tail warp
  int jit_block = 128;                // CTA size of the persistent kernel
  int jit_mode = 1;                   // 0 per-lane fetch, 1 per-warp batches
  std::string jit_source, jit_log;
  sfg_ins* ins;
  sfg_hostop* hostops;
  sfg_binding* binds;
  sfg_rec* recs;
  uint8_t* const_blob;
  const uint8_t* base_blob;  // caller-owned device buffer
  size_t smem;
};

static_assert(sizeof(sfg_ins) == 32, "sfg_ins layout");
static_assert(sizeof(sfg_kernel) == 48, "sfg_kernel layout");
static_assert(sizeof(sfg_hostop) == 72, "sfg_hostop layout");
static_assert(sizeof(sfg_binding) == 16, "sfg_binding layout");
static_assert(sizeof(sfg_rec) == 64, "sfg_rec layout");
static_assert(sizeof(sfg_val) == 64, "sfg_val layout");
static_assert(sizeof(sfg_op) == 32, "sfg_op layout");
static_assert(sizeof(sfg_child) == 144, "sfg_child layout");
static_assert(sizeof(sfg_entry) == 32, "sfg_entry layout");
static_assert(sizeof(sfg_verdict) == 112, "sfg_verdict layout");
static_assert(sizeof(sfg_prog) < 4096, "sfg_prog must fit the kernel parameter space");

// one translation unit: the kernels are defined in these files
#include "mutate.cu"
#include "execute.cu"
#include "triage.cu"
#include "ctxmap.cu"
#include "jit.cu"

static thread_local std::string g_err;

static int fail(const char* where, cudaError_t e) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return 1;
}

#define SFG_CHECK_LAUNCH(name)                               \
  do {                                                       \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) return fail(name, _e);            \
  } while (0)

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
static inline CorpusView CV(const sfg_corpus_dev* c) {
  return CorpusView{(const sfg_entry*)c->meta, (const sfg_val*)c->vals, (const uint8_t*)c->data, c->n, c->n_seeds};
}

template <typename T>
static cudaError_t dupe(T** dst, const void* src, size_t count) {
  *dst = nullptr;
  if (count == 0) return cudaSuccess;
  cudaError_t e = cudaMalloc((void**)dst, count * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
}

static size_t exec_smem(const sfg_prog& P) {
  int maxregs = 1;
  for (int k = 0; k < P.n_kernels; ++k) maxregs = P.kernels[k].regs > maxregs ? P.kernels[k].regs : maxregs;
  const size_t ins = ((size_t)P.total_ins * sizeof(sfg_ins) + 15) & ~(size_t)15;
  return ins + 4 * (size_t)32 * (maxregs * 24 + P.n_edges * 4);
}

template <typename T>
static int scan_impl(const T* in, int64_t n, int stride, int col, uint64_t* out, int out_stride, int out_col,
                     uint64_t* tmp, uint64_t* total, void* stream, const char* name) {
  const int64_t tiles = (n + 2047) / 2048;
  if (n <= 0) {
    if (total) cudaMemsetAsync(total, 0, sizeof(uint64_t), S(stream));
    return 0;
  }
  sfg_scan_tiles<T><<<(unsigned)tiles, 256, 0, S(stream)>>>(in, n, stride, col, tmp);
  SFG_CHECK_LAUNCH(name);
  sfg_scan_tile_sums<<<1, 256, 0, S(stream)>>>(tmp, tiles, total);
  SFG_CHECK_LAUNCH(name);
  sfg_scan_apply<T><<<(unsigned)tiles, 256, 0, S(stream)>>>(in, n, stride, col, tmp, out, out_stride, out_col);
  SFG_CHECK_LAUNCH(name);
  return 0;
}

extern "C" {

int sfg_abi_version(void) { return SFG_ABI_VERSION; }

size_t sfg_layout_probe(int which) {
  switch (which) {
    case 0: return sizeof(sfg_ins);
    case 1: return sizeof(sfg_kernel);
    case 2: return sizeof(sfg_hostop);
    case 3: return sizeof(sfg_binding);
    case 4: return sizeof(sfg_rec);
    case 5: return sizeof(sfg_val);
    case 6: return sizeof(sfg_op);
    case 7: return sizeof(sfg_child);
    case 8: return sizeof(sfg_entry);
    case 9: return sizeof(sfg_verdict);
    case 10: return sizeof(sfg_prog);
    case 11: return offsetof(sfg_prog, kernels);
    case 12: return offsetof(sfg_prog, recent_weight);
    case 13: return offsetof(sfg_prog, copyout_arg);
    default: return 0;
  }
}
const char* sfg_last_error(void) { return g_err.c_str(); }

int sfg_program_create(const void* prog, size_t prog_bytes, const void* ins, size_t n_ins, const void* hostops,
                       size_t n_hostops, const void* binds, size_t n_binds, const void* base_recs, size_t n_recs,
                       const void* const_blob, size_t const_bytes, const void* base_blob_dev, sfg_program** out) {
  if (prog_bytes != sizeof(sfg_prog)) {
    g_err = "sfg_program_create: sfg_prog size mismatch (host " + std::to_string(prog_bytes) + ", device " +
            std::to_string(sizeof(sfg_prog)) + ")";
    return 1;
  }
  sfg_program* p = new sfg_program();
  memcpy(&p->P, prog, sizeof(sfg_prog));
  cudaError_t e;
  if ((e = dupe(&p->ins, ins, n_ins)) != cudaSuccess ||
      (e = dupe(&p->hostops, hostops, n_hostops)) != cudaSuccess ||
      (e = dupe(&p->binds, binds, n_binds)) != cudaSuccess ||
      (e = dupe(&p->recs, base_recs, n_recs)) != cudaSuccess ||
      (e = dupe(&p->const_blob, const_blob, const_bytes)) != cudaSuccess) {
    sfg_program_destroy(p);
    return fail("sfg_program_create", e);
  }
  p->base_blob = (const uint8_t*)base_blob_dev;
  p->smem = exec_smem(p->P);
  const char* jit_env = getenv("SFG_JIT");
  if (!(jit_env && jit_env[0] == '0')) {
    // bound on per-input edge events decides whether counters need overflow checks
    uint64_t events = 0;
    const sfg_hostop* H = (const sfg_hostop*)hostops;
    for (size_t h = 0; h < n_hostops; ++h)
      if (H[h].kind == SFG_H_LAUNCH) {
        const double ev = (double)H[h].grid * (double)H[h].block * (double)p->P.budget;
        events = (ev + (double)events >= 1.8e19) ? ~0ull : events + (uint64_t)ev;
      }
    const int rc = sfg_jit_build(p->P, (const sfg_ins*)ins, events, p->jit_source, p->jit_log, &p->jit_lib,
                                 &p->jit_kernel, &p->jit_tail);
    if (rc != 0) {
      g_err = "sfg_program_create: JIT build failed (" + std::to_string(rc) + "): " + p->jit_log.substr(0, 6000);
      sfg_program_destroy(p);
      return 1;
    }
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (const char* b = getenv("SFG_EXEC_BLOCK")) p->jit_block = atoi(b) >= 32 ? atoi(b) : 128;
    if (const char* md = getenv("SFG_EXEC_MODE")) p->jit_mode = atoi(md);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)p->jit_kernel, p->jit_block, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    p->jit_grid = sms * per_sm;
    if (const char* tk = getenv("SFG_TAIL_K")) p->tail_k = atoi(tk) >= 1 && atoi(tk) <= 32 ? atoi(tk) : 1;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)p->jit_tail, 32, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    p->tail_grid = sms * per_sm;

  }
  e = cudaFuncSetAttribute(sfg_execute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem);
  if (e != cudaSuccess) {
    sfg_program_destroy(p);
    return fail("sfg_program_create: execute smem", e);
  }
  *out = p;
  return 0;
}

int sfg_program_update(sfg_program* p, const void* prog, size_t prog_bytes) {
  if (prog_bytes != sizeof(sfg_prog)) {
    g_err = "sfg_program_update: sfg_prog size mismatch";
    return 1;
  }
  memcpy(&p->P, prog, sizeof(sfg_prog));
  return 0;
}

void sfg_program_destroy(sfg_program* p) {
  if (!p) return;
  if (p->jit_lib) cudaLibraryUnload(p->jit_lib);
  cudaFree(p->ins);
  cudaFree(p->hostops);
  cudaFree(p->binds);
  cudaFree(p->recs);
  cudaFree(p->const_blob);
  delete p;
}

size_t sfg_execute_smem_bytes(const sfg_program* p) { return p->smem; }

int sfg_jit_check(const void* prog, size_t prog_bytes, const void* ins, uint64_t max_edge_events, char* out,
                  size_t cap, size_t* cubin_bytes) {
  if (prog_bytes != sizeof(sfg_prog)) {
    g_err = "sfg_jit_check: sfg_prog size mismatch";
    return 1;
  }
  sfg_prog P;
  memcpy(&P, prog, sizeof P);
  std::string src, log;
  std::vector<char> cubin;
  const int rc = sfg_jit_compile(P, (const sfg_ins*)ins, max_edge_events, src, log, cubin);
  const std::string text = rc ? log + "\n----\n" + src : src;
  if (out && cap) {
    const size_t n = text.size() < cap - 1 ? text.size() : cap - 1;
    memcpy(out, text.data(), n);
    out[n] = 0;
  }
  if (cubin_bytes) *cubin_bytes = cubin.size();
  if (rc) g_err = "sfg_jit_check: compile failed";
  return rc;
}

size_t sfg_program_jit_source(const sfg_program* p, char* buf, size_t cap) {
  if (!p->jit_kernel) return 0;
  if (buf && cap) {
    const size_t n = p->jit_source.size() < cap - 1 ? p->jit_source.size() : cap - 1;
    memcpy(buf, p->jit_source.data(), n);
    buf[n] = 0;
  }
  return p->jit_source.size();
}

int sfg_plan(const sfg_program* p, const sfg_corpus_dev* c, int64_t it0, int n, int32_t* parent, int8_t* picks,
             uint32_t* int_flags, void* stream) {
  if (n <= 0) return 0;
  sfg_plan_kernel<<<blocks_for(n, 128), 128, 0, S(stream)>>>(p->P, CV(c), it0, n, parent, picks, int_flags);
  SFG_CHECK_LAUNCH("sfg_plan");
  return 0;
}

int sfg_mutate(const sfg_program* p, const sfg_corpus_dev* c, int64_t it0, int n, const uint64_t* counts_prefix,
               const uint64_t* counts_base, void* children, void* vals, void* stream) {
  if (n <= 0) return 0;
  sfg_mutate_kernel<<<blocks_for(n, 128), 128, 0, S(stream)>>>(p->P, CV(c), it0, n, counts_prefix, counts_base,
                                                              (sfg_child*)children, (sfg_val*)vals);
  SFG_CHECK_LAUNCH("sfg_mutate");
  return 0;
}

int sfg_apply(const sfg_program* p, const sfg_corpus_dev* c, int n, const void* children, const void* vals,
              const uint64_t* work_base, uint8_t* work, void* stream) {
  if (n <= 0) return 0;
  sfg_apply_kernel<<<blocks_for((int64_t)n * 32, 256), 256, 0, S(stream)>>>(
      p->P, CV(c), n, (const sfg_child*)children, (const sfg_val*)vals, work_base, work, nullptr, nullptr);
  SFG_CHECK_LAUNCH("sfg_apply");
  return 0;
}

int sfg_regen(const sfg_program* p, const sfg_corpus_dev* c, int n_sel, const int32_t* sel, const void* children,
              const void* vals, const uint64_t* dst_off, uint8_t* dst, void* stream) {
  if (n_sel <= 0) return 0;
  sfg_regen_kernel<<<blocks_for((int64_t)n_sel * 32, 256), 256, 0, S(stream)>>>(
      p->P, CV(c), n_sel, sel, (const sfg_child*)children, (const sfg_val*)vals, dst_off, dst);
  SFG_CHECK_LAUNCH("sfg_regen");
  return 0;
}

int sfg_execute(const sfg_program* p, int n, const void* children, const void* vals, const uint64_t* work_base,
                uint8_t* work, void* verdicts, uint32_t* edge_counts, uint8_t* readouts,
                const uint64_t* readout_base, uint64_t* overlay, int* work_counter, uint64_t soft_cap,
                int32_t* deferred, void* stream) {
  if (n <= 0) {
    if (work_counter) cudaMemsetAsync(work_counter, 0, 4 * sizeof(int), S(stream));
    return 0;
  }
  ExecView E{p->ins, p->hostops, p->binds, p->recs, p->base_blob, p->const_blob,
             (const sfg_child*)children, (const sfg_val*)vals, work_base, work,
             (sfg_verdict*)verdicts, edge_counts, readouts, readout_base, overlay, n,
             0ull, deferred, work_counter ? work_counter + 1 : nullptr};
  if (p->jit_kernel) {
    if (work_counter == nullptr) {
      g_err = "sfg_execute: the specialized kernel needs a per-launch work counter";
      return 1;
    }
    if (soft_cap && deferred == nullptr) {
      g_err = "sfg_execute: soft_cap needs a deferred list";
      return 1;
    }
    E.soft_cap = soft_cap;
    cudaError_t e = cudaMemsetAsync(work_counter, 0, 4 * sizeof(int), S(stream));
    if (e != cudaSuccess) return fail("sfg_execute (jit counter)", e);
    int* next = work_counter;
    int mode = p->jit_mode;
    void* args[] = {(void*)&p->P, (void*)&E, (void*)&next, (void*)&mode};
    const unsigned want = blocks_for(n, p->jit_block);
    const unsigned grid = want < (unsigned)p->jit_grid ? want : (unsigned)p->jit_grid;
    e = cudaLaunchKernel((const void*)p->jit_kernel, dim3(grid), dim3(p->jit_block), args, 0, S(stream));
    if (e != cudaSuccess) return fail("sfg_execute (jit)", e);
    return 0;
  }
  if (work_counter) cudaMemsetAsync(work_counter, 0, 4 * sizeof(int), S(stream));
  sfg_execute_kernel<<<blocks_for(n, 128), 128, p->smem, S(stream)>>>(p->P, E);
  SFG_CHECK_LAUNCH("sfg_execute");
  return 0;
}

int sfg_execute_deferred(const sfg_program* p, const sfg_corpus_dev* c, int n, const void* children,
                         const void* vals, const uint64_t* work_base, uint8_t* work, void* verdicts,
                         uint32_t* edge_counts, uint8_t* readouts, const uint64_t* readout_base, uint64_t* overlay,
                         int* work_counter, int32_t* deferred, void* stream) {
  if (n <= 0 || !p->jit_kernel) return 0;  // the interpreter never defers
  // pristine payloads again (the first attempt's stores landed in the work regions)
  sfg_apply_kernel<<<p->jit_grid, 256, 0, S(stream)>>>(p->P, CV(c), n, (const sfg_child*)children,
                                                      (const sfg_val*)vals, work_base, work, deferred,
                                                      work_counter + 1);
  SFG_CHECK_LAUNCH("sfg_execute_deferred/apply");
  ExecView E{p->ins, p->hostops, p->binds, p->recs, p->base_blob, p->const_blob,
             (const sfg_child*)children, (const sfg_val*)vals, work_base, work,
             (sfg_verdict*)verdicts, edge_counts, readouts, readout_base, overlay, n,
             0ull, deferred, work_counter + 1};
  int* next = work_counter + 2;
  int k = p->tail_k;
  void* args[] = {(void*)&p->P, (void*)&E, (void*)&next, (void*)&k};
  // one-warp CTAs: a warp that holds long inputs pins only its own slot
  cudaError_t e = cudaLaunchKernel((const void*)p->jit_tail, dim3((unsigned)p->tail_grid), dim3(32), args, 0, S(stream));
  if (e != cudaSuccess) return fail("sfg_execute_deferred (jit)", e);
  return 0;
}

int sfg_triage_stop(const sfg_program* p, int n, int i_base, const void* verdicts, int32_t* scalars,
                    void* stream) {
  if (n <= 0) return 0;
  sfg_stop_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(p->P, (const sfg_verdict*)verdicts, n, i_base, scalars);
  SFG_CHECK_LAUNCH("sfg_triage_stop");
  return 0;
}

int sfg_triage_absorb(const sfg_program* p, int n, int i_base, const void* verdicts, const uint32_t* edge_counts,
                      const int32_t* scalars, int32_t* first_hit, uint64_t* edge_delta, int32_t* key_first,
                      uint64_t* key_count, uint64_t* entered_cnt, uint64_t* allocs, void* stream) {
  if (n <= 0) return 0;
  sfg_absorb_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(
      p->P, (const sfg_verdict*)verdicts, edge_counts, n, i_base, scalars, first_hit,
      (unsigned long long*)edge_delta, key_first, (unsigned long long*)key_count,
      (unsigned long long*)entered_cnt, allocs);
  SFG_CHECK_LAUNCH("sfg_triage_absorb");
  return 0;
}

int sfg_triage_admit(const sfg_program* p, int n, int i_base, const void* verdicts, const uint32_t* edge_counts,
                     const void* children, const int32_t* scalars, const int32_t* first_hit, const uint8_t* ghit,
                     uint64_t* admit, void* stream) {
  if (n <= 0) return 0;
  sfg_admit_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(p->P, (const sfg_verdict*)verdicts, edge_counts,
                                                             (const sfg_child*)children, n, i_base, scalars,
                                                             first_hit, ghit, admit);
  SFG_CHECK_LAUNCH("sfg_triage_admit");
  return 0;
}

int sfg_commit(const sfg_program* p, const uint64_t* edge_delta, const uint64_t* entered_cnt, uint64_t* edge_total,
               uint8_t* ghit, uint32_t* entered, void* stream) {
  const int ne = p->P.n_edges > 0 ? p->P.n_edges : 1;
  sfg_commit_kernel<<<blocks_for(ne, 256), 256, 0, S(stream)>>>(
      p->P.n_edges, p->P.n_kernels, (const unsigned long long*)edge_delta, (const unsigned long long*)entered_cnt,
      (unsigned long long*)edge_total, ghit, entered);
  SFG_CHECK_LAUNCH("sfg_commit");
  return 0;
}

int sfg_select(const sfg_program* p, const void* children, const void* vals, const uint64_t* admit,
               const uint64_t* pos, int n, void* stage_children, void* stage_vals, void* stream) {
  if (n <= 0) return 0;
  sfg_select_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(p->P, (const sfg_child*)children,
                                                              (const sfg_val*)vals, admit, pos, n,
                                                              (sfg_child*)stage_children, (sfg_val*)stage_vals);
  SFG_CHECK_LAUNCH("sfg_select");
  return 0;
}

int sfg_ctxmap(int n, int n_edges, int i_base, const uint32_t* edge_counts, const int32_t* scalars,
               const uint64_t* edge_ctx, uint8_t* map, int map_bits, uint64_t* new_slots, void* stream) {
  if (n <= 0 || n_edges <= 0) return 0;
  if (map_bits < 2 || map_bits > 34) {
    g_err = "sfg_ctxmap: map_bits out of range";
    return 1;
  }
  const int64_t total = (int64_t)n * n_edges;
  sfg_ctxmap_kernel<<<blocks_for(total, 256), 256, 0, S(stream)>>>(
      n, n_edges, i_base, edge_counts, scalars, edge_ctx, (uint32_t*)map, (1ull << map_bits) - 1,
      (unsigned long long*)new_slots);
  SFG_CHECK_LAUNCH("sfg_ctxmap");
  return 0;
}

int sfg_child_bytes(const sfg_program* p, const void* vals, const uint64_t* admit, int n, uint64_t* bytes,
                    void* stream) {
  if (n <= 0) return 0;
  sfg_child_bytes_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(p->P, (const sfg_val*)vals, admit, n, bytes);
  SFG_CHECK_LAUNCH("sfg_child_bytes");
  return 0;
}

int sfg_compact(const sfg_program* p, const void* children, const void* vals, const uint64_t* admit,
                const uint64_t* pos, const uint64_t* boff, int n, int n_corpus, uint64_t corpus_bytes, void* cmeta,
                void* cvals, void* cchild, int32_t* sel, uint64_t* dst_off, void* stream) {
  if (n <= 0) return 0;
  sfg_compact_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(
      p->P, (const sfg_child*)children, (const sfg_val*)vals, admit, pos, boff, n, n_corpus, corpus_bytes,
      (sfg_entry*)cmeta, (sfg_val*)cvals, (sfg_child*)cchild, sel, dst_off);
  SFG_CHECK_LAUNCH("sfg_compact");
  return 0;
}

int sfg_scan_u32(const uint32_t* in, int64_t n, int stride, int col, uint64_t* out, int out_stride, int out_col,
                 uint64_t* tmp, uint64_t* total, void* stream) {
  return scan_impl(in, n, stride, col, out, out_stride, out_col, tmp, total, stream, "sfg_scan_u32");
}

int sfg_scan_u64(const uint64_t* in, int64_t n, int stride, int col, uint64_t* out, int out_stride, int out_col,
                 uint64_t* tmp, uint64_t* total, void* stream) {
  return scan_impl(in, n, stride, col, out, out_stride, out_col, tmp, total, stream, "sfg_scan_u64");
}

}  // extern "C"
