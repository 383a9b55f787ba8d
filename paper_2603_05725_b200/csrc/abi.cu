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
  int sms = 0;
  int tail_k = 4;                     // long inputs per tail warp (group-parallel pass; at most 32 / group): 1 = lowest latency, 4 = +5 % throughput on C2
  int tail_k_seq = 32;                // inputs per warp of the thread-sequential re-run pass
  int tail_ctas = 1024;               // one-warp CTAs of the long-input pass
  int bulk_persist = 1;               // bulk pass: persistent grid (1) or a CTA per batch (0)
  uint32_t order_mask = ~0u;          // harness args hashed by sfg_order (control_arg_mask)
  int group = 1;                      // lanes per input of the tail pass (group-parallel launches)
  int bulk_group = 1;                 // lanes per input of the bulk pass (1 = thread-sequential)
  int jit_block = 128;                // CTA size of the persistent kernel
  int jit_mode = 1;                   // 0 per-lane fetch, 1 per-warp batches
  std::string jit_source, jit_log;
  sfg_ins* ins;
  sfg_hostop* hostops;
  sfg_binding* binds;
  sfg_rec* recs;
  uint8_t* const_blob;
  size_t tab_bytes[5] = {0, 0, 0, 0, 0};   // bytes of the five tables above (table_free)
  const uint8_t* base_blob;  // caller-owned device buffer
  size_t smem;
  int gen_warps = 4;                  // warps per block of the generic interpreter
  bool gen_ok = true;                 // its shared memory fits
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
#include "order.cu"
#include "jit.cu"

static thread_local std::string g_err;

// Harness arguments that can steer the simulated kernels' control flow: taint of
// every kernel parameter propagated (flow-insensitively, to a fixpoint) through
// moves, arithmetic, conversions and load addresses into setp sources and into
// load/store addresses (the sanitizer's verdict stops a thread at its first
// finding); the launches' bindings map tainted parameters to harness arguments.
// Pure data (e.g. a float scale factor) stays out.
static uint32_t control_arg_mask(const sfg_prog& P, const sfg_ins* ins, const sfg_hostop* H, size_t nh,
                                 const sfg_binding* B) {
  uint32_t args = 0;
  for (size_t h = 0; h < nh; ++h) {
    if (H[h].kind != SFG_H_LAUNCH) continue;
    const sfg_kernel& K = P.kernels[H[h].kernel];
    uint32_t t[4][SFG_MAX_REGS] = {};
    int nr = 0, nf = 0, na = 0;
    for (int q = 0; q < K.n_params && q < 32; ++q) {
      if (K.ptype[q] == 0) t[SFG_CLS_R][nr++] |= 1u << q;
      else if (K.ptype[q] == 1) t[SFG_CLS_F][nf++] |= 1u << q;
      else t[SFG_CLS_A][na++] |= 1u << q;
    }
    uint32_t ctrl = 0;
    for (bool changed = true; changed;) {
      changed = false;
      auto flow = [&](int cls, int r, uint32_t m) {
        if (r < SFG_MAX_REGS && (t[cls][r] | m) != t[cls][r]) { t[cls][r] |= m; changed = true; }
      };
      for (int i = 0; i < K.n_ins; ++i) {
        const sfg_ins& x = ins[K.ins_base + i];
        const bool i1 = x.flags & SFG_F_S1_IMM, i2 = x.flags & SFG_F_S2_IMM;
        auto src = [&](int cls, int r, bool imm) { return imm || r >= SFG_MAX_REGS ? 0u : t[cls][r]; };
        switch (x.op) {
          case SFG_MOV: flow(x.mode, x.dst, src(x.mode, x.s1, i1)); break;
          case SFG_ADD: case SFG_SUB: case SFG_MUL:
            if (x.mode == SFG_CLS_A) flow(SFG_CLS_A, x.dst, src(SFG_CLS_A, x.s1, false) | src(SFG_CLS_R, x.s2, i2));
            else flow(SFG_CLS_R, x.dst, src(SFG_CLS_R, x.s1, i1) | src(SFG_CLS_R, x.s2, i2));
            break;
          case SFG_FADD: case SFG_FSUB: case SFG_FMUL:
            flow(SFG_CLS_F, x.dst, src(SFG_CLS_F, x.s1, i1) | src(SFG_CLS_F, x.s2, i2));
            break;
          case SFG_SETP: {
            const int c = (x.flags & SFG_F_FLOAT) ? SFG_CLS_F : SFG_CLS_R;
            const uint32_t m = src(c, x.s1, i1) | src(c, x.s2, i2);
            if ((ctrl | m) != ctrl) { ctrl |= m; changed = true; }
            flow(SFG_CLS_P, x.dst, m);
            break;
          }
          case SFG_LD: case SFG_ST: {
            // the sanitizer's verdict on the address is a control decision too (a
            // finding stops the thread): whatever reaches an address steers control
            const uint32_t am = src(SFG_CLS_A, x.s1, false);
            if ((ctrl | am) != ctrl) { ctrl |= am; changed = true; }
            if (x.op == SFG_LD) {
              const int c = x.mode == SFG_MK_F32 ? SFG_CLS_F : x.mode == SFG_MK_B64 ? SFG_CLS_A : SFG_CLS_R;
              flow(c, x.dst, am);
            }
            break;
          }
          case SFG_CVT:
            if (x.mode == SFG_CVT_F_FROM_I) flow(SFG_CLS_F, x.dst, src(SFG_CLS_R, x.s1, i1));
            else flow(SFG_CLS_R, x.dst, src(SFG_CLS_F, x.s1, i1));
            break;
          default: break;
        }
      }
    }
    for (int q = 0; q < H[h].n_bind && q < 32; ++q) {
      const sfg_binding& b = B[H[h].bind_base + q];
      if (((ctrl >> q) & 1u) && b.form == SFG_B_ARG && b.idx < 32) args |= 1u << b.idx;
    }
  }
  return args;
}

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

// shared memory of the group-parallel execute kernels: per group a GroupSmem header,
// one conflict tag and one snapshot word per 4 bytes of work region (exec_core.cuh)
constexpr int kExecSmemMax = 96 * 1024;
constexpr int kBulkSmem = 64 * 1024;   // per 128-thread CTA
constexpr int kTailSmem = 16 * 1024;   // per one-warp CTA (up to 4 inputs per warp)

static inline int tag_words(int64_t max_work_bytes) { return (int)((max_work_bytes + 3) / 4); }
static inline CorpusView CV(const sfg_corpus_dev* c) {
  return CorpusView{(const sfg_entry*)c->meta, (const sfg_val*)c->vals, (const uint8_t*)c->data, c->n, c->n_seeds};
}

// Program tables (a few KB each) come from a process-wide free list rather than
// cudaMalloc / cudaFree per program: cudaFree synchronizes the device and, next to a
// caching allocator holding tens of GB, took 0.1-0.4 s at random when a campaign's
// program was destroyed (measured around fuzz_loop calls).
static std::mutex g_tab_mu;
static std::multimap<std::pair<int, size_t>, void*> g_tab_free;   // (device, bytes) -> block

static cudaError_t table_alloc(void** dst, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_tab_mu);
    auto it = g_tab_free.find({dev, bytes});
    if (it != g_tab_free.end()) {
      *dst = it->second;
      g_tab_free.erase(it);
      return cudaSuccess;
    }
  }
  return cudaMalloc(dst, bytes);
}

static void table_free(void* ptr, size_t bytes) {
  if (!ptr) return;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_tab_mu);
  g_tab_free.insert({{dev, bytes}, ptr});
}

template <typename T>
static cudaError_t dupe(T** dst, const void* src, size_t count) {
  *dst = nullptr;
  if (count == 0) return cudaSuccess;
  cudaError_t e = table_alloc((void**)dst, count * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
}

// generic interpreter: instructions + per warp register files and edge counters
static size_t exec_smem(const sfg_prog& P, int warps) {
  int maxregs = 1;
  for (int k = 0; k < P.n_kernels; ++k) maxregs = P.kernels[k].regs > maxregs ? P.kernels[k].regs : maxregs;
  const size_t ins = ((size_t)P.total_ins * sizeof(sfg_ins) + 15) & ~(size_t)15;
  return ins + (size_t)warps * 32 * (maxregs * 24 + P.n_edges * 4);
}
constexpr int kGenSmemMax = 227 * 1024;

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
  p->ins = nullptr; p->hostops = nullptr; p->binds = nullptr; p->recs = nullptr; p->const_blob = nullptr;
  p->tab_bytes[0] = n_ins * sizeof(sfg_ins);
  p->tab_bytes[1] = n_hostops * sizeof(sfg_hostop);
  p->tab_bytes[2] = n_binds * sizeof(sfg_binding);
  p->tab_bytes[3] = n_recs * sizeof(sfg_rec);
  p->tab_bytes[4] = const_bytes;
  if ((e = dupe(&p->ins, ins, n_ins)) != cudaSuccess ||
      (e = dupe(&p->hostops, hostops, n_hostops)) != cudaSuccess ||
      (e = dupe(&p->binds, binds, n_binds)) != cudaSuccess ||
      (e = dupe(&p->recs, base_recs, n_recs)) != cudaSuccess ||
      (e = dupe(&p->const_blob, const_blob, const_bytes)) != cudaSuccess) {
    sfg_program_destroy(p);
    return fail("sfg_program_create", e);
  }
  p->base_blob = (const uint8_t*)base_blob_dev;
  // warps per block of the generic interpreter: as many (<= 4) as fit in shared memory
  p->gen_warps = 4;
  while (p->gen_warps > 1 && exec_smem(p->P, p->gen_warps) > (size_t)kGenSmemMax) --p->gen_warps;
  p->smem = exec_smem(p->P, p->gen_warps);
  const char* jit_env = getenv("SFG_JIT");
  if (!(jit_env && jit_env[0] == '0') && !p->P.jit_off) {
    // bound on per-input edge events decides whether counters need overflow checks
    uint64_t events = 0;
    const sfg_hostop* H = (const sfg_hostop*)hostops;
    for (size_t h = 0; h < n_hostops; ++h)
      if (H[h].kind == SFG_H_LAUNCH) {
        const double ev = (double)H[h].grid * (double)H[h].block * (double)p->P.budget;
        events = (ev + (double)events >= 1.8e19) ? ~0ull : events + (uint64_t)ev;
      }
    // kernels after whose every launch memory is dead: no later launch in COMPUTE and
    // no readouts (the readout copy_outs only run with diff_readback)
    uint32_t dead = 0, alive = 0;
    {
      int last = -1;
      for (size_t h = 0; h < n_hostops; ++h)
        if (H[h].kind == SFG_H_LAUNCH) last = (int)h;
      for (size_t h = 0; h < n_hostops; ++h) {
        if (H[h].kind != SFG_H_LAUNCH) continue;
        if ((int)h == last && !p->P.diff_readback) dead |= 1u << H[h].kernel;
        else alive |= 1u << H[h].kernel;
      }
      dead &= ~alive;
    }
    // the lane's allocator tables at this harness's static bounds (checked against the
    // ceilings at load time, lowering.py): INIT records + one record per array
    // argument (materialized once) and per COMPUTE alloc; the baseline quarantine /
    // free list + one entry per COMPUTE free
    sfgjit::LaneCaps caps;
    {
      int n_ptr = 0, n_alloc = 0, n_free_ops = 0;
      for (int a = 0; a < p->P.n_args; ++a) n_ptr += p->P.arg_kind[a] == SFG_V_ARR;
      for (size_t h = 0; h < n_hostops; ++h) {
        n_alloc += H[h].kind == SFG_H_ALLOC;
        n_free_ops += H[h].kind == SFG_H_FREE;
      }
      auto clampc = [](int v, int hi) { return v < 1 ? 1 : (v > hi ? hi : v); };
      caps.recs = clampc(p->P.n_base_recs + n_ptr + n_alloc, SFG_MAX_LANE_RECS);
      caps.q = clampc(p->P.n_quar + n_free_ops, 32);
      caps.freel = clampc(p->P.n_free + p->P.n_quar + n_free_ops, 32);
      caps.named = clampc(p->P.n_named, SFG_MAX_NAMED);
      caps.args = clampc(p->P.n_args, SFG_MAX_ARGS);
      int np = 1;
      for (int k = 0; k < p->P.n_kernels; ++k) np = p->P.kernels[k].n_params > np ? p->P.kernels[k].n_params : np;
      caps.params = clampc(np, SFG_MAX_ARGS);
    }
    const int rc = sfg_jit_build(p->P, (const sfg_ins*)ins, events, dead, caps, H, n_hostops,
                                 (const sfg_binding*)binds, p->jit_source, p->jit_log, &p->jit_lib,
                                 &p->jit_kernel, &p->jit_tail);
    if (rc != 0) {
      g_err = "sfg_program_create: JIT build failed (" + std::to_string(rc) + "): " + p->jit_log.substr(0, 6000);
      sfg_program_destroy(p);
      return 1;
    }
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // CTA size of the bulk pass: a multiple of 32 within the kernel's launch bounds (128)
    if (const char* b = getenv("SFG_EXEC_BLOCK")) {
      const int v = atoi(b);
      p->jit_block = (v >= 32 && v <= 128 && v % 32 == 0) ? v : 128;
    }
    if (const char* md = getenv("SFG_EXEC_MODE")) p->jit_mode = atoi(md);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)p->jit_kernel, p->jit_block, 0);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    p->jit_grid = sms * per_sm;
    p->sms = sms;
    // group size: the most simulated threads of any COMPUTE launch, rounded up to a
    // power of two, at most a warp (SFG_GROUP overrides; 1 = thread-sequential)
    int maxt = 1;
    for (size_t h = 0; h < n_hostops; ++h)
      if (H[h].kind == SFG_H_LAUNCH && (int64_t)H[h].grid * H[h].block > maxt)
        maxt = (int64_t)H[h].grid * H[h].block > 32 ? 32 : (int)(H[h].grid * H[h].block);
    p->group = 1;
    while (p->group < maxt) p->group <<= 1;
    if (const char* gs = getenv("SFG_GROUP")) {
      const int v = atoi(gs);
      if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32) p->group = v;
    }
    // the bulk pass stays thread-sequential by default: 32 short inputs per warp cost
    // less lane work than one input per group (the per-input setup is per lane);
    // group-parallel pays off for the few long inputs, whose latency bounds a round
    p->bulk_group = 1;
    if (const char* bg = getenv("SFG_BULK_GROUP")) {
      const int v = atoi(bg);
      if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16 || v == 32) p->bulk_group = v < p->group ? v : p->group;
    }
    cudaFuncSetAttribute((const void*)p->jit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kExecSmemMax);
    cudaFuncSetAttribute((const void*)p->jit_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, kExecSmemMax);
    // Reserve the per-thread local memory (stack frame: the per-input allocation
    // table) of both kernels once.  Otherwise the driver grows the device's local
    // memory pool for one kernel and may shrink it for the next, and every such
    // resize synchronizes the device -- which serializes the pipelined rounds.
    {
      size_t need = 0, cur = 0;
      cudaFuncAttributes fa;
      for (cudaKernel_t k : {p->jit_kernel, p->jit_tail})
        if (cudaFuncGetAttributes(&fa, (const void*)k) == cudaSuccess && fa.localSizeBytes > need) need = fa.localSizeBytes;
      need = (need + 1023) & ~(size_t)1023;
      if (cudaDeviceGetLimit(&cur, cudaLimitStackSize) == cudaSuccess && need > cur)
        cudaDeviceSetLimit(cudaLimitStackSize, need);
    }
    if (const char* bp = getenv("SFG_BULK_PERSIST")) p->bulk_persist = atoi(bp) != 0;
    p->order_mask = control_arg_mask(p->P, (const sfg_ins*)ins, H, n_hostops, (const sfg_binding*)binds);
    if (const char* om = getenv("SFG_ORDER_ALL")) if (atoi(om)) p->order_mask = ~0u;
    if (const char* tc = getenv("SFG_TAIL_CTAS")) p->tail_ctas = atoi(tc) >= 1 ? atoi(tc) : 512;
    if (const char* tq = getenv("SFG_TAIL_KSEQ")) p->tail_k_seq = atoi(tq) >= 1 && atoi(tq) <= 32 ? atoi(tq) : 32;
    if (const char* tk = getenv("SFG_TAIL_K")) p->tail_k = atoi(tk) >= 1 && atoi(tk) <= 32 ? atoi(tk) : 4;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)p->jit_tail, 32, kTailSmem);
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    p->tail_grid = sms * per_sm;

  }
  // the generic interpreter (trace mode, one-input INIT/TERM programs) needs its
  // register files in shared memory; with the JIT a program too large for it still
  // runs (sfg_execute_trace then fails)
  e = p->smem <= (size_t)kGenSmemMax
          ? cudaFuncSetAttribute(sfg_execute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->smem)
          : cudaErrorInvalidValue;
  p->gen_ok = e == cudaSuccess;
  if (!p->gen_ok && !p->jit_kernel) {
    sfg_program_destroy(p);
    g_err = "sfg_program_create: the program's registers / edges exceed the interpreter's shared memory";
    return 1;
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
  // p->jit_lib stays loaded: it is shared by every program with the same generated
  // source in this process (jit.cu sfg_jit_build)
  table_free(p->ins, p->tab_bytes[0]);
  table_free(p->hostops, p->tab_bytes[1]);
  table_free(p->binds, p->tab_bytes[2]);
  table_free(p->recs, p->tab_bytes[3]);
  table_free(p->const_blob, p->tab_bytes[4]);
  delete p;
}

size_t sfg_execute_smem_bytes(const sfg_program* p) { return p->smem; }

void sfg_jit_stats(int* compiles, int* disk_hits) {
  if (compiles) *compiles = jit_compiles;
  if (disk_hits) *disk_hits = jit_disk_hits;
}

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
  const int rc = sfg_jit_compile(P, (const sfg_ins*)ins, max_edge_events, 0u, sfgjit::LaneCaps{}, nullptr, 0, nullptr,
                                 src, log, cubin);
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

size_t sfg_stream_state_bytes(void) { return sizeof(SfgStream); }

int sfg_stream_state_init(uint64_t seed, uint64_t stream_id, void* out_host) {
  SfgStream st;
  memset(&st, 0, sizeof st);
  st.ctr[0] = st.ctr[1] = st.ctr[2] = st.ctr[3] = 0;
  st.key0 = seed;
  st.key1 = stream_id;
  st.pos = 4;
  memcpy(out_host, &st, sizeof st);
  return 0;
}

int sfg_plan_seq(const sfg_program* p, const sfg_corpus_dev* c, int64_t it0, int n, const void* state,
                 const uint64_t* counts_base, void* children, void* vals, uint32_t* int_flags, void* states,
                 void* stream) {
  if (n <= 0) return 0;
  sfg_plan_seq_kernel<<<1, 32, 0, S(stream)>>>(p->P, CV(c), it0, n, (const SfgStream*)state, counts_base,
                                                (sfg_child*)children, (sfg_val*)vals, int_flags, (SfgStream*)states);
  SFG_CHECK_LAUNCH("sfg_plan_seq");
  return 0;
}

static int seq_levels(int n) {
  int k = 1;
  while ((1ll << k) <= (int64_t)n) ++k;
  return k;
}

int64_t sfg_seq_scratch_ints(int n, int64_t words) {
  if (n <= 0 || words <= 0) return 0;
  return (int64_t)seq_levels(n) * 2 * words + (n + 1) + 4;
}

int sfg_plan_seq_par(const sfg_program* p, const sfg_corpus_dev* c, int64_t it0, int n, const void* state,
                     int64_t words, const uint64_t* counts_base, void* children, void* vals, uint32_t* int_flags,
                     void* states, int32_t* scratch, int64_t scratch_ints, uint64_t* stats, void* stream) {
  if (n <= 0) return 0;
  if (it0 < 2 || words <= 0 || 2 * words >= (int64_t)0x7FFFFFFF || scratch_ints < sfg_seq_scratch_ints(n, words)) {
    g_err = "sfg_plan_seq_par: bad arguments (it0 >= 2, 0 < 2*words < 2^31, scratch of sfg_seq_scratch_ints)";
    return 1;
  }
  const int K = seq_levels(n);
  const int64_t M = 2 * words;
  int32_t* J = scratch;                       // K levels of M successors
  int32_t* path = scratch + (int64_t)K * M;   // n + 1
  int32_t* q0 = path + n + 1;
  cudaStream_t st = S(stream);
  const SfgStream* start = (const SfgStream*)state;
  unsigned long long* stt = (unsigned long long*)stats;
  sfg_seq_root_kernel<<<1, 32, 0, st>>>(p->P, CV(c), it0, n, start, words, counts_base, (sfg_child*)children,
                                        (sfg_val*)vals, int_flags, (SfgStream*)states, path, q0, stt);
  sfg_seq_walk_kernel<<<blocks_for(M, 128), 128, 0, st>>>(p->P, CV(c), it0, start, words, J);
  const int jb = (int)std::min<int64_t>(blocks_for(M, 256), (int64_t)(p->sms > 0 ? p->sms : 148) * 8);
  for (int k = 0; k + 1 < K; ++k)
    sfg_seq_jump_kernel<<<jb, 256, 0, st>>>(J + (int64_t)k * M, J + (int64_t)(k + 1) * M, M);
  for (int k = K - 1; k >= 0; --k) {
    const int64_t step = 1ll << k;
    const int64_t threads = ((int64_t)n + 2 * step) / (2 * step);
    sfg_seq_path_kernel<<<blocks_for(threads, 128), 128, 0, st>>>(J + (int64_t)k * M, path, q0, n, step);
  }
  sfg_seq_mutate_kernel<<<blocks_for(n, 128), 128, 0, st>>>(p->P, CV(c), it0, n, start, path, q0, counts_base,
                                                            (sfg_child*)children, (sfg_val*)vals, int_flags,
                                                            (SfgStream*)states, stt);
  SFG_CHECK_LAUNCH("sfg_plan_seq_par");
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
  sfg_apply_kernel<<<blocks_for((int64_t)n * kApplyLanes, 256), 256, 0, S(stream)>>>(
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

int sfg_stream_create(int priority, void** out) {
  cudaStream_t s = nullptr;
  const cudaError_t e = cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority);
  if (e != cudaSuccess) return fail("sfg_stream_create", e);
  *out = (void*)s;
  return 0;
}

int sfg_program_group(const sfg_program* p) { return p->jit_kernel ? p->group : 1; }

uint32_t sfg_program_order_mask(const sfg_program* p) { return p->order_mask; }

uint32_t sfg_control_mask(const void* prog, size_t prog_bytes, const void* ins, const void* hostops,
                          size_t n_hostops, const void* binds) {
  if (prog_bytes != sizeof(sfg_prog)) return ~0u;
  sfg_prog P;
  memcpy(&P, prog, sizeof P);
  return control_arg_mask(P, (const sfg_ins*)ins, (const sfg_hostop*)hostops, n_hostops,
                          (const sfg_binding*)binds);
}

size_t sfg_order_scratch_ints(int n) { return (size_t)kOrderBuckets + (size_t)(n > 0 ? n : 0); }

int sfg_order(const sfg_program* p, int n, const void* vals, int32_t* order, int32_t* scratch, const int32_t* rep,
              int32_t* n_live, void* stream) {
  if (n <= 0) return 0;
  int* hist = scratch;
  int* sig = scratch + kOrderBuckets;
  cudaError_t e = cudaMemsetAsync(hist, 0, kOrderBuckets * sizeof(int), S(stream));
  if (e != cudaSuccess) return fail("sfg_order", e);
  sfg_order_hist_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(p->P, (const sfg_val*)vals, n, p->order_mask,
                                                                  hist, sig, rep);
  sfg_order_scan_kernel<<<1, 128, 0, S(stream)>>>(hist, n_live);
  sfg_order_scatter_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(n, sig, hist, order, rep);
  SFG_CHECK_LAUNCH("sfg_order");
  return 0;
}

int sfg_dedupe(const sfg_program* p, int n, const void* children, const void* vals, uint64_t* table, int slots,
               int32_t* rep, void* stream) {
  if (n <= 0) return 0;
  if (slots < 2 * n || (slots & (slots - 1))) {
    g_err = "sfg_dedupe: slots must be a power of two >= 2n";
    return 1;
  }
  cudaError_t e = cudaMemsetAsync(table, 0, (size_t)slots * sizeof(uint64_t), S(stream));
  if (e != cudaSuccess) return fail("sfg_dedupe", e);
  sfg_dedupe_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(p->P, n, (const sfg_child*)children,
                                                              (const sfg_val*)vals, (unsigned long long*)table, slots,
                                                              rep);
  SFG_CHECK_LAUNCH("sfg_dedupe");
  return 0;
}

int sfg_group_schedule(const sfg_program* p, int n, const int32_t* rep, const int32_t* order, const int32_t* n_live,
                       int32_t* full, int32_t* scratch, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t st = S(stream);
  int32_t* cnt = scratch;               // n
  int32_t* fill = scratch + n;          // n
  int32_t* rpos = scratch + 2 * (int64_t)n;
  int64_t* w = (int64_t*)(scratch + (3 * (int64_t)n + 1) / 2 * 2);      // n int64 (8-aligned)
  int64_t* start = w + n;               // n int64
  int64_t* tmp = start + n;             // scan tiles
  cudaError_t e = cudaMemsetAsync(cnt, 0, 2 * (size_t)n * sizeof(int32_t), st);
  if (e != cudaSuccess) return fail("sfg_group_schedule", e);
  sfg_dup_count_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, rep, cnt);
  sfg_group_weights_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, order, n_live, cnt, w);
  const int rc = sfg_scan_u64((const uint64_t*)w, n, 1, 0, (uint64_t*)start, 1, 0, (uint64_t*)tmp,
                              (uint64_t*)(tmp + ((n + 2047) / 2048 + 8)), st);
  if (rc) return rc;
  sfg_group_place_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, order, n_live, start, full, rpos);
  sfg_group_dups_kernel<<<blocks_for(n, 256), 256, 0, st>>>(n, rep, rpos, fill, full);
  SFG_CHECK_LAUNCH("sfg_group_schedule");
  return 0;
}

size_t sfg_group_scratch_ints(int n) {
  const size_t m = (size_t)(n > 0 ? n : 0);
  return 3 * m + 2 + 4 * m + 2 * ((m + 2047) / 2048 + 16);
}

int sfg_dup_fill(const sfg_program* p, int n, const int32_t* rep, void* verdicts, uint32_t* edge_counts,
                 void* stream) {
  if (n <= 0) return 0;
  sfg_dup_fill_kernel<<<blocks_for(n, 256), 256, 0, S(stream)>>>(n, p->P.n_edges, rep, (sfg_verdict*)verdicts,
                                                                edge_counts);
  SFG_CHECK_LAUNCH("sfg_dup_fill");
  return 0;
}


int sfg_execute(const sfg_program* p, const sfg_corpus_dev* c, int n, const void* children, const void* vals,
                const uint64_t* work_base, uint8_t* work, void* verdicts, uint32_t* edge_counts, uint8_t* readouts,
                const uint64_t* readout_base, int* work_counter, uint64_t soft_cap,
                int32_t* deferred, int64_t max_work_bytes, const int32_t* order, const int32_t* n_live,
                void* stream) {
  if (n <= 0) {
    if (work_counter) cudaMemsetAsync(work_counter, 0, 8 * sizeof(int), S(stream));
    return 0;
  }
  ExecView E{p->ins, p->hostops, p->binds, p->recs, p->base_blob, p->const_blob,
             (const sfg_child*)children, (const sfg_val*)vals, work_base, work,
             (sfg_verdict*)verdicts, edge_counts, readouts, readout_base, n,
             0ull, deferred, work_counter ? work_counter + 1 : nullptr,
             deferred ? deferred + n : nullptr, work_counter ? work_counter + 3 : nullptr, 1, 0, order,
             nullptr, 0, nullptr, c ? (const sfg_val*)c->vals : nullptr, c ? (const uint8_t*)c->data : nullptr,
             order ? n_live : nullptr};
  if (n_live && !order) {
    g_err = "sfg_execute: n_live needs the schedule (order) it counts";
    return 1;
  }
  if (p->jit_kernel) {
    if (work_counter == nullptr || (deferred == nullptr && soft_cap != 0)) {
      g_err = "sfg_execute: the specialized kernel needs a per-launch work counter (and deferred lists for soft_cap)";
      return 1;
    }
    E.soft_cap = soft_cap;
    E.group = deferred ? p->bulk_group : 1;  // no lists: nothing can be re-run, so thread-sequential
    size_t smem = 0;
    if (E.group > 1) {
      // tag capacity: the round's largest work region, within the CTA's smem budget
      const int groups = (p->jit_block / 32) * (32 / E.group);
      int cap = tag_words(max_work_bytes);
      const int fit = (int)((kBulkSmem / groups - sizeof(GroupSmem)) / 8) & ~3;
      E.tag_cap = cap < fit ? cap : fit;
      smem = (size_t)groups * group_stride(E.tag_cap);
    }
    cudaError_t e = cudaMemsetAsync(work_counter, 0, 8 * sizeof(int), S(stream));
    if (e != cudaSuccess) return fail("sfg_execute (jit counter)", e);
    int* next = work_counter;
    int mode = p->jit_mode;
    void* args[] = {(void*)&p->P, (void*)&E, (void*)&next, (void*)&mode};
    const int per_cta = E.group > 1 ? (p->jit_block / 32) * (32 / E.group) : p->jit_block;
    const unsigned want = blocks_for(n, per_cta);
    int resident = p->jit_grid;
    if (smem) {
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)p->jit_kernel, p->jit_block, smem) ==
              cudaSuccess && per_sm > 0)
        resident = p->sms * per_sm;
    }
    // persistent (one resident wave) or one CTA per batch: the latter frees SM slots
    // CTA by CTA, so other rounds' long-input warps are not locked out for a whole pass
    const unsigned grid = (!p->bulk_persist || want < (unsigned)resident) ? want : (unsigned)resident;
    e = cudaLaunchKernel((const void*)p->jit_kernel, dim3(grid), dim3(p->jit_block), args, smem, S(stream));
    if (e != cudaSuccess) return fail("sfg_execute (jit)", e);
    return 0;
  }
  if (work_counter) cudaMemsetAsync(work_counter, 0, 8 * sizeof(int), S(stream));
  if (!p->gen_ok) {
    g_err = "the program's registers / edges exceed the generic interpreter's shared memory";
    return 1;
  }
  sfg_execute_kernel<<<blocks_for(n, 32 * p->gen_warps), 32 * p->gen_warps, p->smem, S(stream)>>>(p->P, E);
  SFG_CHECK_LAUNCH("sfg_execute");
  return 0;
}

int sfg_execute_trace(const sfg_program* p, int n, const void* children, const void* vals, const uint64_t* work_base,
                      uint8_t* work, void* verdicts, uint32_t* edge_counts, uint8_t* readouts,
                      const uint64_t* readout_base, uint64_t* trace, uint32_t trace_cap,
                      uint32_t* trace_count, void* stream) {
  if (n <= 0) return 0;
  ExecView E{p->ins, p->hostops, p->binds, p->recs, p->base_blob, p->const_blob,
             (const sfg_child*)children, (const sfg_val*)vals, work_base, work,
             (sfg_verdict*)verdicts, edge_counts, readouts, readout_base, n,
             0ull, nullptr, nullptr, nullptr, nullptr, 1, 0, nullptr, trace, trace_cap, trace_count, nullptr, nullptr};
  if (!p->gen_ok) {
    g_err = "the program's registers / edges exceed the generic interpreter's shared memory";
    return 1;
  }
  sfg_execute_kernel<<<blocks_for(n, 32 * p->gen_warps), 32 * p->gen_warps, p->smem, S(stream)>>>(p->P, E);
  SFG_CHECK_LAUNCH("sfg_execute_trace");
  return 0;
}

int sfg_execute_deferred(const sfg_program* p, const sfg_corpus_dev* c, int n, const void* children,
                         const void* vals, const uint64_t* work_base, uint8_t* work, void* verdicts,
                         uint32_t* edge_counts, uint8_t* readouts, const uint64_t* readout_base,
                         int* work_counter, int32_t* deferred, int64_t max_work_bytes, void* stream) {
  if (n <= 0 || !p->jit_kernel) return 0;  // the interpreter never defers
  ExecView E{p->ins, p->hostops, p->binds, p->recs, p->base_blob, p->const_blob,
             (const sfg_child*)children, (const sfg_val*)vals, work_base, work,
             (sfg_verdict*)verdicts, edge_counts, readouts, readout_base, n,
             0ull, deferred, work_counter + 1, deferred + n, work_counter + 3, p->group, 0, nullptr,
             nullptr, 0, nullptr, nullptr, nullptr};
  for (int pass = 0; pass < 2; ++pass) {
    // pristine payloads again (the earlier attempt's stores landed in the work regions)
    int32_t* list = pass == 0 ? deferred : deferred + n;
    int* count = pass == 0 ? work_counter + 1 : work_counter + 3;
    sfg_apply_kernel<<<p->jit_grid, 256, 0, S(stream)>>>(p->P, CV(c), n, (const sfg_child*)children,
                                                        (const sfg_val*)vals, work_base, work, list, count);
    SFG_CHECK_LAUNCH("sfg_execute_deferred/apply");
    // pass 0: soft-cap list, group-parallel, one input per one-warp CTA (long inputs
    // spread over the SMs); pass 1: thread-sequential re-runs
    int* next = work_counter + (pass == 0 ? 2 : 4);
    int k = pass == 0 ? p->tail_k : p->tail_k_seq;
    int seq = pass;
    size_t smem = 0;
    E.tag_cap = 0;
    if (pass == 0 && p->group > 1) {
      const int per = k < 32 / p->group ? k : 32 / p->group;
      const int cap = tag_words(max_work_bytes);
      const int fit = (int)((kTailSmem / per - sizeof(GroupSmem)) / 8) & ~3;
      E.tag_cap = cap < fit ? cap : fit;
      smem = (size_t)per * group_stride(E.tag_cap);
    }
    void* args[] = {(void*)&p->P, (void*)&E, (void*)&next, (void*)&k, (void*)&seq};
    // persistent one-warp CTAs sized for the usual load (a few hundred long inputs per
    // round, far fewer re-runs): a kernel completes only once every CTA has had a slot,
    // and slots are scarce while other rounds run, so idle CTAs would add latency
    const int want = pass == 0 ? p->tail_ctas : p->tail_ctas / 4 + 1;
    const unsigned grid = (unsigned)(want < p->tail_grid ? want : p->tail_grid);
    cudaError_t e = cudaLaunchKernel((const void*)p->jit_tail, dim3(grid), dim3(32), args, smem, S(stream));
    if (e != cudaSuccess) return fail("sfg_execute_deferred (jit)", e);
  }
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
