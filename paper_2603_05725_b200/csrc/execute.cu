// K3 (generic path): the SIR interpreter runner for exec_core's host-op driver.
//
// Simulated register files live in shared memory, [reg][lane], so a converged
// warp touches 32 consecutive banks; per-edge hit counters likewise [edge][lane].
// Instruction semantics follow executor.py:210-377 (see exec_core.cuh).
#include "exec_core.cuh"

namespace {

struct InterpRunner {
  const sfg_ins* s_ins;
  uint64_t* s_alo;
  uint32_t *s_r, *s_f;
  int32_t *s_ahi, *s_ap;
  uint32_t* s_ecnt;
  int lane, n_edges;
  bool overflow;

  SFG_DEV void begin_input() {
    overflow = false;
    for (int e = 0; e < n_edges; ++e) s_ecnt[e * 32 + lane] = 0;
  }

  // trace mode: event words of the current input (executor.py:122-135)
  //   w0: kind (0 mem, 1 cf) | store << 2 | width << 3 | space << 8 | kernel << 16 | iid or edge << 32
  //   w1: ctaid | tid << 32;  w2, w3: address low / high (mem)
  uint64_t* tr = nullptr;
  uint32_t tr_cap = 0, tr_n = 0;
  int cur_kernel = 0, cur_ctaid = 0, cur_tid = 0;

  SFG_DEV void set_input(const ExecView& E, int i) {
    tr = E.trace ? E.trace + (size_t)i * E.trace_cap * 4 : nullptr;
    tr_cap = E.trace_cap;
    tr_n = 0;
  }
  SFG_DEV void end_input(const ExecView& E, int i) {
    if (tr) E.trace_count[i] = tr_n;
  }
  SFG_DEV void ev(uint64_t w0, uint64_t w2, uint64_t w3) {
    if (tr_n < tr_cap) {
      uint64_t* p = tr + (size_t)tr_n * 4;
      p[0] = w0;
      p[1] = (uint64_t)(uint32_t)cur_ctaid | ((uint64_t)(uint32_t)cur_tid << 32);
      p[2] = w2;
      p[3] = w3;
    }
    ++tr_n;
  }

  SFG_DEV void hit(int e) {
    uint32_t* p = s_ecnt + e * 32 + lane;
    if (*p == 0xFFFFFFFFu) overflow = true; else ++*p;
    if (tr) ev(1ull | ((uint64_t)(uint32_t)cur_kernel << 16) | ((uint64_t)(uint32_t)e << 32), 0, 0);
  }

  SFG_DEV void flush(uint32_t* erow, bool& ovf) {
    for (int e = 0; e < n_edges; ++e) erow[e] = s_ecnt[e * 32 + lane];
    ovf = overflow;
  }

  template <bool PAR>
  SFG_DEV int run_thread(const sfg_prog& P, int kidx, Lane& L, Mem& M, sfg_verdict& V, const Pre& pre, int ctaid,
                         int tid, int grid, int block, uint64_t& total_retired) {
    const sfg_kernel& K = P.kernels[kidx];
    const sfg_ins* kins = s_ins + K.ins_base;
    const int regs = K.regs;
    for (int q = 0; q < regs; ++q) {  // make_thread (executor.py:191-202)
      s_r[q * 32 + lane] = q < pre.nr ? pre.r[q] : 0u;
      s_f[q * 32 + lane] = q < pre.nf ? pre.f[q] : 0u;
      s_alo[q * 32 + lane] = q < pre.na ? (uint64_t)pre.a[q] : 0ull;
      s_ahi[q * 32 + lane] = q < pre.na ? (pre.a[q] < 0 ? -1 : 0) : 0;
      s_ap[q * 32 + lane] = q < pre.na ? pre.ap[q] : 0;
    }
    uint32_t preds = 0;
    int pc = 0;
    uint64_t retired = 0;
    cur_kernel = kidx;
    cur_ctaid = ctaid;
    cur_tid = tid;
    int rc = RUN_EXIT;
    while (true) {
      const sfg_ins I = kins[pc];
      ++retired;
      if (I.op == SFG_EXIT) break;
      if (I.op == SFG_BRA) {
        bool taken = true;
        if (I.flags & SFG_F_PRED) taken = (((preds >> I.s1) & 1u) != 0) != ((I.flags & SFG_F_PNEG) != 0);
        hit(taken ? I.edge_tk : I.edge_ft);
        pc = taken ? I.target : pc + 1;
        if (retired >= P.budget) { rc = RUN_BUDGET; break; }
        continue;
      }
      switch (I.op) {
        case SFG_LD:
        case SFG_ST: {
          const i128 areg = ((i128)s_ahi[I.s1 * 32 + lane] << 64) | (i128)s_alo[I.s1 * 32 + lane];
          const i128 a = areg + (i128)I.imm2;
          const int prov = s_ap[I.s1 * 32 + lane];
          const bool st = I.op == SFG_ST;
          if (tr)  // on_mem_access precedes the sanitizer check (executor.py:244-247)
            ev((uint64_t)(st ? 4 : 0) | ((uint64_t)I.width << 3) | ((uint64_t)I.space << 8) |
                   ((uint64_t)(uint32_t)kidx << 16) | ((uint64_t)(uint32_t)pc << 32),
               (uint64_t)a, (uint64_t)(a >> 64));
          Report rep;
          int rh = -1;
          if (check_access(P, L, a, I.width, I.space, prov, rep, rh)) {
            fill_report(V, P, L, rep, kidx, pc, ctaid, tid, a, I.width, st, I.space, prov);
            rc = RUN_FINDING;
            break;
          }
          const LRec& r = L.rec[rh];
          const int64_t aa = (int64_t)a;
          if (st) {
            uint64_t val;
            if (I.mode == SFG_MK_F32) val = (I.flags & SFG_F_S2_IMM) ? (uint64_t)(uint32_t)I.imm1 : s_f[I.s2 * 32 + lane];
            else if (I.mode == SFG_MK_B64) val = s_alo[I.s2 * 32 + lane];
            else val = (I.flags & SFG_F_S2_IMM) ? (uint64_t)I.imm1 : (uint64_t)s_r[I.s2 * 32 + lane];
            if (!mem_write(M, L, r, aa, I.width, val)) { V.status = SFG_ST_OVERLAY; rc = RUN_FATAL; }
          } else {
            const uint64_t val = mem_read(M, L, r, aa, I.width);
            switch (I.mode) {
              case SFG_MK_F32: s_f[I.dst * 32 + lane] = sfg_quiet((uint32_t)val); break;
              case SFG_MK_B64:
                s_alo[I.dst * 32 + lane] = val;
                s_ahi[I.dst * 32 + lane] = 0;
                s_ap[I.dst * 32 + lane] = 0;
                break;
              default: s_r[I.dst * 32 + lane] = (uint32_t)val; break;  // b8/b16 zero-extend, b32 bits
            }
          }
          break;
        }
        case SFG_MOV:
          if (I.mode == SFG_CLS_R) {
            s_r[I.dst * 32 + lane] = (I.flags & SFG_F_S1_IMM) ? (uint32_t)I.imm1 : s_r[I.s1 * 32 + lane];
          } else if (I.mode == SFG_CLS_F) {
            s_f[I.dst * 32 + lane] = (I.flags & SFG_F_S1_IMM) ? (uint32_t)I.imm1 : s_f[I.s1 * 32 + lane];
          } else if (I.mode == SFG_CLS_A) {
            if (I.flags & SFG_F_S1_IMM) {
              s_alo[I.dst * 32 + lane] = (uint64_t)I.imm1;
              s_ahi[I.dst * 32 + lane] = (I.flags & SFG_F_U64IMM) ? 0 : (I.imm1 < 0 ? -1 : 0);
              s_ap[I.dst * 32 + lane] = 0;
            } else {
              s_alo[I.dst * 32 + lane] = s_alo[I.s1 * 32 + lane];
              s_ahi[I.dst * 32 + lane] = s_ahi[I.s1 * 32 + lane];
              s_ap[I.dst * 32 + lane] = s_ap[I.s1 * 32 + lane];
            }
          } else {
            preds = (preds & ~(1u << I.dst)) | (((preds >> I.s1) & 1u) << I.dst);
          }
          break;
        case SFG_ADD:
        case SFG_SUB:
        case SFG_MUL:
          if (I.mode == SFG_CLS_A) {
            const i128 base = ((i128)s_ahi[I.s1 * 32 + lane] << 64) | (i128)s_alo[I.s1 * 32 + lane];
            const int64_t d = (I.flags & SFG_F_S2_IMM) ? I.imm2 : (int64_t)(int32_t)s_r[I.s2 * 32 + lane];
            const i128 res = I.op == SFG_ADD ? base + (i128)d : base - (i128)d;
            s_alo[I.dst * 32 + lane] = (uint64_t)res;
            s_ahi[I.dst * 32 + lane] = (int32_t)(int64_t)(res >> 64);
            s_ap[I.dst * 32 + lane] = s_ap[I.s1 * 32 + lane];
          } else {
            const uint32_t x = (I.flags & SFG_F_S1_IMM) ? (uint32_t)I.imm1 : s_r[I.s1 * 32 + lane];
            const uint32_t y = (I.flags & SFG_F_S2_IMM) ? (uint32_t)I.imm2 : s_r[I.s2 * 32 + lane];
            s_r[I.dst * 32 + lane] = I.op == SFG_ADD ? x + y : (I.op == SFG_SUB ? x - y : x * y);
          }
          break;
        case SFG_FADD:
        case SFG_FSUB:
        case SFG_FMUL: {
          const uint32_t x = (I.flags & SFG_F_S1_IMM) ? (uint32_t)I.imm1 : s_f[I.s1 * 32 + lane];
          const uint32_t y = (I.flags & SFG_F_S2_IMM) ? (uint32_t)I.imm2 : s_f[I.s2 * 32 + lane];
          s_f[I.dst * 32 + lane] = sfg_fop(I.op, x, y);
          break;
        }
        case SFG_SETP: {
          bool res;
          if (I.flags & SFG_F_FLOAT) {
            const float x = sfg_f((I.flags & SFG_F_S1_IMM) ? (uint32_t)I.imm1 : s_f[I.s1 * 32 + lane]);
            const float y = sfg_f((I.flags & SFG_F_S2_IMM) ? (uint32_t)I.imm2 : s_f[I.s2 * 32 + lane]);
            switch (I.mode) {
              case SFG_CMP_EQ: res = x == y; break;
              case SFG_CMP_NE: res = x != y; break;
              case SFG_CMP_LT: res = x < y; break;
              case SFG_CMP_LE: res = x <= y; break;
              case SFG_CMP_GT: res = x > y; break;
              default: res = x >= y; break;
            }
          } else {
            const int64_t x = (I.flags & SFG_F_S1_IMM) ? I.imm1 : (int64_t)(int32_t)s_r[I.s1 * 32 + lane];
            const int64_t y = (I.flags & SFG_F_S2_IMM) ? I.imm2 : (int64_t)(int32_t)s_r[I.s2 * 32 + lane];
            switch (I.mode) {
              case SFG_CMP_EQ: res = x == y; break;
              case SFG_CMP_NE: res = x != y; break;
              case SFG_CMP_LT: res = x < y; break;
              case SFG_CMP_LE: res = x <= y; break;
              case SFG_CMP_GT: res = x > y; break;
              default: res = x >= y; break;
            }
          }
          preds = (preds & ~(1u << I.dst)) | ((uint32_t)res << I.dst);
          break;
        }
        case SFG_CVT:
          if (I.mode == SFG_CVT_F_FROM_I) {
            s_f[I.dst * 32 + lane] = (I.flags & SFG_F_S1_IMM)
                                         ? (uint32_t)I.imm1
                                         : sfg_b(__int2float_rn((int32_t)s_r[I.s1 * 32 + lane]));
          } else if (I.flags & SFG_F_S1_IMM) {
            s_r[I.dst * 32 + lane] = (uint32_t)I.imm1;
          } else {  // cvt_f32_to_i32 (executor.py:51-65)
            const uint32_t fb = s_f[I.s1 * 32 + lane];
            const float fv = sfg_f(fb);
            int32_t out;
            if (sfg_isnan_bits(fb)) out = 0;
            else if (fv >= 2147483647.0f) out = 2147483647;
            else if (fv <= -2147483648.0f) out = (int32_t)0x80000000u;
            else out = __float2int_rn(fv);
            s_r[I.dst * 32 + lane] = (uint32_t)out;
          }
          break;
        default: {  // SREG
          const int v = I.mode == SFG_SR_TID ? tid : I.mode == SFG_SR_NTID ? block
                      : I.mode == SFG_SR_CTAID ? ctaid : grid;
          s_r[I.dst * 32 + lane] = (uint32_t)v;
          break;
        }
      }
      if (rc != RUN_EXIT) break;
      if (I.edge_ft >= 0) hit(I.edge_ft);
      ++pc;
      if (retired >= P.budget) { rc = RUN_BUDGET; break; }
    }
    total_retired += retired;
    return rc;
  }
};

}  // namespace

extern "C" __global__ void __launch_bounds__(128) sfg_execute_kernel(sfg_prog P, ExecView E) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int nwb = blockDim.x >> 5;
  // instructions for every kernel of the program, then per-warp register files
  sfg_ins* s_ins = reinterpret_cast<sfg_ins*>(smem);
  for (int k = threadIdx.x; k < P.total_ins; k += blockDim.x) s_ins[k] = E.ins[k];
  int maxregs = 1;
  for (int k = 0; k < P.n_kernels; ++k) maxregs = P.kernels[k].regs > maxregs ? P.kernels[k].regs : maxregs;
  const size_t ins_bytes = ((size_t)P.total_ins * sizeof(sfg_ins) + 15) & ~(size_t)15;
  const size_t warp_bytes = (size_t)32 * (maxregs * 24 + P.n_edges * 4);
  uint8_t* wbase = smem + ins_bytes + (size_t)wib * warp_bytes;
  InterpRunner R;
  R.s_ins = s_ins;
  R.s_alo = reinterpret_cast<uint64_t*>(wbase);
  R.s_r = reinterpret_cast<uint32_t*>(wbase + (size_t)32 * maxregs * 8);
  R.s_f = R.s_r + 32 * maxregs;
  R.s_ahi = reinterpret_cast<int32_t*>(R.s_f + 32 * maxregs);
  R.s_ap = R.s_ahi + 32 * maxregs;
  R.s_ecnt = reinterpret_cast<uint32_t*>(R.s_ap + 32 * maxregs);
  R.lane = lane;
  R.n_edges = P.n_edges;
  __syncthreads();
  const int gw = blockIdx.x * nwb + wib;
  const int nw = gridDim.x * nwb;
  for (int base_i = gw * 32; base_i < E.n; base_i += nw * 32) {
    const int i = base_i + lane;
    if (i < E.n) run_input<false>(P, E, i, R, Grp{1, 0, 1u << lane, nullptr, nullptr, 0});
    __syncwarp();
  }
}
