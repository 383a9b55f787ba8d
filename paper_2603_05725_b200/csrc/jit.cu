// SIR -> CUDA C++ specialization of K3, compiled with NVRTC for sm_100a when a
// program is created (the GPU analogue of the paper's instrument-at-load step,
// PAPER.md §3; semantics of executor.py:210-424 preserved instruction by
// instruction).
//
// Per simulated kernel the generator emits one device function in which
//   * every simulated register is a C++ local (r/f: u32 bits, a: 128-bit signed
//     value + provenance tag, p: bool) -> lives in hardware registers,
//   * every basic block is a label; control flow is goto; each static edge's
//     hit counter is a compile-time slot of the runner (registers),
//   * the retired-instruction budget is charged once per block on the fast
//     path; a block that could reach the budget branches to a slow copy that
//     charges and checks per instruction (executor.py:411-415 exactly),
//   * ld/st go through the exec_core sanitizer, with a fast path when static
//     provenance analysis proves the base register carries a pointer
//     parameter's tag and the access lies inside that record's live payload.
// The host-op driver, allocator and sanitizer are exec_core.cuh, shared with
// the generic interpreter (execute.cu).
#include <nvrtc.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <set>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "embedded.inc"  // generated at build time: kEmbeddedNames / kEmbeddedSources / kEmbeddedCount

namespace sfgjit {

enum { TAG_BOT = -2, TAG_TOP = -1, TAG_NONE = 0 };  // q+1 = pointer param q

struct KInfo {
  int base, n, regs, nr, nf, na;
};

static std::string hex64(int64_t v) {
  char b[40];
  snprintf(b, sizeof b, "0x%llxull", (unsigned long long)v);
  return b;
}

static std::string u32lit(int64_t v) {
  char b[24];
  snprintf(b, sizeof b, "0x%08xu", (unsigned)(uint32_t)v);
  return b;
}

static std::string i64lit(int64_t v) {
  char b[48];
  if (v == INT64_MIN) return "(-9223372036854775807ll - 1)";
  snprintf(b, sizeof b, "(%lldll)", (long long)v);
  return b;
}

// blocks: leaders are 0, branch targets and successors of bra/exit (kernel_ir.py:364-401)
static std::vector<int> block_starts(const sfg_ins* I, int n) {
  std::vector<char> lead(n + 1, 0);
  lead[0] = 1;
  for (int i = 0; i < n; ++i) {
    if (I[i].op == SFG_BRA) {
      lead[I[i].target] = 1;
      if (i + 1 < n) lead[i + 1] = 1;
    } else if (I[i].op == SFG_EXIT && i + 1 < n) {
      lead[i + 1] = 1;
    }
  }
  std::vector<int> s;
  for (int i = 0; i < n; ++i)
    if (lead[i]) s.push_back(i);
  return s;
}

static int meet(int a, int b) {
  if (a == TAG_BOT) return b;
  if (b == TAG_BOT) return a;
  return a == b ? a : TAG_TOP;
}

// forward dataflow of a-register provenance tags (static when a param's tag reaches)
static std::vector<std::vector<int>> tag_flow(const sfg_ins* I, int n, const KInfo& K,
                                              const std::vector<int>& starts, std::vector<int>& blk_of) {
  const int nb = (int)starts.size();
  blk_of.assign(n, 0);
  for (int b = 0; b < nb; ++b) {
    const int e = b + 1 < nb ? starts[b + 1] : n;
    for (int i = starts[b]; i < e; ++i) blk_of[i] = b;
  }
  std::vector<std::vector<int>> in(nb, std::vector<int>(K.regs, TAG_BOT));
  for (int q = 0; q < K.regs; ++q) in[0][q] = q < K.na ? q + 1 : TAG_NONE;
  std::vector<std::vector<int>> at(n, std::vector<int>(K.regs, TAG_BOT));  // state before instruction
  bool changed = true;
  while (changed) {
    changed = false;
    for (int b = 0; b < nb; ++b) {
      std::vector<int> st = in[b];
      const int e = b + 1 < nb ? starts[b + 1] : n;
      for (int i = starts[b]; i < e; ++i) {
        at[i] = st;
        const sfg_ins& x = I[i];
        if (x.op == SFG_MOV && x.mode == SFG_CLS_A) st[x.dst] = (x.flags & SFG_F_S1_IMM) ? TAG_NONE : st[x.s1];
        else if ((x.op == SFG_ADD || x.op == SFG_SUB) && x.mode == SFG_CLS_A) st[x.dst] = st[x.s1];
        else if (x.op == SFG_LD && x.mode == SFG_MK_B64) st[x.dst] = TAG_NONE;
      }
      auto flow = [&](int succ) {
        for (int q = 0; q < K.regs; ++q) {
          const int m = meet(in[succ][q], st[q]);
          if (m != in[succ][q]) { in[succ][q] = m; changed = true; }
        }
      };
      const sfg_ins& last = I[e - 1];
      if (last.op == SFG_EXIT) continue;
      if (last.op == SFG_BRA) {
        flow(blk_of[last.target]);
        if ((last.flags & SFG_F_PRED) && e < n) flow(blk_of[e]);
      } else if (e < n) {
        flow(blk_of[e]);
      }
    }
  }
  return at;
}

// Static bounds of one input's allocator tables for this harness (sizes the
// lane's Lane struct in the specialized kernels, exec_core.cuh SFG_LANE_*).
struct LaneCaps {
  int recs = SFG_MAX_LANE_RECS, q = 32, freel = 32, named = SFG_MAX_NAMED, args = SFG_MAX_ARGS,
      params = SFG_MAX_ARGS;
};

struct Gen {
  const sfg_prog& P;
  const sfg_ins* ins;
  std::ostringstream o;
  bool edge_ovf_checks;

  explicit Gen(const sfg_prog& p, const sfg_ins* i) : P(p), ins(i) {}

  std::string r(int i) { return "r" + std::to_string(i); }
  std::string f(int i) { return "f" + std::to_string(i); }
  std::string a(int i) { return "a" + std::to_string(i); }
  std::string t(int i) { return "t" + std::to_string(i); }
  std::string p(int i) { return "p" + std::to_string(i); }

  std::string edge(int e) {
    if (e < 0) return "";
    if (edge_ovf_checks) return "if (++J.ec[" + std::to_string(e) + "] == 0u) J.ovf = true; ";
    return "++J.ec[" + std::to_string(e) + "]; ";
  }

  // retire-adjust string for stops inside a block: fast path adds j+1, slow path already counted
  static std::string radj(bool slow, int j) { return slow ? "" : "ret += " + std::to_string(j + 1) + "; "; }

  void emit_mem(const sfg_ins& x, int kidx, int iid, int j, bool slow, int tag) {
    const int W = x.width;
    const bool st = x.op == SFG_ST;
    if (narrow)   // 64-bit pointer registers (see narrow_ok): the address is exact in int64
      o << "    { const int64_t lo_ = " << a(x.s1) << " + " << i64lit(x.imm2) << "; const i128 A_ = (i128)lo_;\n";
    else
      o << "    { const i128 A_ = " << a(x.s1) << " + (i128)" << i64lit(x.imm2) << "; const int64_t lo_ = (int64_t)A_;\n";
    std::string val;
    if (st) {
      if (x.mode == SFG_MK_F32) val = (x.flags & SFG_F_S2_IMM) ? std::string("(uint64_t)") + u32lit(x.imm1) : "(uint64_t)" + f(x.s2);
      else if (x.mode == SFG_MK_B64) val = "(uint64_t)" + a(x.s2);
      else val = (x.flags & SFG_F_S2_IMM) ? "(uint64_t)" + hex64(x.imm1) : "(uint64_t)" + r(x.s2);
      o << "      const uint64_t sv_ = " << val << ";\n";
    } else {
      o << "      uint64_t v_;\n";
    }
    const std::string W_s = std::to_string(W), SP = std::to_string(x.space);
    // fast path: tagged live own record of the declared space, access inside its payload
    // and naturally aligned in the work region (phys offsets are 16-aligned)
    // (pk<q>_<space>_<W> and pl<q>_<W> are loop-invariant: the payload holds a
    // W-byte access and its last valid offset, computed once per simulated thread)
    auto fast = [&](int q) {
      const std::string Q = std::to_string(q);
      std::string c = "(pk" + Q + "_" + SP + "_" + W_s + (narrow ? "" : " && (i128)lo_ == A_") + " && (uint64_t)(lo_ - pb" +
                      Q + ") <= pl" + Q + "_" + W_s;
      if (W > 1) c += " && ((lo_ - pb" + Q + ") & " + std::to_string(W - 1) + ") == 0";
      return c + ")";
    };
    auto fast_body = [&](int q) {
      const std::string Q = std::to_string(q);
      const char* T = W == 1 ? "uint8_t" : W == 2 ? "uint16_t" : W == 4 ? "uint32_t" : "uint64_t";
      const std::string ptr = std::string("reinterpret_cast<") + (st ? "" : "const ") + T + "*>(pp" + Q + " + (lo_ - pb" + Q + "))";
      // loads from a record no store of this kernel can reach need no tag (no thread
      // of the launch writes it: nothing to conflict with)
      const bool ro = !st && !any_untagged_store && !written[q];
      // stores into a record this kernel never loads, with memory dead after the
      // launch: their order across threads cannot be observed
      const bool wo = st && dead_now && !any_untagged_load && !loaded[q];
      const std::string trk = (ro || wo) ? std::string() :
          "if (PAR && par_track(J.tags, J.ntags, pw" + Q + " + (lo_ - pb" + Q + "), " + W_s + ", " +
          (st ? "true" : "false") + ", J.me, J.waw)) { " + radj(slow, j) + "rc = RUN_CONFLICT; goto done; } ";
      // a write-only store into memory dead after the launch is never read back
      // unless diff readback copies the record out: only the sanitizer check matters
      if (st && wo) return "if (P.diff_readback) *" + ptr + " = (" + T + ")sv_;";
      if (st) return trk + "*" + ptr + " = (" + T + ")sv_;";
      return trk + "v_ = *" + ptr + ";";
    };
    std::string slow_path =
        "{ Report rep_; int rh_ = -1;\n"
        "        if (check_access(P, L, A_, " + W_s + ", " + SP + ", " + t(x.s1) + ", rep_, rh_)) { fill_report(V, P, L, rep_, " +
        std::to_string(kidx) + ", " + std::to_string(iid) + ", ctaid, tid, A_, " + W_s + ", " + (st ? "true" : "false") +
        ", " + SP + ", " + t(x.s1) + "); " + radj(slow, j) + "rc = RUN_FINDING; goto done; }\n";
    slow_path += "        if (PAR && par_access(J, L.rec[rh_], lo_, " + W_s + ", " + (st ? "true" : "false") + ")) { " +
                 radj(slow, j) + "rc = RUN_CONFLICT; goto done; }\n";
    if (st)
      slow_path += "        if (!mem_write(M, L, L.rec[rh_], lo_, " + W_s + ", sv_)) { V.status = SFG_ST_OVERLAY; " +
                   radj(slow, j) + "rc = RUN_FATAL; goto done; } }";
    else
      slow_path += "        v_ = mem_read(M, L, L.rec[rh_], lo_, " + W_s + "); }";
    if (tag > 0) {
      o << "      if " << fast(tag - 1) << " { " << fast_body(tag - 1) << " }\n      else " << slow_path << "\n";
    } else if (tag == TAG_TOP) {
      std::string pre = "      ";
      for (int q = 0; q < cur_na; ++q) {
        o << pre << "if (" << t(x.s1) << " == pt" << q << " && " << fast(q) << ") { " << fast_body(q) << " }\n";
        pre = "      else ";
      }
      o << pre << slow_path << "\n";
    } else {
      o << "      " << slow_path << "\n";
    }
    if (!st) {
      if (x.mode == SFG_MK_F32)
        o << "      " << f(x.dst) << " = " << (fbits[x.dst] ? "sfg_quiet((uint32_t)v_)" : "(uint32_t)v_") << ";\n";
      else if (x.mode == SFG_MK_B64) o << "      " << a(x.dst) << " = (" << AT() << ")(uint64_t)v_; " << t(x.dst) << " = 0;\n";
      else o << "      " << r(x.dst) << " = (uint32_t)v_;\n";
    }
    o << "    }\n";
  }

  // ---------------------------------------------------------------------------
  // Loop summarization.  A simple cycle of blocks whose instructions are register
  // arithmetic, integer setp and branches only (no ld/st) is a pure function of
  // its registers: every register carried from one trip to the next must be a
  // basic induction variable (x += loop-invariant per trip), every exit branch an
  // integer compare of an induction variable (or an invariant) against an
  // invariant.  At a window check of the cycle's head block the summary computes
  // the first trip T whose exit condition holds (closed form over a horizon in
  // which no compared i32 value wraps and the budget cannot be reached), skips
  // trips 0 .. T-2 at once -- induction variables advanced with i32 / pointer
  // wraparound exactly as executor.py:297-318 would, each edge of the cycle
  // counted T-1 times, T-1 trips x trip length retired -- and lets the
  // generated code run trip T-1 (which recomputes every derived register) and
  // the exiting trip T instruction by instruction, so budget exhaustion and
  // exits mid-trip are exactly the reference's (executor.py:411-415).
  struct Opnd {       // r-class (i32) value at a program point, as a function of the trip t
    int kind = 0;     // 0 unknown, 1 invariant expr, 2 IV(x) + offset expr, 3 i64 immediate
    std::string e;    // kind 1: u32 expression; kind 2: u32 offset expression
    int iv = -1;
    int64_t imm = 0;
  };
  struct AVal {       // abstract register value
    int kind = 0;     // 0 unknown, 1 invariant, 2 IV(iv) + e, 4 compare (predicates)
    std::string e;
    int iv = -1;
    int cmp = 0;
    Opnd l, r;
  };
  struct Exit {
    int cmp;          // exits when  l <cmp> r  (already oriented)
    Opnd l, r;
    bool konst;       // predicate invariant over the cycle: exits iff the expr `pe` holds
    std::string pe;
  };
  struct Cycle {
    std::vector<int> blocks;
    int64_t len = 0;
    std::vector<int> edges;                 // edge ids counted once per trip
    std::vector<std::pair<int, std::string>> r_iv, a_iv;  // register, per-trip step expr
    std::vector<Exit> exits;
    std::vector<std::string> guards;        // stable carried registers: current value == invariant
  };

  static int neg_cmp(int c) {
    static const int n[] = {SFG_CMP_NE, SFG_CMP_EQ, SFG_CMP_GE, SFG_CMP_GT, SFG_CMP_LE, SFG_CMP_LT};
    return n[c];
  }

  // successors of block b: (block, edge id)
  struct Succ { int blk, edge; bool taken; };
  std::vector<Succ> succs(const sfg_ins* I, int n, const std::vector<int>& starts, const std::vector<int>& blk_of, int b) {
    const int nb = (int)starts.size();
    const int e = b + 1 < nb ? starts[b + 1] : n;
    const sfg_ins& last = I[e - 1];
    std::vector<Succ> s;
    if (last.op == SFG_EXIT) return s;
    if (last.op == SFG_BRA) {
      s.push_back({blk_of[last.target], last.edge_tk, true});
      if ((last.flags & SFG_F_PRED) && e < n) s.push_back({blk_of[e], last.edge_ft, false});
    } else if (e < n) {
      s.push_back({blk_of[e], last.edge_ft, false});
    }
    return s;
  }

  // analyse one simple cycle (blocks in trip order starting at the head)
  bool analyse_cycle(const sfg_ins* I, int n, const std::vector<int>& starts, const std::vector<int>& blk_of,
                     int regs, Cycle& C) {
    const int nb = (int)starts.size();
    const int R = regs > 0 ? regs : 1;
    // pass 1: which registers (per class) are read before written in the trip, which are written
    std::vector<char> wr(4 * R, 0), er(4 * R, 0);
    auto rd = [&](int cls, int q) { if (!wr[cls * R + q]) er[cls * R + q] = 1; };
    auto wt = [&](int cls, int q) { wr[cls * R + q] = 1; };
    C.len = 0;
    for (size_t bi = 0; bi < C.blocks.size(); ++bi) {
      const int b = C.blocks[bi];
      const int s0 = starts[b], e = b + 1 < nb ? starts[b + 1] : n;
      C.len += e - s0;
      for (int i = s0; i < e; ++i) {
        const sfg_ins& x = I[i];
        const bool i1 = x.flags & SFG_F_S1_IMM, i2 = x.flags & SFG_F_S2_IMM;
        switch (x.op) {
          case SFG_MOV:
            if (!i1 || x.mode == SFG_CLS_P) rd(x.mode, x.s1);
            wt(x.mode, x.dst);
            break;
          case SFG_ADD: case SFG_SUB: case SFG_MUL:
            if (x.mode == SFG_CLS_A) { rd(SFG_CLS_A, x.s1); if (!i2) rd(SFG_CLS_R, x.s2); wt(SFG_CLS_A, x.dst); }
            else { if (!i1) rd(SFG_CLS_R, x.s1); if (!i2) rd(SFG_CLS_R, x.s2); wt(SFG_CLS_R, x.dst); }
            break;
          case SFG_FADD: case SFG_FSUB: case SFG_FMUL:
            if (!i1) rd(SFG_CLS_F, x.s1);
            if (!i2) rd(SFG_CLS_F, x.s2);
            wt(SFG_CLS_F, x.dst);
            break;
          case SFG_SETP: {
            const int c = (x.flags & SFG_F_FLOAT) ? SFG_CLS_F : SFG_CLS_R;
            if (!i1) rd(c, x.s1);
            if (!i2) rd(c, x.s2);
            wt(SFG_CLS_P, x.dst);
            break;
          }
          case SFG_CVT:
            if (!i1) rd(x.mode == SFG_CVT_F_FROM_I ? SFG_CLS_R : SFG_CLS_F, x.s1);
            wt(x.mode == SFG_CVT_F_FROM_I ? SFG_CLS_F : SFG_CLS_R, x.dst);
            break;
          case SFG_SREG: wt(SFG_CLS_R, x.dst); break;
          case SFG_BRA: if (x.flags & SFG_F_PRED) rd(SFG_CLS_P, x.s1); break;
          default: return false;  // ld / st / exit: not a pure register cycle
        }
      }
    }
    // pass 2: abstract values through one trip.  A carried register whose value at
    // the end of the trip is loop-invariant ("stable", e.g. a counter reset inside
    // the cycle) is treated as invariant, guarded at run time by its current value
    // equalling the invariant (then every trip sees the same value).
    std::vector<char> stable(4 * R, 0);
    for (int attempt = 0; attempt < 2; ++attempt) {
    C.edges.clear(); C.exits.clear(); C.r_iv.clear(); C.a_iv.clear(); C.guards.clear();
    bool retry = false;
    std::vector<AVal> v(4 * R);
    for (int c = 0; c < 4; ++c)
      for (int q = 0; q < R; ++q) {
        AVal& a = v[c * R + q];
        if (!wr[c * R + q] || stable[c * R + q]) {
          a.kind = 1;
          a.e = c == SFG_CLS_R ? r(q) : c == SFG_CLS_F ? f(q) : c == SFG_CLS_A ? a_name(q) : p(q);
        } else if (er[c * R + q]) {
          if (c != SFG_CLS_R && c != SFG_CLS_A) return false;  // carried f / p register
          a.kind = 2; a.iv = q; a.e = c == SFG_CLS_R ? "0u" : "(int64_t)0";
        }
      }
    auto Rv = [&](int q) -> AVal& { return v[SFG_CLS_R * R + q]; };
    auto ropnd = [&](const sfg_ins& x, int slot) -> AVal {   // u32 operand
      const bool imm = slot == 1 ? (x.flags & SFG_F_S1_IMM) : (x.flags & SFG_F_S2_IMM);
      if (imm) { AVal a; a.kind = 1; a.e = u32lit(slot == 1 ? x.imm1 : x.imm2); return a; }
      return Rv(slot == 1 ? x.s1 : x.s2);
    };
    auto cmp_opnd = [&](const sfg_ins& x, int slot) -> Opnd {  // src_i64 operand of an int setp
      Opnd o;
      const bool imm = slot == 1 ? (x.flags & SFG_F_S1_IMM) : (x.flags & SFG_F_S2_IMM);
      if (imm) {
        int64_t m = slot == 1 ? x.imm1 : x.imm2;
        const int64_t cl = 1ll << 40;   // i32 values never reach it: the compare is unchanged
        o.kind = 3; o.imm = m > cl ? cl : m < -cl ? -cl : m;
        return o;
      }
      const AVal& a = Rv(slot == 1 ? x.s1 : x.s2);
      if (a.kind == 1) { o.kind = 1; o.e = a.e; }
      else if (a.kind == 2) { o.kind = 2; o.iv = a.iv; o.e = a.e; }
      return o;
    };
    for (size_t bi = 0; bi < C.blocks.size(); ++bi) {
      const int b = C.blocks[bi];
      const int nxt = C.blocks[(bi + 1) % C.blocks.size()];
      const int s0 = starts[b], e = b + 1 < nb ? starts[b + 1] : n;
      for (int i = s0; i < e; ++i) {
        const sfg_ins& x = I[i];
        const bool i1 = x.flags & SFG_F_S1_IMM;
        AVal res;
        switch (x.op) {
          case SFG_MOV:
            if (x.mode == SFG_CLS_R) res = ropnd(x, 1);
            else if (x.mode == SFG_CLS_F) {
              if (i1) { res.kind = 1; res.e = u32lit(x.imm1); } else res = v[SFG_CLS_F * R + x.s1];
            } else if (x.mode == SFG_CLS_A) {
              if (i1) {
                res.kind = 1;
                res.e = (x.flags & SFG_F_U64IMM) ? "(" + AT() + ")(uint64_t)" + hex64(x.imm1) : "(" + AT() + ")" + i64lit(x.imm1);
              } else res = v[SFG_CLS_A * R + x.s1];
            } else res = v[SFG_CLS_P * R + x.s1];
            v[x.mode * R + x.dst] = res;
            break;
          case SFG_ADD: case SFG_SUB: case SFG_MUL: {
            const char* opc = x.op == SFG_ADD ? "+" : x.op == SFG_SUB ? "-" : "*";
            if (x.mode == SFG_CLS_A) {
              if (x.op == SFG_MUL) { v[SFG_CLS_A * R + x.dst] = AVal(); break; }
              std::string o2;
              if (x.flags & SFG_F_S2_IMM) o2 = i64lit(x.imm2);
              else if (Rv(x.s2).kind == 1) o2 = "(int64_t)(int32_t)(" + Rv(x.s2).e + ")";
              const AVal& s = v[SFG_CLS_A * R + x.s1];
              if (!o2.empty() && (s.kind == 1 || s.kind == 2)) {
                res = s;
                res.e = "(" + (s.kind == 1 ? s.e : s.e) + " " + opc + " (" + (s.kind == 1 ? AT() : std::string("int64_t")) +
                        ")" + o2 + ")";
              }
              v[SFG_CLS_A * R + x.dst] = res;
              break;
            }
            const AVal a1 = ropnd(x, 1), a2 = ropnd(x, 2);
            if (a1.kind == 1 && a2.kind == 1) { res.kind = 1; res.e = "(uint32_t)(" + a1.e + " " + opc + " " + a2.e + ")"; }
            else if (x.op != SFG_MUL && a1.kind == 2 && a2.kind == 1) {
              res = a1; res.e = "(uint32_t)(" + a1.e + " " + opc + " " + a2.e + ")";
            } else if (x.op == SFG_ADD && a1.kind == 1 && a2.kind == 2) {
              res = a2; res.e = "(uint32_t)(" + a2.e + " + " + a1.e + ")";
            }
            Rv(x.dst) = res;
            break;
          }
          case SFG_FADD: case SFG_FSUB: case SFG_FMUL: v[SFG_CLS_F * R + x.dst] = AVal(); break;
          case SFG_CVT:
            v[(x.mode == SFG_CVT_F_FROM_I ? SFG_CLS_F : SFG_CLS_R) * R + x.dst] = AVal();
            break;
          case SFG_SREG: {
            static const char* names[] = {"tid", "block", "ctaid", "grid"};
            res.kind = 1; res.e = std::string("(uint32_t)") + names[x.mode];
            Rv(x.dst) = res;
            break;
          }
          case SFG_SETP:
            if (!(x.flags & SFG_F_FLOAT)) {
              const Opnd l = cmp_opnd(x, 1), rr = cmp_opnd(x, 2);
              if (l.kind && rr.kind) { res.kind = 4; res.cmp = x.mode; res.l = l; res.r = rr; }
            }
            v[SFG_CLS_P * R + x.dst] = res;
            break;
          case SFG_BRA: {
            const auto ss = succs(I, n, starts, blk_of, b);
            int stay_tk = -1;  // which direction stays on the cycle: 1 taken, 0 fallthrough
            for (const Succ& sc : ss)
              if (sc.blk == nxt) {
                if (stay_tk >= 0) return false;   // both directions reach the next block
                stay_tk = sc.taken ? 1 : 0;
                if (sc.edge >= 0) C.edges.push_back(sc.edge);
              }
            if (stay_tk < 0) return false;
            if (!(x.flags & SFG_F_PRED)) break;
            // exits when (pneg ? !p : p) != stay_tk, i.e. when p == exit_p
            const bool exit_p = (stay_tk == 1) == ((x.flags & SFG_F_PNEG) != 0);
            const AVal& pv = v[SFG_CLS_P * R + x.s1];
            Exit X;
            if (pv.kind == 1) { X.konst = true; X.pe = exit_p ? pv.e : "!" + pv.e; X.cmp = 0; }
            else if (pv.kind == 4) { X.konst = false; X.cmp = exit_p ? pv.cmp : neg_cmp(pv.cmp); X.l = pv.l; X.r = pv.r; }
            else return false;
            C.exits.push_back(X);
            break;
          }
          default: return false;
        }
        if (i == e - 1 && x.op != SFG_BRA) {   // falls through into the next leader
          if (blk_of[i + 1 < n ? i + 1 : 0] != nxt || i + 1 >= n) return false;
          if (x.edge_ft >= 0) C.edges.push_back(x.edge_ft);
        }
      }
    }
    // carried registers must be basic induction variables: IV(x) + invariant step,
    // or stable (invariant at the end of the trip)
    for (int c : {SFG_CLS_R, SFG_CLS_A})
      for (int q = 0; q < R; ++q) {
        if (!(wr[c * R + q] && er[c * R + q])) continue;
        const AVal& a = v[c * R + q];
        if (stable[c * R + q]) {
          if (a.kind != 1) return false;
          C.guards.push_back((c == SFG_CLS_R ? r(q) : a_name(q)) + " == " + a.e);
          continue;
        }
        if (a.kind == 1 && attempt == 0) { stable[c * R + q] = 1; retry = true; continue; }
        if (a.kind != 2 || a.iv != q) return false;
        (c == SFG_CLS_R ? C.r_iv : C.a_iv).push_back({q, a.e});
      }
    if (!retry) return !C.exits.empty();
    }
    return false;
  }

  std::string a_name(int i) { return a(i); }

  // all summarizable simple cycles through check block h (trip order starting at h)
  std::vector<Cycle> cycles_at(const sfg_ins* I, int n, const std::vector<int>& starts, const std::vector<int>& blk_of,
                               int regs, int h) {
    std::vector<Cycle> out;
    std::vector<int> path{h};
    std::vector<char> on((size_t)starts.size(), 0);
    on[h] = 1;
    int budget = 256;   // DFS steps
    std::function<void(int)> dfs = [&](int b) {
      if (--budget < 0 || out.size() >= 4) return;
      for (const Succ& s : succs(I, n, starts, blk_of, b)) {
        if (s.blk == h) {
          Cycle C;
          C.blocks = path;
          const bool ok_ = analyse_cycle(I, n, starts, blk_of, regs, C);
          if (getenv("SFG_LOOPSUM_DEBUG")) {
            fprintf(stderr, "cycle at %d:", h);
            for (int x : C.blocks) fprintf(stderr, " %d", x);
            fprintf(stderr, " -> %s\n", ok_ ? "summary" : "no");
          }
          if (ok_) out.push_back(C);
        } else if (!on[s.blk] && path.size() < 24) {
          on[s.blk] = 1;
          path.push_back(s.blk);
          dfs(s.blk);
          path.pop_back();
          on[s.blk] = 0;
        }
      }
    };
    dfs(h);
    return out;
  }

  // ---------------------------------------------------------------------------
  // Nest summaries.  A loop at check block h whose body (the blocks on a cycle
  // through h, inner loops included) repeats exactly from one trip to the next up
  // to basic induction registers: the only registers carried from trip to trip are
  // r = r +/- X (X an immediate or a register the body never writes, the def in a
  // block every trip passes once); every other value the body uses is a function
  // of registers the body never writes, of values loaded from records the body
  // never stores to, and of the induction registers through i32 arithmetic whose
  // per-trip change is 0 mod 2^32 (a run-time guard, e.g. row * ldc with
  // ldc = -2^31 and a row step of 8); every exit tests a trip-invariant predicate
  // or, at h, an induction register against an invariant.  Then every trip runs
  // the same instructions on the same addresses and values: the first complete
  // trip after arming is measured (retired instructions, edge counts) and the
  // next k trips are skipped at once -- k below the first trip whose exit test at
  // h holds (closed form, inside the i32 no-wrap horizon) and below the budget --
  // induction registers advanced k steps, edges and retired counted k times;
  // memory is as after one trip.  The remaining trips run instruction by
  // instruction (exits and budget exhaustion exact, executor.py:411-415).
  struct NV { int k = 0; std::string e; };   // 0 read-before-def, 1 invariant (e: expr or ""), 2 per-trip delta e, 3 hard
  struct Nest {
    int h = -1;
    std::vector<int> blocks;
    std::vector<std::pair<int, std::string>> r_iv;   // induction register, per-trip step (u32 expr)
    bool has_x = false;                      // exit at h: iv <x_cmp> rhs (oriented: exits when it holds)
    int x_cmp = 0, x_iv = -1;
    std::string x_rhs;                       // int64 expression
    // u32 expressions that must be 0, each needed only if its block ran in the measured
    // trip (an access / compare the trip does not reach constrains nothing)
    std::vector<std::pair<std::string, int>> guards;
    std::vector<std::pair<std::string, std::pair<int, int>>> distinct;   // ptA != ptB if both blocks ran
    std::vector<int> edges;                  // edges between body blocks (snapshotted per trip)
    std::vector<std::vector<int>> in_edges;  // per body block (index into blocks): its in-edges' snapshot slots, -1: always runs
  };

  static int swap_cmp(int c) {
    static const int m[] = {SFG_CMP_EQ, SFG_CMP_NE, SFG_CMP_GT, SFG_CMP_GE, SFG_CMP_LT, SFG_CMP_LE};
    return m[c];
  }

  bool analyse_nest(const sfg_ins* I, int n, const std::vector<int>& starts, const std::vector<int>& blk_of, int regs,
                    int h, const std::vector<std::vector<int>>& tags, Nest& N) {
    const int nb = (int)starts.size();
    const int R = regs > 0 ? regs : 1;
    auto bend = [&](int b) { return b + 1 < nb ? starts[b + 1] : n; };
    std::vector<std::vector<Succ>> sc(nb);
    std::vector<std::vector<int>> pred(nb);
    for (int b = 0; b < nb; ++b) {
      sc[b] = succs(I, n, starts, blk_of, b);
      for (const Succ& x : sc[b]) pred[x.blk].push_back(b);
    }
    std::vector<char> fw(nb, 0), bw(nb, 0), in(nb, 0);
    std::vector<int> st{h};
    fw[h] = 1;
    while (!st.empty()) {
      const int b = st.back(); st.pop_back();
      for (const Succ& x : sc[b]) if (!fw[x.blk]) { fw[x.blk] = 1; st.push_back(x.blk); }
    }
    st = {h};
    bw[h] = 1;
    while (!st.empty()) {
      const int b = st.back(); st.pop_back();
      for (int q : pred[b]) if (!bw[q]) { bw[q] = 1; st.push_back(q); }
    }
    bool back = false;
    for (int b = 0; b < nb; ++b) in[b] = fw[b] && bw[b];
    for (int q : pred[h]) back |= in[q] != 0;
    if (!back) return false;
    N = Nest();
    N.h = h;
    for (int b = 0; b < nb; ++b) if (in[b]) N.blocks.push_back(b);
    if (N.blocks.size() > 64) return false;
    // register defs in the body
    auto def_cls = [&](const sfg_ins& x, int& c) -> bool {
      switch (x.op) {
        case SFG_MOV: c = x.mode; return true;
        case SFG_ADD: case SFG_SUB: case SFG_MUL: c = x.mode == SFG_CLS_A ? SFG_CLS_A : SFG_CLS_R; return true;
        case SFG_FADD: case SFG_FSUB: case SFG_FMUL: c = SFG_CLS_F; return true;
        case SFG_SETP: c = SFG_CLS_P; return true;
        case SFG_CVT: c = x.mode == SFG_CVT_F_FROM_I ? SFG_CLS_F : SFG_CLS_R; return true;
        case SFG_SREG: c = SFG_CLS_R; return true;
        case SFG_LD: c = x.mode == SFG_MK_F32 ? SFG_CLS_F : x.mode == SFG_MK_B64 ? SFG_CLS_A : SFG_CLS_R; return true;
        default: return false;
      }
    };
    std::vector<int> ndef(4 * R, 0), def_at(4 * R, -1);
    for (int b : N.blocks)
      for (int i = starts[b]; i < bend(b); ++i) {
        int c;
        if (I[i].op == SFG_EXIT) return false;
        if (def_cls(I[i], c)) { ++ndef[c * R + I[i].dst]; def_at[c * R + I[i].dst] = i; }
      }
    // a block every trip passes exactly once
    auto once = [&](int D) -> bool {
      if (D == h) return true;
      std::vector<char> seen(nb, 0);
      std::vector<int> s2;
      for (const Succ& x : sc[D]) if (in[x.blk] && x.blk != h && !seen[x.blk]) { seen[x.blk] = 1; s2.push_back(x.blk); }
      while (!s2.empty()) {
        const int b = s2.back(); s2.pop_back();
        if (b == D) return false;
        for (const Succ& x : sc[b]) if (in[x.blk] && x.blk != h && !seen[x.blk]) { seen[x.blk] = 1; s2.push_back(x.blk); }
      }
      std::fill(seen.begin(), seen.end(), 0);
      for (const Succ& x : sc[h]) {
        if (x.blk == h) return false;
        if (in[x.blk] && x.blk != D && !seen[x.blk]) { seen[x.blk] = 1; s2.push_back(x.blk); }
      }
      while (!s2.empty()) {
        const int b = s2.back(); s2.pop_back();
        for (const Succ& x : sc[b]) {
          if (x.blk == h) return false;
          if (in[x.blk] && x.blk != D && !seen[x.blk]) { seen[x.blk] = 1; s2.push_back(x.blk); }
        }
      }
      return true;
    };
    std::vector<NV> entry(4 * R);
    for (int c = 0; c < 4; ++c)
      for (int q = 0; q < R; ++q) {
        NV& v = entry[c * R + q];
        if (ndef[c * R + q] == 0) {
          v.k = 1;
          v.e = c == SFG_CLS_R ? r(q) : "";
          continue;
        }
        v.k = 0;
        if (c != SFG_CLS_R || ndef[c * R + q] != 1) continue;
        const sfg_ins& x = I[def_at[c * R + q]];
        if (!(x.op == SFG_ADD || x.op == SFG_SUB) || x.mode != SFG_CLS_R) continue;
        const bool i1 = x.flags & SFG_F_S1_IMM, i2 = x.flags & SFG_F_S2_IMM;
        auto inv = [&](bool imm, int64_t iv, int reg) -> std::string {
          if (imm) return u32lit(iv);
          return ndef[SFG_CLS_R * R + reg] == 0 ? r(reg) : std::string();
        };
        std::string step;
        if (!i1 && x.s1 == q) step = inv(i2, x.imm2, x.s2);
        else if (x.op == SFG_ADD && !i2 && x.s2 == q) step = inv(i1, x.imm1, x.s1);
        if (step.empty() || !once(blk_of[def_at[c * R + q]])) continue;
        v.k = 2;
        v.e = x.op == SFG_SUB ? "(uint32_t)(0u - " + step + ")" : step;
        N.r_iv.push_back({q, v.e});
      }
    // the exit test at h: `setp p, iv, rhs` (or rhs, iv) then `bra p` leaving the body
    int x_setp = -1;
    {
      const int e = bend(h);
      const sfg_ins& last = I[e - 1];
      if (last.op == SFG_BRA && (last.flags & SFG_F_PRED)) {
        int stay = -1, outs = 0;
        for (const Succ& x : sc[h]) {
          if (in[x.blk]) stay = x.taken ? 1 : 0;
          else ++outs;
        }
        int sdef = -1;
        for (int i = starts[h]; i < e - 1; ++i)
          if (I[i].op == SFG_SETP && I[i].dst == last.s1) sdef = i;
          else { int c; if (def_cls(I[i], c) && c == SFG_CLS_P && I[i].dst == last.s1) sdef = -2; }
        if (outs == 1 && stay >= 0 && sdef >= 0 && !(I[sdef].flags & SFG_F_FLOAT)) {
          const sfg_ins& x = I[sdef];
          const bool exit_p = (stay == 1) == ((last.flags & SFG_F_PNEG) != 0);
          auto is_iv = [&](int slot) -> int {
            const bool imm = slot == 1 ? (x.flags & SFG_F_S1_IMM) : (x.flags & SFG_F_S2_IMM);
            if (imm) return -1;
            const int q = slot == 1 ? x.s1 : x.s2;
            for (auto& iv : N.r_iv) if (iv.first == q) {
              for (int i = starts[h]; i < sdef; ++i) { int c; if (def_cls(I[i], c) && c == SFG_CLS_R && I[i].dst == q) return -1; }
              return q;
            }
            return -1;
          };
          auto rhs = [&](int slot) -> std::string {
            const bool imm = slot == 1 ? (x.flags & SFG_F_S1_IMM) : (x.flags & SFG_F_S2_IMM);
            if (imm) {
              int64_t m = slot == 1 ? x.imm1 : x.imm2;
              const int64_t cl = 1ll << 40;
              return i64lit(m > cl ? cl : m < -cl ? -cl : m);
            }
            const int q = slot == 1 ? x.s1 : x.s2;
            return ndef[SFG_CLS_R * R + q] == 0 ? "(int64_t)(int32_t)" + r(q) : std::string();
          };
          const int l = is_iv(1), rr = is_iv(2);
          int cmpv = -1;
          std::string rh;
          if (l >= 0 && rr < 0) { rh = rhs(2); cmpv = x.mode; N.x_iv = l; }
          else if (rr >= 0 && l < 0) { rh = rhs(1); cmpv = swap_cmp(x.mode); N.x_iv = rr; }
          if (cmpv >= 0 && !rh.empty()) {
            N.has_x = true;
            N.x_cmp = exit_p ? cmpv : neg_cmp(cmpv);
            N.x_rhs = rh;
            x_setp = sdef;
          }
        }
      }
    }
    // abstract values through a trip, to a fixed point over the body (the back edges
    // into h are cut: h starts every trip with `entry`)
    bool ok = true;
    bool check = false;
    int cur_b = -1;
    std::set<std::pair<std::string, int>> G;
    std::set<std::pair<int, int>> ldt, stt;   // (tag, block)
    auto need_inv = [&](const NV& v) {
      if (v.k == 0 || v.k == 3) ok = false;
      else if (v.k == 2 && check) G.insert({v.e, cur_b});
    };
    auto join = [&](NV& a, const NV& b) -> bool {
      NV old = a;
      if (a.k == 0 || b.k == 0) { a.k = 0; a.e.clear(); }
      else if (a.k == 3 || b.k == 3) { a.k = 3; a.e.clear(); }
      else if (a.k != b.k) { a.k = 3; a.e.clear(); }
      else if (a.e != b.e) { if (a.k == 1) a.e.clear(); else { a.k = 3; a.e.clear(); } }
      return a.k != old.k || a.e != old.e;
    };
    auto transfer = [&](std::vector<NV>& v, int i) {
      const sfg_ins& x = I[i];
      const bool i1 = x.flags & SFG_F_S1_IMM, i2 = x.flags & SFG_F_S2_IMM;
      auto V = [&](int c, int q) -> NV& { return v[c * R + q]; };
      auto rop = [&](int slot) -> NV {
        const bool imm = slot == 1 ? i1 : i2;
        if (imm) { NV t; t.k = 1; t.e = u32lit(slot == 1 ? x.imm1 : x.imm2); return t; }
        const NV t = V(SFG_CLS_R, slot == 1 ? x.s1 : x.s2);
        if (t.k == 0) ok = false;
        return t;
      };
      auto cls_op = [&](int c, int slot) -> NV {   // f / a / p operand
        const bool imm = slot == 1 ? i1 : i2;
        if (imm) { NV t; t.k = 1; return t; }
        const NV t = V(c, slot == 1 ? x.s1 : x.s2);
        if (t.k == 0) ok = false;
        return t;
      };
      NV res;
      res.k = 1;
      switch (x.op) {
        case SFG_MOV:
          if (x.mode == SFG_CLS_R) V(SFG_CLS_R, x.dst) = rop(1);
          else V(x.mode, x.dst) = cls_op(x.mode, 1);
          break;
        case SFG_ADD: case SFG_SUB: case SFG_MUL: {
          if (x.mode == SFG_CLS_A) {
            // a pointer that varies from trip to trip is summarized by the i32 deltas
            // that entered it: invariant iff they are all 0 (checked where it is used)
            if (x.op == SFG_MUL) { ok = false; break; }
            const NV sp = cls_op(SFG_CLS_A, 1);
            const NV ro = i2 ? NV{1, ""} : rop(2);
            NV t;
            if (sp.k == 0 || ro.k == 0) { ok = false; break; }
            if (sp.k == 3 || ro.k == 3) t.k = 3;
            else if (sp.k == 1 && ro.k == 1) t.k = 1;
            else {
              t.k = 2;
              t.e = sp.k == 2 && ro.k == 2 ? "(uint32_t)(" + sp.e + " | " + ro.e + ")" : (sp.k == 2 ? sp.e : ro.e);
            }
            V(SFG_CLS_A, x.dst) = t;
            break;
          }
          const NV a1 = rop(1), a2 = rop(2);
          if (a1.k == 0 || a2.k == 0) { ok = false; break; }
          if (a1.k == 3 || a2.k == 3) { res.k = 3; }
          else if (a1.k == 1 && a2.k == 1) {
            res.k = 1;
            const char* opc = x.op == SFG_ADD ? "+" : x.op == SFG_SUB ? "-" : "*";
            res.e = (a1.e.empty() || a2.e.empty()) ? "" : "(uint32_t)(" + a1.e + " " + opc + " " + a2.e + ")";
          } else if (x.op == SFG_MUL) {
            if (a1.k == 2 && a2.k == 2) { need_inv(a1); need_inv(a2); res.k = 1; }
            else {
              const NV& vv = a1.k == 2 ? a1 : a2;
              const NV& ii = a1.k == 2 ? a2 : a1;
              if (ii.e.empty()) { need_inv(vv); res.k = 1; }
              else { res.k = 2; res.e = "(uint32_t)(" + vv.e + " * " + ii.e + ")"; }
            }
          } else {
            res.k = 2;
            const char* opc = x.op == SFG_ADD ? "+" : "-";
            const std::string d1 = a1.k == 2 ? a1.e : "0u", d2 = a2.k == 2 ? a2.e : "0u";
            res.e = "(uint32_t)(" + d1 + " " + opc + " " + d2 + ")";
          }
          V(SFG_CLS_R, x.dst) = res;
          break;
        }
        case SFG_FADD: case SFG_FSUB: case SFG_FMUL: {
          const NV a1 = cls_op(SFG_CLS_F, 1), a2 = cls_op(SFG_CLS_F, 2);
          res.k = (a1.k == 3 || a2.k == 3) ? 3 : 1;
          V(SFG_CLS_F, x.dst) = res;
          break;
        }
        case SFG_SETP:
          if (x.flags & SFG_F_FLOAT) {
            const NV a1 = cls_op(SFG_CLS_F, 1), a2 = cls_op(SFG_CLS_F, 2);
            res.k = (a1.k == 3 || a2.k == 3) ? 3 : 1;
          } else if (i != x_setp) {
            need_inv(rop(1));
            need_inv(rop(2));
          } else {
            res.k = 3;   // the exit test at h: only its branch may use it (closed form)
          }
          V(SFG_CLS_P, x.dst) = res;
          break;
        case SFG_CVT:
          if (x.mode == SFG_CVT_F_FROM_I) { if (!i1) need_inv(rop(1)); V(SFG_CLS_F, x.dst) = res; }
          else { const NV a1 = cls_op(SFG_CLS_F, 1); res.k = a1.k == 3 ? 3 : 1; V(SFG_CLS_R, x.dst) = res; }
          break;
        case SFG_SREG: {
          static const char* names[] = {"tid", "block", "ctaid", "grid"};
          res.e = std::string("(uint32_t)") + names[x.mode];
          V(SFG_CLS_R, x.dst) = res;
          break;
        }
        case SFG_LD: case SFG_ST: {
          need_inv(cls_op(SFG_CLS_A, 1));
          const int tg = tags[i][x.s1];
          if (tg <= 0) ok = false;
          if (x.op == SFG_LD) {
            ldt.insert({tg, cur_b});
            int c; def_cls(x, c);
            V(c, x.dst) = res;
          } else {
            stt.insert({tg, cur_b});
            if (x.mode == SFG_MK_F32) { if (!i2) { const NV t = cls_op(SFG_CLS_F, 2); if (t.k != 1) ok = false; } }
            else if (x.mode == SFG_MK_B64) need_inv(cls_op(SFG_CLS_A, 2));
            else if (!i2) need_inv(rop(2));
          }
          break;
        }
        case SFG_BRA:
          if ((x.flags & SFG_F_PRED) && check) {
            const NV pv = V(SFG_CLS_P, x.s1);
            const bool is_x = blk_of[i] == h && i == bend(h) - 1 && x_setp >= 0;
            if (!is_x && pv.k != 1) ok = false;
          }
          break;
        default:
          ok = false;
      }
    };
    std::vector<std::vector<NV>> bin(nb);
    std::vector<char> has(nb, 0);
    bin[h] = entry;
    has[h] = 1;
    std::vector<int> work{h};
    int steps = 0;
    while (!work.empty() && ok) {
      if (++steps > 4096) return false;
      const int b = work.back(); work.pop_back();
      std::vector<NV> v = bin[b];
      cur_b = b;
      for (int i = starts[b]; i < bend(b) && ok; ++i) transfer(v, i);
      for (const Succ& x : sc[b]) {
        if (!in[x.blk] || x.blk == h) continue;
        if (!has[x.blk]) { bin[x.blk] = v; has[x.blk] = 1; work.push_back(x.blk); continue; }
        bool ch = false;
        for (int k = 0; k < 4 * R; ++k) ch |= join(bin[x.blk][k], v[k]);
        if (ch) work.push_back(x.blk);
      }
    }
    if (!ok) return false;
    // the check pass over the fixed point: sinks need trip-invariant values
    check = true;
    for (int b : N.blocks) {
      if (!has[b]) return false;
      std::vector<NV> v = bin[b];
      cur_b = b;
      for (int i = starts[b]; i < bend(b) && ok; ++i) transfer(v, i);
      // exits other than h's test need trip-invariant predicates (checked at BRA)
      for (const Succ& x : sc[b]) if (!in[x.blk] && !(I[bend(b) - 1].op == SFG_BRA && (I[bend(b) - 1].flags & SFG_F_PRED)))
        ok = false;   // an unconditional way out of the body cannot be on a cycle
    }
    if (!ok) return false;
    for (auto& lt : ldt)
      for (auto& s2 : stt) {
        if (lt.first == s2.first) return false;   // a record the body both loads and stores
        N.distinct.push_back({"pt" + std::to_string(lt.first - 1) + " != pt" + std::to_string(s2.first - 1),
                              {lt.second, s2.second}});
      }
    for (auto& g : G) N.guards.push_back({"(uint32_t)(" + g.first + ") == 0u", g.second});
    std::set<int> es;
    for (int b : N.blocks) for (const Succ& x : sc[b]) if (x.edge >= 0 && in[x.blk]) es.insert(x.edge);
    N.edges.assign(es.begin(), es.end());
    // a body block ran in a trip iff one of its in-edges from the body was taken (h always)
    N.in_edges.assign(N.blocks.size(), {});
    for (size_t bi = 0; bi < N.blocks.size(); ++bi) {
      const int b = N.blocks[bi];
      if (b == h) { N.in_edges[bi] = {-1}; continue; }
      for (int q : pred[b]) {
        if (!in[q]) continue;
        for (const Succ& x : sc[q]) {
          if (x.blk != b) continue;
          if (x.edge < 0) { N.in_edges[bi] = {-1}; break; }
          N.in_edges[bi].push_back((int)(std::lower_bound(N.edges.begin(), N.edges.end(), x.edge) - N.edges.begin()));
        }
        if (!N.in_edges[bi].empty() && N.in_edges[bi][0] == -1) break;
      }
      if (N.in_edges[bi].empty()) N.in_edges[bi] = {-1};
    }
    return true;
  }

  // arming at the fast entry of h once the thread has run kNestArm instructions
  // since the last attempt: snapshot of the retired count and the body's edges
  std::string nest_arm_code(const Nest& N) {
    std::ostringstream s;
    const std::string H = std::to_string(N.h);
    s << "  else if (ret >= nsn" << H << ") { ns" << H << " = true; nsr" << H << " = ret; nsn" << H
      << " = ret + kNestArm;";
    for (size_t k = 0; k < N.edges.size(); ++k)
      s << " nse" << H << "[" << k << " ^ J.J_dyn] = J.ec[" << N.edges[k] << "];";
    s << " }\n";
    return s.str();
  }

  // at the fast entry of h, one complete trip after arming: skip k trips
  std::string nest_skip_code(const Nest& N, const char* RT) {
    std::ostringstream s;
    const std::string H = std::to_string(N.h);
    s << "  if (ns" << H << " && ret != nsr" << H << ") { // nest summary: blocks";
    for (int b : N.blocks) s << " " << b;
    s << "\n    ns" << H << " = false;\n";
    auto ran = [&](int b) -> std::string {   // block b ran in the measured trip
      const size_t bi = std::find(N.blocks.begin(), N.blocks.end(), b) - N.blocks.begin();
      const std::vector<int>& ie = N.in_edges[bi];
      if (ie.empty() || ie[0] < 0) return "true";
      std::string c = "(";
      for (size_t k = 0; k < ie.size(); ++k)
        c += (k ? " || " : "") + std::string("J.ec[") + std::to_string(N.edges[ie[k]]) + "] != nse" + H + "[" +
             std::to_string(ie[k]) + " ^ J.J_dyn]";
      return c + ")";
    };
    s << "    bool g_ = true;\n";
    for (auto& g : N.guards) s << "    g_ = g_ && (!" << ran(g.second) << " || " << g.first << ");\n";
    for (auto& d : N.distinct)
      s << "    g_ = g_ && (!(" << ran(d.second.first) << " && " << ran(d.second.second) << ") || " << d.first << ");\n";
    s << "    const uint64_t len_ = (uint64_t)(ret - nsr" << H << ");\n"
      << "    int64_t H_ = g_ && HARD > ret ? (int64_t)((uint64_t)(HARD - 1u - ret) / len_) : -1;\n";
    for (auto& iv : N.r_iv) s << "    const uint32_t dn" << iv.first << "_ = " << iv.second << ";\n";
    if (N.has_x) {
      const std::string q = std::to_string(N.x_iv);
      s << "    const int64_t x0_ = (int64_t)(int32_t)" << r(N.x_iv) << ", xd_ = (int64_t)(int32_t)dn" << q << "_;\n"
        << "    H_ = sfg_min64(H_, sfg_wrap_h(x0_, xd_));\n"
        << "    const int64_t T_ = sfg_first_t(" << N.x_cmp << ", x0_ - (" << N.x_rhs << "), xd_, H_);\n"
        << "    const int64_t k_ = T_ < H_ ? T_ : H_;\n";
    } else {
      s << "    const int64_t k_ = H_;\n";
    }
    s << "    if (k_ >= 1) {\n";
    for (auto& iv : N.r_iv)
      s << "      " << r(iv.first) << " = (uint32_t)(" << r(iv.first) << " + (uint32_t)k_ * dn" << iv.first << "_);\n";
    for (size_t k = 0; k < N.edges.size(); ++k)
      s << "      { const uint64_t o_ = (uint64_t)J.ec[" << N.edges[k] << "] + (uint64_t)k_ * (uint64_t)(uint32_t)(J.ec["
        << N.edges[k] << "] - nse" << H << "[" << k << " ^ J.J_dyn]); if (o_ > 0xFFFFFFFFull) J.ovf = true; J.ec["
        << N.edges[k] << "] = (uint32_t)o_; }\n";
    s << "      const " << RT << " sk_ = (" << RT << ")((uint64_t)k_ * len_);\n"
      << "      ret += sk_;\n"
      << "      if (SFT) { HARD = (" << RT << ")(BUD - HARD > sk_ ? HARD + sk_ : BUD); if (HARD == BUD) SFT = false; }\n"
      << "    }\n  }\n";
    s << nest_arm_code(N);
    return s.str();
  }

  // C++ of the summaries at a window check of block h
  std::string summary_code(const std::vector<Cycle>& cs, const char* RT) {
    std::ostringstream s;
    for (const Cycle& C : cs) {
      s << "    { // loop summary: blocks";
      for (int b : C.blocks) s << " " << b;
      s << "\n      const int64_t LEN_ = " << C.len << ";\n"
        << "      int64_t H_ = HARD > ret ? (int64_t)((uint64_t)(HARD - 1u - ret) / (uint64_t)LEN_) : -1;\n";
      for (auto& iv : C.r_iv) s << "      const uint32_t dr" << iv.first << "_ = " << iv.second << ";\n";
      for (auto& iv : C.a_iv) s << "      const int64_t da" << iv.first << "_ = (int64_t)(" << iv.second << ");\n";
      auto val = [&](const Opnd& o, std::string& v0, std::string& d) {
        if (o.kind == 3) { v0 = i64lit(o.imm); d = "0ll"; }
        else if (o.kind == 1) { v0 = "(int64_t)(int32_t)(" + o.e + ")"; d = "0ll"; }
        else { v0 = "(int64_t)(int32_t)(uint32_t)(" + r(o.iv) + " + " + o.e + ")"; d = "(int64_t)(int32_t)dr" + std::to_string(o.iv) + "_"; }
      };
      std::vector<std::string> l0, ld, r0, rdl;
      for (size_t k = 0; k < C.exits.size(); ++k) {
        const Exit& X = C.exits[k];
        std::string a, b, c, d;
        if (!X.konst) { val(X.l, a, b); val(X.r, c, d); }
        l0.push_back(a); ld.push_back(b); r0.push_back(c); rdl.push_back(d);
        if (!X.konst) {
          if (X.l.kind == 2) s << "      H_ = sfg_min64(H_, sfg_wrap_h(" << a << ", " << b << "));\n";
          if (X.r.kind == 2) s << "      H_ = sfg_min64(H_, sfg_wrap_h(" << c << ", " << d << "));\n";
        }
      }
      s << "      if (H_ >= 2";
      for (const std::string& gd : C.guards) s << " && " << gd;
      s << ") {\n        int64_t T_ = SFG_I64MAX;\n";
      for (size_t k = 0; k < C.exits.size(); ++k) {
        const Exit& X = C.exits[k];
        if (X.konst) s << "        if (" << X.pe << ") T_ = 0;\n";
        else
          s << "        T_ = sfg_min64(T_, sfg_first_t(" << X.cmp << ", (" << l0[k] << ") - (" << r0[k] << "), (" << ld[k]
            << ") - (" << rdl[k] << "), H_));\n";
      }
      s << "        const int64_t s_ = (T_ <= H_ ? T_ : H_ + 1) - 1;\n"
        << "        if (s_ >= 2) {\n";
      for (auto& iv : C.r_iv) s << "          " << r(iv.first) << " = (uint32_t)(" << r(iv.first) << " + (uint32_t)s_ * dr" << iv.first << "_);\n";
      for (auto& iv : C.a_iv)
        s << "          " << a(iv.first) << " = " << a(iv.first) << " + (" << AT() << ")s_ * (" << AT() << ")da" << iv.first << "_;\n";
      for (int e : C.edges)
        s << "          { const uint64_t o_ = J.ec[" << e << "]; if (o_ + (uint64_t)s_ > 0xFFFFFFFFull) J.ovf = true; J.ec[" << e
          << "] = (uint32_t)(o_ + (uint64_t)s_); }\n";
      s << "          ret += (" << RT << ")(s_ * LEN_);\n        }\n      }\n    }\n";
    }
    return s.str();
  }

  int cur_na = 0;
  // Pointer registers hold unbounded integers in the reference (executor.py:297-310).
  // A kernel whose pointer registers only ever receive pointer parameters
  // (simulated addresses, < 2^40), small immediates and sums with i32 registers or
  // immediates below 2^31 stays below 2^40 + budget * 2^31 < 2^62 in magnitude
  // for budgets below 2^30: such kernels ("narrow") keep them in int64 and drop
  // the 128-bit arithmetic and high-word checks.  A 64-bit load into a pointer
  // register (values up to 2^64) or any larger immediate keeps the 128-bit form.
  bool narrow = false;
  // fbits[r]: the exact bits of f-register r can be observed (it is copied by a
  // mov or stored).  A loaded f32 is quieted (sNaN -> qNaN, executor.py loads
  // through a double) only then: fadd/fsub/fmul (sfg_fop quiets its first NaN
  // operand itself), float setp and cvt cannot tell a signaling NaN from its
  // quieted form.
  // A store observes its value's bits unless it is write-only into memory that is
  // dead after the launch (the `wo` stores of emit_mem: a pointer parameter's record
  // that no load of the kernel reaches, no untagged load, no later launch or
  // readout) -- then fadd/fsub/fmul results headed only there need no x86 NaN
  // payload fix-up either (sfg_fop_any: any NaN is as good as another to fadd /
  // fmul / setp / cvt and to a store nobody reads).
  // fexact[r]: the NaN payload of f register r matters -- r's bits are observable,
  // or r is an operand of a payload-exact fadd/fsub/fmul (which propagates the
  // payload of its first NaN operand); closed backwards over the arithmetic.
  std::vector<char> fbits, fexact;
  void f_observers(const sfg_ins* I, int n, int regs, const std::vector<std::vector<int>>& tags) {
    fbits.assign(regs > 0 ? regs : 1, 0);
    for (int i = 0; i < n; ++i) {
      const sfg_ins& x = I[i];
      if (x.op == SFG_MOV && x.mode == SFG_CLS_F && !(x.flags & SFG_F_S1_IMM)) fbits[x.s1] = 1;
      if (x.op == SFG_ST && x.mode == SFG_MK_F32 && !(x.flags & SFG_F_S2_IMM)) {
        const int tg = tags[i][x.s1];
        const bool wo = tg > 0 && dead_now && !any_untagged_load && !loaded[tg - 1];
        if (!wo) fbits[x.s2] = 1;
      }
    }
    fexact = fbits;
    for (bool changed = true; changed;) {
      changed = false;
      for (int i = 0; i < n; ++i) {
        const sfg_ins& x = I[i];
        if ((x.op != SFG_FADD && x.op != SFG_FSUB && x.op != SFG_FMUL) || !fexact[x.dst]) continue;
        if (!(x.flags & SFG_F_S1_IMM) && !fexact[x.s1]) fexact[x.s1] = changed = true;
        if (!(x.flags & SFG_F_S2_IMM) && !fexact[x.s2]) fexact[x.s2] = changed = true;
      }
    }
  }
  std::string AT() const { return narrow ? "int64_t" : "i128"; }
  bool narrow_ok(const sfg_ins* I, int n) const {
    if (P.budget >= (1ull << 30)) return false;
    const int64_t small = 1ll << 31, addr = 1ll << 40;
    for (int i = 0; i < n; ++i) {
      const sfg_ins& x = I[i];
      if ((x.op == SFG_LD || x.op == SFG_ST) && (x.imm2 >= small || x.imm2 <= -small)) return false;
      if (x.op == SFG_LD && x.mode == SFG_MK_B64) return false;
      if (x.op == SFG_MOV && x.mode == SFG_CLS_A && (x.flags & SFG_F_S1_IMM) &&
          ((x.flags & SFG_F_U64IMM) || x.imm1 >= addr || x.imm1 <= -addr)) return false;
      if ((x.op == SFG_ADD || x.op == SFG_SUB || x.op == SFG_MUL) && x.mode == SFG_CLS_A) {
        if (x.op == SFG_MUL) return false;
        if ((x.flags & SFG_F_S2_IMM) && (x.imm2 >= small || x.imm2 <= -small)) return false;
      }
    }
    return true;
  }
  // stores of the kernel being emitted: written[q] = some store's base carries the
  // tag of pointer parameter q; any_untagged_store = some store's base has no
  // static tag (could reach any record)
  std::vector<char> written, loaded;
  bool any_untagged_store = false, any_untagged_load = false;
  // bit k: memory is dead after every launch of kernel k (no later launch in the
  // COMPUTE script, no readouts) -- its stores can only be observed by its own loads
  uint32_t dead_kernels = 0;
  LaneCaps caps;
  const sfg_hostop* hostops = nullptr;   // the COMPUTE script (array-argument access masks)
  size_t n_hostops = 0;
  const sfg_binding* binds = nullptr;

  // Array arguments of the COMPUTE script that no launch ever stores through (ro) or
  // loads through (wo), from the kernels' pointer-tag flow: a store / load with no
  // static tag could reach any record and clears every bit.  The bulk pass reads
  // an ro array of an unmutated child straight from its parent's corpus payload
  // and leaves a wo array unbuilt (its bytes are never read), exec_core.cuh.
  void array_masks(uint32_t& ro, uint32_t& wo) {
    ro = wo = 0;
    for (int a = 0; a < P.n_args; ++a)
      if (P.arg_kind[a] == SFG_V_ARR) { ro |= 1u << a; wo |= 1u << a; }
    if (!hostops || !binds) { ro = wo = 0; return; }
    std::vector<std::vector<char>> kw(P.n_kernels), kl(P.n_kernels);
    std::vector<char> kuw(P.n_kernels, 0), kul(P.n_kernels, 0);
    for (int k = 0; k < P.n_kernels; ++k) {
      const sfg_kernel& KD = P.kernels[k];
      KInfo K{KD.ins_base, KD.n_ins, KD.regs, 0, 0, 0};
      for (int q = 0; q < KD.n_params; ++q) {
        if (KD.ptype[q] == 0) ++K.nr;
        else if (KD.ptype[q] == 1) ++K.nf;
        else ++K.na;
      }
      const sfg_ins* I = ins + K.base;
      const std::vector<int> starts = block_starts(I, K.n);
      std::vector<int> blk_of;
      const auto tags = tag_flow(I, K.n, K, starts, blk_of);
      kw[k].assign(K.na > 0 ? K.na : 1, 0);
      kl[k].assign(K.na > 0 ? K.na : 1, 0);
      for (int i = 0; i < K.n; ++i) {
        if (I[i].op != SFG_ST && I[i].op != SFG_LD) continue;
        const int tg = tags[i][I[i].s1];
        const bool st = I[i].op == SFG_ST;
        if (tg > 0) (st ? kw[k] : kl[k])[tg - 1] = 1;
        else if (tg != TAG_BOT) (st ? kuw[k] : kul[k]) = 1;
      }
    }
    for (size_t h = 0; h < n_hostops; ++h) {
      const sfg_hostop& op = hostops[h];
      if (op.kind != SFG_H_LAUNCH) continue;
      const sfg_kernel& KD = P.kernels[op.kernel];
      if (kuw[op.kernel]) ro = 0;
      if (kul[op.kernel]) wo = 0;
      int q = 0;   // pointer-parameter index of binding b
      for (int b = 0; b < op.n_bind && b < KD.n_params; ++b) {
        if (KD.ptype[b] != 2) continue;
        const sfg_binding& B = binds[op.bind_base + b];
        if (B.form == SFG_B_ARG && B.idx >= 0 && B.idx < 32) {
          if (kw[op.kernel][q]) ro &= ~(1u << B.idx);
          if (kl[op.kernel][q]) wo &= ~(1u << B.idx);
        }
        ++q;
      }
    }
  }

  bool dead_now = false;

  std::string src_r(const sfg_ins& x, int slot) {
    const bool imm = slot == 1 ? (x.flags & SFG_F_S1_IMM) : (x.flags & SFG_F_S2_IMM);
    const int64_t v = slot == 1 ? x.imm1 : x.imm2;
    return imm ? u32lit(v) : r(slot == 1 ? x.s1 : x.s2);
  }
  std::string src_f(const sfg_ins& x, int slot) {
    const bool imm = slot == 1 ? (x.flags & SFG_F_S1_IMM) : (x.flags & SFG_F_S2_IMM);
    const int64_t v = slot == 1 ? x.imm1 : x.imm2;
    return imm ? u32lit(v) : f(slot == 1 ? x.s1 : x.s2);
  }
  std::string src_i64(const sfg_ins& x, int slot) {
    const bool imm = slot == 1 ? (x.flags & SFG_F_S1_IMM) : (x.flags & SFG_F_S2_IMM);
    const int64_t v = slot == 1 ? x.imm1 : x.imm2;
    return imm ? i64lit(v) : "(int64_t)(int32_t)" + r(slot == 1 ? x.s1 : x.s2);
  }

  static const char* cmp(int m) {
    static const char* c[] = {"==", "!=", "<", "<=", ">", ">="};
    return c[m];
  }

  // one non-control instruction (everything except BRA/EXIT); j = index in block
  void emit_plain(const sfg_ins& x, int kidx, int iid, int j, bool slow, int tag) {
    switch (x.op) {
      case SFG_MOV:
        if (x.mode == SFG_CLS_R) o << "    " << r(x.dst) << " = " << src_r(x, 1) << ";\n";
        else if (x.mode == SFG_CLS_F) o << "    " << f(x.dst) << " = " << src_f(x, 1) << ";\n";
        else if (x.mode == SFG_CLS_A) {
          if (x.flags & SFG_F_S1_IMM) {
            if (x.flags & SFG_F_U64IMM) o << "    " << a(x.dst) << " = (" << AT() << ")(uint64_t)" << hex64(x.imm1) << "; ";
            else o << "    " << a(x.dst) << " = (" << AT() << ")" << i64lit(x.imm1) << "; ";
            o << t(x.dst) << " = 0;\n";
          } else {
            o << "    " << a(x.dst) << " = " << a(x.s1) << "; " << t(x.dst) << " = " << t(x.s1) << ";\n";
          }
        } else {
          o << "    " << p(x.dst) << " = " << p(x.s1) << ";\n";
        }
        break;
      case SFG_ADD:
      case SFG_SUB:
      case SFG_MUL: {
        const char* opc = x.op == SFG_ADD ? "+" : x.op == SFG_SUB ? "-" : "*";
        if (x.mode == SFG_CLS_A) {
          o << "    " << a(x.dst) << " = " << a(x.s1) << " " << opc << " (" << AT() << ")" << src_i64(x, 2) << "; " << t(x.dst)
            << " = " << t(x.s1) << ";\n";
        } else {
          o << "    " << r(x.dst) << " = (uint32_t)(" << src_r(x, 1) << " " << opc << " " << src_r(x, 2) << ");\n";
        }
        break;
      }
      case SFG_FADD:
      case SFG_FSUB:
      case SFG_FMUL:
        o << "    " << f(x.dst) << " = " << (fexact[x.dst] ? "sfg_fop(" : "sfg_fop_any(") << (int)x.op << ", "
          << src_f(x, 1) << ", " << src_f(x, 2) << ");\n";
        break;
      case SFG_SETP:
        if (x.flags & SFG_F_FLOAT)
          o << "    " << p(x.dst) << " = sfg_f(" << src_f(x, 1) << ") " << cmp(x.mode) << " sfg_f(" << src_f(x, 2) << ");\n";
        else
          o << "    " << p(x.dst) << " = " << src_i64(x, 1) << " " << cmp(x.mode) << " " << src_i64(x, 2) << ";\n";
        break;
      case SFG_CVT:
        if (x.mode == SFG_CVT_F_FROM_I) {
          if (x.flags & SFG_F_S1_IMM) o << "    " << f(x.dst) << " = " << u32lit(x.imm1) << ";\n";
          else o << "    " << f(x.dst) << " = sfg_b(__int2float_rn((int32_t)" << r(x.s1) << "));\n";
        } else {
          if (x.flags & SFG_F_S1_IMM) o << "    " << r(x.dst) << " = " << u32lit(x.imm1) << ";\n";
          else o << "    " << r(x.dst) << " = sfg_cvt_f2i(" << f(x.s1) << ");\n";
        }
        break;
      case SFG_SREG: {
        static const char* names[] = {"tid", "block", "ctaid", "grid"};
        o << "    " << r(x.dst) << " = (uint32_t)" << names[x.mode] << ";\n";
        break;
      }
      case SFG_LD:
      case SFG_ST:
        emit_mem(x, kidx, iid, j, slow, tag);
        break;
      default:
        break;
    }
  }

  void emit_kernel(int kidx) {
    const sfg_kernel& KD = P.kernels[kidx];
    KInfo K{KD.ins_base, KD.n_ins, KD.regs, 0, 0, 0};
    for (int q = 0; q < KD.n_params; ++q) {
      if (KD.ptype[q] == 0) ++K.nr;
      else if (KD.ptype[q] == 1) ++K.nf;
      else ++K.na;
    }
    cur_na = K.na;
    const sfg_ins* I = ins + K.base;
    narrow = narrow_ok(I, K.n);
    const std::vector<int> starts = block_starts(I, K.n);
    std::vector<int> blk_of;
    const auto tags = tag_flow(I, K.n, K, starts, blk_of);
    const int nb = (int)starts.size();
    written.assign(K.na > 0 ? K.na : 1, 0);
    loaded.assign(K.na > 0 ? K.na : 1, 0);
    any_untagged_store = any_untagged_load = false;
    for (int i = 0; i < K.n; ++i) {
      if (I[i].op != SFG_ST && I[i].op != SFG_LD) continue;
      const int tg = tags[i][I[i].s1];
      const bool st = I[i].op == SFG_ST;
      if (tg > 0) (st ? written : loaded)[tg - 1] = 1;
      else if (tg != TAG_BOT) (st ? any_untagged_store : any_untagged_load) = true;  // BOT: unreachable
    }
    dead_now = (dead_kernels >> kidx) & 1u;
    f_observers(I, K.n, K.regs, tags);

    o << "template <bool PAR>\nstatic __device__ __forceinline__ int sim_" << kidx
      << "(JitRunner& J, const sfg_prog& P, Lane& L, Mem& M, sfg_verdict& V, const Pre& pre, int ctaid, int tid, "
         "int grid, int block, uint64_t& total) {\n";
    for (int q = 0; q < K.regs; ++q) {
      o << "  uint32_t " << r(q) << " = " << (q < K.nr ? "pre.r[" + std::to_string(q) + "]" : std::string("0u"))
        << ", " << f(q) << " = " << (q < K.nf ? "pre.f[" + std::to_string(q) + "]" : std::string("0u")) << ";\n";
      o << "  " << AT() << " " << a(q) << " = " << (q < K.na ? "(" + AT() + ")pre.a[" + std::to_string(q) + "]" : std::string("0"))
        << "; int32_t " << t(q) << " = " << (q < K.na ? "pre.ap[" + std::to_string(q) + "]" : std::string("0"))
        << "; bool " << p(q) << " = false;\n";
    }
    for (int q = 0; q < K.na; ++q) {
      const std::string Q = std::to_string(q);
      o << "  const int32_t pt" << Q << " = pre.ap[" << Q << "];\n";
      o << "  int64_t pb" << Q << " = 0, psz" << Q << " = 0, pw" << Q << " = 0; int psp" << Q << " = -1; bool pok" << Q
        << " = false; uint8_t* pp" << Q << " = M.work;\n";
      o << "  if (pt" << Q << " > 0) { const LRec& R_ = L.rec[pt" << Q << " - 1]; pb" << Q << " = R_.base; psz" << Q
        << " = R_.size; psp" << Q << " = R_.space; pok" << Q
        << " = (R_.flags & (R_RES | R_FREED | R_BASE)) == R_RES; pp" << Q << " = M.work + R_.phys; pw" << Q << " = R_.phys; }\n";
      o << "  const bool pk" << Q << "_0 = pok" << Q << " && psp" << Q << " == 0, pk" << Q << "_1 = pok" << Q << " && psp"
        << Q << " == 1, pk" << Q << "_2 = pok" << Q << " && psp" << Q << " == 2;\n";
      // per access width: last valid payload offset, and "the payload holds W bytes"
      // folded into the space flags (unused combinations are dead code)
      for (int W : {1, 2, 4, 8}) {
        const std::string Ws = std::to_string(W);
        o << "  const uint64_t pl" << Q << "_" << Ws << " = (uint64_t)(psz" << Q << " - " << Ws << ");\n";
        for (int sp = 0; sp < 3; ++sp)
          o << "  const bool pk" << Q << "_" << sp << "_" << Ws << " = pk" << Q << "_" << sp << " && psz" << Q
            << " >= " << Ws << ";\n";
      }
    }
    // Retired-budget checks.  The fast copy of a block retires its instructions
    // without per-instruction checks; the budget (or soft cap / poll limit) is tested
    // only at check blocks -- the entry and every target of a backward branch, so
    // every cycle passes one -- against the longest run of instructions the thread
    // can retire before the next check block (paths between check blocks are
    // forward, hence acyclic).  Near the limit the slow copies count and test
    // every instruction (executor.py:411-415) until the next check block.
    std::vector<char> chk(nb, 0);
    chk[0] = 1;
    for (int b = 0; b < nb; ++b) {
      const int e = b + 1 < nb ? starts[b + 1] : K.n;
      const sfg_ins& last = I[e - 1];
      if (last.op == SFG_BRA && blk_of[last.target] <= b) chk[blk_of[last.target]] = 1;
    }
    std::vector<int64_t> span(nb, 0);  // longest checked run from the block's start
    for (int b = nb - 1; b >= 0; --b) {
      const int s0 = starts[b], e = b + 1 < nb ? starts[b + 1] : K.n;
      const sfg_ins& last = I[e - 1];
      const int64_t cost = last.op == SFG_EXIT ? e - s0 - 1 : e - s0;
      int64_t tail = 0;
      auto succ = [&](int sb) { if (!chk[sb]) tail = std::max(tail, span[sb]); };
      if (last.op == SFG_BRA) {
        succ(blk_of[last.target]);
        if ((last.flags & SFG_F_PRED) && e < K.n) succ(blk_of[e]);
      } else if (last.op != SFG_EXIT && e < K.n) {
        succ(blk_of[e]);
      }
      span[b] = cost + tail;
    }
    // slow copies continue in slow copies up to the next check block
    auto dest = [&](int tb) { return std::string(chk[tb] ? "B" : "S") + std::to_string(tb); };
    // 32-bit counters when the budget allows (every limit is <= the budget)
    const bool narrow = P.budget < (1ull << 30);
    const char* RT = narrow ? "uint32_t" : "uint64_t";
    o << "  " << RT << " ret = 0; int rc = RUN_EXIT; const " << RT << " BUD = (" << RT << ")P.budget;\n";
    // fast-path limit: the budget, or the remaining soft cap of the input (deferral)
    o << "  const uint64_t SOFT = J.soft_cap; bool SFT = SOFT != 0ull && (SOFT <= total || SOFT - total < (uint64_t)BUD);\n";
    o << "  " << RT << " HARD = SFT ? (" << RT << ")(SOFT > total ? SOFT - total : 0ull) : BUD;\n";
    // group-parallel mode: stop at poll points every kPoll retired instructions to see
    // whether this thread can still matter (run_launch_group)
    // bulk pass (soft cap on): poll every kStrag retired instructions whether the rest of
    // the warp's batch has finished; a straggler past kStragMin is deferred then
    // loop summaries at the window checks of check blocks (analyse_cycle); a kernel
    // with any runs windowed in every mode so that a long pure-register loop is met
    std::vector<std::vector<Cycle>> sums(nb);
    bool has_sum = false;
    if (loop_summaries)
      for (int b = 0; b < nb; ++b)
        if (chk[b] && span[b] > 0) {
          sums[b] = cycles_at(I, K.n, starts, blk_of, K.regs, b);
          has_sum |= !sums[b].empty();
        }
    for (auto& v : sums) n_summaries += (int)v.size();
    // nest summaries (analyse_nest): loops with memory accesses and inner loops
    std::vector<Nest> nests(nb);
    std::vector<char> has_nest(nb, 0);
    if (loop_summaries && nest_summaries)
      for (int b = 0; b < nb; ++b)
        if (chk[b] && span[b] > 0 && analyse_nest(I, K.n, starts, blk_of, K.regs, b, tags, nests[b])) {
          has_nest[b] = 1;
          has_sum = true;
          ++n_nests;
          if (getenv("SFG_LOOPSUM_DEBUG")) {
            fprintf(stderr, "nest at %d:", b);
            for (int x : nests[b].blocks) fprintf(stderr, " %d", x);
            fprintf(stderr, " ivs %zu exit %d guards %zu distinct %zu edges %zu\n", nests[b].r_iv.size(),
                    (int)nests[b].has_x, nests[b].guards.size(), nests[b].distinct.size(), nests[b].edges.size());
          }
          const std::string H = std::to_string(b);
          o << "  bool ns" << H << " = false; " << RT << " nsr" << H << " = 0, nsn" << H << " = (" << RT
            << ")kNestArm; uint32_t nse" << H << "[" << (nests[b].edges.empty() ? 1 : nests[b].edges.size()) << "];\n";
        }
    o << "  " << RT << " LIM = PAR ? ((HARD > (" << RT << ")kPoll) ? (" << RT << ")kPoll : HARD)\n"
         "            : (((J.done != nullptr || " << (has_sum ? "true" : "false") << ") && HARD > (" << RT << ")kStrag) ? ("
      << RT << ")kStrag : HARD);\n";
    o << "  (void)grid; (void)block; (void)ctaid; (void)tid;\n";
    for (int b = 0; b < nb; ++b) {
      const int s0 = starts[b], e = b + 1 < nb ? starts[b + 1] : K.n;
      const int len = e - s0;
      const std::string sp = std::to_string(span[b]) + (narrow ? "u" : "ull");
      for (int pass = 0; pass < 2; ++pass) {
        const bool slow = pass == 1;
        o << (slow ? "S" : "B") << b << ":\n";
        if (slow && has_nest[b]) o << "  ns" << b << " = false;\n";   // a trip measured across the slow path is void
        if (!slow && chk[b] && span[b] > 0) {
          // a cycle summary at h moves the thread between arrivals: a pending nest measurement is void
          const std::string arm = has_nest[b] ? "      ns" + std::to_string(b) + " = false;\n" : std::string();
          o << "  if (ret + " << sp << " >= LIM) {\n"
            << "    if constexpr (PAR) { if (LIM < HARD) { if (J.poll()) { rc = RUN_ABORT; goto done; }\n"
            << summary_code(sums[b], RT) << arm
            << "      LIM = (HARD - ret > " << sp << " + kPoll) ? ret + " << sp << " + kPoll : HARD; goto B" << b << "; } }\n"
            << "    else { if (LIM < HARD) { if (J.done != nullptr && J.straggler(total + ret)) { rc = RUN_DEFER; goto done; }\n"
            << summary_code(sums[b], RT) << arm
            << "      LIM = (HARD - ret > " << sp << " + kStrag) ? ret + " << sp << " + kStrag : HARD; goto B" << b << "; } }\n"
            << "    if (SFT) { rc = RUN_DEFER; goto done; } goto S" << b << "; }\n";
          if (has_nest[b]) o << nest_skip_code(nests[b], RT);
        }
        for (int i = s0; i < e; ++i) {
          const sfg_ins& x = I[i];
          const int j = i - s0;
          if (slow) o << "  ++ret;\n";
          if (x.op == SFG_EXIT) {
            if (!slow) o << "  ret += " << len << ";\n";
            o << "  goto done;\n";
            break;
          }
          if (x.op == SFG_BRA) {
            const std::string tgt = std::to_string(blk_of[x.target]);
            const std::string nxt = std::to_string(i + 1 < K.n ? blk_of[i + 1] : 0);
            const std::string bud = slow ? "if (ret >= BUD) { rc = RUN_BUDGET; goto done; } " : "ret += " + std::to_string(len) + "; ";
            const int tb = blk_of[x.target], nbk = i + 1 < K.n ? blk_of[i + 1] : 0;
            const std::string gt = slow ? dest(tb) : "B" + tgt, gn = slow ? dest(nbk) : "B" + nxt;
            if (x.flags & SFG_F_PRED) {
              const std::string cond = std::string(x.flags & SFG_F_PNEG ? "!" : "") + p(x.s1);
              o << "  if (" << cond << ") { " << edge(x.edge_tk) << bud << "goto " << gt << "; }\n";
              o << "  else { " << edge(x.edge_ft) << bud << "goto " << gn << "; }\n";
            } else {
              o << "  " << edge(x.edge_tk) << bud << "goto " << gt << ";\n";
            }
            break;
          }
          emit_plain(x, kidx, i, j, slow, tags[i][x.op == SFG_LD || x.op == SFG_ST ? x.s1 : 0]);
          if (i == e - 1) {  // block ends by falling through into the next leader
            o << "  " << edge(x.edge_ft);
            if (slow) o << "if (ret >= BUD) { rc = RUN_BUDGET; goto done; } ";
            else o << "ret += " << len << "; ";
            o << "goto " << (slow ? dest(blk_of[i + 1]) : "B" + std::to_string(blk_of[i + 1])) << ";\n";
          } else if (slow) {
            o << "  if (ret >= BUD) { rc = RUN_BUDGET; goto done; }\n";
          }
        }
      }
    }
    o << "done:\n  total += ret;\n  return rc;\n}\n\n";
  }

  bool loop_summaries = true;
  bool nest_summaries = true;
  uint64_t strag_min = 8192;   // bulk pass: retired count past which the batch's last lane is deferred
  int n_summaries = 0, n_nests = 0;
  int tail_minb = 12;
  int bulk_minb = 4;

  std::string run(int n_edges, uint64_t max_edge_events) {
    edge_ovf_checks = max_edge_events >= 0xFFFFFFFFull;
    const int NE = n_edges > 0 ? n_edges : 1;
    uint32_t ro_mask = 0, wo_mask = 0;
    array_masks(ro_mask, wo_mask);
    if (const char* am = getenv("SFG_ARRAY_ALIAS")) if (atoi(am) == 0) ro_mask = wo_mask = 0;
    o << "#define SFG_RO_ARGS " << ro_mask << "u\n#define SFG_WO_ARGS " << wo_mask << "u\n";
    o << "#define SFG_LANE_RECS " << caps.recs << "\n#define SFG_LANE_Q " << caps.q << "\n#define SFG_LANE_FREE "
      << caps.freel << "\n#define SFG_LANE_NAMED " << caps.named << "\n#define SFG_LANE_ARGS " << caps.args
      << "\n#define SFG_LANE_PARAMS " << caps.params << "\n";
    o << "#include \"exec_core.cuh\"\n\nnamespace {\n\n";
    o << "constexpr uint32_t kPoll = 4096u;\n";
    o << "constexpr uint32_t kNestArm = 4096u;   // retired instructions between nest-summary attempts\n";
    // loop-summary helpers (see analyse_cycle)
    o << "#define SFG_I64MAX 0x7FFFFFFFFFFFFFFFll\n";
    o << "SFG_DEV int64_t sfg_min64(int64_t a, int64_t b) { return a < b ? a : b; }\n"
         "// trips t >= 0 for which x0 + t*d stays inside int32 (x0 an int32 value)\n"
         "SFG_DEV int64_t sfg_wrap_h(int64_t x0, int64_t d) {\n"
         "  if (d > 0) return (2147483647ll - x0) / d;\n"
         "  if (d < 0) return (x0 + 2147483648ll) / (-d);\n"
         "  return SFG_I64MAX;\n}\n"
         "// first t in [0, H] with  a + t*b <cmp> 0  (cmp: == != < <= > >=), else SFG_I64MAX\n"
         "SFG_DEV int64_t sfg_first_t(int cmp, int64_t a, int64_t b, int64_t H) {\n"
         "  int64_t t = SFG_I64MAX;\n"
         "  if (cmp == 4 || cmp == 5) { a = -a; b = -b; cmp = cmp == 4 ? 2 : 3; }\n"
         "  switch (cmp) {\n"
         "    case 0: if (b == 0) t = a == 0 ? 0 : SFG_I64MAX; else if ((-a) % b == 0 && (-a) / b >= 0) t = (-a) / b; break;\n"
         "    case 1: t = a != 0 ? 0 : (b != 0 ? 1 : SFG_I64MAX); break;\n"
         "    case 2: t = a < 0 ? 0 : (b < 0 ? a / (-b) + 1 : SFG_I64MAX); break;\n"
         "    default: t = a <= 0 ? 0 : (b < 0 ? (a + (-b) - 1) / (-b) : SFG_I64MAX); break;\n"
         "  }\n"
         "  return t <= H ? t : SFG_I64MAX;\n}\n";
    o << "constexpr uint32_t kStrag = 2048u;\nconstexpr uint64_t kStragMin = " << strag_min << "ull;\n\n";
    o << "struct JitRunner {\n  uint32_t ec[" << NE << "], ecs[" << NE
      << "];\n  bool ovf, ovfs;\n  uint64_t soft_cap;\n"
      << "  uint32_t* tags = nullptr;\n  int ntags = 0, t = 0;\n  uint32_t me = 0;\n  GroupSmem* gs = nullptr;\n  int* waw = nullptr;\n"
         "  int* done = nullptr;  // bulk: inputs of this warp's batch finished so far\n  int batch_n = 0;\n"
         "  SFG_DEV bool straggler(uint64_t retired) const {\n"
         "    return retired >= kStragMin && *reinterpret_cast<volatile const int*>(done) >= batch_n - 1;\n  }\n"
      << "  SFG_DEV void begin_input() {\n#pragma unroll\n    for (int e = 0; e < " << NE << "; ++e) ec[e] = 0u;\n    ovf = false;\n"
         "    asm volatile(\"mov.u32 %0, 0;\" : \"=r\"(J_dyn));  // opaque 0: keeps ecs[] out of registers\n  }\n"
      // the chunk-start copy lives in local memory (a dynamically indexed array), so
      // it costs no registers in the simulated code
      << "  SFG_DEV void save_edges() {\n#pragma unroll\n    for (int e = 0; e < " << NE << "; ++e) ecs[e ^ J_dyn] = ec[e];\n    ovfs = ovf;\n  }\n"
      << "  SFG_DEV void restore_edges() {\n#pragma unroll\n    for (int e = 0; e < " << NE << "; ++e) ec[e] = ecs[e ^ J_dyn];\n    ovf = ovfs;\n  }\n"
      << "  int J_dyn = 0;\n"
      << "  SFG_DEV void par_begin(const Grp& g, int thread, int nt) {\n"
         "    tags = g.tags; ntags = nt; t = thread; me = (uint32_t)g.gl + 1u; gs = g.sm; waw = &g.sm->waw;\n  }\n"
      << "  SFG_DEV void par_end() {}\n"
      << "  SFG_DEV void set_input(const ExecView&, int) {}\n  SFG_DEV void end_input(const ExecView&, int) {}\n"
      << "  SFG_DEV bool poll() const {\n"
         "    const int s = *reinterpret_cast<volatile const int*>(&gs->stop_min);\n"
         "    const int d = *reinterpret_cast<volatile const int*>(&gs->defer_min);\n"
         "    return *reinterpret_cast<volatile const int*>(&gs->conflict) != 0 || t > (s < d ? s : d);\n  }\n"
      << "  SFG_DEV void flush(uint32_t* row, bool& o) {\n#pragma unroll\n    for (int e = 0; e < " << n_edges
      << "; ++e) row[e] = ec[e];\n    o = ovf;\n  }\n"
      << "  SFG_DEV void flush_group(uint32_t* row, bool& o, unsigned mask, bool leader) {\n"
         "    bool big = false;\n#pragma unroll\n    for (int e = 0; e < " << n_edges << "; ++e) {\n"
         "      const uint32_t lo = __reduce_add_sync(mask, ec[e] & 0xFFFFu), hi = __reduce_add_sync(mask, ec[e] >> 16);\n"
         "      const uint64_t v = ((uint64_t)hi << 16) + lo;\n"
         "      big |= v > 0xFFFFFFFFull;\n"
         "      if (leader) row[e] = (uint32_t)v;\n    }\n"
         "    o = __any_sync(mask, ovf) || big;\n  }\n"
      << "  template <bool PAR>\n  SFG_DEV int run_thread(const sfg_prog& P, int k, Lane& L, Mem& M, sfg_verdict& V, const Pre& pre, int ctaid, "
         "int tid, int grid, int block, uint64_t& total);\n};\n\n";
    for (int k = 0; k < P.n_kernels; ++k) emit_kernel(k);
    o << "template <bool PAR>\nSFG_DEV int JitRunner::run_thread(const sfg_prog& P, int k, Lane& L, Mem& M, sfg_verdict& V, const Pre& pre, "
         "int ctaid, int tid, int grid, int block, uint64_t& total) {\n  switch (k) {\n";
    for (int k = 0; k < P.n_kernels; ++k)
      o << "    case " << k << ": return sim_" << k << "<PAR>(*this, P, L, M, V, pre, ctaid, tid, grid, block, total);\n";
    o << "    default: return RUN_FATAL;\n  }\n}\n\n}  // namespace\n\n";
    // persistent bulk kernel.  Group-parallel (E.group = G > 1): a warp takes 32/G
    // consecutive inputs, one per group of G lanes.  Thread-sequential (G = 1):
    // mode 0 every lane fetches its next input independently; mode 1 a warp fetches
    // 32 consecutive inputs and re-fetches after all 32 finished.
    o << "#define SFG_BULK_MINB " << bulk_minb << "\n";
    o << "extern \"C\" __global__ void __launch_bounds__(128, SFG_BULK_MINB) sfg_jit_execute(const __grid_constant__ sfg_prog P, const __grid_constant__ ExecView E, int* next, int mode) {\n"
         "  extern __shared__ __align__(16) uint8_t smem[];\n"
         "  JitRunner R;\n"
         "  R.soft_cap = E.soft_cap;\n"
         "  const int lane = threadIdx.x & 31;\n"
         "  const int G = E.group;\n"
         "  const int NL = E.n_live ? *E.n_live : E.n;   // inputs in the schedule\n"
         "  if (G <= 1) {\n"
         "    const Grp g{1, 0, 1u << lane, nullptr, nullptr, 0};\n"
         "    if (mode == 0) {\n"
         "      for (int i = atomicAdd(next, 1); i < NL; i = atomicAdd(next, 1)) run_input<false>(P, E, E.order ? E.order[i] : i, R, g);\n"
         "      return;\n"
         "    }\n"
         "    __shared__ int s_done[32];\n"
         "    const int w = threadIdx.x >> 5;\n"
         "    while (true) {\n"
         "      int b = 0;\n"
         "      if (lane == 0) b = atomicAdd(next, 32);\n"
         "      b = __shfl_sync(0xffffffffu, b, 0);\n"
         "      if (b >= NL) break;\n"
         "      if (lane == 0) s_done[w] = 0;\n"
         "      __syncwarp();\n"
         "      if (E.soft_cap) { R.done = &s_done[w]; R.batch_n = NL - b < 32 ? NL - b : 32; }\n"
         "      if (b + lane < NL) {\n"
         "        run_input<false>(P, E, E.order ? E.order[b + lane] : b + lane, R, g);\n"
         "        atomicAdd(&s_done[w], 1);\n"
         "      }\n"
         "      __syncwarp();\n"
         "    }\n"
         "    return;\n"
         "  }\n"
         "  const int per = 32 / G, gi = lane / G;\n"
         "  GroupSmem* sm = reinterpret_cast<GroupSmem*>(smem + (size_t)((threadIdx.x >> 5) * per + gi) * group_stride(E.tag_cap));\n"
         "  const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u) << (gi * G);\n"
         "  const Grp g{G, lane % G, gmask, sm, reinterpret_cast<uint32_t*>(sm + 1), E.tag_cap};\n"
         "  while (true) {\n"
         "    int b = 0;\n"
         "    if (lane == 0) b = atomicAdd(next, per);\n"
         "    b = __shfl_sync(0xffffffffu, b, 0);\n"
         "    if (b >= NL) break;\n"
         "    if (b + gi < NL) run_input<true>(P, E, E.order ? E.order[b + gi] : b + gi, R, g);\n"
         "    __syncwarp();\n"
         "  }\n"
         "}\n\n";
    // tail passes over the deferred inputs with the real budget (sfg_execute_deferred).
    // One-warp CTAs; a warp takes k inputs at a time (at most one per group), so a
    // round's few long inputs spread over many SMs.  seq = 0: the soft-cap list,
    // group-parallel; seq = 1: the inputs that must run thread-sequentially.
    // Its own register cap (launch bounds) raises the number of resident tail warps.
    o << "#define SFG_TAIL_MINB " << tail_minb << "\n"
         "extern \"C\" __global__ void __launch_bounds__(32, SFG_TAIL_MINB) sfg_jit_tail(const __grid_constant__ sfg_prog P, const __grid_constant__ ExecView E, int* next, int k, int seq) {\n"
         "  extern __shared__ __align__(16) uint8_t smem[];\n"
         "  JitRunner R;\n"
         "  R.soft_cap = 0;\n"
         "  const int lane = threadIdx.x;\n"
         "  const int32_t* list = seq ? E.deferred_seq : E.deferred;\n"
         "  const int nd = seq ? *E.n_deferred_seq : *E.n_deferred;\n"
         "  const int G = seq ? 1 : E.group;\n"
         "  int per = 32 / G;\n"
         "  if (k < per) per = k;\n"
         "  const int gi = lane / G;\n"
         "  Grp g{1, 0, 1u << lane, nullptr, nullptr, 0};\n"
         "  if (G > 1) {\n"
         "    GroupSmem* sm = reinterpret_cast<GroupSmem*>(smem + (size_t)gi * group_stride(E.tag_cap));\n"
         "    const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u) << (gi * G);\n"
         "    g = Grp{G, lane % G, gmask, sm, reinterpret_cast<uint32_t*>(sm + 1), E.tag_cap};\n"
         "  }\n"
         "  while (true) {\n"
         "    int b = 0;\n"
         "    if (lane == 0) b = atomicAdd(next, per);\n"
         "    b = __shfl_sync(0xffffffffu, b, 0);\n"
         "    if (b >= nd) break;\n"
         "    if (gi < per && b + gi < nd) {\n"
         "      if (G > 1) run_input<true>(P, E, list[b + gi], R, g);\n"
         "      else run_input<false>(P, E, list[b + gi], R, g);\n"
         "    }\n"
         "    __syncwarp();\n"
         "  }\n"
         "}\n";
    return o.str();
  }
};

}  // namespace sfgjit

static int jit_compiles = 0, jit_disk_hits = 0;   // NVRTC compiles / on-disk cache hits (sfg_jit_stats)

// On-disk cubin cache: NVRTC takes seconds per harness, so a compiled program is
// kept in $SFG_JIT_CACHE (default ~/.cache/sfg_b200_jit; "0" disables), keyed by a
// hash of the generated source and the compile options.  An entry stores the
// source it was compiled from and is used only if that matches exactly.
static std::string jit_cache_dir() {
  const char* d = getenv("SFG_JIT_CACHE");
  if (d && d[0] == '0' && d[1] == 0) return "";
  if (d && d[0]) return d;
  const char* h = getenv("HOME");
  return std::string(h && h[0] ? h : "/tmp") + "/.cache/sfg_b200_jit";
}

static uint64_t fnv1a(const std::string& s) {
  uint64_t x = 1469598103934665603ull;
  for (unsigned char c : s) { x ^= c; x *= 1099511628211ull; }
  return x;
}

static bool jit_cache_load(const std::string& key, std::vector<char>& cubin) {
  const std::string dir = jit_cache_dir();
  if (dir.empty()) return false;
  char name[32];
  snprintf(name, sizeof name, "/%016llx.sfgc", (unsigned long long)fnv1a(key));
  std::ifstream f(dir + name, std::ios::binary);
  if (!f) return false;
  uint64_t n = 0;
  if (!f.read(reinterpret_cast<char*>(&n), 8) || n != key.size()) return false;
  std::string k(n, '\0');
  if (!f.read(&k[0], (std::streamsize)n) || k != key) return false;
  std::vector<char> data((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (data.empty()) return false;
  cubin.swap(data);
  return true;
}

static void jit_cache_store(const std::string& key, const std::vector<char>& cubin) {
  const std::string dir = jit_cache_dir();
  if (dir.empty()) return;
  std::error_code ec;
  std::filesystem::create_directories(dir, ec);
  char name[32];
  snprintf(name, sizeof name, "/%016llx.sfgc", (unsigned long long)fnv1a(key));
  const std::string path = dir + name, tmp = path + ".tmp" + std::to_string((long long)getpid());
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    const uint64_t n = key.size();
    f.write(reinterpret_cast<const char*>(&n), 8);
    f.write(key.data(), (std::streamsize)n);
    f.write(cubin.data(), (std::streamsize)cubin.size());
    if (!f) return;
  }
  std::filesystem::rename(tmp, path, ec);   // atomic: concurrent processes never read a torn entry
}

// Generate and compile; on success `cubin` holds the sm_100a image.  Returns 0 on success.
static int sfg_jit_compile(const sfg_prog& P, const sfg_ins* ins, uint64_t max_edge_events, uint32_t dead_kernels,
                           const sfgjit::LaneCaps& caps, const sfg_hostop* hostops, size_t n_hostops,
                           const sfg_binding* binds, std::string& source,
                           std::string& log, std::vector<char>& cubin) {
  sfgjit::Gen g(P, ins);
  g.dead_kernels = dead_kernels;
  g.caps = caps;
  g.hostops = hostops;
  g.n_hostops = n_hostops;
  g.binds = binds;
  if (const char* ls = getenv("SFG_LOOPSUM")) g.loop_summaries = atoi(ls) != 0;
  if (const char* ns = getenv("SFG_NESTSUM")) g.nest_summaries = atoi(ns) != 0;
  if (const char* sm = getenv("SFG_STRAG_MIN")) g.strag_min = strtoull(sm, nullptr, 10) ? strtoull(sm, nullptr, 10) : 8192;
  if (const char* tb = getenv("SFG_TAIL_MINB")) g.tail_minb = atoi(tb) >= 1 ? atoi(tb) : 12;
  if (const char* bb = getenv("SFG_BULK_MINB")) g.bulk_minb = atoi(bb) >= 1 ? atoi(bb) : 4;
  source = g.run(P.n_edges, max_edge_events);
  // process-wide cache: identical programs (same generated source) compile once;
  // then the on-disk cache across processes
  static std::mutex mu;
  static std::map<std::string, std::vector<char>> cache;
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-default-device",
                        "-lineinfo", "-DSFG_JIT=1", "--device-int128", "--maxrregcount=255"};
  std::string key;
  for (const char* op : opts) key += std::string(op) + " ";
  {
    int ver[2] = {0, 0};
    nvrtcVersion(&ver[0], &ver[1]);
    key += "nvrtc " + std::to_string(ver[0]) + "." + std::to_string(ver[1]) + "\n";
    for (int e = 0; e < kEmbeddedCount; ++e) key += kEmbeddedSources[e];
  }
  key += source;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(source);
    if (it != cache.end()) {
      cubin = it->second;
      return 0;
    }
  }
  if (jit_cache_load(key, cubin)) {
    std::lock_guard<std::mutex> lk(mu);
    cache[source] = cubin;
    jit_disk_hits++;
    return 0;
  }
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, source.c_str(), "sfg_jit.cu", kEmbeddedCount, kEmbeddedSources, kEmbeddedNames) !=
      NVRTC_SUCCESS) {
    log = "nvrtcCreateProgram failed";
    return 1;
  }
  const nvrtcResult cr = nvrtcCompileProgram(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t lsz = 0;
  nvrtcGetProgramLogSize(prog, &lsz);
  log.assign(lsz, '\0');
  if (lsz) nvrtcGetProgramLog(prog, &log[0]);
  if (cr != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return 2;
  }
  size_t csz = 0;
  nvrtcGetCUBINSize(prog, &csz);
  cubin.resize(csz);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  jit_compiles++;
  jit_cache_store(key, cubin);
  std::lock_guard<std::mutex> lk(mu);
  cache[source] = cubin;
  return 0;
}

// Generate, compile and load the specialized execute kernels (bulk + tail).  Returns 0 on success.
static int sfg_jit_build(const sfg_prog& P, const sfg_ins* ins, uint64_t max_edge_events, uint32_t dead_kernels,
                         const sfgjit::LaneCaps& caps, const sfg_hostop* hostops, size_t n_hostops,
                         const sfg_binding* binds, std::string& source,
                         std::string& log, cudaLibrary_t* lib_out, cudaKernel_t* kern_out, cudaKernel_t* tail_out) {
  std::vector<char> cubin;
  const int rc = sfg_jit_compile(P, ins, max_edge_events, dead_kernels, caps, hostops, n_hostops, binds, source, log,
                                 cubin);
  if (rc) return rc;
  // Loaded libraries stay loaded for the process, one per distinct program on each
  // device: unloading a module whose kernels use a large local-memory frame makes the
  // driver shrink and later regrow the context's local-memory pool, which stalled the
  // next campaign's first launches for 0.1-0.4 s (measured around fuzz_loop calls).
  struct Loaded { cudaLibrary_t lib; cudaKernel_t kern, tail; };
  static std::mutex lmu;
  static std::map<std::pair<int, std::string>, Loaded> loaded;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(lmu);
    auto it = loaded.find({dev, source});
    if (it != loaded.end()) {
      *lib_out = it->second.lib;
      *kern_out = it->second.kern;
      *tail_out = it->second.tail;
      return 0;
    }
  }
  cudaError_t e = cudaLibraryLoadData(lib_out, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) {
    log += std::string("\ncudaLibraryLoadData: ") + cudaGetErrorString(e);
    return 3;
  }
  e = cudaLibraryGetKernel(kern_out, *lib_out, "sfg_jit_execute");
  if (e == cudaSuccess) e = cudaLibraryGetKernel(tail_out, *lib_out, "sfg_jit_tail");
  if (e != cudaSuccess) {
    log += std::string("\ncudaLibraryGetKernel: ") + cudaGetErrorString(e);
    return 4;
  }
  std::lock_guard<std::mutex> lk(lmu);
  loaded[{dev, source}] = Loaded{*lib_out, *kern_out, *tail_out};
  return 0;
}
