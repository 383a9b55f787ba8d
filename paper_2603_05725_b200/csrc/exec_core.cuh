// K3 core: per-input memory model, sanitizer and COMPUTE host-op driver shared
// by the generic interpreter (execute.cu) and the per-harness JIT kernels (jit.cu).
//
// K3: execute + sanitize + cover, one fuzz input per lane.
//
// Each lane runs its input's COMPUTE host-op script (campaign.py:483-561) and
// interprets every launch's simulated threads strictly sequentially
// (block-major, thread-major, run-to-completion, first-bug-stop, per-thread
// retired budget; executor.py:390-424), so results are bit-identical with the
// reference interpreter.  32 inputs of the same harness share a warp.
//
// Memory model per input (no per-input copy of the 16+ MiB image):
//   * allocation records: the post-INIT baseline table (constant) + this
//     input's own allocations/frees, in a small local-memory table; shadow
//     codes are derived analytically from it (device_memory.py:347-393 proves
//     shadow == f(registry, quarantine)), so nothing is staged per granule;
//   * payload bytes: the input's materialized arrays and COMPUTE allocs live in
//     its work region (written by sfg_apply_kernel); INIT buffers are read from
//     the shared baseline blob; a write copies the touched 256-byte chunk into
//     the input's copy-on-write overlay at the tail of its work region first
//     (the reference's dirty-chunk restore, device_memory.py:551-618, becomes
//     "start every input with an empty overlay").
//   * simulated register files live in shared memory, [reg][lane] so that a
//     converged warp touches 32 consecutive banks; per-edge hit counters too.
//
// Sanitizer order = sanitizer.py:145-187 (SPACE_MISMATCH -> TEMPORAL_UAF ->
// shadow scan (SPATIAL_OOB / freed) -> PROVENANCE_ESCAPE -> WILD_ACCESS), with
// a provenance fast path that is provably equivalent when the tagged record's
// live payload contains the whole access.
#pragma once
#include "common.cuh"

namespace {

constexpr uint8_t SH_RZ = 0xFA, SH_FREED = 0xFD, SH_UNALLOC = 0xFF;
// Per-input table capacities.  The generic interpreter uses the ceilings; the
// specialized kernels define them from the harness's static bounds (jit.cu
// LaneCaps: INIT records + one record per array argument and COMPUTE alloc, the
// baseline quarantine / free list + one entry per COMPUTE free), so a lane's
// tables are a few hundred bytes and stay in L1 instead of spilling to DRAM.
#ifndef SFG_LANE_RECS
#define SFG_LANE_RECS SFG_MAX_LANE_RECS
#endif
#ifndef SFG_LANE_Q
#define SFG_LANE_Q 32
#endif
#ifndef SFG_LANE_FREE
#define SFG_LANE_FREE 32
#endif
#ifndef SFG_LANE_NAMED
#define SFG_LANE_NAMED SFG_MAX_NAMED
#endif
#ifndef SFG_LANE_ARGS
#define SFG_LANE_ARGS SFG_MAX_ARGS
#endif
#ifndef SFG_LANE_PARAMS   // kernel parameters of a launch (bound values by class)
#define SFG_LANE_PARAMS SFG_MAX_ARGS
#endif
// Array arguments no launch stores through / loads through (jit.cu array_masks;
// 0 for the generic interpreter): the bulk pass reads an unmutated read-only array
// straight from the parent's corpus payload and does not build a write-only one.
#ifndef SFG_RO_ARGS
#define SFG_RO_ARGS 0u
#endif
#ifndef SFG_WO_ARGS
#define SFG_WO_ARGS 0u
#endif
constexpr int kMaxQ = SFG_LANE_Q;
constexpr int kMaxFree = SFG_LANE_FREE;

enum : uint8_t { R_FREED = 1, R_RES = 2, R_BASE = 4 };

struct LRec {            // 48 bytes
  int64_t base, size, slot_start, slot_end;
  int64_t phys;          // baseline: blob offset, own: work-region offset
  int32_t id;            // >0 campaign id (baseline), <0 -(k+1) own k-th allocation
  int16_t label;
  uint8_t space, flags;
};

struct Lane {
  LRec rec[SFG_LANE_RECS];
  int nrec, nalloc, nq, nfree, nov;
  int64_t cursor[3], qbytes[3];
  int16_t quar[kMaxQ];
  sfg_free fl[kMaxFree];
  int64_t named_addr[SFG_LANE_NAMED];
  int16_t named_rec[SFG_LANE_NAMED];
  int16_t mat_rec[SFG_LANE_ARGS];
  uint64_t ro_cursor;
};

}  // namespace

struct ExecView {
  const sfg_ins* ins;
  const sfg_hostop* hostops;
  const sfg_binding* binds;
  const sfg_rec* base_recs;
  const uint8_t* base_blob;
  const uint8_t* const_blob;
  const sfg_child* children;
  const sfg_val* vals;
  const uint64_t* work_base;
  uint8_t* work;
  sfg_verdict* verdicts;
  uint32_t* edge_counts;       // [n][n_edges]
  uint8_t* readouts;
  const uint64_t* readout_base;
  int n;
  // long-input deferral (specialized kernel only): an input whose retired count
  // would reach soft_cap is abandoned and appended to deferred[] (count in
  // *n_deferred); the tail pass re-materializes and re-runs it from scratch with
  // the real budget, 32 long inputs per warp.  soft_cap 0 = off.
  uint64_t soft_cap;
  int32_t* deferred;
  int* n_deferred;
  // inputs that must run thread-sequentially (a cross-thread memory conflict was
  // seen in group-parallel mode, or the work region exceeds the tag capacity)
  int32_t* deferred_seq;
  int* n_deferred_seq;
  // group-parallel mode: the simulated threads of one launch run on G lanes at once
  // (G = 1: one lane runs them one after another); tag_cap = per-group conflict-tag
  // words in shared memory (4 bytes of work region per word)
  int group;
  int tag_cap;
  // bulk-pass schedule: the j-th fetched input is order[j] (sfg_order), null = j
  const int32_t* order;
  // trace mode (generic interpreter only, sfg_execute_trace): ExecHooks events
  // (executor.py:122-135) of input i into trace[i * trace_cap ...], 4 words each;
  // trace_count[i] = events produced (may exceed trace_cap: truncated)
  uint64_t* trace;
  uint32_t trace_cap;
  uint32_t* trace_count;
  // in-kernel materialization (the bulk pass, sfg_execute with a corpus): each input's
  // arrays are built from its parent's payload right before its COMPUTE phase, by the
  // rule of sfg_apply (campaign.py:440-450); null: the work regions are already built
  const sfg_val* mat_vals;
  const uint8_t* mat_data;
  // bulk pass: the schedule (order) holds *n_live inputs (duplicates left out,
  // sfg_dedupe); null = all n
  const int32_t* n_live;
};

namespace {

typedef __int128 i128;

// sanitizer slow path, allocator walk and report assembly: rare, called from every
// memory access site of the specialized kernel -> out of line (code size / compile time)
#define SFG_SLOW __device__ __noinline__

// space bases 0x1000_0000 / 0x2000_0000 / 0x3000_0000 (device_memory.py:41-45)
SFG_DEV int64_t sbase(int s) { return (int64_t)(s + 1) << 28; }

struct Report {
  int cls, mech, shadow;       // shadow -1 none
  int rec;                     // attributed lane record, -1 none
};

// ---------------------------------------------------------------------------
// allocation registry (device_memory.py:397-517), analytic shadow

SFG_DEV int space_of(const sfg_prog& P, i128 a) {
  for (int s = 0; s < 3; ++s)
    if (a >= (i128)sbase(s) && a < (i128)(sbase(s) + P.space_size[s])) return s;
  return -1;
}

SFG_DEV int resolve_payload(const Lane& L, int sp, int64_t a) {
  for (int k = 0; k < L.nrec; ++k) {
    const LRec& r = L.rec[k];
    if ((r.flags & R_RES) && r.space == sp && r.base <= a && a < r.base + r.size) return k;
  }
  return -1;
}

SFG_DEV int resolve_slot(const Lane& L, int sp, int64_t a) {
  for (int k = 0; k < L.nrec; ++k) {
    const LRec& r = L.rec[k];
    if ((r.flags & R_RES) && r.space == sp && r.slot_start <= a && a < r.slot_end) return k;
  }
  return -1;
}

struct Scan { int kind; int64_t gaddr; int code; };  // kind 0 none, 1 spatial, 2 freed, 3 wild

// _scan_shadow (sanitizer.py:102-142) on shadow codes derived from the registry
SFG_SLOW Scan scan_shadow(const sfg_prog& P, const Lane& L, i128 a, int64_t width) {
  const int sp = space_of(P, a);
  if (sp < 0) return {3, 0, SH_UNALLOC};
  const int64_t g = P.granule;
  const int64_t sb = sbase(sp);
  const int64_t addr = (int64_t)a;
  const int64_t end = addr + width;
  int64_t gi = (addr - sb) / g;
  while (true) {
    const int64_t gstart = sb + gi * g;
    if (gstart >= end) return {0, 0, 0};
    if (gi * g >= P.space_size[sp]) return {3, gstart, SH_UNALLOC};
    const int k = resolve_slot(L, sp, gstart);
    if (k < 0) return {3, gstart, SH_UNALLOC};
    const LRec& r = L.rec[k];
    const int64_t pay_end = r.base + ((r.size + g - 1) / g) * g;
    if (gstart < r.base || gstart >= pay_end) return {1, gstart, SH_RZ};
    if (r.flags & R_FREED) return {2, gstart, SH_FREED};
    const int64_t full_end = r.base + (r.size / g) * g;
    if (gstart < full_end) {       // run of addressable granules: jump past it
      gi = (full_end - sb) / g;
      continue;
    }
    const int64_t code = r.size % g;  // partial tail granule
    const int64_t lo = (addr > gstart ? addr : gstart) - gstart;
    const int64_t hi = (end < gstart + g ? end : gstart + g) - gstart;
    if (lo >= code || hi > code) return {1, gstart, (int)code};
    ++gi;
  }
}

// check_access (sanitizer.py:145-187).  prov: lane record index + 1, 0 none.
SFG_SLOW bool check_access(const sfg_prog& P, const Lane& L, i128 a, int64_t width, int decl, int prov,
                          Report& rep, int& hit) {
  // fast path: the tagged live record contains the whole access in its declared space
  if (prov > 0) {
    const LRec& t = L.rec[prov - 1];
    if ((t.flags & (R_RES | R_FREED)) == R_RES && t.space == decl && a >= (i128)t.base &&
        a + width <= (i128)(t.base + t.size)) {
      hit = prov - 1;
      return false;
    }
  }
  const int sp = space_of(P, a);
  int r = sp >= 0 ? resolve_payload(L, sp, (int64_t)a) : -1;
  if (r >= 0 && L.rec[r].space != decl) { rep = {SFG_C_SPACE_MISMATCH, SFG_MECH_REGISTRY, -1, r}; return true; }
  if (r >= 0 && (L.rec[r].flags & R_FREED)) { rep = {SFG_C_TEMPORAL_UAF, SFG_MECH_SHADOW, SH_FREED, r}; return true; }
  const Scan v = scan_shadow(P, L, a, width);
  if (v.kind == 1) {
    rep = {SFG_C_SPATIAL_OOB, SFG_MECH_SHADOW, v.code, r >= 0 ? r : resolve_slot(L, space_of(P, v.gaddr), v.gaddr)};
    return true;
  }
  if (v.kind == 2) {
    rep = {SFG_C_TEMPORAL_UAF, SFG_MECH_SHADOW, v.code, resolve_slot(L, space_of(P, v.gaddr), v.gaddr)};
    return true;
  }
  if (prov > 0) {
    const LRec& t = L.rec[prov - 1];
    if (!(a >= (i128)t.base && a + width <= (i128)(t.base + t.size))) {
      rep = {SFG_C_PROVENANCE_ESCAPE, SFG_MECH_PROVENANCE, v.kind ? v.code : -1, prov - 1};
      return true;
    }
  }
  if (v.kind == 3) { rep = {SFG_C_WILD_ACCESS, SFG_MECH_SHADOW, v.code, -1}; return true; }
  hit = r;
  return false;
}


// _alloc_common (device_memory.py:407-440), scope 0; returns record index or -status
SFG_DEV int lane_alloc(const sfg_prog& P, Lane& L, int sp, int64_t size, int label, int64_t phys) {
  const int64_t g = P.granule, rz = P.redzone;
  const int64_t slot = rz + ((size + g - 1) / g) * g + rz;
  int best = -1;
  for (int k = 0; k < L.nfree; ++k)
    if (L.fl[k].space == sp && L.fl[k].scope == 0 && L.fl[k].slot == slot && (best < 0 || L.fl[k].off < L.fl[best].off))
      best = k;
  int64_t off;
  if (best >= 0) {
    off = L.fl[best].off;
    L.fl[best] = L.fl[--L.nfree];
  } else {
    if (L.cursor[sp] + slot > P.scope_size[sp]) return -SFG_ST_OUT_OF_SPACE;
    off = L.cursor[sp];
    L.cursor[sp] += slot;
  }
  if (L.nrec >= SFG_LANE_RECS) return -SFG_ST_LANE_RECS;
  LRec& r = L.rec[L.nrec];
  r.slot_start = sbase(sp) + off;
  r.slot_end = r.slot_start + slot;
  r.base = r.slot_start + rz;
  r.size = size;
  r.phys = phys;
  r.id = -(++L.nalloc);
  r.label = (int16_t)label;
  r.space = (uint8_t)sp;
  r.flags = R_RES;
  return L.nrec++;
}

// out of space: the figures of OutOfSpaceError's message (device_memory.py:426-430)
// -- space, slot bytes needed, bytes remaining in scope 0 -- into the verdict
SFG_DEV void oos_detail(const sfg_prog& P, const Lane& L, sfg_verdict& V, int sp, int64_t size) {
  if (V.status != SFG_ST_OUT_OF_SPACE) return;
  const int64_t g = P.granule;
  V.space = (uint8_t)sp;
  V.alloc_size = P.redzone + ((size + g - 1) / g) * g + P.redzone;
  V.alloc_base = P.scope_size[sp] - L.cursor[sp];
}

// free (device_memory.py:442-487); returns 0 ok, 1 invalid free, 2 invalid free of an
// allocation already freed, -status fatal
SFG_DEV int lane_free(const sfg_prog& P, Lane& L, int64_t addr) {
  const int sp = space_of(P, addr);
  if (sp < 0) return 1;
  int k = -1;
  for (int j = 0; j < L.nrec; ++j)
    if ((L.rec[j].flags & R_RES) && L.rec[j].space == sp && L.rec[j].base == addr) k = j;
  if (k < 0) return 1;
  if (L.rec[k].flags & R_FREED) return 2;
  LRec& r = L.rec[k];
  r.flags |= R_FREED;
  if (L.nq >= kMaxQ) return -SFG_ST_LANE_RECS;
  L.quar[L.nq++] = (int16_t)k;
  L.qbytes[sp] += r.slot_end - r.slot_start;
  while (L.qbytes[sp] > P.qcap[sp]) {  // _evict_one: first quarantined record of this space
    int qi = 0;
    while (qi < L.nq && L.rec[L.quar[qi]].space != sp) ++qi;
    const int e = L.quar[qi];
    for (int j = qi; j + 1 < L.nq; ++j) L.quar[j] = L.quar[j + 1];
    --L.nq;
    LRec& v = L.rec[e];
    v.flags &= ~R_RES;
    if (L.nfree >= kMaxFree) return -SFG_ST_LANE_RECS;
    L.fl[L.nfree++] = sfg_free{v.slot_start - sbase(sp), v.slot_end - v.slot_start, sp, 0};
    L.qbytes[sp] -= v.slot_end - v.slot_start;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// payload bytes

struct Mem {
  const ExecView* E;
  uint8_t* work;               // this input's work region
  const uint8_t* blob;         // baseline payloads, padded to a multiple of SFG_OV_CHUNK
  int64_t* ov_idx;             // copy-on-write overlay: blob chunk index of each copied chunk
  uint8_t* ov_data;            // ... and the chunks (ov_cap of them)
  int ov_cap;
};

// overlay slot holding blob chunk c, or -1
SFG_DEV int ov_find(const Mem& M, const Lane& L, int64_t c) {
  for (int k = 0; k < L.nov; ++k)
    if (M.ov_idx[k] == c) return k;
  return -1;
}

SFG_DEV uint8_t base_byte(const Mem& M, const Lane& L, const LRec& r, int64_t a) {
  const int64_t o = r.phys + (a - r.base);
  const int k = L.nov ? ov_find(M, L, o / SFG_OV_CHUNK) : -1;
  return k >= 0 ? M.ov_data[(size_t)k * SFG_OV_CHUNK + (o % SFG_OV_CHUNK)] : M.blob[o];
}

SFG_SLOW uint64_t mem_read(const Mem& M, const Lane& L, const LRec& r, int64_t a, int w) {
  uint64_t v = 0;
  if (!(r.flags & R_BASE)) {
    const uint8_t* p = M.work + r.phys + (a - r.base);
    if ((((uintptr_t)p) & (w - 1)) == 0) {
      if (w == 4) return *reinterpret_cast<const uint32_t*>(p);
      if (w == 8) return *reinterpret_cast<const uint64_t*>(p);
      if (w == 2) return *reinterpret_cast<const uint16_t*>(p);
      return *p;
    }
    for (int k = 0; k < w; ++k) v |= (uint64_t)p[k] << (8 * k);
    return v;
  }
  for (int k = 0; k < w; ++k) v |= (uint64_t)base_byte(M, L, r, a + k) << (8 * k);
  return v;
}

SFG_SLOW bool mem_write(const Mem& M, Lane& L, const LRec& r, int64_t a, int w, uint64_t v) {
  if (!(r.flags & R_BASE)) {
    uint8_t* p = M.work + r.phys + (a - r.base);
    if ((((uintptr_t)p) & (w - 1)) == 0) {
      if (w == 4) *reinterpret_cast<uint32_t*>(p) = (uint32_t)v;
      else if (w == 8) *reinterpret_cast<uint64_t*>(p) = v;
      else if (w == 2) *reinterpret_cast<uint16_t*>(p) = (uint16_t)v;
      else *p = (uint8_t)v;
      return true;
    }
    for (int k = 0; k < w; ++k) p[k] = (uint8_t)(v >> (8 * k));
    return true;
  }
  // INIT buffer: write into the input's copy of the touched chunk (copied on first
  // write); false = the overlay is full (the host grows ov_cap and re-runs the round)
  for (int k = 0; k < w; ++k) {
    const int64_t o = r.phys + (a + k - r.base);
    const int64_t c = o / SFG_OV_CHUNK;
    int j = ov_find(M, L, c);
    if (j < 0) {
      if (L.nov >= M.ov_cap) return false;
      j = L.nov++;
      M.ov_idx[j] = c;
      const uint4* src = reinterpret_cast<const uint4*>(M.blob + c * SFG_OV_CHUNK);
      uint4* dst = reinterpret_cast<uint4*>(M.ov_data + (size_t)j * SFG_OV_CHUNK);
      for (int q = 0; q < SFG_OV_CHUNK / 16; ++q) dst[q] = src[q];
    }
    M.ov_data[(size_t)j * SFG_OV_CHUNK + (o % SFG_OV_CHUNK)] = (uint8_t)(v >> (8 * k));
  }
  return true;
}

// direct payload access for the JIT fast path (own, work-backed records only)
SFG_DEV uint64_t ld_work(const uint8_t* p, int w) {
  if ((((uintptr_t)p) & (w - 1)) == 0) {
    if (w == 4) return *reinterpret_cast<const uint32_t*>(p);
    if (w == 8) return *reinterpret_cast<const uint64_t*>(p);
    if (w == 2) return *reinterpret_cast<const uint16_t*>(p);
    return *p;
  }
  uint64_t v = 0;
  for (int k = 0; k < w; ++k) v |= (uint64_t)p[k] << (8 * k);
  return v;
}

SFG_DEV void st_work(uint8_t* p, int w, uint64_t v) {
  if ((((uintptr_t)p) & (w - 1)) == 0) {
    if (w == 4) *reinterpret_cast<uint32_t*>(p) = (uint32_t)v;
    else if (w == 8) *reinterpret_cast<uint64_t*>(p) = v;
    else if (w == 2) *reinterpret_cast<uint16_t*>(p) = (uint16_t)v;
    else *p = (uint8_t)v;
    return;
  }
  for (int k = 0; k < w; ++k) p[k] = (uint8_t)(v >> (8 * k));
}

// ---------------------------------------------------------------------------

SFG_SLOW void fill_report(sfg_verdict& V, const sfg_prog& P, const Lane& L, const Report& rep, int kernel,
                         int iid, int ctaid, int tid, i128 a, int width, bool store, int space, int prov) {
  V.status = SFG_ST_FINDING;
  V.bug_class = rep.cls;
  V.kernel = kernel;
  V.iid = iid;
  V.ctaid = ctaid;
  V.tid = tid;
  V.width = width;
  V.shadow = rep.shadow;
  V.addr_lo = (int64_t)(uint64_t)a;
  V.addr_hi = (int64_t)(a >> 64);
  V.is_store = store;
  V.space = (uint8_t)(space < 0 ? 255 : space);
  V.mech = (uint8_t)rep.mech;
  V.prov = prov > 0 ? L.rec[prov - 1].id : 0;
  if (rep.rec >= 0) {
    const LRec& r = L.rec[rep.rec];
    V.alloc = r.id;
    V.label = r.label;
    V.alloc_base = r.base;
    V.alloc_size = r.size;
    V.alloc_state = (r.flags & R_FREED) ? 1 : 0;
  } else {
    V.alloc = 0;
    V.label = -1;
    V.alloc_base = 0;
    V.alloc_size = 0;
    V.alloc_state = 255;
  }
  const int g = kernel < 0 ? P.total_ins : P.kernels[kernel].ins_base + iid;
  const int site = rep.rec >= 0 ? L.rec[rep.rec].label : P.n_labels;
  V.key = (rep.cls * (P.total_ins + 1) + g) * (P.n_labels + 1) + site;
}

// host copy check (sanitizer.py:190-196): declared space = the space the address lands in
SFG_DEV bool host_check(const sfg_prog& P, const Lane& L, sfg_verdict& V, int64_t addr, int64_t width, bool store,
                        int& hit) {
  Report rep;
  const int sp = space_of(P, addr);
  const int decl = sp < 0 ? 0 : sp;
  if (check_access(P, L, addr, width, decl, 0, rep, hit)) {
    fill_report(V, P, L, rep, -1, -1, -1, -1, addr, (int)width, store, decl, 0);
    return true;
  }
  return false;
}

SFG_DEV void edge_hit(uint32_t* ecnt, int e, bool& overflow) {
  uint32_t* p = ecnt + e * 32 + (threadIdx.x & 31);
  if (*p == 0xFFFFFFFFu) overflow = true; else ++*p;
}


// bound launch arguments, per register class in parameter order (executor.py:167-188)
struct Pre {
  uint32_t r[SFG_LANE_PARAMS], f[SFG_LANE_PARAMS];
  int64_t a[SFG_LANE_PARAMS];
  int32_t ap[SFG_LANE_PARAMS];
  int nr, nf, na;
};

enum { RUN_EXIT = 0, RUN_FINDING = 1, RUN_BUDGET = 2, RUN_FATAL = 3, RUN_DEFER = 4, RUN_CONFLICT = 5, RUN_ABORT = 6 };

// ---------------------------------------------------------------------------
// group-parallel launches (JIT runner only)
//
// executor.py:405-424 runs the simulated threads of a launch one after another
// (ctaid-major), each to completion, first stop wins.  A group of G lanes runs
// G consecutive simulated threads at once instead, and the attempt is kept only
// if it provably equals the sequential run:
//   * every work-region word carries a tag (writer lane, reader lane / many) in
//     shared memory; a word written by one thread and read or written by another
//     is a conflict -> the input is re-run thread-sequentially (deferred_seq);
//     stores into INIT (baseline) buffers are conflicts too;
//   * threads are independent otherwise (own registers, own budget,
//     executor.py:414), so the stop is the smallest stopping thread index s;
//     threads after s are discarded (their edge counts rolled back, their
//     retired counts dropped) and threads <= s are exactly the sequential ones;
//   * a lane polls the group state every few thousand retired instructions and
//     quits once its thread can no longer matter.
// Chunks of G threads run in order, so a launch with more threads than lanes
// sees every earlier chunk's stores.  A chunk with a conflict is undone (its
// work-region snapshot restored, edge counts rolled back) and re-run in place
// by the group's first lane, thread after thread.

struct GroupSmem {
  int stop_min;    // smallest stopping thread index of the chunk
  int defer_min;   // smallest thread that reached the soft cap
  int conflict;
  int seq_rc;      // sequential re-run of a conflicting chunk: LG_* outcome
  unsigned long long seq_retired;
  int seq_nov;
  int waw;         // some word written by several threads of the chunk (and read by none)
  sfg_verdict V;   // the stopping thread's verdict, broadcast to the group
  // uint32_t tags[tag_cap], then uint32_t snapshot[tag_cap] of the work region
};

struct Grp {
  int G;           // lanes per input
  int gl;          // this lane's index in the group
  unsigned mask;   // the group's lanes
  GroupSmem* sm;
  uint32_t* tags;
  int tag_cap;
};

__host__ __device__ inline size_t group_stride(int tag_cap) {
  return (sizeof(GroupSmem) + (size_t)tag_cap * 8 + 15) & ~(size_t)15;
}

// record an access of [off, off+w) of the work region by lane `me` (1-based).
// Tag: bits 0-7 writer (lane + 1, 0xFF several), bits 8-15 reader (lane + 1, 0xFF
// several).  true = conflict: a word read by one thread and written by another
// (either order), or read after several threads wrote it.  A word written by
// several threads and read by none is not a conflict but sets *waw: only the
// final memory differs from the sequential run, which matters iff memory is
// read later (run_launch_group decides).
SFG_DEV bool par_track(uint32_t* tags, int ntags, int64_t off, int w, bool st, uint32_t me, int* waw) {
  if (off < 0) return true;
  const int64_t w0 = off >> 2, w1 = (off + w - 1) >> 2;
  if (w1 >= ntags) return true;
  for (int64_t x = w0; x <= w1; ++x) {
    uint32_t old = *reinterpret_cast<volatile uint32_t*>(&tags[x]);
    while (true) {
      const uint32_t wr = old & 0xFFu, rd = (old >> 8) & 0xFFu;
      uint32_t nw;
      if (st) {
        if (rd && rd != me) return true;
        if (wr && wr != me) {
          *waw = 1;
          nw = old | 0xFFu;
        } else {
          nw = (old & ~0xFFu) | me;
        }
      } else {
        if (wr && wr != me) return true;
        if (rd == me || rd == 0xFFu) break;
        nw = (old & ~0xFF00u) | ((rd ? 0xFFu : me) << 8);
      }
      if (nw == old) break;
      const uint32_t prev = atomicCAS(&tags[x], old, nw);
      if (prev == old) break;
      old = prev;
    }
  }
  return false;
}

// slow-path access (check_access passed, record r) in group-parallel mode
template <class Runner>
SFG_DEV bool par_access(const Runner& R, const LRec& r, int64_t lo, int w, bool st) {
  if (r.flags & R_BASE) return st;  // INIT buffers: reads are shared, writes go through the overlay
  return par_track(R.tags, R.ntags, r.phys + (lo - r.base), w, st, R.me, R.waw);
}

// One input's COMPUTE phase (campaign.py:483-561).  Runner supplies the simulated
// thread execution: begin_input(), run_thread(...) -> RUN_*, flush(row).
enum { LG_OK = 0, LG_STOP = 1, LG_DEFER = 2, LG_SEQ = 3 };

// One launch's simulated threads on the lanes of a group, G at a time (see above).
template <class Runner>
SFG_DEV int run_launch_group(const sfg_prog& P, const sfg_hostop& op, Lane& L, Mem& M, sfg_verdict& V,
                             const Pre& pre, Runner& R, const Grp& g, uint64_t& total_retired, int ntags,
                             int& reruns, bool mem_dead) {
  const int T = op.grid * op.block;
  uint32_t* wk = reinterpret_cast<uint32_t*>(M.work);  // 16-aligned, work_bytes a multiple of 16
  uint32_t* snap = g.tags + g.tag_cap;
  for (int c0 = 0; c0 < T; c0 += g.G) {
    for (int x = g.gl; x < ntags; x += g.G) {
      g.tags[x] = 0u;
      snap[x] = wk[x];
    }
    if (g.gl == 0) {
      g.sm->stop_min = 0x7FFFFFFF;
      g.sm->defer_min = 0x7FFFFFFF;
      g.sm->conflict = 0;
      g.sm->waw = 0;
    }
    __syncwarp(g.mask);
    R.save_edges();
    const int t = c0 + g.gl;
    int rc = RUN_EXIT;
    uint64_t tr = 0;
    sfg_verdict Vt = V;
    if (t < T) {
      R.par_begin(g, t, ntags);
      rc = R.template run_thread<true>(P, op.kernel, L, M, Vt, pre, t / op.block, t % op.block, op.grid, op.block, tr);
      R.par_end();
      if (rc == RUN_FINDING || rc == RUN_BUDGET || rc == RUN_FATAL) atomicMin(&g.sm->stop_min, t);
      else if (rc == RUN_DEFER) atomicMin(&g.sm->defer_min, t);
      else if (rc == RUN_CONFLICT) atomicOr(&g.sm->conflict, 1);
    }
    __syncwarp(g.mask);
    const int s = *reinterpret_cast<volatile int*>(&g.sm->stop_min);
    const int d = *reinterpret_cast<volatile int*>(&g.sm->defer_min);
    // several writers of a word: harmless if nothing reads memory afterwards -- the
    // phase stops here (s), or this is the last chunk of the last launch and no
    // readout is taken (campaign.py:516-517 skips copy_out values without diff_readback)
    const bool waw = *reinterpret_cast<volatile int*>(&g.sm->waw) != 0;
    const int cf = *reinterpret_cast<volatile int*>(&g.sm->conflict) ||
                   (waw && s == 0x7FFFFFFF && !(mem_dead && c0 + g.G >= T));
    __syncwarp(g.mask);
    if (cf) {
      // undo the chunk and re-run it thread-sequentially on the first lane
      ++reruns;
      for (int x = g.gl; x < ntags; x += g.G) wk[x] = snap[x];
      R.restore_edges();
      __syncwarp(g.mask);
      if (g.gl == 0) {
        int lg = LG_OK;
        uint64_t before = total_retired;
        for (int tt = c0; tt < T && tt < c0 + g.G; ++tt) {
          const int r2 = R.template run_thread<false>(P, op.kernel, L, M, V, pre, tt / op.block, tt % op.block,
                                                      op.grid, op.block, total_retired);
          if (r2 == RUN_EXIT) continue;
          if (r2 == RUN_BUDGET) V.status = SFG_ST_BUDGET;
          lg = r2 == RUN_DEFER ? LG_DEFER : LG_STOP;  // finding / budget / fatal stop the phase
          break;
        }
        g.sm->seq_rc = lg;
        g.sm->seq_retired = total_retired - before;
        g.sm->seq_nov = L.nov;
        g.sm->V = V;
      }
      __syncwarp(g.mask);
      const int lg = g.sm->seq_rc;
      if (g.gl != 0) {
        total_retired += g.sm->seq_retired;
        L.nov = g.sm->seq_nov;  // overlay entries (INIT-buffer stores) are shared
        V = g.sm->V;
      }
      __syncwarp(g.mask);
      if (lg != LG_OK) return lg;
      continue;
    }
    if (d < s) return LG_DEFER;
    const bool keep = t < T && t <= s;
    if (!keep) R.restore_edges();
    uint64_t sum = keep ? tr : 0ull;
    for (int o = g.G >> 1; o; o >>= 1) sum += __shfl_xor_sync(g.mask, sum, o);
    total_retired += sum;
    if (s != 0x7FFFFFFF) {
      if (t == s) {
        if (rc == RUN_BUDGET) Vt.status = SFG_ST_BUDGET;
        g.sm->V = Vt;
      }
      __syncwarp(g.mask);
      V = g.sm->V;
      __syncwarp(g.mask);
      return LG_STOP;
    }
  }
  return LG_OK;
}

// GRP: group-parallel launches (g.G > 1, specialized kernel only) vs one lane
// running the simulated threads one after another
template <bool GRP, class Runner>
SFG_DEV void run_input(const sfg_prog& P, const ExecView& E, int i, Runner& R, const Grp& g) {
  const sfg_child& ch = E.children[i];
  const sfg_val* cv = E.vals + (size_t)i * P.n_args;
  uint64_t t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  Lane L;
  const uint64_t ovb = sfg_ov_bytes(P.ov_cap);
  uint8_t* wk = E.work + E.work_base[i];
  uint64_t pri_tot = 0;
  if (P.copy_src_mask) sfg_pristine_off(&P, cv, ch.work_bytes, 0, &pri_tot);
  int64_t* ovi = reinterpret_cast<int64_t*>(wk + ch.work_bytes - pri_tot - ovb);
  Mem M{&E, wk, E.base_blob, ovi, reinterpret_cast<uint8_t*>(ovi) + (((uint64_t)P.ov_cap * 8ull + 15ull) & ~15ull),
        P.ov_cap};
  sfg_verdict V{};
  V.status = SFG_ST_OK;
  V.key = -1;
  V.label = -1;
  V.shadow = -1;
  V.alloc_state = 255;
  V.space = 255;
  // baseline allocator state (the restored snapshot, device_memory.py:574-618)
  L.nrec = P.n_base_recs;
  for (int k = 0; k < P.n_base_recs; ++k) {
    const sfg_rec& b = E.base_recs[k];
    LRec& r = L.rec[k];
    r.base = b.base; r.size = b.size; r.slot_start = b.slot_start; r.slot_end = b.slot_end;
    r.phys = b.phys; r.id = b.id; r.label = b.label; r.space = b.space;
    r.flags = (uint8_t)(R_BASE | (b.state ? R_FREED : 0) | (b.resident ? R_RES : 0));
  }
  L.nalloc = 0;
  L.nov = 0;
  L.nq = P.n_quar;
  for (int k = 0; k < P.n_quar; ++k) L.quar[k] = (int16_t)P.quar[k];
  L.nfree = P.n_free;
  for (int k = 0; k < P.n_free; ++k) L.fl[k] = P.freel[k];
  for (int s = 0; s < 3; ++s) { L.cursor[s] = P.cursor[s]; L.qbytes[s] = P.qbytes[s]; }
  for (int k = 0; k < P.n_named; ++k) { L.named_addr[k] = P.named[k].addr; L.named_rec[k] = (int16_t)P.named[k].rec; }
  for (int k = 0; k < P.n_args; ++k) L.mat_rec[k] = -1;
  L.ro_cursor = 0;
  R.begin_input();
  R.set_input(E, i);
  uint64_t total_retired = 0;
  uint8_t* ro = (P.diff_readback && E.readouts) ? E.readouts + E.readout_base[i] : nullptr;
  const uint64_t arrays_end = ch.work_bytes - (uint64_t)P.named_work_bytes - ovb - pri_tot;
  const int ntags = (int)((ch.work_bytes + 3) / 4);
  int defer_kind = 0;  // 1: soft cap reached (deferred), 2: re-run thread-sequentially (deferred_seq)
  int seq_reruns = 0;  // group-parallel chunks undone and re-run sequentially (diagnostics)
  if (GRP && ntags > g.tag_cap) defer_kind = 2;
  uint32_t alias = 0;               // arrays whose record reads the parent's payload in place
  const sfg_val* mpv = nullptr;     // the parent's values (in-kernel materialization)
  if (E.mat_data != nullptr && defer_kind == 0) {
    mpv = E.mat_vals + (size_t)(ch.parent < 0 ? 0 : ch.parent) * P.n_args;
    const int gl = GRP ? g.gl : 0, gn = GRP ? g.G : 1;
    for (int a = 0; a < P.n_args; ++a) {
      if (cv[a].kind != SFG_V_ARR) continue;
      const sfg_op* op = nullptr;
      for (int k = 0; k < ch.n_ops; ++k)
        if (ch.ops[k].arg == a) op = &ch.ops[k];
      if ((P.copy_src_mask >> a) & 1u)   // the test case's own bytes for copy_in (campaign.py:404-409)
        emit_child(wk + sfg_pristine_off(&P, cv, ch.work_bytes, a, nullptr), cv[a].nbytes,
                   E.mat_data + mpv[a].data_off, mpv[a].nbytes, cv[a], op, gl, gn);
      const uint64_t msz = sfg_mat_size(cv[a]);
      if (!GRP) {
        // never loaded (and no readback of it): its bytes are never read
        if (((SFG_WO_ARGS >> a) & 1u) && !P.diff_readback) continue;
        // never stored, data unchanged by the child's op, within the parent's bytes:
        // the materialized contents ARE the parent's payload prefix (emit_child)
        const uint64_t lim = cv[a].nbytes < mpv[a].nbytes ? cv[a].nbytes : mpv[a].nbytes;
        if (((SFG_RO_ARGS >> a) & 1u) && msz <= lim &&
            (op == nullptr || (op->kind != SFG_M_ARRAY_EXTREME && op->kind != SFG_M_ARRAY_ELEM))) {
          alias |= 1u << a;
          continue;
        }
      }
      emit_child(wk + cv[a].data_off, msz, E.mat_data + mpv[a].data_off, mpv[a].nbytes, cv[a], op, gl, gn);
    }
    if constexpr (GRP) __syncwarp(g.mask);
  }

  bool stop = defer_kind != 0;
  for (int h = 0; h < P.n_hostops && !stop; ++h) {
    const sfg_hostop& op = E.hostops[h];
    if (op.kind == SFG_H_SYNC) continue;
    if (op.kind == SFG_H_ALLOC) {
      if (op.size <= 0) { V.status = SFG_ST_ZERO_ALLOC; break; }
      const int64_t phys = (int64_t)arrays_end + op.work_off;
      const int k = lane_alloc(P, L, op.space, op.size, op.label, phys);
      if (k < 0) { V.status = -k; oos_detail(P, L, V, op.space, op.size); break; }
      for (int64_t b = 0; b < op.size; ++b) M.work[phys + b] = 0;
      L.named_addr[op.buf] = L.rec[k].base;
      L.named_rec[op.buf] = (int16_t)k;
      continue;
    }
    if (op.kind == SFG_H_COPY_IN) {
      const int64_t addr = L.named_addr[op.buf];
      int64_t len = op.size;
      const sfg_val* src_v = nullptr;
      const uint8_t* src_p = nullptr;   // array source: its pristine copy
      if (op.src_form == SFG_SRC_ARG) {
        src_v = &cv[op.src_arg];
        if (src_v->kind == SFG_V_ARR) {   // value.data (campaign.py:404-409)
          len = src_v->nbytes;
          src_p = M.work + sfg_pristine_off(&P, cv, ch.work_bytes, op.src_arg, nullptr);
        } else {
          len = 4;
        }
      }
      if (len == 0) continue;
      int hit = -1;
      if (host_check(P, L, V, addr, len, true, hit)) break;
      const LRec& r = L.rec[hit];
      for (int64_t b = 0; b < len; ++b) {
        uint8_t byte = 0;
        if (op.src_form == SFG_SRC_SEQ32) byte = (uint8_t)((uint32_t)(b >> 2) >> (8 * (b & 3)));
        else if (op.src_form == SFG_SRC_HEX) byte = E.const_blob[op.blob_off + b];
        else if (op.src_form == SFG_SRC_ARG) byte = src_p ? src_p[b] : (uint8_t)(src_v->bits >> (8 * b));
        if (!mem_write(M, L, r, addr + b, 1, byte)) { V.status = SFG_ST_OVERLAY; stop = true; break; }
      }
      continue;
    }
    if (op.kind == SFG_H_COPY_OUT_NAMED || op.kind == SFG_H_COPY_OUT_ARG) {
      int64_t addr, len;
      if (op.kind == SFG_H_COPY_OUT_ARG) {
        if (!P.diff_readback) continue;
        if (L.mat_rec[op.arg_ref] < 0) continue;
        addr = L.rec[L.mat_rec[op.arg_ref]].base;
        len = cv[op.arg_ref].nbytes;
      } else {
        addr = L.named_addr[op.buf];
        len = op.size;
      }
      if (len == 0) continue;
      int hit = -1;
      if (host_check(P, L, V, addr, len, false, hit)) break;
      if (ro != nullptr) {
        const LRec& r = L.rec[hit];
        for (int64_t b = 0; b < len; ++b) ro[L.ro_cursor + b] = (uint8_t)mem_read(M, L, r, addr + b, 1);
        L.ro_cursor += (len + 15) & ~15ll;
      }
      continue;
    }
    if (op.kind == SFG_H_FREE) {
      const int64_t addr = L.named_addr[op.buf];
      const int res = lane_free(P, L, addr);
      if (res < 0) { V.status = -res; break; }
      if (res == 2 && P.term_phase) continue;  // TERM teardown is idempotent (campaign.py:538-541)
      if (res >= 1) {  // invalid_free_report (sanitizer.py:199-205)
        const int sp = space_of(P, addr);
        int r = sp >= 0 ? resolve_payload(L, sp, addr) : -1;
        if (r < 0 && sp >= 0) r = resolve_slot(L, sp, addr);
        Report rep{SFG_C_INVALID_FREE, SFG_MECH_REGISTRY, -1, r};
        fill_report(V, P, L, rep, -1, -1, -1, -1, addr, 0, false, sp, 0);
        break;
      }
      continue;
    }
    // ---- launch: bind arguments (campaign.py:452-479), materializing arrays lazily
    Pre pre;
    pre.nr = pre.nf = pre.na = 0;
    for (int b = 0; b < op.n_bind && !stop; ++b) {
      const sfg_binding& B = E.binds[op.bind_base + b];
      if (B.form == SFG_B_LIT_I32) { pre.r[pre.nr++] = (uint32_t)B.lit; continue; }
      if (B.form == SFG_B_LIT_F32) { pre.f[pre.nf++] = (uint32_t)B.lit; continue; }
      if (B.form == SFG_B_BUF) {
        pre.a[pre.na] = L.named_addr[B.idx];
        pre.ap[pre.na++] = L.named_rec[B.idx] + 1;
        continue;
      }
      const sfg_val& v = cv[B.idx];
      if (v.kind == SFG_V_I32) { pre.r[pre.nr++] = v.bits; continue; }
      if (v.kind == SFG_V_F32) { pre.f[pre.nf++] = sfg_quiet(v.bits); continue; }
      if (L.mat_rec[B.idx] < 0) {
        const int64_t size = (int64_t)sfg_mat_size(v);
        // an aliased array's record addresses the parent's payload (phys relative to the work region)
        const int64_t phys = ((alias >> B.idx) & 1u)
                                 ? (int64_t)((uintptr_t)(E.mat_data + mpv[B.idx].data_off) - (uintptr_t)wk)
                                 : (int64_t)v.data_off;
        const int k = lane_alloc(P, L, v.space, size, P.label_arg_base + B.idx, phys);
        if (k < 0) { V.status = -k; oos_detail(P, L, V, v.space, size); stop = true; break; }
        L.mat_rec[B.idx] = (int16_t)k;
      }
      const LRec& r = L.rec[L.mat_rec[B.idx]];
      pre.a[pre.na] = r.base + v.base_offset;
      pre.ap[pre.na++] = L.mat_rec[B.idx] + 1;
    }
    if (stop) break;
    V.entered |= 1u << op.kernel;
    V.launches++;
    if constexpr (GRP) {
      __syncwarp(g.mask);  // host-op stores (made identically by every lane) visible to all
      // memory is dead after this launch: no later launch and no readout taken
      bool later_launch = false;
      for (int h2 = h + 1; h2 < P.n_hostops; ++h2) later_launch |= E.hostops[h2].kind == SFG_H_LAUNCH;
      const bool mem_dead = !later_launch && ro == nullptr;
      const int lg = run_launch_group(P, op, L, M, V, pre, R, g, total_retired, ntags, seq_reruns, mem_dead);
      if (lg == LG_STOP) stop = true;
      else if (lg == LG_DEFER) { defer_kind = 1; stop = true; }
      else if (lg == LG_SEQ) { defer_kind = 2; stop = true; }
      continue;
    }
    for (int ctaid = 0; ctaid < op.grid && !stop; ++ctaid) {
      for (int tid = 0; tid < op.block && !stop; ++tid) {
        const int rc = R.template run_thread<false>(P, op.kernel, L, M, V, pre, ctaid, tid, op.grid, op.block,
                                                    total_retired);
        if (rc == RUN_BUDGET) { V.status = SFG_ST_BUDGET; stop = true; }
        else if (rc == RUN_DEFER) { defer_kind = 1; stop = true; }
        else if (rc != RUN_EXIT) stop = true;  // finding (V filled) or fatal (V.status set)
      }
    }
  }
  if (defer_kind) {  // nothing of this attempt is kept
    if (g.gl == 0) {
      if (defer_kind == 1) E.deferred[atomicAdd(E.n_deferred, 1)] = i;
      else E.deferred_seq[atomicAdd(E.n_deferred_seq, 1)] = i;
    }
    return;
  }
  R.end_input(E, i);
  V.retired = total_retired;
  V.allocs = L.nalloc;
  uint32_t* erow = E.edge_counts + (size_t)i * P.n_edges;
  bool overflow = false;
  if constexpr (GRP) R.flush_group(erow, overflow, g.mask, g.gl == 0);
  else R.flush(erow, overflow);
  if (overflow && V.status < SFG_ST_OUT_OF_SPACE) V.status = SFG_ST_COUNTER;
  uint64_t t_end;
  uint32_t smid;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  V.where = (uint64_t)(smid & 0xff) | ((uint64_t)(seq_reruns > 0) << 8) | ((t_end - t_start) << 9);
  if (g.gl == 0) E.verdicts[i] = V;
}

}  // namespace
