// Device table and record layouts shared by the CUDA kernels and the host
// packer (paper_2603_05725_b200/lowering.py mirrors every struct below with a
// numpy structured dtype; tests/test_layout.py checks the sizes/offsets).
//
// Everything is plain-old-data, little-endian, naturally aligned.
#pragma once
#ifdef __CUDACC_RTC__
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned long uintptr_t;
#else
#include <stdint.h>
#endif

#define SFG_ABI_VERSION 5

#define SFG_MAX_ARGS 16      // argspecs per harness
#define SFG_MAX_OPS 3        // MutationConfig.max_ops ceiling (reference default 3)
#define SFG_MAX_KERNELS 16
#define SFG_MAX_NAMED 32     // named host buffers (INIT + COMPUTE allocs)
#define SFG_MAX_BASE_RECS 32 // allocation records alive after INIT
#define SFG_MAX_FREE 32      // baseline free-list entries
#define SFG_MAX_LANE_RECS 40 // baseline + per-input allocation records
#define SFG_MAX_REGS 64      // kernel register_count ceiling (the generic interpreter's register files)
#define SFG_MAX_EDGES 1024   // static edges over all kernels
#define SFG_OV_CHUNK 256     // copy-on-write granule of INIT-buffer writes (device_memory.py:551-618 dirty chunks)

// opcodes == sir.Opcode
enum { SFG_MOV = 0, SFG_ADD, SFG_SUB, SFG_MUL, SFG_FADD, SFG_FSUB, SFG_FMUL, SFG_SETP,
       SFG_BRA, SFG_LD, SFG_ST, SFG_CVT, SFG_SREG, SFG_EXIT };

// sfg_ins.mode
enum { SFG_CLS_R = 0, SFG_CLS_F = 1, SFG_CLS_A = 2, SFG_CLS_P = 3 };           // MOV/ADD dst class
enum { SFG_CMP_EQ = 0, SFG_CMP_NE, SFG_CMP_LT, SFG_CMP_LE, SFG_CMP_GT, SFG_CMP_GE };
enum { SFG_MK_B8 = 0, SFG_MK_B16, SFG_MK_B32, SFG_MK_B64, SFG_MK_F32 };          // LD/ST kind
enum { SFG_SR_TID = 0, SFG_SR_NTID, SFG_SR_CTAID, SFG_SR_NCTAID };
enum { SFG_CVT_F_FROM_I = 0, SFG_CVT_I_FROM_F = 1 };

// sfg_ins.flags
#define SFG_F_S1_IMM 0x01
#define SFG_F_S2_IMM 0x02
#define SFG_F_PRED 0x04
#define SFG_F_PNEG 0x08
#define SFG_F_FLOAT 0x10     // SETP compares f32
#define SFG_F_U64IMM 0x20    // MOV %a, imm with imm in [2^63, 2^64)

typedef struct sfg_ins {     // 32 bytes
  uint8_t op, mode, flags, dst;
  uint8_t s1, s2, space, width;
  int32_t target;            // BRA: target pc (kernel-relative)
  int16_t edge_ft;           // edge id for pc -> pc+1 when it crosses a block, else -1
  int16_t edge_tk;           // BRA: edge id for the taken transition
  int64_t imm1;              // s1 immediate (prepared: wrapped i32 / f32 bits / i64) or const result
  int64_t imm2;              // s2 immediate, LD/ST byte offset
} sfg_ins;

typedef struct sfg_kernel {  // 48 bytes
  int32_t ins_base, n_ins, regs, n_params;
  int32_t edge_base, n_edges, n_blocks, name_idx;
  uint8_t ptype[16];         // 0 i32, 1 f32, 2 ptr
} sfg_kernel;

// host-op kinds (COMPUTE script)
enum { SFG_H_ALLOC = 0, SFG_H_COPY_IN, SFG_H_COPY_OUT_NAMED, SFG_H_COPY_OUT_ARG, SFG_H_FREE,
       SFG_H_LAUNCH, SFG_H_SYNC };
enum { SFG_SRC_ZEROS = 0, SFG_SRC_SEQ32, SFG_SRC_HEX, SFG_SRC_ARG };
enum { SFG_B_ARG = 0, SFG_B_BUF, SFG_B_LIT_I32, SFG_B_LIT_F32 };

typedef struct sfg_hostop {  // 72 bytes
  int32_t kind, buf, space, kernel;
  int64_t size;              // alloc bytes / copy_out bytes / copy_in bytes
  int32_t src_form, src_arg; // copy_in source
  int64_t blob_off;          // copy_in hex payload (offset into the const blob)
  int32_t arg_ref, grid, block, bind_base;
  int32_t n_bind, label, work_off, pad;  // work_off: offset of a COMPUTE alloc in the named-work area
} sfg_hostop;

typedef struct sfg_binding { // 16 bytes
  int32_t form, idx;
  int64_t lit;               // lit_i32: wrapped value; lit_f32: f32 bits of f32(float(lit))
} sfg_binding;

typedef struct sfg_rec {     // 64 bytes: an allocation record alive after INIT
  int64_t base, size, slot_start, slot_end;
  int64_t phys;              // payload offset into the baseline blob
  int32_t id;                // campaign alloc id
  int16_t label;
  uint8_t space, state;      // state: 0 LIVE, 1 FREED (quarantined)
  uint8_t resident, scope, pad[14];
} sfg_rec;

typedef struct sfg_free {    // 24 bytes: one free-list slot (offset within its space)
  int64_t off, slot;
  int32_t space, scope;
} sfg_free;

typedef struct sfg_named { int64_t addr; int32_t id, rec; } sfg_named;  // rec: baseline rec index

#define SFG_NO_OVERRIDE ((int64_t)0x8000000000000000ll)

// per-argument typed value (corpus entries and round children), 64 bytes
enum { SFG_V_I32 = 0, SFG_V_F32 = 1, SFG_V_ARR = 2 };
typedef struct sfg_val {
  uint8_t kind, elem, space, ndim;   // elem: 0 i32, 1 f32
  uint32_t bits;                     // scalar value bits
  uint64_t data_off;                 // array payload offset in its arena
  uint32_t nbytes, count;            // len(data), product(extents)
  int64_t base_offset;
  int64_t size_override;             // SFG_NO_OVERRIDE == None
  uint32_t ext[4];
  uint64_t pad;
} sfg_val;

// mutation ops (decoded to MutationOp text on the host)
enum { SFG_M_INT_BOUNDARY = 0, SFG_M_INT_BYTE, SFG_M_FLOAT_SIGN, SFG_M_FLOAT_EXPONENT,
       SFG_M_FLOAT_MANTISSA, SFG_M_FLOAT_BYTE, SFG_M_FLOAT_ARITH, SFG_M_ARRAY_EXTREME,
       SFG_M_ARRAY_DIM, SFG_M_ARRAY_EMPTY, SFG_M_PTR_SPACE, SFG_M_PTR_OFFSET, SFG_M_ARRAY_ELEM };
typedef struct sfg_op {      // 32 bytes
  uint8_t kind, arg, sub, byte;    // sub: which/mode/pattern/target/ndim; byte: byte idx or exp bit
  uint8_t inner, isub, ibyte, pad; // ARRAY_ELEM inner op
  uint32_t mask;             // mask / mantissa mask / delta_bits / extent 0
  uint32_t imask;            // inner mask / extent 1
  uint32_t index, pad2;      // ARRAY_ELEM element index
  int64_t delta;             // int_byte add delta / ptr_offset delta / inner add delta
} sfg_op;

typedef struct sfg_child {   // 144 bytes: per-input mutation result (values live in a sfg_val table)
  uint64_t rng_seed;
  int64_t it;                // global iteration id
  int32_t parent;            // corpus index (-1: seed iteration)
  int32_t n_ops;
  uint64_t work_bytes;       // bytes of the input's work region
  uint64_t readout_bytes;    // diff_readback: bytes of copy_out payloads
  uint64_t pad;
  sfg_op ops[SFG_MAX_OPS];
} sfg_child;

typedef struct sfg_entry {   // 32 bytes: corpus entry metadata
  int64_t admitted_iteration;
  uint64_t rng_seed;
  int32_t is_seed, parent;   // parent: corpus index of the entry's parent (-1 seeds)
  int64_t it;                // iteration that produced it (0 for seeds)
} sfg_entry;

// execution status
enum { SFG_ST_OK = 0, SFG_ST_FINDING = 1, SFG_ST_BUDGET = 2, SFG_ST_DEFERRED = 3,
       SFG_ST_OUT_OF_SPACE = 16, SFG_ST_ZERO_ALLOC = 17, SFG_ST_LANE_RECS = 18,
       SFG_ST_OVERLAY = 19, SFG_ST_COUNTER = 20 };
enum { SFG_C_SPATIAL_OOB = 0, SFG_C_TEMPORAL_UAF, SFG_C_SPACE_MISMATCH, SFG_C_PROVENANCE_ESCAPE,
       SFG_C_WILD_ACCESS, SFG_C_INVALID_FREE };
enum { SFG_MECH_SHADOW = 0, SFG_MECH_REGISTRY, SFG_MECH_PROVENANCE };

// alloc-id encoding inside the device: >0 baseline campaign id, <0 -(k+1) for the
// input's k-th allocation (fixed up by the host with the round's id prefix), 0 none
typedef struct sfg_verdict { // 112 bytes
  int32_t status, bug_class, kernel, iid;     // kernel: -1 host op
  int32_t ctaid, tid, width, shadow;          // shadow: -1 none
  int64_t addr_lo, addr_hi;                   // signed 128-bit faulting address
  uint8_t is_store, space, mech, alloc_state; // space 255: none; alloc_state 0 LIVE 1 FREED 255 none
  int32_t prov, alloc, label;                 // label -1: none
  int64_t alloc_base, alloc_size;
  uint64_t retired;
  int32_t launches, allocs;
  uint32_t entered;                           // bit k: kernel k launched
  int32_t key;                                // dedupe slot, -1 none
  uint64_t where;                             // diagnostics: SM id (bits 0-7), sequential re-run (bit 8), ns (bits 9-63)
} sfg_verdict;

// program-wide scalars passed by value to every kernel
typedef struct sfg_prog {
  // memory config (reference MemConfig)
  int64_t space_size[3];     // total bytes per space (scope size * scopes)
  int64_t scope_size[3];
  int64_t qcap[3];
  int32_t granule, redzone;
  // baseline allocator state after INIT
  int64_t cursor[3];         // scope-0 bump cursor per space (offset within space)
  int64_t qbytes[3];
  int32_t n_base_recs, n_free, n_quar, n_named;
  int32_t quar[SFG_MAX_BASE_RECS];        // baseline rec indices in FIFO order
  sfg_named named[SFG_MAX_NAMED];
  sfg_free freel[SFG_MAX_FREE];
  // harness
  int32_t n_args, n_mutable, n_int_args, n_kernels;
  uint8_t arg_kind[SFG_MAX_ARGS], arg_elem[SFG_MAX_ARGS], arg_fixed[SFG_MAX_ARGS];
  int8_t mutable_args[SFG_MAX_ARGS];
  int8_t int_slot[SFG_MAX_ARGS];         // arg -> rotation-count column, -1 if not i32
  int32_t n_hostops, n_edges, n_labels, n_keys;
  int32_t label_arg_base, total_ins, named_work_bytes, ov_cap;  // ov_cap: copy-on-write chunks per input
  sfg_kernel kernels[SFG_MAX_KERNELS];
  // mutation / campaign config
  int32_t max_ops, mut_granule, mut_redzone, window;
  double recent_weight;
  uint64_t master_seed, keybase;
  uint64_t budget;
  int32_t diff_readback, stop_first, stop_class, n_copyout_arg;  // stop_class -1: none
  int64_t readout_bytes_fixed;     // sum of named copy_out sizes in COMPUTE
  int8_t copyout_arg[SFG_MAX_ARGS];  // arg refs of COMPUTE `copy_out arg:k`, in script order
  // parent scheduling: 0 = schedule_next (campaign.py:593-603, one random() draw);
  // k > 0 = fixed fan-out, input it mutates corpus entry ((it - 1) / k) mod n (no draw;
  // BASELINE.json configs[3]: k children per seed of a large seed corpus)
  int32_t fanout;
  // array args that are the source of a COMPUTE `copy_in <buf> arg:k`: their
  // unmodified bytes (the test case's data, campaign.py:404-409) are kept in a
  // pristine copy at the very end of the work region
  uint32_t copy_src_mask;
  // the script is a TERM phase (campaign.py:538-541: freeing an already freed
  // allocation is skipped); jit_off: run on the generic interpreter (no NVRTC) --
  // the one-input INIT-launch / TERM programs
  int32_t term_phase, jit_off;
} sfg_prog;

// Tail of every input's work region: the copy-on-write overlay of INIT buffers,
// int64 blob-chunk index[ov_cap] (16-aligned) then ov_cap chunks of SFG_OV_CHUNK bytes.
#ifdef __CUDACC__
__host__ __device__
#endif
static inline uint64_t sfg_ov_bytes(int32_t cap) {
  return cap <= 0 ? 0ull : (((uint64_t)cap * 8ull + 15ull) & ~15ull) + (uint64_t)cap * SFG_OV_CHUNK;
}

// Work region of one input: array args at their materialized sizes | COMPUTE named
// allocs | copy-on-write overlay | pristine copies of copy_in source arrays.
// Offset of arg a's pristine copy given the input's values (vals[n_args]).
#ifdef __CUDACC__
__host__ __device__
#endif
static inline uint64_t sfg_pristine_off(const sfg_prog* P, const sfg_val* v, uint64_t work_bytes, int a,
                                        uint64_t* total) {
  uint64_t tot = 0, off = 0;
  for (int k = 0; k < P->n_args; ++k)
    if ((P->copy_src_mask >> k) & 1u) {
      if (k == a) off = tot;
      tot += ((uint64_t)v[k].nbytes + 15ull) & ~15ull;
    }
  if (total) *total = tot;
  return work_bytes - tot + off;
}
