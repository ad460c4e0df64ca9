// rb_internal.cuh -- device-side data model of librbgpu (not part of the ABI).
//
// Layout in HBM (one rb_rel per relation, uploaded once):
//   CODES  col: int32 codes[n]
//   MASK   col: uint8 mask[n]
//   TOKENS col: int64 offsets[n+1], int32 ids[nnz]            (from the host)
//               int32 len[n] (-1 = missing), uint4 sig[n] (128-bit token
//               signature), uint2 hash[n] (64-bit id-list hash)  (derived on device)
//   CHARS  col: int64 offsets[n+1], u8|u32 chars[nnz]         (from the host)
//               int32 len[n] (-1 = missing), uint4 bag[n] (16 x u8 saturating
//               character-bucket counts)                        (derived on device)
//
// The derived per-tuple features are what the pair kernel streams: they are
// fixed-size, 16-byte aligned and read with 128-bit loads.  The ragged
// arrays are touched only by the exact interpreter for surviving pairs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rbgpu.h"

namespace rb {

constexpr int MAX_COLS = 64;
constexpr int MAX_EQ = 6;      // equality features filtered in the pair loop
constexpr int MAX_TOK = 2;     // token-set features (jaccard / exact_token)
constexpr int MAX_STR = 2;     // string features (edit)
constexpr int MAX_CONST = 8;   // t.attr = const masks
constexpr int MAX_FSLOTS = 4;  // slots sharing one token / string feature
constexpr int MAX_RULES = RB_MAX_CHECKPOINTS;
constexpr int MAX_LEV = 3;     // multiplicity levels of the outer token signature

constexpr int BLOCK = 256;     // threads per CTA = outer rows per item
constexpr int TJ = 128;        // inner tuples per shared-memory tile
constexpr int QCAP = 256;      // survivor queue entries per warp
constexpr int NWARPS = BLOCK / 32;
constexpr int64_t CHUNK = 16384;  // inner columns per work item

enum RunMode : int32_t { MODE_SYM = 0, MODE_ASYM = 1, MODE_CROSS = 2 };

struct DevColumn {
    int32_t kind;
    int32_t width;
    const int32_t* codes;
    const uint8_t* mask;
    const int64_t* offsets;
    const void* data;
    const int32_t* len;
    const uint4* sig;
    const uint2* hash;
    const uint4* bag;
};

struct DevSlot {
    int32_t kind;
    int32_t lhs;
    int32_t rhs;
    int32_t flags;
    const int32_t* tab0;
    const int32_t* tab1;
    int32_t len0;
    int32_t len1;
};

struct TokSlotF {
    int32_t kind;
    int32_t bit;
    const int32_t* tab0;  // minsmall (jaccard)
    const int32_t* tab1;  // mink (jaccard)
    int32_t len0;
    int32_t len1;
};

struct StrSlotF {
    int32_t bit;
    int32_t pad;
    const int32_t* maxgap;
    const int32_t* maxd;
    int32_t len0;
    int32_t len1;
};

// Phase-1 filter program: exact equality / const tests and exact-safe bounds
// for the similarity slots.  A bit of `maybe` cleared here is a predicate
// that is certainly false; survivors are re-evaluated exactly.
struct FilterPlan {
    int32_t n_eq, n_tok, n_str, n_const, n_rules, pad;
    const int32_t* eq_outer[MAX_EQ];
    const int32_t* eq_inner[MAX_EQ];
    uint64_t eq_slots[MAX_EQ];
    const uint8_t* const_mask[MAX_CONST];
    uint64_t const_slots[MAX_CONST];
    const int64_t* tok_ooff[MAX_TOK];
    const int32_t* tok_oids[MAX_TOK];
    const int32_t* tok_olen[MAX_TOK];
    const uint2* tok_ohash[MAX_TOK];
    const int32_t* tok_ilen[MAX_TOK];
    const uint4* tok_isig[MAX_TOK];
    const uint2* tok_ihash[MAX_TOK];
    int32_t tok_nslots[MAX_TOK];
    TokSlotF tok_slot[MAX_TOK][MAX_FSLOTS];
    uint64_t tok_rules[MAX_TOK];
    const int32_t* str_olen[MAX_STR];
    const uint4* str_obag[MAX_STR];
    const int32_t* str_ilen[MAX_STR];
    const uint4* str_ibag[MAX_STR];
    int32_t str_nslots[MAX_STR];
    StrSlotF str_slot[MAX_STR][MAX_FSLOTS];
    uint64_t str_rules[MAX_STR];
    uint64_t need[MAX_RULES];  // slot bits each rule's precondition needs
};

// Exact interpreter program (evaluate_pair, engine.py:93-132).
struct VerifyProg {
    const int4* ins;  // {op, slot | checkpoint ordinal, fail_jump, rule}
    const DevSlot* slots;
    const DevColumn* cols;
    const int32_t* cp_rule;  // checkpoint ordinal -> index into path.rule_ids
    int32_t n_ins;
    int32_t n_slots;
};

struct RunParams {
    const int32_t* refs;  // position -> tid; nullptr = identity
    int64_t n;
    int32_t mode;
    uint32_t flags;
    const int4* items;  // {row0, col0, col1, row_hi}
    int32_t n_items;
    unsigned int* item_counter;
    int32_t* out_t;
    int32_t* out_s;
    int32_t* out_r;
    unsigned long long* out_count;
    long long cap;
    unsigned long long* stat_pairs;
    unsigned long long* stat_surv;
    unsigned long long* slot_evals;
    int32_t* scratch;
    int64_t scratch_stride;
};

// device-side helpers shared by kernels
__host__ __device__ inline uint32_t sig_bit(int32_t id) { return ((uint32_t)id * 0x9E3779B1u) >> 25; }
__host__ __device__ inline uint32_t bag_bucket(uint32_t c) { return (c * 0x9E3779B1u) >> 28; }
__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// launchers (rb_kernels.cu)
cudaError_t launch_token_features(const int64_t* offsets, const int32_t* ids, const uint8_t* missing, int64_t n,
                                  int32_t* len, uint4* sig, uint2* hash, cudaStream_t st);
cudaError_t launch_char_features(const int64_t* offsets, const void* chars, int32_t width, const uint8_t* missing,
                                 int64_t n, int32_t* len, uint4* bag, cudaStream_t st);
cudaError_t launch_pair_kernel(const FilterPlan& F, const VerifyProg& V, const RunParams& R, int grid,
                               cudaStream_t st);
int pair_kernel_blocks_per_sm();

}  // namespace rb
