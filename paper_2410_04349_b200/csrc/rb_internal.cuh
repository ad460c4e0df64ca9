// rb_internal.cuh -- host-side view of the device data model (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <string>

#include "../../include/rbgpu.h"
#include "rb_device.cuh"

namespace rb {

// launchers (rb_kernels.cu)
cudaError_t launch_token_features(const int64_t* offsets, const int32_t* ids, const uint8_t* missing, int64_t n,
                                  int32_t* len, uint4* sig, uint2* hash, cudaStream_t st);
cudaError_t launch_char_features(const int64_t* offsets, const void* chars, int32_t width, const uint8_t* missing,
                                 int64_t n, int32_t* len, uint4* bag, cudaStream_t st);
// components of one composite key, read on one side (t or s) of the pair
struct CompositeSpec {
    int n;
    const int32_t* codes[MAX_EQ + MAX_TOK * MAX_FSLOTS];  // eq code column, or null for a token list
    const int32_t* len[MAX_EQ + MAX_TOK * MAX_FSLOTS];    // token list length (-1 missing)
    const uint2* hash[MAX_EQ + MAX_TOK * MAX_FSLOTS];     // token list hash
};
cudaError_t launch_refs_check(const int32_t* refs, int64_t n, int64_t limit, unsigned long long* bad,
                              cudaStream_t st);
cudaError_t launch_composite_key(int64_t n, const CompositeSpec& spec, int32_t* out, cudaStream_t st);
cudaError_t launch_pair_kernel(const FilterPlan& F, const VerifyProg& V, const RunParams& R, int grid,
                               cudaStream_t st);
int pair_kernel_blocks_per_sm();
// RB_EXACT_STATS: first-touch slot evaluations over every pair of `parts`
struct StatPart {
    int64_t base, n, split, rbase;
};
cudaError_t launch_exact_stats(const VerifyProg& V, const int32_t* refs, const StatPart* parts, int n_parts,
                               int64_t row_lo, int64_t row_hi, uint32_t flags, int32_t* scratch, int64_t stride,
                               unsigned long long* evals, int grid, int block, cudaStream_t st);

// NVRTC specialisation (rb_jit.cu).  A JitKernel is looked up (or compiled
// once per process) from the program's shape; `ok` false means the generic
// kernel is used.
struct JitKernel {
    bool ok = false;
    cudaKernel_t kernel = nullptr;
    int blocks_per_sm = 1;
    int rows = 1;  // outer rows per thread
    bool defer = false;  // survivors go to a buffer decided by `verify` (see RunParams::surv)
    bool gated = false;  // compiled with the stage-1 gate (counts gate passes in RunParams::stat_gate)
    bool packed = false;  // takes MODE_PACKED items (several tiny partitions per item)
    cudaKernel_t verify = nullptr;
    int verify_blocks_per_sm = 1;
    double compile_ms = 0;
    std::string key;
    std::string log;
};
// force_rows > 0 compiles that many outer rows per thread (the small-partition variant);
// packed: the variant also takes MODE_PACKED items (deferred kernels only)
JitKernel jit_pair_kernel(const FilterPlan& F, int device, int force_rows = 0, bool packed = false);
cudaError_t launch_jit_kernel(const JitKernel& k, const FilterPlan& F, const VerifyProg& V, const RunParams& R,
                              int grid, cudaStream_t st);
cudaError_t launch_jit_verify(const JitKernel& k, const VerifyProg& V, const RunParams& R, int grid, cudaStream_t st);

}  // namespace rb
