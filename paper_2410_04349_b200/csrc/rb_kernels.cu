// rb_kernels.cu -- sm_100a kernels of the rule-evaluation path.
//
// 1. token_features / char_features: one pass over the ragged columns at
//    upload time, producing the fixed-size per-tuple features the pair
//    kernel streams (length, 128-bit token signature, 64-bit id-list hash,
//    16-bucket character histogram).
// 2. pair_kernel: the generic build of pair_body (rb_device.cuh); the
//    NVRTC-specialised build of the same body is made by rb_jit.cu.
//    Persistent CTAs pull work items (an outer row block x an inner column
//    chunk) from a global counter -- the analogue of the reference's interval
//    claiming and stealing (engine.py:139-207).  Each thread owns one outer
//    tuple in registers; inner tuples are staged through shared memory and
//    read as warp broadcasts.  Per pair the thread runs the phase-1 filter
//    with warp-uniform skipping (__any_sync) of feature classes no live rule
//    needs; maybe-pairs go to a per-warp queue (ballot + popc compaction)
//    that the warp drains through the exact path interpreter
//    (evaluate_pair, engine.py:93-132), one pair per lane, appending rows
//    with one warp-aggregated atomicAdd.
#include <climits>

#include "rb_internal.cuh"

namespace rb {

// ---------------------------------------------------------------------------
// upload-time feature kernels

__global__ void token_features_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ ids,
                                      const uint8_t* __restrict__ missing, int64_t n, int32_t* __restrict__ len,
                                      uint4* __restrict__ sig, uint2* __restrict__ hash) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = offsets[r], b = offsets[r + 1];
        uint32_t s[4] = {0, 0, 0, 0};
        uint64_t h = mix64((uint64_t)(b - a));
        for (int64_t k = a; k < b; k++) {
            const int32_t id = ids[k];
            const uint32_t bit = sig_bit(id);
            s[bit >> 5] |= 1u << (bit & 31);
            h = mix64(h ^ (uint32_t)id);
        }
        len[r] = (missing && missing[r]) ? -1 : (int32_t)(b - a);
        sig[r] = make_uint4(s[0], s[1], s[2], s[3]);
        hash[r] = make_uint2((uint32_t)h, (uint32_t)(h >> 32));
    }
}

__global__ void char_features_kernel(const int64_t* __restrict__ offsets, const void* __restrict__ chars,
                                     int32_t width, const uint8_t* __restrict__ missing, int64_t n,
                                     int32_t* __restrict__ len, uint4* __restrict__ bag) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = offsets[r], b = offsets[r + 1];
        uint32_t cnt[16];
#pragma unroll
        for (int q = 0; q < 16; q++) cnt[q] = 0;
        for (int64_t k = a; k < b; k++) {
            const uint32_t c = width == 1 ? ((const uint8_t*)chars)[k] : ((const uint32_t*)chars)[k];
            const uint32_t q = bag_bucket(c);
#pragma unroll
            for (int z = 0; z < 16; z++)
                if (z == (int)q) cnt[z] = min(cnt[z] + 1, 255u);
        }
        uint32_t w[4];
#pragma unroll
        for (int z = 0; z < 4; z++)
            w[z] = cnt[4 * z] | (cnt[4 * z + 1] << 8) | (cnt[4 * z + 2] << 16) | (cnt[4 * z + 3] << 24);
        const bool miss = missing && missing[r];
        len[r] = miss ? -1 : (int32_t)(b - a);
        // a missing row gets a saturated bag: against any present string its
        // length gap already exceeds the gap table (the pair filter needs no
        // separate presence test)
        bag[r] = miss ? make_uint4(~0u, ~0u, ~0u, ~0u) : make_uint4(w[0], w[1], w[2], w[3]);
    }
}

cudaError_t launch_token_features(const int64_t* offsets, const int32_t* ids, const uint8_t* missing, int64_t n,
                                  int32_t* len, uint4* sig, uint2* hash, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int grid = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    token_features_kernel<<<grid, 256, 0, st>>>(offsets, ids, missing, n, len, sig, hash);
    return cudaGetLastError();
}

cudaError_t launch_char_features(const int64_t* offsets, const void* chars, int32_t width, const uint8_t* missing,
                                 int64_t n, int32_t* len, uint4* bag, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int grid = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    char_features_kernel<<<grid, 256, 0, st>>>(offsets, chars, width, missing, n, len, bag);
    return cudaGetLastError();
}

// Rule-level composite keys: one 31-bit hash per tuple over the equality
// codes and token-list hashes of every equality-type test (eq code,
// exact_token) one rule requires, so the pair filter tests the whole
// conjunction with one compare.  Equal components give equal keys; unequal
// ones collide with probability 2^-31 and are caught by the exact pass.  A
// missing code or a missing / empty token list (the test is false) gives -1.
__global__ void composite_key_kernel(int64_t n, CompositeSpec spec, int32_t* __restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h = 0x243F6A8885A308D3ull;
        bool ok = true;
        for (int k = 0; k < spec.n; k++) {
            uint32_t v;
            if (spec.codes[k]) {
                const int32_t c = spec.codes[k][r];
                ok &= c >= 0;
                v = (uint32_t)c;
            } else {
                ok &= spec.len[k][r] > 0;
                v = spec.hash[k][r].x;
            }
            h = mix64(h ^ ((uint64_t)k << 40) ^ v);
        }
        out[r] = ok ? (int32_t)(h & 0x7fffffffu) : -1;
    }
}

cudaError_t launch_composite_key(int64_t n, const CompositeSpec& spec, int32_t* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int grid = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
    composite_key_kernel<<<grid, 256, 0, st>>>(n, spec, out);
    return cudaGetLastError();
}

// RB_EXACT_STATS: every pair of every part through the exact interpreter,
// counting each slot's first touch per pair (evaluate_pair, engine.py:93-132)
// into shared counters; one global add per slot and block.
__global__ void exact_stats_kernel(VerifyProg V, const int32_t* __restrict__ refs, const StatPart* __restrict__ parts,
                                   int n_parts, int64_t row_lo, int64_t row_hi, uint32_t flags, int32_t* scratch,
                                   int64_t stride, unsigned long long* evals) {
    __shared__ unsigned long long cnt[RB_MAX_SLOTS];
    for (int k = threadIdx.x; k < RB_MAX_SLOTS; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    int32_t* scr = scratch + (int64_t)(blockIdx.x * blockDim.x + threadIdx.x) * stride;
    const bool sym = (flags & RB_SYMMETRIC) != 0, enumerate = (flags & RB_ENUMERATE) != 0;
    for (int p = blockIdx.x; p < n_parts; p += gridDim.x) {
        const StatPart P = parts[p];
        const bool cross = P.split >= 0;
        const int64_t rlo = max((int64_t)0, row_lo), rhi = min(row_hi, cross ? P.split : P.n);
        for (int64_t i = rlo; i < rhi; i++) {
            const int64_t pi = P.base + i;
            const int32_t ti = refs ? __ldg(refs + pi) : (int32_t)pi;
            int64_t jlo, jhi;
            if (cross) {
                jlo = P.rbase;
                jhi = P.rbase + (P.n - P.split);
            } else {
                jlo = P.base + (sym ? i + 1 : 0);
                jhi = P.base + P.n;
            }
            for (int64_t pj = jlo + threadIdx.x; pj < jhi; pj += blockDim.x) {
                if (!cross && pj == pi) continue;
                const int32_t si = refs ? __ldg(refs + pj) : (int32_t)pj;
                interpret(V, ti, si, enumerate, scr, cnt);
            }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < V.n_slots && k < RB_MAX_SLOTS; k += blockDim.x)
        if (cnt[k]) atomicAdd(evals + k, cnt[k]);
}

cudaError_t launch_exact_stats(const VerifyProg& V, const int32_t* refs, const StatPart* parts, int n_parts,
                               int64_t row_lo, int64_t row_hi, uint32_t flags, int32_t* scratch, int64_t stride,
                               unsigned long long* evals, int grid, int block, cudaStream_t st) {
    if (n_parts <= 0) return cudaSuccess;
    exact_stats_kernel<<<grid, block, 0, st>>>(V, refs, parts, n_parts, row_lo, row_hi, flags, scratch, stride, evals);
    return cudaGetLastError();
}

// Range check of a run's tuple refs (replaces a host scan of every ref).
__global__ void refs_check_kernel(const int32_t* __restrict__ refs, int64_t n, int64_t limit,
                                  unsigned long long* bad) {
    bool ok = true;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = refs[k];
        ok &= r >= 0 && (int64_t)r < limit;
    }
    if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1ull);
}

cudaError_t launch_refs_check(const int32_t* refs, int64_t n, int64_t limit, unsigned long long* bad,
                              cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int grid = (int)((n + 255) / 256 < 148 * 8 ? (n + 255) / 256 : 148 * 8);
    refs_check_kernel<<<grid, 256, 0, st>>>(refs, n, limit, bad);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// the generic pair kernel (shape read from the kernel parameters)

template <typename Mask>
__global__ void __launch_bounds__(BLOCK, 2)
    pair_kernel(const __grid_constant__ FilterPlan F, const __grid_constant__ VerifyProg V,
                const __grid_constant__ RunParams R) {
    pair_body<Mask, 1>(F, V, R);
}

int pair_kernel_blocks_per_sm() {
    int a = 0, b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, pair_kernel<uint32_t>, BLOCK, 0) != cudaSuccess) a = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, pair_kernel<uint64_t>, BLOCK, 0) != cudaSuccess) b = 1;
    const int nb = a < b ? a : b;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_pair_kernel(const FilterPlan& F, const VerifyProg& V, const RunParams& R, int grid,
                               cudaStream_t st) {
    if (F.n_rules <= 32)
        pair_kernel<uint32_t><<<grid, BLOCK, 0, st>>>(F, V, R);
    else
        pair_kernel<uint64_t><<<grid, BLOCK, 0, st>>>(F, V, R);
    return cudaGetLastError();
}

}  // namespace rb
