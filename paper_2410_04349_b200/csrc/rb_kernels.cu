// rb_kernels.cu -- sm_100a kernels of the rule-evaluation path.
//
// 1. token_features / char_features: one pass over the ragged columns at
//    upload time, producing the fixed-size per-tuple features the pair
//    kernel streams (length, 128-bit token signature, 64-bit id-list hash,
//    16-bucket character histogram).
// 2. pair_kernel: persistent CTAs pull work items (an outer row block x an
//    inner column chunk) from a global counter -- the analogue of the
//    reference's interval claiming and stealing (engine.py:139-207).  Each
//    thread owns one outer tuple in registers; inner tuples are staged
//    through shared memory and read as warp broadcasts.  Per pair the
//    thread runs the phase-1 filter (exact equality / const tests plus
//    exact-safe bounds for jaccard, exact_token and edit), with warp-uniform
//    skipping (__any_sync) of feature classes no live rule needs.  Pairs
//    that may satisfy a rule are pushed into a per-warp shared-memory queue
//    (ballot + popc compaction) and, when it fills, the warp drains it by
//    running the exact path interpreter (evaluate_pair, engine.py:93-132),
//    one pair per lane, and appends rows with one warp-aggregated atomicAdd.
//
// Exactness of the filters (all are bounds on the reference's quantities):
//  * token signature: bit(id) = top-7 bits of id*phi.  With the outer set's
//    bits split into multiplicity levels, u = sum_l popc(level_l & sig_s)
//    counts the outer tokens whose bit is present in the inner signature,
//    so u >= |A n B|; u < mink[n+m] proves jaccard < delta.
//  * id-list hash: different hashes prove different lists (exact_token).
//  * character histogram: 16 buckets of saturating u8 counts; saturation is
//    1-Lipschitz so D' = sum |ha-hb| <= D, and lev >= ceil((D'+|la-lb|)/2)
//    (bag distance), so a bound above maxd[L] proves the edit test fails.
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
        len[r] = (missing && missing[r]) ? -1 : (int32_t)(b - a);
        bag[r] = make_uint4(w[0], w[1], w[2], w[3]);
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

// ---------------------------------------------------------------------------
// exact interpreter (survivors only)

__device__ __forceinline__ uint32_t char_at(const DevColumn& c, int64_t k) {
    return c.width == 1 ? __ldg((const uint8_t*)c.data + k) : __ldg((const uint32_t*)c.data + k);
}

// Banded Levenshtein with cutoff k (Ukkonen): exact when the distance is
// <= k, otherwise returns k+1.  Rows run over the shorter string, the
// single DP row (longer string) lives in this thread's scratch slice.
__device__ int lev_bounded(const DevColumn& ca, int64_t a0, int la, const DevColumn& cb, int64_t b0, int lb, int k,
                           int32_t* row) {
    const DevColumn* cs = &ca;
    const DevColumn* cl = &cb;
    int64_t s0 = a0, l0 = b0;
    int n = la, m = lb;
    if (n > m) {
        cs = &cb;
        cl = &ca;
        s0 = b0;
        l0 = a0;
        n = lb;
        m = la;
    }
    const int INF = k + 1;
    if (m - n > k) return INF;
    if (n == 0) return m;
    for (int j = 0; j <= m; j++) row[j] = min(j, INF);
    for (int i = 1; i <= n; i++) {
        const uint32_t ai = char_at(*cs, s0 + i - 1);
        const int jlo = max(1, i - k), jhi = min(m, i + k);
        int diag = row[jlo - 1];
        int left = (jlo == 1) ? min(i, INF) : INF;
        if (jlo == 1) row[0] = min(i, INF);
        int rmin = (jlo == 1) ? left : INF;
        for (int j = jlo; j <= jhi; j++) {
            const int up = row[j];
            int v = diag + (ai == char_at(*cl, l0 + j - 1) ? 0 : 1);
            v = min(v, up + 1);
            v = min(v, left + 1);
            v = min(v, INF);
            diag = up;
            row[j] = v;
            left = v;
            rmin = min(rmin, v);
        }
        if (rmin > k) return INF;
    }
    return row[m];
}

__device__ int intersect_ids(const int32_t* __restrict__ a, int n, const int32_t* __restrict__ b, int m) {
    int i = 0, j = 0, inter = 0;
    while (i < n && j < m) {
        const int32_t x = __ldg(a + i), y = __ldg(b + j);
        inter += (x == y);
        i += (x <= y);
        j += (y <= x);
    }
    return inter;
}

__device__ bool exact_slot(const VerifyProg& V, int s, int32_t ti, int32_t si, int32_t* scratch) {
    const DevSlot sl = V.slots[s];
    const DevColumn& ca = V.cols[sl.lhs];
    const DevColumn& cb = V.cols[sl.rhs];
    switch (sl.kind) {
        case RB_SLOT_EQ_CODE: {
            const int32_t x = __ldg(ca.codes + ti);
            return x >= 0 && x == __ldg(cb.codes + si);
        }
        case RB_SLOT_EQ_CONST:
            return __ldg(ca.mask + ti) != 0;
        case RB_SLOT_JACCARD: {
            const int n = __ldg(ca.len + ti), m = __ldg(cb.len + si);
            if (n < 0 || m < 0 || (n | m) == 0) return false;
            const int small = min(n, m), big = max(n, m);
            if (big < sl.len0 && small < __ldg(sl.tab0 + big)) return false;
            const int inter = intersect_ids((const int32_t*)ca.data + ca.offsets[ti], n,
                                            (const int32_t*)cb.data + cb.offsets[si], m);
            return n + m < sl.len1 && inter >= __ldg(sl.tab1 + n + m);
        }
        case RB_SLOT_EXACT: {
            const int n = __ldg(ca.len + ti), m = __ldg(cb.len + si);
            if (n < 0 || m < 0 || (n | m) == 0 || n != m) return false;
            const int32_t* a = (const int32_t*)ca.data + ca.offsets[ti];
            const int32_t* b = (const int32_t*)cb.data + cb.offsets[si];
            for (int k = 0; k < n; k++)
                if (__ldg(a + k) != __ldg(b + k)) return false;
            return true;
        }
        case RB_SLOT_EDIT: {
            const int la = __ldg(ca.len + ti), lb = __ldg(cb.len + si);
            if (la < 0 || lb < 0) return false;
            const int L = max(la, lb);
            if (L == 0) return true;
            if (L >= sl.len0 || L >= sl.len1) return false;  // cannot happen: tables cover the columns
            if (abs(la - lb) > __ldg(sl.tab0 + L)) return false;
            const int k = __ldg(sl.tab1 + L);
            if (k < 0) return false;
            const int d = lev_bounded(ca, ca.offsets[ti], la, cb, cb.offsets[si], lb, k, scratch);
            return d <= k;
        }
    }
    return false;
}

// Returns the mask of checkpoint ordinals reached (first one only unless
// enumerating).  engine.py:531-559.
__device__ uint64_t interpret(const VerifyProg& V, int32_t ti, int32_t si, bool enumerate, int32_t* scratch,
                              unsigned long long* slot_evals) {
    uint64_t reuse = 0, value = 0, hit = 0;
    int ip = 0;
    while (ip < V.n_ins) {
        const int4 ins = __ldg(V.ins + ip);
        if (ins.x == 1) {
            hit |= 1ull << ins.y;
            if (!enumerate) break;
            ip++;
            continue;
        }
        const uint64_t bit = 1ull << ins.y;
        bool truth;
        if (reuse & bit) {
            truth = (value & bit) != 0;
        } else {
            truth = exact_slot(V, ins.y, ti, si, scratch);
            reuse |= bit;
            if (truth) value |= bit;
            if (slot_evals) atomicAdd(slot_evals + ins.y, 1ull);
        }
        ip = truth ? ip + 1 : ins.z;
    }
    return hit;
}

__device__ void drain_queue(const VerifyProg& V, const RunParams& R, const int2* q, int qn, const int* cp_rule,
                            int32_t* scratch) {
    const int lane = threadIdx.x & 31;
    const bool enumerate = (R.flags & RB_ENUMERATE) != 0;
    const bool sym = (R.flags & RB_SYMMETRIC) != 0;
    for (int base = 0; base < qn; base += 32) {
        const int k = base + lane;
        uint64_t hit = 0;
        int32_t ti = 0, si = 0;
        if (k < qn) {
            const int2 e = q[k];
            ti = e.x;
            si = e.y;
            hit = interpret(V, ti, si, enumerate, scratch, (R.flags & RB_STATS) ? R.slot_evals : nullptr);
        }
        const int cnt = __popcll(hit);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        unsigned long long at = 0;
        if (lane == 31) at = atomicAdd(R.out_count, (unsigned long long)total);
        at = __shfl_sync(0xffffffffu, at, 31) + (unsigned long long)(incl - cnt);
        int32_t a = ti, b = si;
        if (sym && a > b) {
            a = si;
            b = ti;
        }
        while (hit) {
            const int ord = __ffsll((long long)hit) - 1;
            hit &= hit - 1;
            if (at < (unsigned long long)R.cap) {
                R.out_t[at] = a;
                R.out_s[at] = b;
                R.out_r[at] = cp_rule[ord];
            }
            at++;
        }
    }
}

// ---------------------------------------------------------------------------
// the pair kernel

struct __align__(16) Tile {
    int32_t eq[MAX_EQ][TJ];
    uint4 toksig[MAX_TOK][TJ];
    uint2 tokhash[MAX_TOK][TJ];
    int32_t toklen[MAX_TOK][TJ];
    uint4 strbag[MAX_STR][TJ];
    int32_t strlen_[MAX_STR][TJ];
    int32_t tid[TJ];
};

__device__ __forceinline__ uint64_t alive_rules(const FilterPlan& F, uint64_t maybe) {
    uint64_t alive = 0;
    for (int r = 0; r < F.n_rules; r++)
        if ((maybe & F.need[r]) == F.need[r]) alive |= 1ull << r;
    return alive;
}

__global__ void __launch_bounds__(BLOCK, 2)
    pair_kernel(const __grid_constant__ FilterPlan F, const __grid_constant__ VerifyProg V,
                const __grid_constant__ RunParams R) {
    __shared__ Tile T;
    __shared__ int2 queue[NWARPS][QCAP];
    __shared__ int cp_rule[MAX_RULES];
    __shared__ int s_item;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const unsigned FULL = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;
    int2* q = queue[warp];
    int qn = 0;
    unsigned long long my_pairs = 0, my_surv = 0;
    int32_t* scratch = R.scratch + (int64_t)(blockIdx.x * BLOCK + threadIdx.x) * R.scratch_stride;

    for (int k = threadIdx.x; k < MAX_RULES; k += BLOCK) cp_rule[k] = V.cp_rule[k];

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = (int)atomicAdd(R.item_counter, 1u);
        __syncthreads();
        const int it = s_item;
        if (it >= R.n_items) break;
        const int4 item = R.items[it];
        const int64_t i = (int64_t)item.x + threadIdx.x;
        const int64_t col0 = item.y, col1 = item.z;
        const bool row_ok = i < (int64_t)item.w;

        // ---- outer tuple -> registers
        int32_t ti = 0;
        uint64_t maybe0 = 0;
        int32_t ocode[MAX_EQ];
        int32_t olen[MAX_TOK];
        uint32_t lev[MAX_TOK][MAX_LEV][4];
        uint2 ohash[MAX_TOK];
        bool nofilt[MAX_TOK];
        int nlev[MAX_TOK];
        int32_t oslen[MAX_STR];
        uint4 obag[MAX_STR];
        if (row_ok) {
            ti = R.refs ? R.refs[i] : (int32_t)i;
            maybe0 = ~0ull;
            if (R.mode == MODE_SYM)
                {
                    const int64_t lo = col0 > i + 1 ? col0 : i + 1;
                    my_pairs += (unsigned long long)(col1 > lo ? col1 - lo : 0);
                }
            else if (R.mode == MODE_ASYM)
                my_pairs += (unsigned long long)((col1 - col0) - ((i >= col0 && i < col1) ? 1 : 0));
            else
                my_pairs += (unsigned long long)(col1 - col0);
        }
#pragma unroll
        for (int f = 0; f < MAX_EQ; f++) {
            ocode[f] = INT_MIN;
            if (f < F.n_eq && row_ok) {
                const int32_t c = __ldg(F.eq_outer[f] + ti);
                if (c >= 0)
                    ocode[f] = c;
                else
                    maybe0 &= ~F.eq_slots[f];
            }
        }
#pragma unroll
        for (int k = 0; k < MAX_CONST; k++)
            if (k < F.n_const && row_ok && !__ldg(F.const_mask[k] + ti)) maybe0 &= ~F.const_slots[k];
#pragma unroll
        for (int f = 0; f < MAX_TOK; f++) {
            olen[f] = -1;
            nofilt[f] = false;
            nlev[f] = 0;
            ohash[f] = make_uint2(0, 0);
#pragma unroll
            for (int l = 0; l < MAX_LEV; l++)
#pragma unroll
                for (int w = 0; w < 4; w++) lev[f][l][w] = 0;
            if (f < F.n_tok && row_ok) {
                olen[f] = __ldg(F.tok_olen[f] + ti);
                ohash[f] = __ldg(F.tok_ohash[f] + ti);
                const int64_t a = __ldg(F.tok_ooff[f] + ti), b = __ldg(F.tok_ooff[f] + ti + 1);
                for (int64_t k = a; k < b; k++) {
                    const uint32_t bit = sig_bit(__ldg(F.tok_oids[f] + k));
                    const uint32_t m = 1u << (bit & 31);
                    const uint32_t wsel = bit >> 5;
                    bool placed = false;
#pragma unroll
                    for (int l = 0; l < MAX_LEV; l++) {
#pragma unroll
                        for (int w = 0; w < 4; w++) {
                            if (!placed && w == (int)wsel && !(lev[f][l][w] & m)) {
                                lev[f][l][w] |= m;
                                placed = true;
                                nlev[f] = max(nlev[f], l + 1);
                            }
                        }
                    }
                    if (!placed) nofilt[f] = true;
                }
            }
            nlev[f] = __reduce_max_sync(FULL, (unsigned)nlev[f]);
        }
#pragma unroll
        for (int f = 0; f < MAX_STR; f++) {
            oslen[f] = -1;
            obag[f] = make_uint4(0, 0, 0, 0);
            if (f < F.n_str && row_ok) {
                oslen[f] = __ldg(F.str_olen[f] + ti);
                obag[f] = __ldg(F.str_obag[f] + ti);
            }
        }
        const int64_t i_row = row_ok ? i : INT64_MAX;

        // ---- stream inner tiles
        for (int64_t jt = col0; jt < col1; jt += TJ) {
            const int tn = (int)(col1 - jt < TJ ? col1 - jt : TJ);
            __syncthreads();
            for (int k = threadIdx.x; k < tn; k += BLOCK) {
                const int64_t j = jt + k;
                const int32_t sj = R.refs ? __ldg(R.refs + j) : (int32_t)j;
                T.tid[k] = sj;
#pragma unroll
                for (int f = 0; f < MAX_EQ; f++)
                    if (f < F.n_eq) T.eq[f][k] = __ldg(F.eq_inner[f] + sj);
#pragma unroll
                for (int f = 0; f < MAX_TOK; f++)
                    if (f < F.n_tok) {
                        T.toklen[f][k] = __ldg(F.tok_ilen[f] + sj);
                        T.toksig[f][k] = __ldg(F.tok_isig[f] + sj);
                        T.tokhash[f][k] = __ldg(F.tok_ihash[f] + sj);
                    }
#pragma unroll
                for (int f = 0; f < MAX_STR; f++)
                    if (f < F.n_str) {
                        T.strlen_[f][k] = __ldg(F.str_ilen[f] + sj);
                        T.strbag[f][k] = __ldg(F.str_ibag[f] + sj);
                    }
            }
            __syncthreads();

            for (int jj = 0; jj < tn; jj++) {
                const int64_t j = jt + jj;
                bool valid;
                if (R.mode == MODE_SYM)
                    valid = j > i_row;
                else if (R.mode == MODE_ASYM)
                    valid = row_ok && j != i;
                else
                    valid = row_ok;
                uint64_t maybe = valid ? maybe0 : 0ull;
#pragma unroll
                for (int f = 0; f < MAX_EQ; f++)
                    if (f < F.n_eq && ocode[f] != T.eq[f][jj]) maybe &= ~F.eq_slots[f];
                uint64_t alive = alive_rules(F, maybe);

#pragma unroll
                for (int f = 0; f < MAX_TOK; f++) {
                    if (f < F.n_tok && __any_sync(FULL, (alive & F.tok_rules[f]) != 0)) {
                        const int m = T.toklen[f][jj];
                        const uint4 is = T.toksig[f][jj];
                        const int n = olen[f];
                        int u = 0;
#pragma unroll
                        for (int l = 0; l < MAX_LEV; l++)
                            if (l < nlev[f])
                                u += __popc(lev[f][l][0] & is.x) + __popc(lev[f][l][1] & is.y) +
                                     __popc(lev[f][l][2] & is.z) + __popc(lev[f][l][3] & is.w);
                        if (nofilt[f]) u = INT_MAX;
                        const bool dead = n < 0 || m < 0 || (n | m) == 0;
                        const int small = min(n, m), big = max(n, m);
                        u = min(u, small);
                        for (int z = 0; z < F.tok_nslots[f]; z++) {
                            const TokSlotF& ts = F.tok_slot[f][z];
                            bool ok;
                            if (dead) {
                                ok = false;
                            } else if (ts.kind == RB_SLOT_JACCARD) {
                                ok = (big >= ts.len0 || small >= __ldg(ts.tab0 + big)) &&
                                     (n + m >= ts.len1 || u >= __ldg(ts.tab1 + n + m));
                            } else {
                                const uint2 h = T.tokhash[f][jj];
                                ok = n == m && h.x == ohash[f].x && h.y == ohash[f].y;
                            }
                            if (!ok) maybe &= ~(1ull << ts.bit);
                        }
                        alive = alive_rules(F, maybe);
                    }
                }
#pragma unroll
                for (int f = 0; f < MAX_STR; f++) {
                    if (f < F.n_str && __any_sync(FULL, (alive & F.str_rules[f]) != 0)) {
                        const int la = oslen[f], lb = T.strlen_[f][jj];
                        const uint4 ib = T.strbag[f][jj];
                        const int L = max(la, lb);
                        const int gap = abs(la - lb);
                        const int D = (int)(__vsadu4(obag[f].x, ib.x) + __vsadu4(obag[f].y, ib.y) +
                                            __vsadu4(obag[f].z, ib.z) + __vsadu4(obag[f].w, ib.w));
                        const int lower = max(gap, (D + gap + 1) >> 1);
                        for (int z = 0; z < F.str_nslots[f]; z++) {
                            const StrSlotF& ss = F.str_slot[f][z];
                            bool ok;
                            if (la < 0 || lb < 0)
                                ok = false;
                            else if (L == 0 || L >= ss.len0 || L >= ss.len1)
                                ok = true;
                            else
                                ok = gap <= __ldg(ss.maxgap + L) && lower <= __ldg(ss.maxd + L);
                            if (!ok) maybe &= ~(1ull << ss.bit);
                        }
                        alive = alive_rules(F, maybe);
                    }
                }

                const bool surv = alive != 0;
                const unsigned bal = __ballot_sync(FULL, surv);
                if (bal) {
                    if (surv) q[qn + __popc(bal & lt_mask)] = make_int2(ti, T.tid[jj]);
                    qn += __popc(bal);
                    my_surv += surv ? 1 : 0;
                    if (qn > QCAP - 32) {
                        __syncwarp();
                        drain_queue(V, R, q, qn, cp_rule, scratch);
                        __syncwarp();
                        qn = 0;
                    }
                }
            }
        }
        if (qn) {
            __syncwarp();
            drain_queue(V, R, q, qn, cp_rule, scratch);
            __syncwarp();
            qn = 0;
        }
    }

    // ---- statistics
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_pairs += __shfl_down_sync(FULL, my_pairs, o);
        my_surv += __shfl_down_sync(FULL, my_surv, o);
    }
    if (lane == 0) {
        atomicAdd(R.stat_pairs, my_pairs);
        atomicAdd(R.stat_surv, my_surv);
    }
}

int pair_kernel_blocks_per_sm() {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pair_kernel, BLOCK, 0) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_pair_kernel(const FilterPlan& F, const VerifyProg& V, const RunParams& R, int grid,
                               cudaStream_t st) {
    pair_kernel<<<grid, BLOCK, 0, st>>>(F, V, R);
    return cudaGetLastError();
}

}  // namespace rb
