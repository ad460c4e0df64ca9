// rb_device.cuh -- all device code of the pair evaluation, self-contained so
// that it compiles both with nvcc (the generic kernel, built into
// librbgpu.so) and with NVRTC at program-creation time (a kernel specialised
// to one program's shape: number of equality / token / string features and
// slots per feature become compile-time constants, so the per-pair loop has
// no dispatch left -- query compilation, the way a database compiles a plan).
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
// The derived per-tuple features are what the pair kernel streams: fixed-size,
// 16-byte aligned, read with 128-bit loads.  The ragged arrays are touched
// only by the exact interpreter for surviving pairs.
//
// Exactness of the phase-1 filters (each is a bound on the reference's own
// quantity, so a pair is dropped only when a predicate is certainly false):
//  * token signature: bit(id) = top-7 bits of id*phi.  u = popc(sig_t & sig_s)
//    + (|t| - popc(sig_t)) counts every outer token whose bit is present in
//    the inner signature plus every outer token that shares its bit with an
//    earlier one, so u >= |A n B|; u < mink[n+m] proves jaccard < delta.
//    For short token rows both signatures are folded to 64 bits (bit b and
//    b+64 merged) -- the same argument holds on the folded bits.
//  * id-list hash: different hashes prove different lists (exact_token).
//  * character histogram: 16 buckets of saturating u8 counts; saturation is
//    1-Lipschitz so D' = sum |ha-hb| <= D, and lev >= ceil((D'+|la-lb|)/2)
//    (bag distance), so a bound above maxd[L] proves the edit test fails.
#pragma once

#ifdef __CUDACC_RTC__
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned long long uintptr_t;
#define INT_MIN (-2147483647 - 1)
#define INT_MAX 2147483647
#define INT64_MAX 9223372036854775807LL
#define RB_SLOT_EQ_CODE 0
#define RB_SLOT_EQ_CONST 1
#define RB_SLOT_JACCARD 2
#define RB_SLOT_EXACT 3
#define RB_SLOT_EDIT 4
#define RB_SYMMETRIC 1u
#define RB_ENUMERATE 2u
#define RB_STATS 4u
#define RB_MAX_SLOTS 64
#define RB_MAX_CHECKPOINTS 64
#endif

namespace rb {

constexpr int MAX_COLS = 64;
#ifndef SPEC_PREANY
#define SPEC_PREANY 1  // gated kernels: the stage-1 pre-vote in tile_loop (RB_PREANY=0 at run time: off)
#endif
#ifndef SPEC_PACKED
#define SPEC_PACKED 0  // 1: the kernel also takes MODE_PACKED items (batches of tiny partitions)
#endif

constexpr int MAX_EQ = 6;      // equality features filtered in the pair loop
constexpr int MAX_TOK = 2;     // token-set features (jaccard / exact_token)
constexpr int MAX_STR = 2;     // string features (edit)
constexpr int MAX_CONST = 8;   // t.attr = const masks
constexpr int MAX_FSLOTS = 4;  // slots sharing one token / string feature
constexpr int MAX_RULES = RB_MAX_CHECKPOINTS;
constexpr int SMEM_TAB = 2048; // int32 threshold-table entries staged in shared memory

constexpr int BLOCK = 256;     // threads per CTA = outer rows per item
constexpr int TJ = 128;        // inner tuples per shared-memory tile
constexpr int QCAP = 256;      // survivor queue entries per warp
constexpr int NWARPS = BLOCK / 32;
constexpr int64_t CHUNK = 16384;  // inner columns per work item

// MODE_PACKED: several whole partitions of a batch back to back in one item
// (rows [row0, row_hi), parts [part, pad0)); a row pairs only with the later
// rows (symmetric) or the other rows (asymmetric) of its own partition.  Only
// the packed kernel variant (SPEC_PACKED) is given such items.
enum RunMode : int32_t { MODE_SYM = 0, MODE_ASYM = 1, MODE_CROSS = 2, MODE_PACKED = 3 };

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

// One filtered slot on a token / string feature.  Its exact tables are
// staged in shared memory at [off0, off0+cap0) and [off1, off1+cap1); a
// length beyond a cap is simply not filtered (left to the exact pass).
struct FSlot {
    uint64_t kill;  // rules whose precondition contains this slot (+ rules it rules out by implication)
    int32_t kind;
    int32_t off0, cap0;
    int32_t off1, cap1;
    int32_t w2;      // jaccard in 2-D mode: need[n][m] at off0 + n*w2 + (m+1)
    int32_t slot;    // the path slot it filters
    int32_t stage2;  // evaluated after the stage-1 gate (see FilterPlan::gate)
    double delta;    // threshold (implied kills between slots of one feature)
};

// Phase-1 filter program.  Per pair the kernel keeps the set of rules that
// may still hold ("alive"); a predicate proven false kills every rule that
// needs it.  Equality / const tests are exact; token and string slots use
// exact-safe bounds.  Survivors are re-evaluated exactly.
struct FilterPlan {
    int32_t n_eq, n_tok, n_str, n_const, n_rules, n_tab;
    int32_t full_tab;  // every shared table covers its column's longest row
    int32_t rows;      // outer rows per thread of the kernel that will run (items cover BLOCK * rows)
    int32_t tok2d;     // jaccard thresholds as one 2-D table need[n][m] per slot (see FSlot)
    uint64_t all_rules;
    const int32_t* tab_src;  // n_tab int32 entries copied to shared memory
    const int32_t* eq_outer[MAX_EQ];
    const int32_t* eq_inner[MAX_EQ];
    uint64_t eq_kill[MAX_EQ];
    uint64_t eq_slots[MAX_EQ];   // path slots the feature tests (a composite key: several)
    int32_t eq_stage2[MAX_EQ];   // evaluated after the stage-1 gate
    // Stage-1 gate: a few selective tests whose (implied) kills cover every
    // rule run first; a warp with no live pair left skips all other tests.
    int32_t gate;
    // eq_any: the stage-1 equality keys are sparse (a regated plan: the unit's
    // own key is implied, the rest rarely match), so a pair first ORs their
    // compares; with no key equal its rules drop to eq_free (the rules no
    // stage-1 key kills) in one step, and the per-key kills run only behind a
    // warp vote when some lane's row matched a key
    int32_t eq_any;
    uint64_t eq_free;
    const uint8_t* const_mask[MAX_CONST];
    uint64_t const_kill[MAX_CONST];
    const int64_t* tok_ooff[MAX_TOK];
    const int32_t* tok_oids[MAX_TOK];
    const int32_t* tok_olen[MAX_TOK];
    const uint2* tok_ohash[MAX_TOK];
    const int32_t* tok_ilen[MAX_TOK];
    const uint4* tok_isig[MAX_TOK];
    const uint2* tok_ihash[MAX_TOK];
    int32_t tok_nslots[MAX_TOK];  // slots on the feature: the first tok_njac are jaccard, the rest exact_token
    int32_t tok_njac[MAX_TOK];
    int32_t tok_always[MAX_TOK];  // some rule reaches this feature with nothing filtered before it
    int32_t tok_sig64[MAX_TOK];   // short token rows: fold the signature to 64 bits (half the popcounts)
    uint64_t tok_rules[MAX_TOK];
    uint64_t tok_kill[MAX_TOK];  // OR of the feature's slot kills: an outer row without tokens fails them all
    FSlot tok_slot[MAX_TOK][MAX_FSLOTS];
    int32_t tok_off[MAX_TOK];  // 2-D mode: interleaved need[n][m][z] table (see rb_program_create)
    int32_t tok_w2[MAX_TOK];
    int32_t tok_njp[MAX_TOK];  // jaccard slots per entry, padded to 1, 2 or 4
    const int32_t* str_olen[MAX_STR];
    const uint4* str_obag[MAX_STR];
    const int32_t* str_ilen[MAX_STR];
    const uint4* str_ibag[MAX_STR];
    int32_t str_nslots[MAX_STR];
    uint64_t str_rules[MAX_STR];
    uint64_t str_kill[MAX_STR];  // a missing outer string fails every slot on the feature
    int32_t str_always[MAX_STR];
    int32_t str_fold[MAX_STR];  // 8-bucket (folded) bags for this string feature
    FSlot str_slot[MAX_STR][MAX_FSLOTS];
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

// One work item: outer rows [row0, row_hi) x inner columns [col0, col1) of
// the concatenated refs array, in one partition's pair space.
struct __align__(16) Item {
    int32_t row0, col0, col1, row_hi;
    int32_t mode;  // RunMode of the item's partition
    int32_t part;  // index of the partition in the batch
    int32_t pad0, pad1;
};

struct RunParams {
    const int32_t* refs;  // position -> tid; nullptr = identity
    int64_t n;
    uint32_t flags;
    const Item* items;
    int32_t n_items;
    unsigned int* item_counter;
    int32_t* out_t;
    int32_t* out_s;
    int32_t* out_r;
    int32_t* out_p;  // partition index per row (batched runs), may be null
    unsigned long long* out_count;
    long long cap;
    unsigned long long* stat_pairs;
    unsigned long long* stat_surv;
    unsigned long long* stat_gate;  // warp iterations that passed the stage-1 gate (gated kernels)
    unsigned long long* slot_evals;
    int32_t* scratch;
    int64_t scratch_stride;
    // deferred verification (specialised kernel): phase 1 appends its
    // survivors {t, s, part} here; rb_verify_kernel_spec decides them
    int4* surv;
    long long surv_cap;
    unsigned long long* surv_count;
    const unsigned long long* bad_refs;  // non-zero: a tuple ref is out of range, evaluate nothing
    const int32_t* part_off;  // packed items: start position of every part of the batch (+ the end)
    const int32_t* part_end;  // packed items: end position of every part (parts of a pack are adjacent)
};

// the part of a packed item (parts [lo, hi)) holding position pos
static __device__ __forceinline__ int find_part(const RunParams& R, int lo, int hi, int64_t pos) {
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(R.part_off + mid) <= pos)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// device-side helpers shared by kernels
__host__ __device__ inline uint32_t sig_bit(int32_t id) { return ((uint32_t)id * 0x9E3779B1u) >> 25; }
__host__ __device__ inline uint32_t bag_bucket(uint32_t c) { return (c * 0x9E3779B1u) >> 28; }
__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// exact interpreter (survivors only)

static __device__ __forceinline__ uint32_t char_at(const DevColumn& c, int64_t k) {
    return c.width == 1 ? __ldg((const uint8_t*)c.data + k) : __ldg((const uint32_t*)c.data + k);
}

// Four bytes of a u8 column starting at any byte offset (two aligned loads).
static __device__ __forceinline__ uint32_t load4_u8(const DevColumn& c, int64_t k) {
    const uint8_t* p = (const uint8_t*)c.data + k;
    const uint32_t* w = (const uint32_t*)((uintptr_t)p & ~(uintptr_t)3);
    const uint32_t sh = (uint32_t)((uintptr_t)p & 3) * 8;
    return __funnelshift_r(__ldg(w), __ldg(w + 1), sh);
}

// Length of the common run s[i..] == l[i+d..] starting at i (returns the
// first mismatching i, capped by both ends).  u8 columns compare four
// characters per step.
static __device__ __forceinline__ int slide(const DevColumn& cs, int64_t s0, int n, const DevColumn& cl, int64_t l0,
                                            int m, int i, int d) {
    if (cs.width == 1 && cl.width == 1) {
        while (i + 4 <= n && i + d + 4 <= m) {
            const uint32_t x = load4_u8(cs, s0 + i) ^ load4_u8(cl, l0 + i + d);
            if (x) return i + ((__ffs(x) - 1) >> 3);
            i += 4;
        }
    }
    while (i < n && i + d < m && char_at(cs, s0 + i) == char_at(cl, l0 + i + d)) i++;
    return i;
}

// Myers' bit-vector Levenshtein distance (Myers 1999, the block form with
// the horizontal delta carried from word to word): the shorter string is the
// pattern, 64 of its positions per machine word; every character of the other
// string advances all W = ceil(n/64) words by ~15 integer ops, so a pair costs
// O(ceil(n/64) m) word steps instead of the band's O(n k) cells.  The
// pattern's match masks Peq[c] live in the thread's scratch slice: an
// open-addressed table of its distinct characters (at most MYERS_DCAP) and
// MYERS_DCAP x W masks.  Stops as soon as the last row's score minus the
// columns left exceeds k (the final score cannot come back under k).
// Returns the exact distance when <= k, k+1 when above, -1 when the pattern
// does not fit (longer than MYERS_NMAX or more than MYERS_DCAP distinct
// characters): the caller then runs the banded DP.
#define MYERS_NMAX 1024
#define MYERS_DCAP 48
#define MYERS_HS 64  // hash slots (power of two > MYERS_DCAP)
static __device__ __forceinline__ int myers_slot(const int32_t* hkey, uint32_t c) {
    uint32_t h = (c * 0x9E3779B1u) >> 26;  // 6 bits: MYERS_HS slots
    while (true) {
        const int32_t k = hkey[h];
        if (k == (int32_t)c || k == -1) return (int)h;
        h = (h + 1) & (MYERS_HS - 1);
    }
}
static __device__ int lev_myers(const DevColumn& cs, int64_t s0, int n, const DevColumn& cl, int64_t l0, int m,
                                int k, int32_t* scr) {
    if (n > MYERS_NMAX) return -1;
    const int W = (n + 63) >> 6;
    int32_t* hkey = scr;
    int32_t* hidx = scr + MYERS_HS;
    uint64_t* peq = (uint64_t*)(scr + 2 * MYERS_HS);  // 8-byte aligned: the slice is 128-byte aligned
    for (int h = 0; h < MYERS_HS; h++) hkey[h] = -1;
    int D = 0;
    for (int i = 0; i < n; i++) {
        const uint32_t c = char_at(cs, s0 + i);
        const int h = myers_slot(hkey, c);
        int idx = hidx[h];
        if (hkey[h] == -1) {
            if (D == MYERS_DCAP) return -1;
            hkey[h] = (int32_t)c;
            hidx[h] = idx = D++;
            for (int w = 0; w < W; w++) peq[idx * W + w] = 0;
        }
        peq[idx * W + (i >> 6)] |= 1ull << (i & 63);
    }
    uint64_t Pv[MYERS_NMAX / 64], Mv[MYERS_NMAX / 64];
    for (int w = 0; w < W; w++) {
        Pv[w] = ~0ull;
        Mv[w] = 0;
    }
    const int last = (n - 1) & 63;
    int score = n;
    for (int j = 0; j < m; j++) {
        const uint32_t c = char_at(cl, l0 + j);
        const int h = myers_slot(hkey, c);
        const uint64_t* eqv = hkey[h] == -1 ? nullptr : peq + hidx[h] * W;
        int hin = 1;  // the top row D[0][j] = j rises by one per column
        for (int w = 0; w < W; w++) {
            uint64_t Eq = eqv ? eqv[w] : 0ull;
            const uint64_t pv = Pv[w], mv = Mv[w];
            const uint64_t Xv = Eq | mv;
            if (hin < 0) Eq |= 1ull;
            const uint64_t Xh = (((Eq & pv) + pv) ^ pv) | Eq;
            uint64_t Ph = mv | ~(Xh | pv);
            uint64_t Mh = pv & Xh;
            const int high = (w == W - 1) ? last : 63;
            const int hout = (int)((Ph >> high) & 1ull) - (int)((Mh >> high) & 1ull);
            Ph <<= 1;
            Mh <<= 1;
            if (hin < 0)
                Mh |= 1ull;
            else if (hin > 0)
                Ph |= 1ull;
            Pv[w] = Mh | ~(Xv | Ph);
            Mv[w] = Ph & Xv;
            hin = hout;
        }
        score += hin;
        if (score - (m - 1 - j) > k) return k + 1;
    }
    return score <= k ? score : k + 1;
}

// Bounded Levenshtein: exact when the distance is <= k, otherwise k+1.
// For k <= 31 (every threshold the configs use) it is Landau-Vishkin /
// Ukkonen's diagonal algorithm: for e = 0..k edits keep, per diagonal
// d = j - i, the furthest row reachable with e edits, then slide along
// matching characters.  Cost O(k^2 + slide length) instead of the band's
// O(n k) cells; near-duplicate strings slide almost all the way at e = 0.
// Wider bounds first try the same diagonal algorithm up to 31 edits (a
// near duplicate is decided there), then Myers' bit-vector algorithm; a
// pattern Myers cannot hold runs a banded DP over the thread's slice of
// the global scratch.
static __device__ int lev_bounded(const DevColumn& ca, int64_t a0, int la, const DevColumn& cb, int64_t b0, int lb, int k,
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
    {
        const int kd = min(k, 31);  // the diagonal algorithm's own bound
        constexpr int OFF = 32, NEG = -(1 << 30);
        int fr0[2 * OFF + 1], fr1[2 * OFF + 1];  // furthest row per diagonal, index OFF + d
        int* prev = fr0;
        int* cur = fr1;
        const int dfin = m - n;
        int i = slide(*cs, s0, n, *cl, l0, m, 0, 0);
        if (dfin == 0 && i >= n) return 0;
        prev[OFF] = i;
        for (int e = 1; e <= kd; e++) {
            for (int d = -e; d <= e; d++) {
                int best = NEG;
                if (d >= -(e - 1) && d <= e - 1) best = prev[OFF + d] + 1;                      // substitution
                if (d + 1 >= -(e - 1) && d + 1 <= e - 1) best = max(best, prev[OFF + d + 1] + 1);  // skip s[i]
                if (d - 1 >= -(e - 1) && d - 1 <= e - 1) best = max(best, prev[OFF + d - 1]);      // skip l[j]
                if (d > m || -d > n || best < 0) {
                    cur[OFF + d] = NEG;
                    continue;
                }
                i = min(best, min(n, m - d));
                i = slide(*cs, s0, n, *cl, l0, m, i, d);
                cur[OFF + d] = i;
                if (d == dfin && i >= n) return e;
            }
            int* t = prev;
            prev = cur;
            cur = t;
        }
        if (k <= 31) return INF;
    }
    const int dm = lev_myers(*cs, s0, n, *cl, l0, m, k, row);
    if (dm >= 0) return dm;
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

static __device__ int intersect_ids(const int32_t* __restrict__ a, int n, const int32_t* __restrict__ b, int m) {
    int i = 0, j = 0, inter = 0;
    while (i < n && j < m) {
        const int32_t x = __ldg(a + i), y = __ldg(b + j);
        inter += (x == y);
        i += (x <= y);
        j += (y <= x);
    }
    return inter;
}

static __device__ bool exact_slot(const VerifyProg& V, int s, int32_t ti, int32_t si, int32_t* scratch) {
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
static __device__ uint64_t interpret(const VerifyProg& V, int32_t ti, int32_t si, bool enumerate, int32_t* scratch,
                              unsigned long long* slot_evals, uint64_t* touched = nullptr) {
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
    if (touched) *touched = reuse;
    return hit;
}

// Per-slot first-touch counts of a warp's pairs, added with one shared-memory
// atomic per touched slot (a ballot per slot instead of one global atomic per
// evaluation: 538M survivors x a few slots contended on 64 global counters).
static __device__ __forceinline__ void count_touched(uint64_t touched, unsigned long long* evals) {
    const unsigned FULL = 0xffffffffu;
    uint64_t any = ((uint64_t)__reduce_or_sync(FULL, (unsigned)(touched >> 32)) << 32) |
                   (uint64_t)__reduce_or_sync(FULL, (unsigned)touched);
    while (any) {
        const int s = __ffsll((long long)any) - 1;
        any &= any - 1;
        const unsigned n = __popc(__ballot_sync(FULL, (touched >> s) & 1ull));
        if ((threadIdx.x & 31) == 0) atomicAdd(evals + s, (unsigned long long)n);
    }
}

// Warp-collective: every lane decides one pair (valid lanes only) with the
// exact interpreter and the warp appends the reached checkpoints' rows with
// one atomicAdd.  engine.py:531-559 + CandidateSink.reserve (214-246).
// evals: per-slot counters the warp adds its first touches to (RB_STATS):
// shared-memory counters of the block in the verify kernel, else null
static __device__ __forceinline__ void verify_emit(const VerifyProg& V, const RunParams& R, bool valid, int32_t ti,
                                                   int32_t si, int part, const int* cp_rule, int32_t* scratch,
                                                   unsigned long long* evals = nullptr) {
    const int lane = threadIdx.x & 31;
    const bool enumerate = (R.flags & RB_ENUMERATE) != 0;
    const bool sym = (R.flags & RB_SYMMETRIC) != 0;
    uint64_t hit = 0;
    if (evals) {
        uint64_t touched = 0;
        if (valid) hit = interpret(V, ti, si, enumerate, scratch, nullptr, &touched);
        count_touched(touched, evals);
    } else if (valid) {
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
    if (total == 0) return;
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
            if (R.out_p) R.out_p[at] = part;
        }
        at++;
    }
}

static __device__ __noinline__ void drain_queue(const VerifyProg& V, const RunParams& R, const int2* q, int qn, int part, const int* cp_rule,
                            int32_t* scratch) {
    const int lane = threadIdx.x & 31;
    for (int base = 0; base < qn; base += 32) {
        const int k = base + lane;
        const int2 e = k < qn ? q[k] : make_int2(0, 0);
        verify_emit(V, R, k < qn, e.x, e.y, part, cp_rule, scratch);
    }
}

// Deferred form: the warp appends its queue to the global survivor buffer
// (one atomicAdd, coalesced 16-byte stores).  Entries past the capacity are
// counted but not stored; the host then re-runs with room for all of them.
// part_hi >= 0: a packed item (parts [part, part_hi)); its queue entries
// carry the outer position instead of the tid
static __device__ __forceinline__ void flush_survivors(const RunParams& R, const int2* q, int qn, int part,
                                                       int part_hi = -1) {
    const int lane = threadIdx.x & 31;
    unsigned long long at = 0;
    if (lane == 0) at = atomicAdd(R.surv_count, (unsigned long long)qn);
    at = __shfl_sync(0xffffffffu, at, 0);
    for (int k = lane; k < qn; k += 32)
        if (at + k < (unsigned long long)R.surv_cap) {
            const int2 e = q[k];
            if (part_hi >= 0)
                R.surv[at + k] = make_int4(R.refs ? __ldg(R.refs + e.x) : e.x, e.y, find_part(R, part, part_hi, e.x), 0);
            else
                R.surv[at + k] = make_int4(e.x, e.y, part, 0);
        }
}

// Phase 2 as its own kernel: every thread decides one buffered survivor.
// Runs at full occupancy with its own register budget, so the pair kernel
// keeps no interpreter state.
__device__ __forceinline__ void verify_body(const VerifyProg& V, const RunParams& R) {
    __shared__ int cp_rule[RB_MAX_CHECKPOINTS];
    __shared__ unsigned long long evals[RB_MAX_SLOTS];
    for (int k = threadIdx.x; k < RB_MAX_CHECKPOINTS; k += blockDim.x) cp_rule[k] = V.cp_rule[k];
    for (int k = threadIdx.x; k < RB_MAX_SLOTS; k += blockDim.x) evals[k] = 0;
    __syncthreads();
    const bool stats = (R.flags & RB_STATS) != 0;
    const unsigned long long cnt = *R.surv_count;
    const long long n = (long long)(cnt < (unsigned long long)R.surv_cap ? cnt : (unsigned long long)R.surv_cap);
    int32_t* scratch = R.scratch + (int64_t)(blockIdx.x * blockDim.x + threadIdx.x) * R.scratch_stride;
    const long long stride = (long long)gridDim.x * blockDim.x;
    // whole warps iterate together (verify_emit is warp-collective)
    for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
        const long long k = base + (threadIdx.x & 31);
        const int4 e = k < n ? R.surv[k] : make_int4(0, 0, 0, 0);
        verify_emit(V, R, k < n, e.x, e.y, e.z, cp_rule, scratch, stats ? evals : nullptr);
    }
    if (stats) {
        __syncthreads();
        for (int k = threadIdx.x; k < V.n_slots && k < RB_MAX_SLOTS; k += blockDim.x)
            if (evals[k]) atomicAdd(R.slot_evals + k, evals[k]);
    }
}

// ---------------------------------------------------------------------------
// the pair kernel

// One inner tuple's streamed features, stored record-wise so that the pair
// loop reads every field of tuple jj at a constant offset from one running
// shared-memory address (eq codes and token length share a 32-byte line).
// 160-byte stride: the tile fill (thread k writes record k) hits 8 banks
// instead of 1.
struct __align__(16) Rec {
    // equality codes at [0, n_eq), token-row lengths right after them at
    // [n_eq, n_eq + n_tok): with few features one 16-byte load fetches all
    int32_t head[MAX_EQ + MAX_TOK];
    uint4 toksig[MAX_TOK];
    uint2 tokhash[MAX_TOK];
    int32_t strlen_[MAX_STR];
    int32_t tid;
    int32_t pad0;
    uint4 strbag[MAX_STR];
    int32_t strm2[MAX_STR][MAX_FSLOTS];  // 2*maxd[|s|] per edit slot (see the string filter)
};

// byte offset of a Rec field (the pre-vote's explicit shared-memory loads)
#define RB_REC_OFF(field) ((uint32_t)(uintptr_t)(&((const Rec*)nullptr)->field))

struct __align__(16) Tile {
    Rec r[TJ];
};

// Shape of the filter program: compile-time constants in a specialised
// (NVRTC) build, kernel-parameter reads in the generic build.
#ifdef RB_SPEC
#define RB_NEQ SPEC_NEQ
#define RB_NCONST SPEC_NCONST
#define RB_NTOK SPEC_NTOK
#define RB_NSTR SPEC_NSTR
#define RB_TOK_NS(f) ((f) == 0 ? SPEC_TOK0_NS : SPEC_TOK1_NS)
#define RB_TOK_NJ(f) ((f) == 0 ? SPEC_TOK0_NJ : SPEC_TOK1_NJ)
#define RB_TOK_ALWAYS(f) ((f) == 0 ? SPEC_TOK0_ALWAYS : SPEC_TOK1_ALWAYS)
#define RB_TOK_SIG64(f) ((f) == 0 ? SPEC_TOK0_SIG64 : SPEC_TOK1_SIG64)
#define RB_TOK_NJP(f) (RB_TOK_NJ(f) <= 1 ? 1 : RB_TOK_NJ(f) <= 2 ? 2 : 4)
#define RB_STR_NS(f) ((f) == 0 ? SPEC_STR0_NS : SPEC_STR1_NS)
#define RB_STR_ALWAYS(f) ((f) == 0 ? SPEC_STR0_ALWAYS : SPEC_STR1_ALWAYS)
#define RB_STR_FOLD(f) ((f) == 0 ? SPEC_STR0_FOLD : SPEC_STR1_FOLD)
#define RB_FULLTAB SPEC_FULLTAB
#define RB_TOK2D SPEC_TOK2D
// rule masks are compile-time constants too: a failed test becomes one
// predicated LOP3 on the live-rule mask
#define RB_PICK6(f, P) ((f) == 0 ? P##0 : (f) == 1 ? P##1 : (f) == 2 ? P##2 : (f) == 3 ? P##3 : (f) == 4 ? P##4 : P##5)
#define RB_PICK8(f, P) ((f) < 6 ? RB_PICK6(f, P) : (f) == 6 ? P##6 : P##7)
#define RB_PICK2(f, P) ((f) == 0 ? P##0 : P##1)
#define RB_PICK4(z, P) ((z) == 0 ? P##0 : (z) == 1 ? P##1 : (z) == 2 ? P##2 : P##3)
#define RB_ALL_RULES SPEC_ALL_RULES
#define RB_EQ_KILL(f) RB_PICK6(f, SPEC_EQ_KILL_)
#define RB_CONST_KILL(k) RB_PICK8(k, SPEC_CONST_KILL_)
#define RB_TOK_ROWKILL(f) RB_PICK2(f, SPEC_TOK_ROWKILL_)
#define RB_STR_ROWKILL(f) RB_PICK2(f, SPEC_STR_ROWKILL_)
#define RB_TOK_RULES(f) RB_PICK2(f, SPEC_TOK_RULES_)
#define RB_STR_RULES(f) RB_PICK2(f, SPEC_STR_RULES_)
#define RB_TOK_KILL(f, z) ((f) == 0 ? RB_PICK4(z, SPEC_TOK0_KILL_) : RB_PICK4(z, SPEC_TOK1_KILL_))
#define RB_STR_KILL(f, z) ((f) == 0 ? RB_PICK4(z, SPEC_STR0_KILL_) : RB_PICK4(z, SPEC_STR1_KILL_))
#define RB_GATE SPEC_GATE
#ifndef SPEC_EQ_ANY
#define SPEC_EQ_ANY 0
#endif
#define RB_EQ_STAGE2(f) RB_PICK6(f, SPEC_EQ_STAGE2_)
#define RB_TOK_STAGE2(f, z) ((f) == 0 ? RB_PICK4(z, SPEC_TOK0_STAGE2_) : RB_PICK4(z, SPEC_TOK1_STAGE2_))
// edit tables' shared-memory offsets as immediates: the lookup is one LEA + LDS [R + imm]
#define RB_STR_OFF(f, z) ((f) == 0 ? RB_PICK4(z, SPEC_STR0_OFF_) : RB_PICK4(z, SPEC_STR1_OFF_))
#else
#define RB_NEQ F.n_eq
#define RB_NCONST F.n_const
#define RB_NTOK F.n_tok
#define RB_NSTR F.n_str
#define RB_TOK_NS(f) F.tok_nslots[f]
#define RB_TOK_NJ(f) F.tok_njac[f]
#define RB_TOK_ALWAYS(f) F.tok_always[f]
#define RB_TOK_SIG64(f) F.tok_sig64[f]
#define RB_TOK_NJP(f) F.tok_njp[f]
#define RB_STR_NS(f) F.str_nslots[f]
#define RB_STR_ALWAYS(f) F.str_always[f]
#define RB_STR_FOLD(f) F.str_fold[f]
#define RB_FULLTAB F.full_tab
#define RB_TOK2D F.tok2d
#define RB_ALL_RULES F.all_rules
#define RB_EQ_KILL(f) F.eq_kill[f]
#define RB_CONST_KILL(k) F.const_kill[k]
#define RB_TOK_ROWKILL(f) F.tok_kill[f]
#define RB_STR_ROWKILL(f) F.str_kill[f]
#define RB_TOK_RULES(f) F.tok_rules[f]
#define RB_STR_RULES(f) F.str_rules[f]
#define RB_TOK_KILL(f, z) F.tok_slot[f][z].kill
#define RB_STR_KILL(f, z) F.str_slot[f][z].kill
#define RB_STR_OFF(f, z) F.str_slot[f][z].off0
// the generic kernel evaluates every test in one stage
#define RB_GATE 0
#define RB_EQ_STAGE2(f) 0
#define RB_TOK_STAGE2(f, z) 0
#endif

// Shared tables start at TAB_BASE so that the (discarded) lookups of pairs
// with a missing side, whose lengths are -1, stay inside the array.
constexpr int TAB_BASE = 2;

// 32-bit shared-memory load: the address is one register add away.
static __device__ __forceinline__ int lds_s32(uint32_t addr) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
static __device__ __forceinline__ int4 lds_s32x4(uint32_t addr) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
// non-volatile forms for the read-only tile inside the pair loop: the
// compiler may schedule and combine them freely
static __device__ __forceinline__ int lds_ro(uint32_t addr) {
    int v;
    asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
static __device__ __forceinline__ uint2 lds_ro2(uint32_t addr) {
    uint2 v;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
static __device__ __forceinline__ uint4 lds_ro4(uint32_t addr) {
    uint4 v;
    asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
static __device__ __forceinline__ int2 lds_s32x2(uint32_t addr) {
    int2 v;
    asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
// 2*maxd[len] of an edit slot from its {G, M2} table (rb_program_create);
// lengths past a partial table are not filtered; a missing string gets -1
static __device__ __forceinline__ int str_m2(const int32_t* tab, const FSlot& fs, int off, int len) {
    if (len < 0) return -1;
    if ((unsigned)len >= (unsigned)fs.cap0) return INT_MAX;
    return tab[off + 2 * len + 1];
}

// buckets i and i+8 summed with byte saturation (x,y), z = w = 0: the
// 8-bucket bag; saturation is 1-Lipschitz, so the bag distance of folded
// bags is still a lower bound of the 16-bucket one
static __device__ __forceinline__ uint4 fold_bag(uint4 b) {
    return make_uint4(__vaddus4(b.x, b.z), __vaddus4(b.y, b.w), 0u, 0u);
}

// sum over the four bytes of |a_i - b_i|, plus c (VABSDIFF4 with accumulate)
static __device__ __forceinline__ uint32_t vsad4_acc(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("vabsdiff4.u32.u32.u32.add %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

template <bool B>
struct BoolC {
    static constexpr bool value = B;
};

// The set of rules still possible for a pair.  Integer masks (u32 / u64)
// take runtime kill masks; RuleBits<N> is the specialised form for short
// paths: one bool per rule, kill masks are compile-time constants, so every
// test folds into a predicate AND (ISETP ... .AND) instead of a SEL / LOP3
// on a mask register, and "any rule alive" is a short predicate OR.
template <int NR>
struct RuleBits {
    bool b[NR];
};

template <typename M>
__device__ __forceinline__ void m_init(M& m, uint64_t all) { m = (M)all; }
template <typename M>
__device__ __forceinline__ void m_kill(M& m, bool fail, uint64_t kill) {
    if (fail) m &= ~(M)kill;
}
template <typename M>
__device__ __forceinline__ bool m_any(const M& m) { return m != 0; }
template <typename M>
__device__ __forceinline__ bool m_hits(const M& m, uint64_t rules) { return (m & (M)rules) != 0; }
template <typename M>
__device__ __forceinline__ M m_gate(bool valid, const M& m) { return valid ? m : (M)0; }

template <int NR>
__device__ __forceinline__ void m_init(RuleBits<NR>& m, uint64_t all) {
#pragma unroll
    for (int k = 0; k < NR; k++) m.b[k] = ((all >> k) & 1ull) != 0;
}
template <int NR>
__device__ __forceinline__ void m_kill(RuleBits<NR>& m, bool fail, uint64_t kill) {
#pragma unroll
    for (int k = 0; k < NR; k++)
        if ((kill >> k) & 1ull) m.b[k] = m.b[k] & !fail;
}
template <int NR>
__device__ __forceinline__ bool m_any(const RuleBits<NR>& m) {
    bool a = false;
#pragma unroll
    for (int k = 0; k < NR; k++) a = a | m.b[k];
    return a;
}
template <int NR>
__device__ __forceinline__ bool m_hits(const RuleBits<NR>& m, uint64_t rules) {
    bool a = false;
#pragma unroll
    for (int k = 0; k < NR; k++)
        if ((rules >> k) & 1ull) a = a | m.b[k];
    return a;
}
template <int NR>
__device__ __forceinline__ RuleBits<NR> m_gate(bool valid, const RuleBits<NR>& m) {
    RuleBits<NR> o;
#pragma unroll
    for (int k = 0; k < NR; k++) o.b[k] = valid & m.b[k];
    return o;
}

// One outer tuple held in registers for a whole work item.
template <typename Mask>
struct Outer {
    int64_t i;
    int32_t ti;
    bool ok;
    Mask alive0;  // rules still possible after the t-only tests
    Mask alive_c; // rules still possible after the t-only constant tests alone
    int32_t jj_lo, jj_skip;
#if SPEC_PACKED
    int32_t jj_hi;       // packed items: first invalid tile column
    int32_t pbeg, pend;  // packed items: the row's valid inner positions [pbeg, pend) (minus i itself)
#endif
    int32_t ocode[MAX_EQ];
    int32_t olen[MAX_TOK], orem[MAX_TOK];
    uint32_t orow[MAX_TOK];  // 2-D jaccard: shared-memory byte address of need[n][0][0]
    uint32_t lev[MAX_TOK][4];
    uint2 ohash[MAX_TOK];
    int32_t oslen[MAX_STR];
    uint4 obag[MAX_STR];
    int32_t om2[MAX_STR][MAX_FSLOTS];  // 2*maxd[|t|] per edit slot

    __device__ __forceinline__ void load(const FilterPlan& F, const RunParams& R, const int32_t* tab, int mode,
                                         int64_t i_, int64_t row_hi, int64_t col0, int64_t col1,
                                         unsigned long long& my_pairs, int part_lo = 0, int part_hi = -1) {
        i = i_;
        ok = i < row_hi;
#if SPEC_PACKED
        pbeg = pend = 0;
        if (mode == MODE_PACKED && ok) {
            // symmetric: the later rows of its own partition; asymmetric: every other row of it
            const int k = find_part(R, part_lo, part_hi, i);
            pbeg = (R.flags & RB_SYMMETRIC) ? (int32_t)i + 1 : __ldg(R.part_off + k);
            pend = __ldg(R.part_end + k);
            my_pairs += (unsigned long long)(pend - pbeg - (pbeg <= i ? 1 : 0));
        }
#endif
        ti = 0;
        m_init(alive0, 0);
        m_init(alive_c, 0);
        if (ok) {
            ti = R.refs ? R.refs[i] : (int32_t)i;
            m_init(alive0, RB_ALL_RULES);
            m_init(alive_c, RB_ALL_RULES);
            if (mode == MODE_PACKED) {
                // counted above
            } else if (mode == MODE_SYM) {
                const int64_t lo = col0 > i + 1 ? col0 : i + 1;
                my_pairs += (unsigned long long)(col1 > lo ? col1 - lo : 0);
            } else if (mode == MODE_ASYM) {
                my_pairs += (unsigned long long)((col1 - col0) - ((i >= col0 && i < col1) ? 1 : 0));
            } else {
                my_pairs += (unsigned long long)(col1 - col0);
            }
        }
#pragma unroll
        for (int f = 0; f < MAX_EQ; f++) {
            ocode[f] = INT_MIN;  // never equals an inner code (those are >= -2)
            if (f < RB_NEQ && ok) {
                const int32_t c = __ldg(F.eq_outer[f] + ti);
                if (c >= 0)
                    ocode[f] = c;
                else
                    m_kill(alive0, true, RB_EQ_KILL(f));
            }
        }
#pragma unroll
        for (int k = 0; k < MAX_CONST; k++)
            if (k < RB_NCONST && ok && !__ldg(F.const_mask[k] + ti)) {
                m_kill(alive0, true, RB_CONST_KILL(k));
                m_kill(alive_c, true, RB_CONST_KILL(k));
            }
#pragma unroll
        for (int f = 0; f < MAX_TOK; f++) {
            olen[f] = -1;
            orem[f] = 0;
            ohash[f] = make_uint2(0, 0);
#pragma unroll
            for (int w = 0; w < 4; w++) lev[f][w] = 0;
            // inactive rows still run the (discarded) lookups: point them at the guard entries
            const uint32_t guard = (uint32_t)__cvta_generic_to_shared(tab + TAB_BASE);
            orow[f] = guard;
            if (RB_TOK2D && f < RB_NTOK)  // keep vector loads aligned: inactive rows read row n = 0
                orow[f] = (uint32_t)__cvta_generic_to_shared(tab + F.tok_off[f] + RB_TOK_NJP(f));
            if (f < RB_NTOK && ok) {
                olen[f] = __ldg(F.tok_olen[f] + ti);
                ohash[f] = __ldg(F.tok_ohash[f] + ti);
                // jaccard and exact_token are false for a missing or empty t side.
                // Such rows also fail the in-loop tests on their own (need[0][.]
                // is INF; the hash below matches no empty / missing inner row),
                // which the specialised loop relies on instead of alive0.
                m_kill(alive0, olen[f] <= 0, RB_TOK_ROWKILL(f));
                if (olen[f] <= 0) ohash[f].x = ~(uint32_t)mix64(0);
                if (RB_TOK2D) {
                    const int nn = olen[f] > 0 ? olen[f] : 0;
                    orow[f] = (uint32_t)__cvta_generic_to_shared(
                        tab + F.tok_off[f] + (nn * F.tok_w2[f] + 1) * RB_TOK_NJP(f));
                }
                const int64_t a = __ldg(F.tok_ooff[f] + ti), b = __ldg(F.tok_ooff[f] + ti + 1);
                const uint32_t fold = RB_TOK_SIG64(f) ? 1u : 3u;  // 64-bit mode: bit b and b+64 coincide
                for (int64_t k = a; k < b; k++) {
                    const uint32_t bit = sig_bit(__ldg(F.tok_oids[f] + k));
                    const uint32_t m = 1u << (bit & 31);
                    const uint32_t wsel = (bit >> 5) & fold;
#pragma unroll
                    for (int w = 0; w < 4; w++) {
                        if (w == (int)wsel) {
                            if (lev[f][w] & m) orem[f]++;  // shares its bit with an earlier token
                            lev[f][w] |= m;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int f = 0; f < MAX_STR; f++) {
            oslen[f] = -1;
            obag[f] = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int z = 0; z < MAX_FSLOTS; z++) om2[f][z] = -1;
            if (f < RB_NSTR && ok) {
                oslen[f] = __ldg(F.str_olen[f] + ti);
                obag[f] = __ldg(F.str_obag[f] + ti);
                m_kill(alive0, oslen[f] < 0, RB_STR_ROWKILL(f));  // missing t side: edit is false
                if (oslen[f] < 0) obag[f] = make_uint4(0, 0, 0, 0);  // with gap = |s| + 1 the bag bound fails on its own
                if (RB_STR_FOLD(f)) obag[f] = fold_bag(obag[f]);
#pragma unroll
                for (int z = 0; z < MAX_FSLOTS; z++)
                    if (z < RB_STR_NS(f)) om2[f][z] = str_m2(tab, F.str_slot[f][z], RB_STR_OFF(f, z), oslen[f]);
            }
        }
    }

    // valid(jj) <=> jj >= jj_lo && jj != jj_skip, for the tile starting at jt
    __device__ __forceinline__ bool tile(int mode, int64_t jt) {
        jj_lo = 0;
        jj_skip = -1;
#if SPEC_PACKED
        jj_hi = TJ + 1;
        if (mode == MODE_PACKED) {
            const int64_t d = (int64_t)pbeg - jt, e = (int64_t)pend - jt, x = i - jt;
            jj_lo = d < 0 ? 0 : (d > TJ + 1 ? TJ + 1 : (int)d);
            jj_hi = e < 0 ? 0 : (e > TJ + 1 ? TJ + 1 : (int)e);
            jj_skip = (pbeg <= i && x >= 0 && x < TJ) ? (int)x : -1;
            if (!ok || jj_hi <= jj_lo) jj_lo = TJ + 1;
            return false;
        }
#endif
        if (!ok) {
            jj_lo = TJ + 1;
        } else if (mode == MODE_SYM) {
            const int64_t d = i - jt + 1;
            jj_lo = d < 0 ? 0 : (d > TJ + 1 ? TJ + 1 : (int)d);
        } else if (mode == MODE_ASYM) {
            const int64_t d = i - jt;
            jj_skip = (d >= 0 && d < TJ) ? (int)d : -1;
        }
        return jj_lo == 0 && jj_skip < 0;
    }
};

// The per-pair filter over one shared tile for ROWS outer tuples per thread.
// AllValid: every (outer, jj) pair of the warp is inside the pair space.
template <typename Mask, int ROWS, bool AllValid, bool DEFER>
__device__ __forceinline__ void tile_loop(const FilterPlan& F, const VerifyProg& V, const RunParams& R, const Tile& T,
                                          const int32_t* tab, Outer<Mask> (&o)[ROWS], int jj0, int tn, int2* q, int& qn,
                                          int part, int part_hi, const int* cp_rule, int32_t* scratch,
                                          unsigned long long& my_surv, unsigned& gate_hits, unsigned& gate_iters) {
    const unsigned FULL = 0xffffffffu;
    const unsigned lt_mask = (1u << (threadIdx.x & 31)) - 1u;
    const uint32_t tab_s = (uint32_t)__cvta_generic_to_shared(tab);
    // the tile's shared-memory address, made opaque to the compiler so the
    // pre-vote's record address is one add per inner tuple (not the shared
    // window base re-derived in uniform registers every iteration)
    uint32_t rec_s;
    asm volatile("mov.u32 %0, %1;" : "=r"(rec_s) : "r"((uint32_t)__cvta_generic_to_shared(&T.r[0])));
#ifdef RB_SPEC
    // The specialised loop starts every pair from the constant rule set (or
    // the row's constant-test survivors): a row whose t side is missing or
    // empty fails the per-pair tests by construction (see Outer::load), and
    // any pair let through here is still decided by the exact interpreter.
    Mask all_rules;
    m_init(all_rules, RB_ALL_RULES);
#endif
#if RB_GATE
    gate_iters += (unsigned)(tn - jj0);
#endif
#if defined(RB_SPEC) && SPEC_UNROLL > 1
#pragma unroll SPEC_UNROLL
#endif
    for (int jj = jj0; jj < tn; jj++) {
#if defined(RB_SPEC) && RB_GATE && !SPEC_EQ_ANY && SPEC_PREANY
        {
            // Stage-1 pre-vote: whether any rule of any row survives the stage-1
            // tests, as one sum of products of the test outcomes (rule k lives
            // iff every stage-1 test whose kill set holds k passes).  The same
            // condition as the gate below, without building the rule masks:
            // most warp iterations stop here after the compares, popcounts and
            // a few predicate ops; the rest re-run the tests and build the masks.
            bool anyw = false;
            const uint32_t ra = rec_s + (uint32_t)jj * (uint32_t)sizeof(Rec);  // this inner tuple's record
#pragma unroll
            for (int r = 0; r < ROWS; r++) {
#if SPEC_PACKED
                const bool valid = AllValid || (jj >= o[r].jj_lo && jj != o[r].jj_skip && jj < o[r].jj_hi);
#else
                const bool valid = AllValid || (jj >= o[r].jj_lo && jj != o[r].jj_skip);
#endif
                bool peq[MAX_EQ];
#pragma unroll
                for (int f = 0; f < MAX_EQ; f++) {
                    peq[f] = true;
                    if (f < RB_NEQ && !RB_EQ_STAGE2(f) && RB_EQ_KILL(f))
                        peq[f] = o[r].ocode[f] == lds_ro(ra + RB_REC_OFF(head) + 4u * f);
                }
                bool ptk[MAX_TOK][MAX_FSLOTS];
#pragma unroll
                for (int f = 0; f < MAX_TOK; f++) {
                    int u = 0;
                    uint32_t a = 0;
                    if (f < RB_NTOK && RB_TOK_NJ(f) > 0) {
                        const uint32_t sa = ra + RB_REC_OFF(toksig) + 16u * f;
                        uint4 is;
                        if (RB_TOK_SIG64(f)) {
                            const uint2 h2 = lds_ro2(sa);
                            is = make_uint4(h2.x, h2.y, 0u, 0u);
                        } else {
                            is = lds_ro4(sa);
                        }
                        u = RB_TOK_SIG64(f) ? __popc(o[r].lev[f][0] & is.x) + __popc(o[r].lev[f][1] & is.y) + o[r].orem[f]
                                            : __popc(o[r].lev[f][0] & is.x) + __popc(o[r].lev[f][1] & is.y) +
                                                  __popc(o[r].lev[f][2] & is.z) + __popc(o[r].lev[f][3] & is.w) +
                                                  o[r].orem[f];
                        a = o[r].orow[f] + ((uint32_t)(lds_ro(ra + RB_REC_OFF(head) + 4u * (RB_NEQ + f)) * RB_TOK_NJP(f)) << 2);
                    }
#pragma unroll
                    for (int z = 0; z < MAX_FSLOTS; z++) {
                        ptk[f][z] = true;
                        if (f < RB_NTOK && z < RB_TOK_NS(f) && !RB_TOK_STAGE2(f, z) && RB_TOK_KILL(f, z))
                            ptk[f][z] = z < RB_TOK_NJ(f) ? u >= lds_s32(a + 4u * z)
                                                         : (uint32_t)lds_ro(ra + RB_REC_OFF(tokhash) + 8u * f) ==
                                                               o[r].ohash[f].x;
                    }
                }
                bool any_r = false;
#pragma unroll
                for (int k = 0; k < 64; k++) {
                    if (!(((uint64_t)RB_ALL_RULES >> k) & 1)) continue;
                    bool ok = RB_NCONST == 0 || m_hits(o[r].alive_c, 1ull << k);
#pragma unroll
                    for (int f = 0; f < MAX_EQ; f++)
                        if (f < RB_NEQ && !RB_EQ_STAGE2(f) && (((uint64_t)RB_EQ_KILL(f) >> k) & 1)) ok = ok && peq[f];
#pragma unroll
                    for (int f = 0; f < MAX_TOK; f++)
#pragma unroll
                        for (int z = 0; z < MAX_FSLOTS; z++)
                            if (f < RB_NTOK && z < RB_TOK_NS(f) && !RB_TOK_STAGE2(f, z) &&
                                (((uint64_t)RB_TOK_KILL(f, z) >> k) & 1))
                                ok = ok && ptk[f][z];
                    any_r = any_r || ok;
                }
                anyw = anyw || (valid && any_r);
            }
            if (!__any_sync(FULL, anyw)) continue;
        }
#endif
        Mask alive[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; r++) {
#ifdef RB_SPEC
            const Mask& base = RB_NCONST == 0 ? all_rules : o[r].alive_c;
#else
            const Mask& base = o[r].alive0;
#endif
#if SPEC_PACKED
            alive[r] = AllValid ? base : m_gate(jj >= o[r].jj_lo && jj != o[r].jj_skip && jj < o[r].jj_hi, base);
#else
            alive[r] = AllValid ? base : m_gate(jj >= o[r].jj_lo && jj != o[r].jj_skip, base);
#endif
#if defined(RB_SPEC) && SPEC_EQ_ANY
        }
        {
            bool hit[ROWS];
            bool any_hit = false;
#pragma unroll
            for (int r = 0; r < ROWS; r++) {
                hit[r] = false;
#pragma unroll
                for (int f = 0; f < MAX_EQ; f++)
                    if (f < RB_NEQ && !RB_EQ_STAGE2(f) && RB_EQ_KILL(f)) hit[r] |= o[r].ocode[f] == T.r[jj].head[f];
                m_kill(alive[r], !hit[r], ~(uint64_t)SPEC_EQ_FREE);
                any_hit |= hit[r];
            }
            if (__any_sync(FULL, any_hit)) {
#pragma unroll
                for (int r = 0; r < ROWS; r++) {
#pragma unroll
                    for (int f = 0; f < MAX_EQ; f++)
                        if (f < RB_NEQ && !RB_EQ_STAGE2(f) && RB_EQ_KILL(f))
                            m_kill(alive[r], hit[r] && o[r].ocode[f] != T.r[jj].head[f], RB_EQ_KILL(f));
                }
            }
        }
#else
#pragma unroll
            for (int f = 0; f < MAX_EQ; f++)
                if (f < RB_NEQ && !RB_EQ_STAGE2(f)) m_kill(alive[r], o[r].ocode[f] != T.r[jj].head[f], RB_EQ_KILL(f));
        }
#endif
        // token tests kept for stage 2 (always-evaluated features only)
        int u_keep[ROWS][MAX_TOK];
        int need_keep[ROWS][MAX_TOK][4];
        uint32_t hash_keep[MAX_TOK];

#pragma unroll
        for (int f = 0; f < MAX_TOK; f++) {
            if (f >= RB_NTOK) continue;
            bool need = false;
#pragma unroll
            for (int r = 0; r < ROWS; r++) need |= m_hits(alive[r], RB_TOK_RULES(f));
            if (!RB_TOK_ALWAYS(f) && !__any_sync(FULL, need)) continue;
            const int m = T.r[jj].head[RB_NEQ + f];
            const uint32_t mo = (uint32_t)(m * RB_TOK_NJP(f)) << 2;  // byte offset of column m within a need[n] row
            const uint4 is = T.r[jj].toksig[f];
            const uint2 h = T.r[jj].tokhash[f];
#pragma unroll
            for (int r = 0; r < ROWS; r++) {
                // u >= |A n B| (see the header); rows with n <= 0 were killed at load
                const int u = RB_TOK_SIG64(f)
                                  ? __popc(o[r].lev[f][0] & is.x) + __popc(o[r].lev[f][1] & is.y) + o[r].orem[f]
                                  : __popc(o[r].lev[f][0] & is.x) + __popc(o[r].lev[f][1] & is.y) +
                                        __popc(o[r].lev[f][2] & is.z) + __popc(o[r].lev[f][3] & is.w) + o[r].orem[f];
                const int n = o[r].olen[f];
                int need2d[4] = {0, 0, 0, 0};
                u_keep[r][f] = u;
                hash_keep[f] = h.x;
                bool split = false;  // a stage-2 Jaccard slot: load only the stage-1 thresholds now
#pragma unroll
                for (int z = 0; z < MAX_FSLOTS; z++) split |= RB_GATE && z < RB_TOK_NJ(f) && RB_TOK_STAGE2(f, z);
                if (RB_TOK2D && RB_TOK_NJ(f) > 0 && split) {
                    const uint32_t a = o[r].orow[f] + mo;
#pragma unroll
                    for (int z = 0; z < MAX_FSLOTS; z++)
                        if (z < RB_TOK_NJ(f) && !RB_TOK_STAGE2(f, z)) need2d[z] = lds_s32(a + 4u * z);
                } else if (RB_TOK2D && RB_TOK_NJ(f) > 0) {  // one vector load: every jaccard slot's need[n][m]
                    const uint32_t a = o[r].orow[f] + mo;
                    if (RB_TOK_NJP(f) == 1) {
                        need2d[0] = lds_s32(a);
                    } else if (RB_TOK_NJP(f) == 2) {
                        const int2 v = lds_s32x2(a);
                        need2d[0] = v.x;
                        need2d[1] = v.y;
                    } else {
                        const int4 v = lds_s32x4(a);
                        need2d[0] = v.x;
                        need2d[1] = v.y;
                        need2d[2] = v.z;
                        need2d[3] = v.w;
                    }
                }
#pragma unroll
                for (int z = 0; z < 4; z++) need_keep[r][f][z] = need2d[z];
#pragma unroll
                for (int z = 0; z < MAX_FSLOTS; z++) {
                    if (z < RB_TOK_NS(f) && !RB_TOK_STAGE2(f, z)) {
                        const FSlot& fs = F.tok_slot[f][z];
                        bool ok;
                        if (z < RB_TOK_NJ(f)) {  // jaccard: exact integer tables
                            if (RB_TOK2D) {
                                // need[n][m]: INF unless the length tests pass, else mink[n+m]
                                ok = u >= need2d[z];
                            } else {
                                const bool live = m >= 0;
                                const int small = min(n, m), big = max(n, m);
                                const int ms =
                                    (RB_FULLTAB || (unsigned)big < (unsigned)fs.cap0) ? tab[fs.off0 + big] : 0;
                                const int mk =
                                    (RB_FULLTAB || (unsigned)(n + m) < (unsigned)fs.cap1) ? tab[fs.off1 + n + m] : 0;
                                ok = live & (small >= ms) & (min(u, small) >= mk);
                            }
                        } else {  // exact_token: the id-list hash (seeded with the length) must match;
                            // 32 of its bits suffice to drop all but ~2^-32 of the unequal pairs
                            ok = h.x == o[r].ohash[f].x;
                        }
                        m_kill(alive[r], !ok, RB_TOK_KILL(f, z));
                    }
                }
            }
        }
#if RB_GATE
        {
            // stage-1 tests cover every rule: a warp with no live pair skips the rest
            bool any = false;
#pragma unroll
            for (int r = 0; r < ROWS; r++) any |= m_any(alive[r]);
            if (!__any_sync(FULL, any)) continue;
            gate_hits++;
#pragma unroll
            for (int r = 0; r < ROWS; r++) {
#pragma unroll
                for (int f = 0; f < MAX_EQ; f++)
                    if (f < RB_NEQ && RB_EQ_STAGE2(f))
                        m_kill(alive[r], o[r].ocode[f] != T.r[jj].head[f], RB_EQ_KILL(f));
#pragma unroll
                for (int f = 0; f < MAX_TOK; f++) {
#pragma unroll
                    for (int z = 0; z < MAX_FSLOTS; z++) {
                        if (f < RB_NTOK && z < RB_TOK_NS(f) && RB_TOK_STAGE2(f, z)) {
                            // 2-D Jaccard tables or the exact_token hash (stage 2 needs TOK2D)
                            // a stage-2 Jaccard threshold is read only now (rarely)
                            const uint32_t mo2 = (uint32_t)(T.r[jj].head[RB_NEQ + f] * RB_TOK_NJP(f)) << 2;
                            const bool ok = z < RB_TOK_NJ(f) ? u_keep[r][f] >= lds_s32(o[r].orow[f] + mo2 + 4u * z)
                                                             : hash_keep[f] == o[r].ohash[f].x;
                            m_kill(alive[r], !ok, RB_TOK_KILL(f, z));
                        }
                    }
                }
            }
        }
#endif
#pragma unroll
        for (int f = 0; f < MAX_STR; f++) {
            if (f >= RB_NSTR) continue;
            bool need = false;
#pragma unroll
            for (int r = 0; r < ROWS; r++) need |= m_hits(alive[r], RB_STR_RULES(f));
            if (!RB_STR_ALWAYS(f) && !__any_sync(FULL, need)) continue;
            const int lb = T.r[jj].strlen_[f];
            const uint4 ib = T.r[jj].strbag[f];
#pragma unroll
            for (int r = 0; r < ROWS; r++) {
                const int la = o[r].oslen[f];
                // t = bag distance + |la - lb| in five accumulating SAD steps;
                // lev <= maxd[L] implies t <= 2*maxd[L] <= max(2*maxd[la], 2*maxd[lb])
                // (L is one of la, lb), so no max, no table lookup per pair
                const uint32_t t2 = vsad4_acc(o[r].obag[f].y, ib.y, vsad4_acc(o[r].obag[f].x, ib.x, __sad(la, lb, 0u)));
                const int t = RB_STR_FOLD(f) ? (int)t2
                                             : (int)vsad4_acc(o[r].obag[f].w, ib.w, vsad4_acc(o[r].obag[f].z, ib.z, t2));
#pragma unroll
                for (int z = 0; z < MAX_FSLOTS; z++) {
                    if (z < RB_STR_NS(f)) {
                        const bool ok = t <= max(o[r].om2[f][z], T.r[jj].strm2[f][z]);
                        m_kill(alive[r], !ok, RB_STR_KILL(f, z));
                    }
                }
            }
        }

        // ---- survivors -> the warp's queue (ballot + popc compaction)
        bool any_surv = false;
#pragma unroll
        for (int r = 0; r < ROWS; r++) any_surv |= m_any(alive[r]);
        if (__any_sync(FULL, any_surv)) {
#pragma unroll
            for (int r = 0; r < ROWS; r++) {
                const bool surv = m_any(alive[r]);
                const unsigned bal = __ballot_sync(FULL, surv);
                if (surv) q[qn + __popc(bal & lt_mask)] = make_int2(part_hi >= 0 ? (int)o[r].i : o[r].ti, T.r[jj].tid);
                qn += __popc(bal);
                my_surv += surv ? 1 : 0;
            }
            if (qn > QCAP - 32 * ROWS) {
                __syncwarp();
                if (DEFER)
                    flush_survivors(R, q, qn, part, part_hi);
                else
                    drain_queue(V, R, q, qn, part, cp_rule, scratch);
                __syncwarp();
                qn = 0;
            }
        }
    }
}

// Mask = uint32_t when the path has <= 32 checkpoints, else uint64_t.
// ROWS outer tuples per thread: a work item covers BLOCK * ROWS outer rows.
template <typename Mask, int ROWS, bool DEFER = false>
__device__ __forceinline__ void pair_body(const FilterPlan& F, const VerifyProg& V, const RunParams& R) {
    __shared__ Tile T;
    __shared__ int2 queue[NWARPS][QCAP];
    __shared__ __align__(16) int32_t tab[SMEM_TAB];
    __shared__ int cp_rule[MAX_RULES];
    __shared__ int s_item;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const unsigned FULL = 0xffffffffu;
    int2* q = queue[warp];
    int qn = 0;
    unsigned long long my_pairs = 0, my_surv = 0;
    unsigned gate_hits = 0, gate_iters = 0;  // stage-1 gate passes / inner tuples visited (per warp)
    int32_t* scratch = R.scratch + (int64_t)(blockIdx.x * BLOCK + threadIdx.x) * R.scratch_stride;

    if (R.bad_refs && *R.bad_refs) return;  // the host reports the bad ref
    for (int k = threadIdx.x; k < MAX_RULES; k += BLOCK) cp_rule[k] = V.cp_rule[k];
    for (int k = threadIdx.x; k < F.n_tab; k += BLOCK) tab[k] = F.tab_src[k];

    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_item = (int)atomicAdd(R.item_counter, 1u);
        __syncthreads();
        const int it = s_item;
        if (it >= R.n_items) break;
        const Item item = R.items[it];
        const int64_t col0 = item.col0, col1 = item.col1;
        const int part = item.part;
        const int part_hi = SPEC_PACKED && item.mode == MODE_PACKED ? item.pad0 : -1;

        Outer<Mask> o[ROWS];
#pragma unroll
        for (int r = 0; r < ROWS; r++)
            // a warp owns 32 * ROWS consecutive outer rows, so its rows meet the
            // symmetric diagonal together (tight jj0 skip, more all-valid tiles)
            o[r].load(F, R, tab, item.mode, (int64_t)item.row0 + (warp * ROWS + r) * 32 + lane, (int64_t)item.row_hi,
                      col0, col1,
                      my_pairs, part, part_hi);

        for (int64_t jt = col0; jt < col1; jt += TJ) {
            const int tn = (int)(col1 - jt < TJ ? col1 - jt : TJ);
            __syncthreads();
            for (int k = threadIdx.x; k < tn; k += BLOCK) {
                const int64_t j = jt + k;
                const int32_t sj = R.refs ? __ldg(R.refs + j) : (int32_t)j;
                T.r[k].tid = sj;
#pragma unroll
                for (int f = 0; f < MAX_EQ; f++)
                    if (f < RB_NEQ) T.r[k].head[f] = __ldg(F.eq_inner[f] + sj);
#pragma unroll
                for (int f = 0; f < MAX_TOK; f++)
                    if (f < RB_NTOK) {
                        T.r[k].head[RB_NEQ + f] = __ldg(F.tok_ilen[f] + sj);
                        uint4 sg = __ldg(F.tok_isig[f] + sj);
                        if (RB_TOK_SIG64(f)) sg = make_uint4(sg.x | sg.z, sg.y | sg.w, 0u, 0u);
                        T.r[k].toksig[f] = sg;
                        T.r[k].tokhash[f] = __ldg(F.tok_ihash[f] + sj);
                    }
#pragma unroll
                for (int f = 0; f < MAX_STR; f++)
                    if (f < RB_NSTR) {
                        const int lb = __ldg(F.str_ilen[f] + sj);
                        T.r[k].strlen_[f] = lb;
                        const uint4 bg = __ldg(F.str_ibag[f] + sj);
                        T.r[k].strbag[f] = RB_STR_FOLD(f) ? fold_bag(bg) : bg;
#pragma unroll
                        for (int z = 0; z < MAX_FSLOTS; z++)
                            if (z < RB_STR_NS(f)) T.r[k].strm2[f][z] = str_m2(tab, F.str_slot[f][z], RB_STR_OFF(f, z), lb);
                    }
            }
            __syncthreads();

            bool all_valid = true;
            int lo = TJ + 1;
#pragma unroll
            for (int r = 0; r < ROWS; r++) {
                all_valid &= o[r].tile(item.mode, jt);
                lo = min(lo, o[r].jj_lo);
            }
            // the warp's first inner position with a valid pair: the symmetric
            // triangle's diagonal tiles (and small partitions) skip the dead part
            const int jj0 = __reduce_min_sync(FULL, lo);
            if (jj0 >= tn) continue;
#if SPEC_PACKED
            int hi = 0;
#pragma unroll
            for (int r = 0; r < ROWS; r++) hi = max(hi, o[r].jj_lo <= TJ ? o[r].jj_hi : 0);
            const int tn_w = min(tn, (int)__reduce_max_sync(FULL, (unsigned)hi));  // the warp's last valid column + 1
#else
            const int tn_w = tn;
#endif
            if (__all_sync(FULL, all_valid))
                tile_loop<Mask, ROWS, true, DEFER>(F, V, R, T, tab, o, 0, tn, q, qn, part, part_hi, cp_rule, scratch, my_surv,
                                                   gate_hits, gate_iters);
            else
                tile_loop<Mask, ROWS, false, DEFER>(F, V, R, T, tab, o, jj0, tn_w, q, qn, part, part_hi, cp_rule, scratch,
                                                    my_surv, gate_hits, gate_iters);
        }
        if (qn) {
            __syncwarp();
            if (DEFER)
                flush_survivors(R, q, qn, part, part_hi);
            else
                drain_queue(V, R, q, qn, part, cp_rule, scratch);
            __syncwarp();
            qn = 0;
        }
    }

    // ---- statistics
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
        my_pairs += __shfl_down_sync(FULL, my_pairs, o2);
        my_surv += __shfl_down_sync(FULL, my_surv, o2);
    }
    if (lane == 0) {
        atomicAdd(R.stat_pairs, my_pairs);
        atomicAdd(R.stat_surv, my_surv);
#if RB_GATE
        if (R.stat_gate) {  // warp-uniform counts
            atomicAdd(R.stat_gate, (unsigned long long)gate_hits);
            atomicAdd(R.stat_gate + 1, (unsigned long long)gate_iters);
        }
#endif
    }
}

}  // namespace rb

#ifdef RB_SPEC
extern "C" __global__ void __launch_bounds__(rb::BLOCK, SPEC_MINBLOCKS)
    rb_pair_kernel_spec(const __grid_constant__ rb::FilterPlan F, const __grid_constant__ rb::VerifyProg V,
                        const __grid_constant__ rb::RunParams R) {
    rb::pair_body<SPEC_MASK, SPEC_ROWS, SPEC_DEFER != 0>(F, V, R);
}

extern "C" __global__ void __launch_bounds__(rb::BLOCK) rb_verify_kernel_spec(const __grid_constant__ rb::VerifyProg V,
                                                                           const __grid_constant__ rb::RunParams R) {
    rb::verify_body(V, R);
}
#endif
