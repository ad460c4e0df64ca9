/*
 * rb_oracle.c -- CPU restatement of the reference engine's per-pair
 * semantics.  TEST INFRASTRUCTURE ONLY: used by tests/, by
 * __graft_entry__.smoke() as the checker and by bench.py's cpu_baseline /
 * --impl reference leg.  The product path (librbgpu.so) never links it.
 *
 * What it restates (reference file:line under /root/reference/pkg/src/ruleblock):
 *   evaluate_pair / _walk_survivors   engine.py:93-132, 508-559
 *       reuse bit -> fail_jump -> first checkpoint (or every one when
 *       enumerating); symmetric rows canonicalised to (min tid, max tid)
 *   pair ranges                       engine.py:411-449, 475-506, 684-719
 *       symmetric i<j, asymmetric i!=j, cross left x right
 *   comparisons / slot_evals          engine.py:486, 558 (first-touch counts)
 *   _eq_code_slot / _eq_const_slot    encode.py:191-219
 *   _edit_slot                        encode.py:222-240 (float64 prefilter)
 *   _jaccard_slot                     encode.py:243-261 (float64 prefilter)
 *   _exact_token_slot                 encode.py:264-278
 *   fallback slots (no prefilter)     encode.py:281-288 -> measures.py:45-70
 *   levenshtein_u32                   _kernels.py:29-51 (two-row DP)
 *   jaccard_sorted                    _kernels.py:54-73 (sorted merge, float64)
 *   sorted_equal                      _kernels.py:76-83
 * Thresholds are compared in float64 with the reference's own expressions,
 * NOT through the integer tables the GPU uses -- so this oracle checks the
 * tables too.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/rbgpu.h"

typedef struct orc_column {
    int32_t kind;
    int32_t width;
    const void* data;
    const int64_t* offsets;
    const uint8_t* missing;
} orc_column;

typedef struct orc_prog {
    const orc_column* cols;
    const int32_t *op, *slot, *fail, *rule;
    int32_t n_ins;
    const rb_slot* slots;
    int32_t n_slots;
} orc_prog;

static inline uint32_t char_at(const orc_column* c, int64_t k) {
    return c->width == 1 ? ((const uint8_t*)c->data)[k] : ((const uint32_t*)c->data)[k];
}

/* _kernels.py:29-51: full two-row DP (int64 cells) */
static int64_t levenshtein(const orc_column* ca, int64_t a0, int64_t n, const orc_column* cb, int64_t b0, int64_t m,
                           int64_t* prev, int64_t* cur) {
    if (n == 0) return m;
    if (m == 0) return n;
    for (int64_t j = 0; j <= m; j++) prev[j] = j;
    for (int64_t i = 1; i <= n; i++) {
        cur[0] = i;
        uint32_t ai = char_at(ca, a0 + i - 1);
        for (int64_t j = 1; j <= m; j++) {
            int64_t best = prev[j - 1] + (ai == char_at(cb, b0 + j - 1) ? 0 : 1);
            if (prev[j] + 1 < best) best = prev[j] + 1;
            if (cur[j - 1] + 1 < best) best = cur[j - 1] + 1;
            cur[j] = best;
        }
        int64_t* t = prev;
        prev = cur;
        cur = t;
    }
    return prev[m];
}

/* _kernels.py:54-73 (returns the intersection; the caller divides) */
static int64_t intersect_sorted(const int32_t* a, int64_t n, const int32_t* b, int64_t m) {
    int64_t i = 0, j = 0, inter = 0;
    while (i < n && j < m) {
        if (a[i] == b[j]) {
            inter++;
            i++;
            j++;
        } else if (a[i] < b[j]) {
            i++;
        } else {
            j++;
        }
    }
    return inter;
}

typedef struct scratch {
    int64_t* prev;
    int64_t* cur;
    int64_t cap;
} scratch;

static int eval_slot(const orc_prog* P, int s, int64_t t, int64_t u, scratch* sc) {
    const rb_slot* sl = &P->slots[s];
    const orc_column* ca = &P->cols[sl->lhs];
    const orc_column* cb = &P->cols[sl->rhs];
    const double delta = sl->delta;
    const int prefilter = (sl->flags & RB_SLOT_PREFILTER) != 0;
    switch (sl->kind) {
        case RB_SLOT_EQ_CODE: {
            int32_t x = ((const int32_t*)ca->data)[t];
            return x >= 0 && x == ((const int32_t*)cb->data)[u];
        }
        case RB_SLOT_EQ_CONST:
            return ((const uint8_t*)ca->data)[t] != 0;
        case RB_SLOT_EDIT: {
            if (ca->missing[t] || cb->missing[u]) return 0;
            int64_t a0 = ca->offsets[t], la = ca->offsets[t + 1] - a0;
            int64_t b0 = cb->offsets[u], lb = cb->offsets[u + 1] - b0;
            int64_t longest = la >= lb ? la : lb, shortest = la >= lb ? lb : la;
            if (longest == 0) return 1;
            if (prefilter && (double)(longest - shortest) > (1.0 - delta) * (double)longest) return 0;
            if (longest + 1 > sc->cap) {
                sc->cap = 2 * (longest + 1);
                sc->prev = (int64_t*)realloc(sc->prev, sizeof(int64_t) * sc->cap);
                sc->cur = (int64_t*)realloc(sc->cur, sizeof(int64_t) * sc->cap);
            }
            int64_t lev = levenshtein(ca, a0, la, cb, b0, lb, sc->prev, sc->cur);
            return 1.0 - (double)lev / (double)longest >= delta;
        }
        case RB_SLOT_JACCARD: {
            if (ca->missing[t] || cb->missing[u]) return 0;
            int64_t a0 = ca->offsets[t], n = ca->offsets[t + 1] - a0;
            int64_t b0 = cb->offsets[u], m = cb->offsets[u + 1] - b0;
            if (n == 0 && m == 0) return 0;
            int64_t small = n <= m ? n : m, big = n <= m ? m : n;
            if (prefilter && (double)small < delta * (double)big) return 0;
            const int32_t* ia = (const int32_t*)ca->data + a0;
            const int32_t* ib = (const int32_t*)cb->data + b0;
            int64_t inter = intersect_sorted(ia, n, ib, m);
            return (double)inter / (double)(n + m - inter) >= delta;
        }
        case RB_SLOT_EXACT: {
            if (ca->missing[t] || cb->missing[u]) return 0;
            int64_t a0 = ca->offsets[t], n = ca->offsets[t + 1] - a0;
            int64_t b0 = cb->offsets[u], m = cb->offsets[u + 1] - b0;
            if (n == 0 && m == 0) return 0;
            if (n != m) return 0;
            return memcmp((const int32_t*)ca->data + a0, (const int32_t*)cb->data + b0, sizeof(int32_t) * n) == 0;
        }
    }
    return 0;
}

typedef struct sink {
    int32_t *t, *s, *r;
    int64_t cap;
    int64_t count;
} sink;

static void emit(sink* out, int32_t a, int32_t b, int32_t rule) {
    int64_t at;
#pragma omp atomic capture
    at = out->count++;
    if (at < out->cap) {
        out->t[at] = a;
        out->s[at] = b;
        out->r[at] = rule;
    }
}

/* engine.py:531-559 for one pair */
static void walk_pair(const orc_prog* P, int32_t ti, int32_t si, uint32_t flags, sink* out, int64_t* evals,
                      scratch* sc) {
    uint64_t reuse = 0, value = 0;
    int32_t ip = 0;
    while (ip < P->n_ins) {
        if (P->op[ip] == 1) {
            int32_t a = ti, b = si;
            if ((flags & RB_SYMMETRIC) && a > b) {
                a = si;
                b = ti;
            }
            emit(out, a, b, P->rule[ip]);
            if (!(flags & RB_ENUMERATE)) return;
            ip++;
            continue;
        }
        int s = P->slot[ip];
        uint64_t bit = 1ull << s;
        int truth;
        if (reuse & bit) {
            truth = (value & bit) != 0;
        } else {
            truth = eval_slot(P, s, ti, si, sc);
            reuse |= bit;
            if (truth) value |= bit;
            evals[s]++;
        }
        ip = truth ? ip + 1 : P->fail[ip];
    }
}

/*
 * Evaluate the pairs owned by outer positions [row_lo, row_hi) of
 * refs[0..n).  split < 0: partition (symmetric i<j / asymmetric i!=j);
 * split >= 0: cross, outer in [0, split), inner in [split, n).
 * Returns the number of rows produced (rows beyond cap are counted, not
 * stored).
 */
int64_t orc_run(const orc_column* cols, int32_t n_cols, const int32_t* op, const int32_t* slot, const int32_t* fail,
                const int32_t* rule, int32_t n_ins, const rb_slot* slots, int32_t n_slots, const int32_t* refs,
                int64_t n, int64_t split, int64_t row_lo, int64_t row_hi, uint32_t flags, int32_t nthreads,
                int32_t* out_t, int32_t* out_s, int32_t* out_r, int64_t cap, int64_t* comparisons,
                int64_t* slot_evals) {
    (void)n_cols;
    orc_prog P = {cols, op, slot, fail, rule, n_ins, slots, n_slots};
    sink out = {out_t, out_s, out_r, cap, 0};
    int64_t total_cmp = 0;
    if (split >= 0 && row_hi > split) row_hi = split;
    if (row_hi > n) row_hi = n;
    for (int s = 0; s < n_slots; s++) slot_evals[s] = 0;
    if (nthreads > 0) {
#ifdef _OPENMP
        extern void omp_set_num_threads(int);
        omp_set_num_threads(nthreads);
#endif
    }
#pragma omp parallel reduction(+ : total_cmp)
    {
        int64_t evals[RB_MAX_SLOTS] = {0};
        scratch sc = {NULL, NULL, 0};
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = row_lo; i < row_hi; i++) {
            int32_t ti = refs ? refs[i] : (int32_t)i;
            int64_t j0, j1;
            if (split >= 0) {
                j0 = split;
                j1 = n;
            } else if (flags & RB_SYMMETRIC) {
                j0 = i + 1;
                j1 = n;
            } else {
                j0 = 0;
                j1 = n;
            }
            for (int64_t j = j0; j < j1; j++) {
                if (split < 0 && !(flags & RB_SYMMETRIC) && j == i) continue;
                int32_t si = refs ? refs[j] : (int32_t)j;
                total_cmp++;
                walk_pair(&P, ti, si, flags, &out, evals, &sc);
            }
        }
        for (int s = 0; s < n_slots; s++) {
#pragma omp atomic
            slot_evals[s] += evals[s];
        }
        free(sc.prev);
        free(sc.cur);
    }
    *comparisons = total_cmp;
    return out.count;
}

/*
 * Witness of each given pair (t[k], s[k]) in evaluation order t-then-s:
 * rule_out[k] = the rule of the first checkpoint reached (engine.py:531-559,
 * not enumerating), -1 when no rule holds.  Used to check every row a device
 * run emitted (the caller passes t = lower position).
 */
void orc_witness_pairs(const orc_column* cols, const int32_t* op, const int32_t* slot, const int32_t* fail,
                       const int32_t* rule, int32_t n_ins, const rb_slot* slots, int32_t n_slots, const int32_t* t,
                       const int32_t* s, int64_t n_pairs, int32_t nthreads, int32_t* rule_out) {
    orc_prog P = {cols, op, slot, fail, rule, n_ins, slots, n_slots};
    if (nthreads > 0) {
#ifdef _OPENMP
        extern void omp_set_num_threads(int);
        omp_set_num_threads(nthreads);
#endif
    }
#pragma omp parallel
    {
        int64_t evals[RB_MAX_SLOTS] = {0};
        scratch sc = {NULL, NULL, 0};
        int32_t one_t, one_s, one_r;
#pragma omp for schedule(dynamic, 256)
        for (int64_t k = 0; k < n_pairs; k++) {
            sink out = {&one_t, &one_s, &one_r, 1, 0};
            walk_pair(&P, t[k], s[k], 0u, &out, evals, &sc);
            rule_out[k] = out.count ? one_r : -1;
        }
        free(sc.prev);
        free(sc.cur);
    }
}

/* struct layout check for the ctypes mirror */
int32_t orc_slot_size(void) { return (int32_t)sizeof(rb_slot); }
int32_t orc_column_size(void) { return (int32_t)sizeof(orc_column); }
