// rb_api.cu -- the C ABI (include/rbgpu.h): contexts, device-resident
// relations and programs, run orchestration and results.
//
// Host-side work here is bookkeeping only: it copies plain arrays to HBM,
// derives the phase-1 filter plan from the instruction list (which slots
// each rule's checkpoint needs: the EVALs whose subtree encloses it,
// planner/plan.py:269-300), builds the work-item list and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "rb_state.cuh"

using namespace rb;

namespace rb {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

}  // namespace rb

using rb::g_err;

// Stage-1 gate (specialised kernel): for each rule, in checkpoint order, not
// yet ruled out by a chosen test, choose the equality key or always-evaluated
// token slot holding its earliest path slot.  If every rule is covered, the
// other equality / token tests run only for warps with a live pair after
// stage 1.  `implied`: path slots known to hold for every pair of the run
// (the equality root of the branch whose partitions are being evaluated:
// every pair of a non-missing group shares the key).  An equality feature
// testing only implied slots can never fail: it kills nothing, is never
// chosen for stage 1 and is compiled out, so a rule it guarded is gated by
// its next test (e.g. the Jaccard of `zip = ∧ address jaccard` inside a zip
// partition).  Exactness is unaffected: the filter only prunes, the
// interpreter re-decides every survivor.
void rb::choose_gate(FilterPlan& F, const std::vector<uint64_t>& need, const std::vector<int>& first_pos, int n_slots,
                     uint64_t implied, const std::vector<int>* cls) {
    if (implied) {
        for (int f = 0; f < F.n_eq; f++)
            if (F.eq_slots[f] && (F.eq_slots[f] & ~implied) == 0) F.eq_kill[f] = 0;
        // a token / string feature is "always" needed when some rule using it
        // has no slot filtered before it; an implied slot filters nothing
        if (cls && (int)cls->size() >= n_slots) {
            for (int f = 0; f < F.n_tok; f++)
                for (size_t r = 0; r < need.size() && !F.tok_always[f]; r++) {
                    bool uses = false, earlier = false;
                    for (int s = 0; s < n_slots; s++) {
                        if (!(need[r] & (1ull << s))) continue;
                        if ((*cls)[s] == 1 + f) uses = true;
                        if ((*cls)[s] >= 0 && (*cls)[s] < 1 + f && !((implied >> s) & 1)) earlier = true;
                    }
                    if (uses && !earlier) F.tok_always[f] = 1;
                }
            for (int f = 0; f < F.n_str; f++)
                for (size_t r = 0; r < need.size() && !F.str_always[f]; r++) {
                    bool uses = false, earlier = false;
                    for (int s = 0; s < n_slots; s++) {
                        if (!(need[r] & (1ull << s))) continue;
                        if ((*cls)[s] == 1 + MAX_TOK + f) uses = true;
                        if ((*cls)[s] >= 0 && (*cls)[s] < 1 + MAX_TOK + f && !((implied >> s) & 1)) earlier = true;
                    }
                    if (uses && !earlier) F.str_always[f] = 1;
                }
        }
    }
    const char* env_gate = std::getenv("RB_GATE");
    bool covered_all = !(env_gate && env_gate[0] == '0');
    uint64_t covered = 0;
    std::vector<char> eq_chosen(F.n_eq, 0);
    std::vector<std::vector<char>> tok_chosen(F.n_tok, std::vector<char>(MAX_FSLOTS, 0));
    for (size_t r = 0; r < need.size() && covered_all; r++) {
        if ((covered >> r) & 1) continue;
        int best_pos = INT32_MAX, bf = -1, bz = -1;  // bz < 0: equality key bf
        for (int f = 0; f < F.n_eq; f++) {
            if (!((F.eq_kill[f] >> r) & 1) || !(F.eq_slots[f] & need[r])) continue;
            for (int sl2 = 0; sl2 < n_slots; sl2++)
                if (((F.eq_slots[f] & need[r] & ~implied) >> sl2) & 1 && first_pos[sl2] < best_pos) {
                    best_pos = first_pos[sl2];
                    bf = f;
                    bz = -1;
                }
        }
        for (int f = 0; f < F.n_tok; f++) {
            if (!F.tok_always[f]) continue;
            for (int z = 0; z < F.tok_nslots[f]; z++) {
                const FSlot& fs = F.tok_slot[f][z];
                if (((fs.kill >> r) & 1) && ((need[r] >> fs.slot) & 1) && first_pos[fs.slot] < best_pos) {
                    best_pos = first_pos[fs.slot];
                    bf = f;
                    bz = z;
                }
            }
        }
        if (bf < 0) {
            covered_all = false;
            break;
        }
        if (bz < 0) {
            eq_chosen[bf] = 1;
            covered |= F.eq_kill[bf];
        } else {
            tok_chosen[bf][bz] = 1;
            covered |= F.tok_slot[bf][bz].kill;
        }
    }
    F.gate = covered_all && F.n_rules > 0 ? 1 : 0;
    for (int f = 0; f < F.n_eq; f++) F.eq_stage2[f] = F.gate && !eq_chosen[f] && F.eq_kill[f];
    // a regated plan's remaining stage-1 keys are other attributes than the
    // unit's own key: sparse, so they may be ORed first (FilterPlan::eq_any).
    // Measured on config 4 (i): 1.488 s with, 1.471 s without -- the
    // compiler's predicated kills already cost about what the OR chain does --
    // so it is opt-in (RB_EQ_ANY=1)
    F.eq_any = 0;
    F.eq_free = F.all_rules;
    const char* eq_any_on = std::getenv("RB_EQ_ANY");
    if (implied && eq_any_on && std::atoi(eq_any_on) != 0) {
        int n1 = 0;
        uint64_t killed = 0;
        for (int f = 0; f < F.n_eq; f++)
            if (!F.eq_stage2[f] && F.eq_kill[f]) {
                n1++;
                killed |= F.eq_kill[f];
            }
        if (n1 >= 2) {
            F.eq_any = 1;
            F.eq_free = F.all_rules & ~killed;
        }
    }
    for (int f = 0; f < F.n_tok; f++)
        for (int z = 0; z < F.tok_nslots[f]; z++) F.tok_slot[f][z].stage2 = F.gate && F.tok_always[f] && !tok_chosen[f][z];
    // Even with nothing deferred the gate pays when stage 1 is selective:
    // one vote then replaces the token / string feature votes (config 4:
    // 9.3e11 with, 7.9e11 without); it costs one vote per inner tuple when
    // stage 1 never fails inside the partitions (config 5: 7.0e11 vs 7.4e11).
}

extern "C" {

const char* rb_last_error(void) { return g_err.c_str(); }
const char* rb_version(void) { return "rbgpu 0.1 sm_100a"; }

int rb_ctx_create(int device, rb_ctx** out) {
    if (!out) return fail(RB_ERR_INVALID, "rb_ctx_create: out is NULL");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(RB_ERR_INVALID, "device %d out of range (%d devices)", device, ndev);
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) return fail(RB_ERR_CUDA, "device %d is sm_%d%d; librbgpu is built for sm_100a", device,
                                     prop.major, prop.minor);
    rb_ctx* c = new (std::nothrow) rb_ctx();
    if (!c) return fail(RB_ERR_OOM, "host allocation failed");
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->mem_total = prop.totalGlobalMem;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev_mid);
    if (e != cudaSuccess) {
        delete c;
        return fail(RB_ERR_CUDA, "context setup: %s", cudaGetErrorString(e));
    }
    c->own_stream = true;
    c->blocks_per_sm = pair_kernel_blocks_per_sm();
    cudaMemPool_t mp;
    if (cudaDeviceGetDefaultMemPool(&mp, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    if (cudaMallocHost(&c->host_ctr, sizeof(unsigned long long) * (16 + RB_MAX_SLOTS)) != cudaSuccess) {
        cudaGetLastError();
        c->host_ctr = nullptr;
    }
    *out = c;
    return RB_OK;
}

int rb_ctx_set_stream(rb_ctx* c, void* stream) {
    if (!c) return fail(RB_ERR_INVALID, "null ctx");
    CK(cudaSetDevice(c->device));
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    c->stream = (cudaStream_t)stream;
    c->own_stream = false;
    return RB_OK;
}

int rb_ctx_destroy(rb_ctx* c) {
    if (!c) return RB_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->items.release(c->stream);
    c->refs.release(c->stream);
    c->counters.release(c->stream);
    c->scratch.release(c->stream);
    c->surv.release(c->stream);
    c->offs.release(c->stream);
    for (DevBuf* b : {&c->col_k0, &c->col_k1, &c->col_flag, &c->col_temp, &c->col_r1, &c->col_r2, &c->col_cnt,
                      &c->col_out[0], &c->col_out[1], &c->col_out[2]})
        b->release(c->stream);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->ev_mid) cudaEventDestroy(c->ev_mid);
    for (auto& e : c->pool)
        for (int k = 0; k < 3; k++) dev_free(e.d[k], c->stream);
    c->pool.clear();
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->host_ctr) cudaFreeHost(c->host_ctr);
    c->host_items.release();
    c->host_offs.release();
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return RB_OK;
}

// ---------------------------------------------------------------------------
// relation

int rb_relation_create(rb_ctx* c, int64_t n, rb_rel** out) {
    if (!c || !out) return fail(RB_ERR_INVALID, "rb_relation_create: null argument");
    if (n < 0 || n > INT32_MAX) return fail(RB_ERR_INVALID, "relation size %lld out of range", (long long)n);
    rb_rel* r = new (std::nothrow) rb_rel();
    if (!r) return fail(RB_ERR_OOM, "host allocation failed");
    r->ctx = c;
    r->n = n;
    *out = r;
    return RB_OK;
}

// pad: zeroed bytes after the data (word-wise readers may touch them)
static cudaError_t upload(rb_rel* r, const void* src, size_t bytes, void** dst, size_t pad = 0) {
    *dst = nullptr;
    const size_t alloc = std::max<size_t>(bytes + pad, 16);  // never hand out null for an empty array
    cudaError_t e = dev_alloc(dst, alloc, r->ctx->stream);
    if (e != cudaSuccess) return e;
    r->allocs.push_back(*dst);
    if (!src || bytes == 0) return cudaMemsetAsync(*dst, 0, alloc, r->ctx->stream);
    e = cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, r->ctx->stream);
    if (e == cudaSuccess && alloc > bytes) e = cudaMemsetAsync((char*)*dst + bytes, 0, alloc - bytes, r->ctx->stream);
    return e;
}

static int add_column(rb_rel* r, const DevColumn& dc, int64_t max_len, int32_t* col, double mean_len = 0) {
    if ((int)r->cols.size() >= MAX_COLS) return fail(RB_ERR_LIMIT, "relation has more than %d columns", MAX_COLS);
    r->cols.push_back(dc);
    r->max_len.push_back(max_len);
    r->mean_len.push_back(mean_len);
    r->cols_dirty = true;
    if (col) *col = (int32_t)r->cols.size() - 1;
    return RB_OK;
}

int rb_relation_add_codes(rb_rel* r, const int32_t* codes, int32_t* col) {
    if (!r || (!codes && r->n)) return fail(RB_ERR_INVALID, "rb_relation_add_codes: null argument");
    CK(cudaSetDevice(r->ctx->device));
    DevColumn dc{};
    dc.kind = RB_COL_CODES;
    void* p;
    CK(upload(r, codes, sizeof(int32_t) * r->n, &p));
    dc.codes = (const int32_t*)p;
    return add_column(r, dc, 0, col);
}

int rb_relation_add_mask(rb_rel* r, const uint8_t* mask, int32_t* col) {
    if (!r || (!mask && r->n)) return fail(RB_ERR_INVALID, "rb_relation_add_mask: null argument");
    CK(cudaSetDevice(r->ctx->device));
    DevColumn dc{};
    dc.kind = RB_COL_MASK;
    void* p;
    CK(upload(r, mask, r->n, &p));
    dc.mask = (const uint8_t*)p;
    return add_column(r, dc, 0, col);
}

static int check_offsets(const int64_t* offsets, int64_t n, int64_t* max_len) {
    if (offsets[0] != 0) return fail(RB_ERR_INVALID, "offsets[0] must be 0");
    // longest row and first non-monotone row; large columns are scanned by
    // several host threads (a 10M-row column is 80 MB of offsets, ~10 ms on one
    // core, ahead of its upload)
    auto scan = [offsets](int64_t lo, int64_t hi, int64_t* m_out, int64_t* bad_out) {
        int64_t m = 0, bad = -1;
        for (int64_t i = lo; i < hi; i++) {
            const int64_t l = offsets[i + 1] - offsets[i];
            if (l < 0) {
                bad = i;
                break;
            }
            m = l > m ? l : m;
        }
        *m_out = m;
        *bad_out = bad;
    };
    const int nt = n >= (1 << 20) ? (int)std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency())) : 1;
    std::vector<int64_t> ms((size_t)nt, 0), bads((size_t)nt, -1);
    {
        std::vector<std::thread> th;
        for (int t = 1; t < nt; t++)
            th.emplace_back(scan, n * t / nt, n * (t + 1) / nt, &ms[(size_t)t], &bads[(size_t)t]);
        scan(0, n / nt, &ms[0], &bads[0]);
        for (auto& x : th) x.join();
    }
    int64_t m = 0;
    for (int t = 0; t < nt; t++) {
        if (bads[(size_t)t] >= 0) return fail(RB_ERR_INVALID, "offsets not monotone at row %lld", (long long)bads[(size_t)t]);
        m = std::max(m, ms[(size_t)t]);
    }
    if (m > INT32_MAX / 2) return fail(RB_ERR_LIMIT, "row of %lld elements is too long", (long long)m);
    *max_len = m;
    return RB_OK;
}

int rb_relation_add_tokens(rb_rel* r, const int64_t* offsets, const int32_t* ids, const uint8_t* missing,
                           int32_t* col) {
    if (!r || !offsets) return fail(RB_ERR_INVALID, "rb_relation_add_tokens: null argument");
    int64_t max_len;
    if (int rc = check_offsets(offsets, r->n, &max_len)) return rc;
    const int64_t nnz = offsets[r->n];
    if (nnz && !ids) return fail(RB_ERR_INVALID, "rb_relation_add_tokens: ids is NULL");
    CK(cudaSetDevice(r->ctx->device));
    DevColumn dc{};
    dc.kind = RB_COL_TOKENS;
    void *d_off, *d_ids, *d_miss = nullptr, *d_len, *d_sig, *d_hash;
    CK(upload(r, offsets, sizeof(int64_t) * (r->n + 1), &d_off));
    CK(upload(r, ids, sizeof(int32_t) * nnz, &d_ids));
    if (missing) CK(upload(r, missing, r->n, &d_miss));
    CK(upload(r, nullptr, sizeof(int32_t) * r->n, &d_len));
    CK(upload(r, nullptr, sizeof(uint4) * r->n, &d_sig));
    CK(upload(r, nullptr, sizeof(uint2) * r->n, &d_hash));
    CK(launch_token_features((const int64_t*)d_off, (const int32_t*)d_ids, (const uint8_t*)d_miss, r->n,
                             (int32_t*)d_len, (uint4*)d_sig, (uint2*)d_hash, r->ctx->stream));
    dc.offsets = (const int64_t*)d_off;
    dc.data = d_ids;
    dc.len = (const int32_t*)d_len;
    dc.sig = (const uint4*)d_sig;
    dc.hash = (const uint2*)d_hash;
    return add_column(r, dc, max_len, col, r->n ? (double)nnz / (double)r->n : 0.0);
}

int rb_relation_add_chars(rb_rel* r, const int64_t* offsets, const void* chars, int32_t width,
                          const uint8_t* missing, int32_t* col) {
    if (!r || !offsets) return fail(RB_ERR_INVALID, "rb_relation_add_chars: null argument");
    if (width != 1 && width != 4) return fail(RB_ERR_INVALID, "char width must be 1 or 4, got %d", width);
    int64_t max_len;
    if (int rc = check_offsets(offsets, r->n, &max_len)) return rc;
    const int64_t nnz = offsets[r->n];
    if (nnz && !chars) return fail(RB_ERR_INVALID, "rb_relation_add_chars: chars is NULL");
    CK(cudaSetDevice(r->ctx->device));
    DevColumn dc{};
    dc.kind = RB_COL_CHARS;
    dc.width = width;
    void *d_off, *d_chars, *d_miss = nullptr, *d_len, *d_bag;
    CK(upload(r, offsets, sizeof(int64_t) * (r->n + 1), &d_off));
    CK(upload(r, chars, (size_t)width * nnz, &d_chars, 16));  // the edit verifier reads u8 text four bytes at a time
    if (missing) CK(upload(r, missing, r->n, &d_miss));
    CK(upload(r, nullptr, sizeof(int32_t) * r->n, &d_len));
    CK(upload(r, nullptr, sizeof(uint4) * r->n, &d_bag));
    CK(launch_char_features((const int64_t*)d_off, d_chars, width, (const uint8_t*)d_miss, r->n, (int32_t*)d_len,
                            (uint4*)d_bag, r->ctx->stream));
    dc.offsets = (const int64_t*)d_off;
    dc.data = d_chars;
    dc.len = (const int32_t*)d_len;
    dc.bag = (const uint4*)d_bag;
    return add_column(r, dc, max_len, col, r->n ? (double)nnz / (double)r->n : 0.0);
}

int rb_relation_destroy(rb_rel* r) {
    if (!r) return RB_OK;
    cudaSetDevice(r->ctx->device);
    cudaStreamSynchronize(r->ctx->stream);
    for (void* p : r->allocs) dev_free(p, r->ctx->stream);
    dev_free(r->d_cols, r->ctx->stream);
    delete r;
    return RB_OK;
}

// ---------------------------------------------------------------------------
// program

int rb_program_create(rb_ctx* c, rb_rel* rel, const int32_t* op, const int32_t* slot, const int32_t* failj,
                      const int32_t* rule, int32_t n_ins, const rb_slot* slots, int32_t n_slots,
                      const int32_t* tables, int64_t n_tables, rb_prog** out) {
    if (!c || !rel || !out || (n_ins && (!op || !slot || !failj || !rule)) || (n_slots && !slots))
        return fail(RB_ERR_INVALID, "rb_program_create: null argument");
    // a relation is shared by every context of its device (e.g. one per
    // worker stream): its uploads, ordered on the owner's stream, finish first
    if (rel->ctx->device != c->device) return fail(RB_ERR_INVALID, "relation lives on another device");
    if (rel->ctx != c) CK(cudaStreamSynchronize(rel->ctx->stream));
    if (n_slots > RB_MAX_SLOTS) return fail(RB_ERR_LIMIT, "%d slots exceed the limit of %d", n_slots, RB_MAX_SLOTS);
    if (n_tables < 0 || (n_tables && !tables)) return fail(RB_ERR_INVALID, "bad table buffer");
    const int ncols = (int)rel->cols.size();

    // ---- validate slots
    for (int s = 0; s < n_slots; s++) {
        const rb_slot& sl = slots[s];
        if (sl.lhs < 0 || sl.lhs >= ncols || sl.rhs < 0 || sl.rhs >= ncols)
            return fail(RB_ERR_INVALID, "slot %d: column out of range", s);
        const int kl = rel->cols[sl.lhs].kind, kr = rel->cols[sl.rhs].kind;
        bool ok = false;
        switch (sl.kind) {
            case RB_SLOT_EQ_CODE: ok = kl == RB_COL_CODES && kr == RB_COL_CODES; break;
            case RB_SLOT_EQ_CONST: ok = kl == RB_COL_MASK; break;
            case RB_SLOT_JACCARD:
            case RB_SLOT_EXACT: ok = kl == RB_COL_TOKENS && kr == RB_COL_TOKENS; break;
            case RB_SLOT_EDIT: ok = kl == RB_COL_CHARS && kr == RB_COL_CHARS; break;
            default: return fail(RB_ERR_INVALID, "slot %d: unknown kind %d", s, sl.kind);
        }
        if (!ok) return fail(RB_ERR_INVALID, "slot %d: column kinds do not fit slot kind %d", s, sl.kind);
        if (sl.kind == RB_SLOT_JACCARD || sl.kind == RB_SLOT_EDIT) {
            if (sl.tab0 < 0 || sl.tab1 < 0 || sl.len0 < 1 || sl.len1 < 1 || sl.tab0 + sl.len0 > n_tables ||
                sl.tab1 + sl.len1 > n_tables)
                return fail(RB_ERR_INVALID, "slot %d: table range outside the table buffer", s);
            const int64_t lm = std::max(rel->max_len[sl.lhs], rel->max_len[sl.rhs]);
            const int64_t need0 = lm + 1, need1 = sl.kind == RB_SLOT_EDIT ? lm + 1 : 2 * lm + 1;
            if (sl.len0 < need0 || sl.len1 < need1)
                return fail(RB_ERR_INVALID, "slot %d: tables cover lengths < %lld", s, (long long)lm);
        }
    }

    // ---- instructions: checkpoint ordinals and each rule's needed slots
    std::vector<int4> ins(std::max(n_ins, 1));
    std::vector<int32_t> cp_rule(MAX_RULES, 0);
    std::vector<uint64_t> need;
    for (int k = 0; k < n_ins; k++) {
        if (op[k] == 1) {
            if ((int)need.size() >= MAX_RULES)
                return fail(RB_ERR_LIMIT, "more than %d checkpoints in the path", MAX_RULES);
            if (rule[k] < 0) return fail(RB_ERR_INVALID, "instruction %d: bad rule index", k);
            uint64_t m = 0;
            for (int p = 0; p < k; p++)
                if (op[p] == 0 && failj[p] > k) m |= 1ull << slot[p];
            cp_rule[need.size()] = rule[k];
            ins[k] = make_int4(1, (int)need.size(), -1, rule[k]);
            need.push_back(m);
        } else if (op[k] == 0) {
            if (slot[k] < 0 || slot[k] >= n_slots) return fail(RB_ERR_INVALID, "instruction %d: bad slot", k);
            if (failj[k] <= k || failj[k] > n_ins) return fail(RB_ERR_INVALID, "instruction %d: bad fail_jump", k);
            ins[k] = make_int4(0, slot[k], failj[k], -1);
        } else {
            return fail(RB_ERR_INVALID, "instruction %d: bad op %d", k, op[k]);
        }
    }

    CK(cudaSetDevice(c->device));
    rb_prog* P = new (std::nothrow) rb_prog();
    if (!P) return fail(RB_ERR_OOM, "host allocation failed");
    P->ctx = c;
    P->rel = rel;
    P->n_slots = n_slots;
    auto up = [&](const void* src, size_t bytes, void** dst) -> cudaError_t {
        *dst = nullptr;
        cudaError_t e = dev_alloc(dst, bytes, c->stream);
        if (e != cudaSuccess) return e;
        P->allocs.push_back(*dst);
        return cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, c->stream);
    };
    auto bail = [&](cudaError_t e) {
        for (void* p : P->allocs) dev_free(p, c->stream);
        delete P;
        return fail(e == cudaErrorMemoryAllocation ? RB_ERR_OOM : RB_ERR_CUDA, "program upload: %s",
                    cudaGetErrorString(e));
    };
    void *d_ins, *d_slots, *d_tables, *d_cp, *d_cols;
    cudaError_t e;
    if ((e = up(ins.data(), sizeof(int4) * ins.size(), &d_ins))) return bail(e);
    if ((e = up(cp_rule.data(), sizeof(int32_t) * cp_rule.size(), &d_cp))) return bail(e);
    std::vector<int32_t> tab(tables ? tables : (const int32_t*)nullptr,
                             tables ? tables + n_tables : (const int32_t*)nullptr);
    if (tab.empty()) tab.push_back(0);
    if ((e = up(tab.data(), sizeof(int32_t) * tab.size(), &d_tables))) return bail(e);
    const int32_t* T = (const int32_t*)d_tables;
    std::vector<DevSlot> ds(std::max(n_slots, 1));
    for (int s = 0; s < n_slots; s++) {
        const rb_slot& sl = slots[s];
        ds[s] = DevSlot{sl.kind, sl.lhs, sl.rhs, sl.flags, T + sl.tab0, T + sl.tab1, sl.len0, sl.len1};
        if (sl.kind == RB_SLOT_EDIT)
            P->lmax_edit = std::max<int64_t>(P->lmax_edit, std::max(rel->max_len[sl.lhs], rel->max_len[sl.rhs]));
    }
    if ((e = up(ds.data(), sizeof(DevSlot) * ds.size(), &d_slots))) return bail(e);
    if ((e = up(rel->cols.data(), sizeof(DevColumn) * rel->cols.size(), &d_cols))) return bail(e);

    // ---- phase-1 filter plan
    FilterPlan& F = P->F;
    memset(&F, 0, sizeof F);
    F.n_rules = (int)need.size();
    F.all_rules = need.size() >= 64 ? ~0ull : ((1ull << need.size()) - 1);
    auto kill_of = [&](int s) {  // rules whose precondition contains slot s
        uint64_t m = 0;
        for (size_t r = 0; r < need.size(); r++)
            if (need[r] & (1ull << s)) m |= 1ull << r;
        return m;
    };
    // shared-memory threshold tables: every filtered jaccard / edit slot gets
    // a prefix of its two tables; lengths beyond the prefix are not filtered
    struct TabReq {
        bool tok;
        int feat, z;
        int64_t src0, len0, src1, len1;
        int64_t nmax, mmax;  // jaccard: longest token row on the t / s side
    };
    std::vector<TabReq> treq;
    std::map<std::pair<int, int>, int> eqf, tokf, strf;
    std::map<int, int> constf;
    // filter class of each slot, in evaluation order: 0 eq/const, 1+f token
    // feature f, 1+MAX_TOK+f string feature f; -1 not filtered
    std::vector<int> cls(n_slots, -1);

    // ---- rule-level composite keys: the equality-type tests one rule needs
    // (eq codes, exact_token) become one key column, tested with one compare
    // (composite_key_kernel).  covered[s]: rules whose key contains slot s.
    std::vector<uint64_t> covered(n_slots, 0);
    {
        const char* env_ck = std::getenv("RB_COMPOSITE");
        const bool enable = !(env_ck && env_ck[0] == '0');
        constexpr int MAXC = MAX_EQ + MAX_TOK * MAX_FSLOTS;
        std::map<uint64_t, uint64_t> groups;  // component slots -> rules
        for (size_t r = 0; r < need.size() && enable; r++) {
            uint64_t m = 0;
            int cnt = 0;
            for (int s = 0; s < n_slots && cnt < MAXC; s++)
                if (((need[r] >> s) & 1) && (slots[s].kind == RB_SLOT_EQ_CODE || slots[s].kind == RB_SLOT_EXACT)) {
                    m |= 1ull << s;
                    cnt++;
                }
            if (cnt >= 2) groups[m] |= 1ull << r;
        }
        for (auto& g : groups) {
            if (F.n_eq >= MAX_EQ) break;
            CompositeSpec so{}, si{};
            bool same = true;
            for (int s = 0; s < n_slots; s++) {
                if (!((g.first >> s) & 1)) continue;
                const rb_slot& sl = slots[s];
                const DevColumn& L = rel->cols[sl.lhs];
                const DevColumn& R = rel->cols[sl.rhs];
                same &= sl.lhs == sl.rhs;
                if (sl.kind == RB_SLOT_EQ_CODE) {
                    so.codes[so.n] = L.codes;
                    si.codes[si.n] = R.codes;
                } else {
                    so.len[so.n] = L.len;
                    so.hash[so.n] = L.hash;
                    si.len[si.n] = R.len;
                    si.hash[si.n] = R.hash;
                }
                so.n++;
                si.n++;
            }
            void* d_o = nullptr;
            void* d_i = nullptr;
            if ((e = dev_alloc(&d_o, sizeof(int32_t) * std::max<int64_t>(rel->n, 1), c->stream))) return bail(e);
            P->allocs.push_back(d_o);
            if ((e = launch_composite_key(rel->n, so, (int32_t*)d_o, c->stream))) return bail(e);
            d_i = d_o;
            if (!same) {
                if ((e = dev_alloc(&d_i, sizeof(int32_t) * std::max<int64_t>(rel->n, 1), c->stream))) return bail(e);
                P->allocs.push_back(d_i);
                if ((e = launch_composite_key(rel->n, si, (int32_t*)d_i, c->stream))) return bail(e);
            }
            const int f = F.n_eq++;
            F.eq_outer[f] = (const int32_t*)d_o;
            F.eq_inner[f] = (const int32_t*)d_i;
            F.eq_kill[f] = g.second;
            F.eq_slots[f] = g.first;
            for (int s = 0; s < n_slots; s++)
                if ((g.first >> s) & 1) covered[s] |= g.second;
        }
    }

    for (int s = 0; s < n_slots; s++) {
        const rb_slot& sl = slots[s];
        uint64_t kill = kill_of(s);
        if (sl.kind == RB_SLOT_EQ_CODE || sl.kind == RB_SLOT_EXACT) {
            kill &= ~covered[s];  // those rules test it through their composite key
            if (!kill) {
                if (covered[s]) cls[s] = 0;
                continue;
            }
        }
        const DevColumn& L = rel->cols[sl.lhs];
        const DevColumn& R = rel->cols[sl.rhs];
        const auto key = std::make_pair(sl.lhs, sl.rhs);
        if (sl.kind == RB_SLOT_EQ_CODE) {
            auto it = eqf.find(key);
            int f;
            if (it != eqf.end()) {
                f = it->second;
            } else {
                if (F.n_eq >= MAX_EQ) continue;  // left unfiltered: decided by the exact pass
                f = eqf[key] = F.n_eq++;
                F.eq_outer[f] = L.codes;
                F.eq_inner[f] = R.codes;
            }
            F.eq_kill[f] |= kill;
            F.eq_slots[f] |= 1ull << s;
            cls[s] = 0;
        } else if (sl.kind == RB_SLOT_EQ_CONST) {
            auto it = constf.find(sl.lhs);
            int f;
            if (it != constf.end()) {
                f = it->second;
            } else {
                if (F.n_const >= MAX_CONST) continue;
                f = constf[sl.lhs] = F.n_const++;
                F.const_mask[f] = L.mask;
            }
            F.const_kill[f] |= kill;
            cls[s] = 0;
        } else if (sl.kind == RB_SLOT_JACCARD || sl.kind == RB_SLOT_EXACT) {
            auto it = tokf.find(key);
            int f;
            if (it != tokf.end()) {
                f = it->second;
            } else {
                if (F.n_tok >= MAX_TOK) continue;
                f = tokf[key] = F.n_tok++;
                F.tok_ooff[f] = L.offsets;
                F.tok_oids[f] = (const int32_t*)L.data;
                F.tok_olen[f] = L.len;
                F.tok_ohash[f] = L.hash;
                F.tok_ilen[f] = R.len;
                F.tok_isig[f] = R.sig;
                F.tok_ihash[f] = R.hash;
            }
            if (F.tok_nslots[f] >= MAX_FSLOTS) continue;
            // keep jaccard slots ahead of exact_token slots on each feature
            int at = F.tok_nslots[f]++;
            if (sl.kind == RB_SLOT_JACCARD) {
                for (int z = at; z > F.tok_njac[f]; z--) F.tok_slot[f][z] = F.tok_slot[f][z - 1];
                for (auto& t : treq)
                    if (t.feat == f && t.tok) t.z += (t.z >= F.tok_njac[f]) ? 1 : 0;
                at = F.tok_njac[f]++;
            }
            FSlot& fs = F.tok_slot[f][at];
            fs = FSlot{};
            fs.kill = kill;
            fs.kind = sl.kind;
            fs.slot = s;
            fs.delta = sl.delta;
            if (sl.kind == RB_SLOT_JACCARD)
                treq.push_back({true, f, at, sl.tab0, sl.len0, sl.tab1, sl.len1, rel->max_len[sl.lhs],
                                rel->max_len[sl.rhs]});
            F.tok_rules[f] |= kill;
            F.tok_kill[f] |= kill;
            cls[s] = 1 + f;
            // fold to 64-bit signatures when rows are short on both sides (<= 12
            // tokens on average): half the popcounts, few extra maybe-pairs
            {
                const double tl = rel->mean_len[sl.lhs], tr = rel->mean_len[sl.rhs];
                const char* env = std::getenv("RB_SIG64");
                F.tok_sig64[f] = env ? (env[0] == '1') : (tl <= 12.0 && tr <= 12.0);
            }
        } else if (sl.kind == RB_SLOT_EDIT) {
            auto it = strf.find(key);
            int f;
            if (it != strf.end()) {
                f = it->second;
            } else {
                if (F.n_str >= MAX_STR) continue;
                f = strf[key] = F.n_str++;
                F.str_olen[f] = L.len;
                F.str_obag[f] = L.bag;
                F.str_ilen[f] = R.len;
                F.str_ibag[f] = R.bag;
            }
            if (F.str_nslots[f] >= MAX_FSLOTS) continue;
            const int at = F.str_nslots[f]++;
            FSlot& fs = F.str_slot[f][at];
            fs.kill = kill;
            fs.kind = sl.kind;
            fs.slot = s;
            fs.delta = sl.delta;
            treq.push_back({false, f, at, sl.tab0, sl.len0, sl.tab1, sl.len1, 0, 0});
            F.str_rules[f] |= kill;
            F.str_kill[f] |= kill;
            cls[s] = 1 + MAX_TOK + f;
        }
    }
    // a token feature is "always" needed when some rule using it has no slot
    // filtered before it: then every warp with a valid pair evaluates it
    for (int f = 0; f < F.n_tok; f++) {
        for (size_t r = 0; r < need.size(); r++) {
            bool uses = false, earlier = false;
            for (int s = 0; s < n_slots; s++) {
                if (!(need[r] & (1ull << s))) continue;
                if (cls[s] == 1 + f) uses = true;
                if (cls[s] >= 0 && cls[s] < 1 + f) earlier = true;
            }
            if (uses && !earlier) F.tok_always[f] = 1;
        }
    }
    for (int f = 0; f < F.n_str; f++) {
        for (size_t r = 0; r < need.size(); r++) {
            bool uses = false, earlier = false;
            for (int s = 0; s < n_slots; s++) {
                if (!(need[r] & (1ull << s))) continue;
                if (cls[s] == 1 + MAX_TOK + f) uses = true;
                if (cls[s] >= 0 && cls[s] < 1 + MAX_TOK + f) earlier = true;
            }
            if (uses && !earlier) F.str_always[f] = 1;
        }
    }
    // ---- folded bags: for long strings with tight edit thresholds, buckets i
    // and i+8 are summed (saturating) -- still a bag-distance lower bound, half
    // the byte-SAD work per pair, and far above maxd for unrelated strings
    for (int f = 0; f < F.n_str; f++) {
        double dmin = 1.0;
        for (int z = 0; z < F.str_nslots[f]; z++) dmin = std::min(dmin, F.str_slot[f][z].delta);
        const int s0 = F.str_slot[f][0].slot;
        const double mean = std::min(rel->mean_len[slots[s0].lhs], rel->mean_len[slots[s0].rhs]);
        const char* env_fold = std::getenv("RB_FOLD_BAG");
        F.str_fold[f] = (env_fold ? env_fold[0] == '1' : (mean >= 48.0 && dmin >= 0.9)) ? 1 : 0;
    }

    // ---- implied kills: a failed test also rules out every rule that needs
    // a test implying it.  The threshold tables are monotone in delta, so a
    // Jaccard (edit) slot failing implies every slot on the same feature
    // with a higher delta fails; an equality key failing implies every key
    // over a superset of its slots fails (a component of a composite key);
    // an exact_token slot failing implies the composite keys containing it.
    {
        uint64_t tk[MAX_TOK][MAX_FSLOTS], sk[MAX_STR][MAX_FSLOTS], ek[MAX_EQ];
        for (int f = 0; f < F.n_tok; f++)
            for (int z = 0; z < F.tok_nslots[f]; z++) tk[f][z] = F.tok_slot[f][z].kill;
        for (int f = 0; f < F.n_str; f++)
            for (int z = 0; z < F.str_nslots[f]; z++) sk[f][z] = F.str_slot[f][z].kill;
        for (int f = 0; f < F.n_eq; f++) ek[f] = F.eq_kill[f];
        for (int f = 0; f < F.n_tok; f++)
            for (int z = 0; z < F.tok_njac[f]; z++)
                for (int y = 0; y < F.tok_njac[f]; y++)
                    if (y != z && F.tok_slot[f][y].delta >= F.tok_slot[f][z].delta) F.tok_slot[f][z].kill |= tk[f][y];
        for (int f = 0; f < F.n_str; f++)
            for (int z = 0; z < F.str_nslots[f]; z++)
                for (int y = 0; y < F.str_nslots[f]; y++)
                    if (y != z && F.str_slot[f][y].delta >= F.str_slot[f][z].delta) F.str_slot[f][z].kill |= sk[f][y];
        for (int a = 0; a < F.n_eq; a++)
            for (int b = 0; b < F.n_eq; b++)
                if (a != b && F.eq_slots[a] && (F.eq_slots[a] & ~F.eq_slots[b]) == 0) F.eq_kill[a] |= ek[b];
        for (int f = 0; f < F.n_tok; f++)
            for (int z = F.tok_njac[f]; z < F.tok_nslots[f]; z++)
                for (int b = 0; b < F.n_eq; b++)
                    if ((F.eq_slots[b] >> F.tok_slot[f][z].slot) & 1) F.tok_slot[f][z].kill |= ek[b];
    }
    // ---- stage-1 gate (specialised kernel): see choose_gate
    {
        std::vector<int> first_pos(n_slots, INT32_MAX);  // earliest instruction of each slot
        for (int k = 0; k < n_ins; k++)
            if (op[k] == 0 && first_pos[slot[k]] == INT32_MAX) first_pos[slot[k]] = k;
        P->gate_need = need;
        P->gate_first_pos = first_pos;
        P->gate_cls.assign(cls.begin(), cls.end());
        choose_gate(F, need, first_pos, n_slots, 0);
    }
    std::vector<int32_t> stab(TAB_BASE, 0);  // guard entries: lookups of missing (-1) lengths land here
    {
        // jaccard slots prefer one 2-D table need[n][m] (n in [0,nmax], m in
        // [-1,mmax]) folding both length tests: a single lookup per pair
        int64_t total1d = TAB_BASE, total2d = TAB_BASE;
        for (auto& t : treq) {
            total1d += t.len0 + t.len1;
            // 2-D: the jaccard slots of one token feature share one interleaved table
            const int njp = t.tok ? (F.tok_njac[t.feat] <= 1 ? 1 : F.tok_njac[t.feat] <= 2 ? 2 : 4) : 0;
            total2d += t.tok ? (t.z == 0 ? (t.nmax + 1) * ((t.mmax + 2) | 1) * njp + 4 : 0) : t.len0 + t.len1 + 4;
        }
        F.tok2d = total2d <= SMEM_TAB ? 1 : 0;
        const bool full = F.tok2d || total1d <= SMEM_TAB;
        const int64_t per = treq.empty() ? 0 : std::max<int64_t>(1, (SMEM_TAB - TAB_BASE) / (2 * (int64_t)treq.size()));
        const int32_t INF = 1 << 30;
        for (auto& t : treq) {
            FSlot& fs = t.tok ? F.tok_slot[t.feat][t.z] : F.str_slot[t.feat][t.z];
            if (t.tok && F.tok2d) {
                // need[n][m][z] for the feature's jaccard slots z, interleaved so
                // one vector load per pair fetches every slot's threshold:
                // entry (n, m, z) at tok_off[f] + ((n * w2) + m + 1) * njp + z
                const int f = t.feat;
                const int njp = F.tok_njac[f] <= 1 ? 1 : F.tok_njac[f] <= 2 ? 2 : 4;
                // row stride (in entries) padded to an odd count: lanes of a warp
                // read rows n of different outer tuples at the same column m, and
                // an odd stride spreads them over distinct shared-memory banks
                const int64_t w2 = (t.mmax + 2) | 1;
                if (t.z == 0) {
                    while (stab.size() % 4) stab.push_back(INF);  // 16-byte alignment of vector entries
                    F.tok_off[f] = (int32_t)stab.size();
                    F.tok_w2[f] = (int32_t)w2;
                    F.tok_njp[f] = njp;
                    stab.resize(stab.size() + (size_t)((t.nmax + 1) * w2 * njp), INF);
                }
                const int32_t* minsmall = tables + t.src0;
                const int32_t* mink = tables + t.src1;
                for (int64_t nn = 0; nn <= t.nmax; nn++)
                    for (int64_t mm = -1; mm <= t.mmax; mm++) {
                        int32_t v = INF;
                        if (mm >= 0 && (nn | mm) != 0) {
                            const int64_t small = std::min(nn, mm), big = std::max(nn, mm);
                            const int32_t ms = big < t.len0 ? minsmall[big] : 0;
                            const int32_t mk = nn + mm < t.len1 ? mink[nn + mm] : INF;
                            if (small >= ms && mk <= small) v = mk;
                        }
                        stab[(size_t)(F.tok_off[f] + (nn * w2 + mm + 1) * njp + t.z)] = v;
                    }
                fs.w2 = (int32_t)w2;
                fs.off0 = fs.off1 = F.tok_off[f];
                fs.cap0 = fs.cap1 = (int32_t)((t.nmax + 1) * w2 * njp);
                continue;
            }
            if (!t.tok) {
                // edit: one interleaved int2 table {G, M2}[L] with
                //   G  = min(maxgap[L], maxd[L])  (gap test; not read by the current filter)
                //   M2 = 2 * maxd[L]              (ceil((bag + gap) / 2) <= maxd)
                // The pair filter tests bag + gap <= max(M2[la], M2[lb]) with
                // both values looked up once per tuple (str_m2); M2[0] = 0
                // lets two empty strings through.  A guard entry {-1, -1}
                // precedes the table.
                const int32_t* maxgap = tables + t.src0;
                const int32_t* maxd = tables + t.src1;
                const int64_t lim = std::min(t.len0, t.len1);
                const int64_t c = full ? lim : std::min(lim, std::max<int64_t>(1, per - 2));
                if (stab.size() & 1) stab.push_back(0);  // 8-byte alignment
                stab.push_back(-1);
                stab.push_back(-1);
                fs.off0 = (int32_t)stab.size();
                fs.cap0 = (int32_t)c;
                for (int64_t L = 0; L < c; L++) {
                    if (L == 0) {  // two empty strings match: t = 0 passes; M2 stays monotone in L
                        stab.push_back(INF);
                        stab.push_back(0);
                    } else {
                        stab.push_back(std::min(maxgap[L], maxd[L]));
                        stab.push_back(maxd[L] < 0 ? -1 : 2 * maxd[L]);
                    }
                }
                fs.off1 = fs.off0;
                fs.cap1 = fs.cap0;
                continue;
            }
            const int64_t c0 = full ? t.len0 : std::min(t.len0, per);
            const int64_t c1 = full ? t.len1 : std::min(t.len1, per);
            fs.off0 = (int32_t)stab.size();
            fs.cap0 = (int32_t)c0;
            stab.insert(stab.end(), tables + t.src0, tables + t.src0 + c0);
            fs.off1 = (int32_t)stab.size();
            fs.cap1 = (int32_t)c1;
            stab.insert(stab.end(), tables + t.src1, tables + t.src1 + c1);
        }
        F.full_tab = full ? 1 : 0;
    }
    void* d_stab;
    if ((e = up(stab.data(), sizeof(int32_t) * stab.size(), &d_stab))) return bail(e);
    F.tab_src = (const int32_t*)d_stab;
    F.n_tab = (int32_t)stab.size();
    P->V.ins = (const int4*)d_ins;
    P->V.slots = (const DevSlot*)d_slots;
    P->V.cols = (const DevColumn*)d_cols;
    P->V.cp_rule = (const int32_t*)d_cp;
    P->V.n_ins = n_ins;
    P->V.n_slots = n_slots;
    if ((e = cudaStreamSynchronize(c->stream))) return bail(e);
    P->jit = jit_pair_kernel(P->F, c->device);
    {  // the program's shape key, and what earlier programs of this shape learned
        uint64_t h = 1469598103934665603ull;
        auto mix = [&](const void* p, size_t bytes) {
            const unsigned char* b = (const unsigned char*)p;
            for (size_t k = 0; k < bytes; k++) h = (h ^ b[k]) * 1099511628211ull;
        };
        mix(op, sizeof(int32_t) * n_ins);
        mix(slot, sizeof(int32_t) * n_ins);
        mix(failj, sizeof(int32_t) * n_ins);
        mix(rule, sizeof(int32_t) * n_ins);
        mix(slots, sizeof(rb_slot) * n_slots);
        if (n_tables) mix(tables, sizeof(int32_t) * n_tables);
        mix(&rel->n, sizeof rel->n);
        for (size_t k = 0; k < rel->cols.size(); k++) {
            mix(&rel->cols[k].kind, sizeof rel->cols[k].kind);
            mix(&rel->max_len[k], sizeof rel->max_len[k]);
        }
        P->shape_key = h;
        std::lock_guard<std::mutex> lock(c->mu);
        const char* learn = std::getenv("RB_LEARN");  // RB_LEARN=0: every program starts cold (tests)
        auto it = (learn && std::atoi(learn) == 0) ? c->learned.end() : c->learned.find(h);
        if (it != c->learned.end()) {
            const Learned& L = it->second;
            P->gate_off = L.gate_off;
            P->last_rows = L.last_rows;
            P->rows_by_items = L.rows_by_items;
            P->last_surv = L.last_surv;
            P->surv_rate = L.surv_rate;
            P->range_plans = L.range_plans;
        }
    }
    *out = P;
    return RB_OK;
}

int rb_program_kernel_info(const rb_prog* P, int32_t* specialized, double* compile_ms, const char** log) {
    if (!P) return fail(RB_ERR_INVALID, "rb_program_kernel_info: null program");
    if (specialized) *specialized = P->jit.ok ? 1 : 0;
    if (compile_ms) *compile_ms = P->jit.compile_ms;
    if (log) *log = P->jit.log.c_str();
    return RB_OK;
}

int rb_program_destroy(rb_prog* P) {
    if (!P) return RB_OK;
    cudaSetDevice(P->ctx->device);
    cudaStreamSynchronize(P->ctx->stream);
    for (void* p : P->allocs) dev_free(p, P->ctx->stream);
    delete P;
    return RB_OK;
}

// ---------------------------------------------------------------------------
// runs

}  // extern "C"

// RB_HOST_TIMING=1: host-side phase times of every run on stderr (diagnostics)
static double host_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

namespace {
int edit_stride(const rb_prog* P) {
    if (P->lmax_edit < 0) return 0;
    // a slice holds the banded DP row, or Myers' pattern table for bounds
    // above 31 (rb_device.cuh lev_myers: 2 x MYERS_HS slots + MYERS_DCAP x W
    // 64-bit masks, W = ceil(min(L, MYERS_NMAX) / 64))
    int64_t need = P->lmax_edit + 2;
    if (P->lmax_edit > 31) need = std::max<int64_t>(need, 2 * 64 + 2 * 48 * ((std::min<int64_t>(P->lmax_edit, 1024) + 63) / 64));
    return (int)((need + 31) & ~(int64_t)31);
}

int run_impl(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, int64_t total, const std::vector<Part>& parts,
             int64_t row_lo, int64_t row_hi, uint32_t flags, bool want_parts, rb_result** out, bool refs_on_device,
             uint64_t implied);

// RB_EXACT_STATS: after the run, one pass of the exact interpreter over
// every pair of its parts counts each slot's first touches; they replace
// the run's survivor-only counts.
int exact_stats(rb_ctx* c, rb_prog* P, const int32_t* d_refs, const std::vector<Part>& parts, int64_t row_lo,
                int64_t row_hi, uint32_t flags, int64_t* slot_evals) {
    std::lock_guard<std::mutex> lock(c->mu);
    cudaStream_t st = c->stream;
    std::vector<StatPart> sp(parts.size());
    for (size_t k = 0; k < parts.size(); k++) sp[k] = StatPart{parts[k].base, parts[k].n, parts[k].split, parts[k].rbase};
    const int block = 256, grid = std::max(1, std::min<int>((int)sp.size(), c->sm_count * 4));
    const int64_t stride = std::max(1, edit_stride(P));
    if (cudaError_t e = c->scratch.grow(sizeof(int32_t) * (size_t)stride * grid * block, st))
        return fail(RB_ERR_OOM, "exact stats scratch: %s", cudaGetErrorString(e));
    StatPart* d_parts = nullptr;
    unsigned long long* d_ev = nullptr;
    cudaError_t e = dev_alloc((void**)&d_parts, sizeof(StatPart) * std::max<size_t>(1, sp.size()), st);
    if (!e) e = dev_alloc((void**)&d_ev, sizeof(unsigned long long) * RB_MAX_SLOTS, st);
    unsigned long long h_ev[RB_MAX_SLOTS];
    if (!e && !sp.empty()) e = cudaMemcpyAsync(d_parts, sp.data(), sizeof(StatPart) * sp.size(), cudaMemcpyHostToDevice, st);
    if (!e) e = cudaMemsetAsync(d_ev, 0, sizeof(unsigned long long) * RB_MAX_SLOTS, st);
    if (!e) e = launch_exact_stats(P->V, d_refs, d_parts, (int)sp.size(), row_lo, row_hi, flags, (int32_t*)c->scratch.p,
                                   stride, d_ev, grid, block, st);
    if (!e) e = cudaMemcpyAsync(h_ev, d_ev, sizeof h_ev, cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    dev_free(d_parts, st);
    dev_free(d_ev, st);
    if (e) return fail(RB_ERR_CUDA, "exact stats: %s", cudaGetErrorString(e));
    for (int s = 0; s < RB_MAX_SLOTS; s++) slot_evals[s] = (int64_t)h_ev[s];
    return RB_OK;
}
}  // namespace

int rb::run(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, int64_t total, const std::vector<Part>& parts,
            int64_t row_lo, int64_t row_hi, uint32_t flags, bool want_parts, rb_result** out, bool refs_on_device,
            uint64_t implied) {
    int rc = run_impl(c, rel, P, refs, total, parts, row_lo, row_hi, flags, want_parts, out, refs_on_device, implied);
    if (rc == RB_OK) {  // keep what this run taught the program for later programs of its shape
        std::lock_guard<std::mutex> lock(c->mu);
        std::lock_guard<std::mutex> lock2(P->ranges_mu);
        Learned& L = c->learned[P->shape_key];
        L.gate_off = P->gate_off;
        L.last_rows = P->last_rows;
        L.rows_by_items = P->rows_by_items;
        L.last_surv = P->last_surv;
        L.surv_rate = P->surv_rate;
        L.range_plans = P->range_plans;
    }
    if (rc != RB_OK || !(flags & RB_EXACT_STATS)) return rc;
    const int32_t* d_refs = refs ? (refs_on_device ? refs : (const int32_t*)c->refs.p) : nullptr;
    rc = exact_stats(c, P, d_refs, parts, row_lo, row_hi, flags, (*out)->stats.slot_evals);
    if (rc != RB_OK) {
        rb_result_destroy(*out);
        *out = nullptr;
    }
    return rc;
}

namespace {
__global__ void remap_parts_kernel(int32_t* __restrict__ p, int64_t k, const int32_t* __restrict__ map) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = map[p[i]];
}
}  // namespace

int rb::run_mixed(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, int64_t total,
                  const std::vector<Part>& parts, uint32_t flags, bool want_parts, rb_result** out,
                  bool refs_on_device, uint64_t implied) {
    // size classes: a "large" unit fills at least one 3-row item (768 outer
    // rows) and one column chunk's worth of inner tuples
    const int64_t big = 3 * (int64_t)BLOCK;
    std::vector<int32_t> ia, ib;
    for (size_t k = 0; k < parts.size(); k++) {
        const Part& q = parts[k];
        const int64_t rows = q.split >= 0 ? q.split : q.n, cols = q.split >= 0 ? q.n - q.split : q.n;
        (rows >= big && cols >= big ? ib : ia).push_back((int32_t)k);
    }
    // measured on config 4 (i) at 10M: no gain (the large units' rate is set by
    // their pairs -- every pair of a zip partition reaches the address Jaccard --
    // not by the variant), and two runs per batch cost launches: opt-in
    const char* mixed = std::getenv("RB_MIXED");
    const bool on = mixed && std::atoi(mixed) != 0;
    if (!on || ia.empty() || ib.empty())
        return run(c, rel, P, refs, total, parts, 0, INT64_MAX, flags, want_parts, out, refs_on_device, implied);
    std::vector<Part> pa, pb;
    for (int32_t k : ia) pa.push_back(parts[(size_t)k]);
    for (int32_t k : ib) pb.push_back(parts[(size_t)k]);
    rb_result *ra = nullptr, *rbg = nullptr;
    int rc = run(c, rel, P, refs, total, pb, 0, INT64_MAX, flags, want_parts, &rbg, refs_on_device, implied);
    if (rc != RB_OK) return rc;
    rc = run(c, rel, P, refs, total, pa, 0, INT64_MAX, flags, want_parts, &ra, refs_on_device, implied);
    if (rc != RB_OK) {
        rb_result_destroy(rbg);
        return rc;
    }
    return merge_results(c, ra, rbg, want_parts, ia, ib, out);
}

int rb::merge_results(rb_ctx* c, rb_result* ra, rb_result* rbg, bool want_parts, const std::vector<int32_t>& ia,
                      const std::vector<int32_t>& ib, rb_result** out) {
    std::lock_guard<std::mutex> lock(c->mu);
    cudaStream_t st = c->stream;
    rb_result* res = new (std::nothrow) rb_result();
    if (!res) {
        rb_result_destroy(ra);
        rb_result_destroy(rbg);
        return fail(RB_ERR_OOM, "host allocation failed");
    }
    res->ctx = c;
    res->stream = st;
    const int64_t k = ra->count + rbg->count;
    res->cap = std::max<int64_t>(k, 1);
    res->count = k;
    cudaError_t e = cudaSuccess;
    int32_t** dst[4] = {&res->d_t, &res->d_s, &res->d_r, &res->d_p};
    int32_t* srca[4] = {ra->d_t, ra->d_s, ra->d_r, ra->d_p};
    int32_t* srcb[4] = {rbg->d_t, rbg->d_s, rbg->d_r, rbg->d_p};
    long long pcap = 0;
    const bool pooled = c->pool_take(res->cap, &res->d_t, &res->d_s, &res->d_r, &pcap);
    if (pooled) res->cap = pcap;
    for (int q = 0; q < 4 && !e; q++) {
        if (q == 3 && !want_parts) break;
        if (!(pooled && q < 3)) e = dev_alloc((void**)dst[q], sizeof(int32_t) * (size_t)res->cap, st);
        if (!e && ra->count) e = cudaMemcpyAsync(*dst[q], srca[q], sizeof(int32_t) * ra->count, cudaMemcpyDeviceToDevice, st);
        if (!e && rbg->count)
            e = cudaMemcpyAsync(*dst[q] + ra->count, srcb[q], sizeof(int32_t) * rbg->count, cudaMemcpyDeviceToDevice, st);
    }
    int32_t* d_map = nullptr;
    if (!e && want_parts && k) {  // sub-run part indices -> the batch's
        std::vector<int32_t> map(ia);
        map.insert(map.end(), ib.begin(), ib.end());
        e = dev_alloc((void**)&d_map, sizeof(int32_t) * map.size(), st);
        if (!e) e = cudaMemcpyAsync(d_map, map.data(), sizeof(int32_t) * map.size(), cudaMemcpyHostToDevice, st);
        // rows of ra index ia (map[0..|ia|)), rows of rbg index ib (map[|ia|..))
        const int grid = (int)std::min<int64_t>((k + 255) / 256, (int64_t)c->sm_count * 8);
        if (!e && ra->count) {
            remap_parts_kernel<<<grid, 256, 0, st>>>(res->d_p, ra->count, d_map);
            e = cudaGetLastError();
        }
        if (!e && rbg->count) {
            remap_parts_kernel<<<grid, 256, 0, st>>>(res->d_p + ra->count, rbg->count, d_map + ia.size());
            e = cudaGetLastError();
        }
    }
    if (!e) e = cudaStreamSynchronize(st);
    dev_free(d_map, st);
    res->stats = rbg->stats;
    rb_stats& S = res->stats;
    const rb_stats& A = ra->stats;
    S.comparisons += A.comparisons;
    S.survivors += A.survivors;
    S.emitted += A.emitted;
    S.kernel_ms += A.kernel_ms;
    S.pair_ms += A.pair_ms;
    S.launches += A.launches;
    S.retries += A.retries;
    S.jit_compile_ms += A.jit_compile_ms;
    S.specialized = std::min(S.specialized, A.specialized);
    for (int s = 0; s < RB_MAX_SLOTS; s++) S.slot_evals[s] += A.slot_evals[s];
    {
        // the sub-results go back to the context (their buffers feed the pool)
        c->mu.unlock();
        rb_result_destroy(ra);
        rb_result_destroy(rbg);
        c->mu.lock();
    }
    if (e) {
        for (int q = 0; q < 4; q++) dev_free(*dst[q], st);
        delete res;
        return fail(RB_ERR_CUDA, "merging the size classes of a batch: %s", cudaGetErrorString(e));
    }
    *out = res;
    return RB_OK;
}

namespace {
int run_impl(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, int64_t total, const std::vector<Part>& parts,
             int64_t row_lo, int64_t row_hi, uint32_t flags, bool want_parts, rb_result** out, bool refs_on_device,
             uint64_t implied) {
    if (!c || !rel || !P || !out) return fail(RB_ERR_INVALID, "run: null argument");
    // every run on a context shares its scratch (items, counters, survivor
    // buffer, output pool) and its program's adaptive state: one at a time
    std::lock_guard<std::mutex> ctx_lock(c->mu);
    if (P->rel != rel || P->ctx != c || rel->ctx->device != c->device)
        return fail(RB_ERR_INVALID, "run: program/relation/context mismatch");
    if (total < 0 || total > INT32_MAX) return fail(RB_ERR_INVALID, "run: partition size out of range");
    // tuple refs are range-checked on the device (refs_check_kernel, ahead of
    // the pair kernel, which then does nothing); the host scans only to name
    // the bad position (bad_refs below)
    auto bad_refs = [&]() {
        if (refs_on_device) return fail(RB_ERR_INVALID, "tuple ref outside the relation");
        for (int64_t k = 0; k < total; k++)
            if (refs[k] < 0 || refs[k] >= rel->n)
                return fail(RB_ERR_INVALID, "tuple ref %d at position %lld outside the relation", refs[k],
                            (long long)k);
        return fail(RB_ERR_INVALID, "tuple ref outside the relation");
    };
    if (!refs && total > rel->n) {
        return fail(RB_ERR_INVALID, "identity partition of %lld tuples exceeds the relation", (long long)total);
    }
    *out = nullptr;
    static const bool timing = std::getenv("RB_HOST_TIMING") != nullptr;
    double tm[8] = {timing ? host_ms() : 0};
    int ntm = 1;
    auto mark = [&]() {
        if (timing && ntm < 8) tm[ntm++] = host_ms();
    };
    auto report = [&]() {
        if (!timing) return;
        fprintf(stderr, "rb run: parts %zu items %zu |", parts.size(), (size_t)c->host_items.size());
        for (int k = 1; k < ntm; k++) fprintf(stderr, " %.3f", tm[k] - tm[k - 1]);
        fprintf(stderr, " ms\n");
    };
    CK(cudaSetDevice(c->device));
    rb_result* res = new (std::nothrow) rb_result();
    if (!res) return fail(RB_ERR_OOM, "host allocation failed");
    res->stream = c->stream;
    auto cleanup = [&](int rc) {
        dev_free(res->d_t, c->stream);
        dev_free(res->d_s, c->stream);
        dev_free(res->d_r, c->stream);
        dev_free(res->d_p, c->stream);
        delete res;
        return rc;
    };

    // ---- work items: BLOCK * rows outer rows x `chunk` inner columns, per part
    PinnedVec<Item>& items = c->host_items;
    // the items of parts [p0, p1), written at `at` (when non-null); returns their count
    auto part_items = [&](size_t p0, size_t p1, int64_t rows_per_item, int64_t chunk, Item* at) {
        size_t k = 0;
        for (size_t pi = p0; pi < p1; pi++) {
            const Part& pt = parts[pi];
            const bool cross = pt.split >= 0;
            const int32_t mode = cross ? MODE_CROSS : ((flags & RB_SYMMETRIC) ? MODE_SYM : MODE_ASYM);
            const int64_t end = cross ? pt.rbase + (pt.n - pt.split) : pt.base + pt.n;
            const int64_t rlo = pt.base + std::max<int64_t>(0, row_lo);
            const int64_t rhi = pt.base + std::min<int64_t>(row_hi, cross ? pt.split : pt.n);
            for (int64_t r0 = rlo; r0 < rhi; r0 += rows_per_item) {
                const int64_t rend = std::min<int64_t>(r0 + rows_per_item, rhi);
                int64_t c0 = cross ? pt.rbase : (mode == MODE_SYM ? r0 + 1 : pt.base);
                for (; c0 < end; c0 += chunk, k++) {
                    if (!at) continue;
                    Item& it = at[k];
                    it.row0 = (int32_t)r0;
                    it.col0 = (int32_t)c0;
                    it.col1 = (int32_t)std::min<int64_t>(c0 + chunk, end);
                    it.row_hi = (int32_t)rend;
                    it.mode = mode;
                    it.part = (int32_t)pi;
                    it.pad0 = it.pad1 = 0;
                }
            }
        }
        return k;
    };
    // A batch of many parts (one item or more each) is laid out by several
    // host threads: count per part range, then fill at the ranges' offsets
    // (same order as one thread).  Writing ~10^5 items is memory-bound work.
    const char* env_par = std::getenv("RB_ITEM_THREADS_MIN");
    const size_t par_min = env_par ? (size_t)std::max(1ll, std::atoll(env_par)) : 16384;
    // packed variant: runs of tiny partitions share items, larger parts and cross blocks get their own
    bool packed_items = false;
    const char* env_pack = std::getenv("RB_PACK_MAX");
    const int64_t pack_max = env_pack ? std::atoll(env_pack) : 64;
    // the items of parts [p0, p1) in the packed layout (packs never cross p1),
    // written at `at` when non-null; returns their count
    auto packed_items_of = [&](size_t p0, size_t p1, int64_t rows_per_item, int64_t chunk, Item* at) {
        size_t k = 0, first = 0, n_in = 0;  // the open pack: parts [first, first + n_in)
        int64_t rows = 0;
        auto close = [&]() {
            if (!n_in) return;
            if (at) {
                const Part& a = parts[first];
                const Part& b = parts[first + n_in - 1];
                Item& it = at[k];
                it.row0 = (int32_t)a.base;
                it.col0 = (int32_t)((flags & RB_SYMMETRIC) ? a.base + 1 : a.base);
                it.col1 = it.row_hi = (int32_t)(b.base + b.n);
                it.mode = MODE_PACKED;
                it.part = (int32_t)first;
                it.pad0 = (int32_t)(first + n_in);
                it.pad1 = 0;
            }
            k++;
            n_in = 0;
            rows = 0;
        };
        for (size_t pi = p0; pi < p1; pi++) {
            const Part& pt = parts[pi];
            if (pt.split < 0 && pt.n >= 2 && pt.n <= pack_max && pt.n <= rows_per_item) {  // a pack fits one item
                // a pack covers consecutive positions: parts must follow each other in refs
                if (n_in && (rows + pt.n > rows_per_item ||
                             parts[first + n_in - 1].base + parts[first + n_in - 1].n != pt.base))
                    close();
                if (!n_in) first = pi;
                n_in++;
                rows += pt.n;
                continue;
            }
            close();
            k += part_items(pi, pi + 1, rows_per_item, chunk, at ? at + k : nullptr);
        }
        close();
        return k;
    };
    auto build_items = [&](int64_t rows_per_item, int64_t chunk) {
        items.clear();
        const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
        const size_t nt = parts.size() >= par_min ? std::min<size_t>(hw, parts.size()) : 1;
        std::vector<size_t> cut(nt + 1), off(nt + 1, 0);
        for (size_t t = 0; t <= nt; t++) cut[t] = parts.size() * t / nt;
        std::vector<std::thread> pool;
        std::vector<size_t> cnt(nt, 0);
        auto run_all = [&](auto&& fn) {
            pool.clear();
            for (size_t t = 1; t < nt; t++) pool.emplace_back(fn, t);
            fn(0);
            for (auto& th : pool) th.join();
        };
        auto layout = [&](size_t t, Item* at) {
            return packed_items ? packed_items_of(cut[t], cut[t + 1], rows_per_item, chunk, at)
                                : part_items(cut[t], cut[t + 1], rows_per_item, chunk, at);
        };
        run_all([&](size_t t) { cnt[t] = layout(t, nullptr); });
        for (size_t t = 0; t < nt; t++) off[t + 1] = off[t] + cnt[t];
        if (off[nt] > items.cap && !items.grow(std::max(off[nt], 2 * items.cap))) return;
        run_all([&](size_t t) { layout(t, items.p + off[t]); });
        items.n = off[nt];
    };
    // Kernel variant: a 3-row kernel's 768-row items would leave threads idle
    // on small partitions (batches whose average part is shorter use a 2-row
    // variant), and a program whose gate proved useless runs ungated.  The
    // variants are compiled on first use.
    // Batches of tiny partitions (average <= RB_PACK_MAX tuples, 64 by
    // default; 0 disables) run the packed variant: whole partitions of up to
    // that size go back to back into one item, so every warp of a CTA has rows.
    const JitKernel* jp = &P->jit;
    // a run whose pairs all satisfy some slots (`implied`) uses a filter plan
    // regated without them (rb::choose_gate), compiled per variant on first
    // use (the process-wide NVRTC cache keys on the plan)
    FilterPlan Fi;
    JitKernel Ji;
    const FilterPlan* Fp = &P->F;
    if (implied && P->jit.ok && !P->gate_need.empty()) {
        Fi = P->F;
        choose_gate(Fi, P->gate_need, P->gate_first_pos, P->n_slots, implied, &P->gate_cls);
        const bool packed_v = P->jit.defer && parts.size() > 1 && pack_max >= 2 &&
                              total / (int64_t)parts.size() <= pack_max;
        Ji = jit_pair_kernel(Fi, c->device, packed_v ? 2 : 0, packed_v);
        if (Ji.ok && !packed_v && Ji.rows > 2 && !parts.empty() &&
            total / (int64_t)parts.size() < (int64_t)BLOCK * Ji.rows)
            Ji = jit_pair_kernel(Fi, c->device, 2);
        if (Ji.ok && (!packed_v || Ji.packed)) {
            jp = &Ji;
            Fp = &Fi;
        }
    }
    if (jp == &P->jit && P->jit.ok && P->jit.defer && parts.size() > 1 && pack_max >= 2 &&
        total / (int64_t)parts.size() <= pack_max) {
        static std::mutex packed_mu;
        std::lock_guard<std::mutex> lock(packed_mu);
        if (!P->jit_packed_tried) {
            P->jit_packed = jit_pair_kernel(P->F, c->device, 2, true);
            P->jit_packed_tried = true;
        }
        if (P->jit_packed.ok && P->jit_packed.packed) jp = &P->jit_packed;
    }
    if (P->jit.ok && jp == &P->jit) {
        const bool small = P->jit.rows > 2 && !parts.empty() &&
                           total / (int64_t)parts.size() < (int64_t)BLOCK * P->jit.rows;
        const bool nogate = P->gate_off && P->jit.gated;
        if (small || nogate) {
            static std::mutex variant_mu;  // programs may be shared by host threads
            std::lock_guard<std::mutex> lock(variant_mu);
            JitKernel& slot = nogate ? (small ? P->jit_small_nogate : P->jit_nogate) : P->jit_small;
            bool& tried = nogate ? (small ? P->jit_small_nogate_tried : P->jit_nogate_tried) : P->jit_small_tried;
            if (!tried) {
                FilterPlan Fv = P->F;
                if (nogate) {
                    Fv.gate = 0;
                    for (int f = 0; f < MAX_EQ; f++) Fv.eq_stage2[f] = 0;
                    for (int f = 0; f < MAX_TOK; f++)
                        for (int z = 0; z < MAX_FSLOTS; z++) Fv.tok_slot[f][z].stage2 = 0;
                }
                slot = jit_pair_kernel(Fv, c->device, small ? 2 : 0);
                tried = true;
            }
            if (slot.ok) jp = &slot;
        }
    }
    const JitKernel& J = *jp;
    packed_items = J.ok && J.packed;
    const int64_t rows_per_item = (int64_t)BLOCK * (J.ok ? J.rows : 1);
    mark();  // [1] variant selection
    build_items(rows_per_item, CHUNK);
    {
        // small runs: narrower column chunks until every CTA has work (down to one tile)
        const size_t target = 2 * (size_t)c->sm_count * (size_t)(J.ok ? J.blocks_per_sm : c->blocks_per_sm);
        for (int64_t chunk = CHUNK / 2; items.size() < target && chunk >= TJ; chunk /= 2)
            build_items(rows_per_item, chunk);
    }
    if (items.failed) {
        items.failed = false;
        return cleanup(fail(RB_ERR_OOM, "pinned host buffer for %zu work items", items.size() + 1));
    }
    int n_items = (int)items.size();
    const int64_t n = total;
    if (n_items == 0) {
        *out = res;
        return RB_OK;
    }

    if (cudaError_t e = c->items.grow(sizeof(Item) * items.size(), c->stream)) return cleanup(fail(RB_ERR_CUDA, "items: %s", cudaGetErrorString(e)));
    if (refs && !refs_on_device)
        if (cudaError_t e = c->refs.grow(sizeof(int32_t) * n, c->stream)) return cleanup(fail(RB_ERR_CUDA, "refs: %s", cudaGetErrorString(e)));
    // counters: [0] item counter (u32, padded), [1] out_count, [2] pairs, [3] survivors, [4..68) slot evals,
    // [68] entries appended to the deferred survivor buffer
    const size_t n_counters = 8 + RB_MAX_SLOTS;
    const size_t SURV = 4 + RB_MAX_SLOTS;
    const size_t BAD = 5 + RB_MAX_SLOTS;   // set by refs_check_kernel
    const size_t GATE = 6 + RB_MAX_SLOTS;  // warp iterations past the stage-1 gate, then all gated iterations
    // deferred verification: buffered survivors up to this many entries (16 B each); a
    // run that needs more falls back to the generic kernel, which decides them in place
    // RB_SURV_LIMIT / RB_SURV_MIN override both bounds (tests drive the retry and fallback paths with them)
    const char* env_lim = std::getenv("RB_SURV_LIMIT");
    const char* env_min = std::getenv("RB_SURV_MIN");
    // survivor buffer limit: 16 B per entry; 2^30 entries (17 GB) on a GPU with
    // HBM to spare (B200: 180 GB) so a pass with hundreds of millions of
    // survivors streams in one range instead of several serialised ones
    const long long SURV_LIMIT = env_lim ? std::max(1ll, std::atoll(env_lim)) : (c->mem_total >= (96ull << 30) ? 1ll << 30 : 1ll << 28);
    const long long SURV_MIN = env_min ? std::max(1ll, std::atoll(env_min)) : 1ll << 24;
    const bool defer = J.ok && J.defer;
    // capacity: the program's last survivor count, or whatever the context's
    // (pooled) buffer already holds, at least SURV_MIN entries (256 MB)
    long long scap = defer ? std::min(SURV_LIMIT, std::max<long long>({SURV_MIN, P->last_surv + P->last_surv / 4,
                                                                      env_min ? 0ll
                                                                              : (long long)(c->surv.bytes / sizeof(int4))}))
                           : 0;
    if (cudaError_t e = c->counters.grow(sizeof(unsigned long long) * n_counters, c->stream))
        return cleanup(fail(RB_ERR_CUDA, "counters: %s", cudaGetErrorString(e)));

    const int bps = J.ok ? J.blocks_per_sm : c->blocks_per_sm;
    const int grid = std::max(1, std::min(n_items, c->sm_count * bps));
    const int gridg = c->sm_count * c->blocks_per_sm;  // generic kernel (fallback)
    const int grid_v = c->sm_count * (J.ok ? J.verify_blocks_per_sm : 1);  // deferred verification
    int64_t stride = 0;
    if (P->lmax_edit >= 0) {
        stride = edit_stride(P);
        const size_t slices = (size_t)std::max(grid, std::max(gridg, grid_v)) * BLOCK;
        if (cudaError_t e = c->scratch.grow(sizeof(int32_t) * stride * slices, c->stream))
            return cleanup(fail(RB_ERR_OOM, "edit scratch (%lld B): %s",
                                (long long)(sizeof(int32_t) * stride * slices), cudaGetErrorString(e)));
    }

    if (packed_items) {  // start and end position of every part: the packed items' row -> part lookup
        PinnedVec<int32_t>& po = c->host_offs;  // pinned: the copy stays asynchronous
        const size_t np = parts.size();
        po.clear();
        if (2 * np + 1 > po.cap && !po.grow(2 * np + 1))
            return cleanup(fail(RB_ERR_OOM, "pinned part offsets (%zu)", 2 * np + 1));
        for (size_t k = 0; k < np; k++) {
            po.p[k] = (int32_t)parts[k].base;
            po.p[np + 1 + k] = (int32_t)(parts[k].base + parts[k].n);
        }
        po.p[np] = (int32_t)total;
        po.n = 2 * np + 1;
        if (cudaError_t e = c->offs.grow(sizeof(int32_t) * po.n, c->stream))
            return cleanup(fail(RB_ERR_CUDA, "part offsets: %s", cudaGetErrorString(e)));
        CK(cudaMemcpyAsync(c->offs.p, po.p, sizeof(int32_t) * po.n, cudaMemcpyHostToDevice, c->stream));
    }
    mark();  // [2] items built, device buffers sized
    CK(cudaMemcpyAsync(c->items.p, items.data(), sizeof(Item) * items.size(), cudaMemcpyHostToDevice, c->stream));
    if (refs && !refs_on_device)
        CK(cudaMemcpyAsync(c->refs.p, refs, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
    const int32_t* d_refs = refs_on_device ? refs : (const int32_t*)c->refs.p;

    // output rows: the previous run's count + 25%, at least RB_OUT_MIN (1M; tests lower it
    // to drive the grow-in-place path)
    const char* env_out = std::getenv("RB_OUT_MIN");
    const int n_items_now = (int)items.size();
    long long prev_rows = P->last_rows;
    {  // the previous run over the same items (a size class of a mixed batch alternates with another)
        std::lock_guard<std::mutex> lock(P->ranges_mu);
        auto it = P->rows_by_items.find(n_items_now);
        if (it != P->rows_by_items.end()) prev_rows = it->second;
    }
    long long cap = std::max<long long>(env_out ? std::max(1ll, std::atoll(env_out)) : 1 << 20,
                                        prev_rows + prev_rows / 4);
    unsigned long long* ctr = (unsigned long long*)c->counters.p;
    res->ctx = c;
    unsigned long long stack_ctr[n_counters];
    unsigned long long* host_ctr = c->host_ctr ? c->host_ctr : stack_ctr;

    if (defer) {
        // ---- deferred verification, streamed over item ranges.  Each range:
        // pair kernel -> (survivor count) -> verify kernel.  A range whose
        // survivors overflow the buffer is rolled back and re-run with a
        // larger buffer (up to SURV_LIMIT) or split in half, so any survivor
        // volume streams through a bounded buffer; the output buffer grows
        // (keeping its rows) before a verify that could overflow it.
        if (!env_out && c->pool_take(cap, &res->d_t, &res->d_s, &res->d_r, &cap)) {
        } else {
            cudaError_t e = dev_alloc((void**)&res->d_t, sizeof(int32_t) * cap, c->stream);
            if (!e) e = dev_alloc((void**)&res->d_s, sizeof(int32_t) * cap, c->stream);
            if (!e) e = dev_alloc((void**)&res->d_r, sizeof(int32_t) * cap, c->stream);
            if (e) return cleanup(fail(RB_ERR_OOM, "output buffer of %lld rows: %s", cap, cudaGetErrorString(e)));
        }
        if (want_parts)
            if (cudaError_t e = dev_alloc((void**)&res->d_p, sizeof(int32_t) * cap, c->stream))
                return cleanup(fail(RB_ERR_OOM, "part buffer of %lld rows: %s", cap, cudaGetErrorString(e)));
        res->cap = cap;
        if (cudaError_t e = c->surv.grow(sizeof(int4) * (size_t)scap, c->stream))
            return cleanup(fail(RB_ERR_OOM, "survivor buffer of %lld entries: %s", scap, cudaGetErrorString(e)));
        std::vector<unsigned long long> base(n_counters, 0);  // counters after the last completed range
        CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * n_counters, c->stream));
        if (refs) {
            CK(launch_refs_check(d_refs, n, rel->n, &ctr[BAD], c->stream));
            res->stats.launches += 1;
        }
        RunParams R{};
        R.bad_refs = refs ? &ctr[BAD] : nullptr;
        R.refs = refs ? d_refs : nullptr;
        R.n = n;
        R.flags = flags;
        R.item_counter = (unsigned int*)&ctr[0];
        R.out_count = &ctr[1];
        R.stat_pairs = &ctr[2];
        R.stat_surv = &ctr[3];
        R.slot_evals = &ctr[4];
        R.scratch = (int32_t*)c->scratch.p;
        R.scratch_stride = stride;
        R.surv_count = &ctr[SURV];
        R.stat_gate = &ctr[GATE];
        R.part_off = packed_items ? (const int32_t*)c->offs.p : nullptr;
        R.part_end = packed_items ? (const int32_t*)c->offs.p + parts.size() + 1 : nullptr;
        const long long per_row = (flags & RB_ENUMERATE) ? std::max(1, P->F.n_rules) : 1;
        // Ranges are sized from the survivors per item seen so far (the
        // program's previous run, else a probe of 1/64 of the items), so a
        // range rarely overflows the buffer; one that does is rolled back and
        // re-run larger or in halves (the `ranges` stack).
        std::vector<std::pair<int, int>> ranges, done_ranges, plan;
        std::vector<long long> done_counts;  // survivors of each completed range
        size_t replay = 0;
        // the plan's key: the item count, the run's tuple count and flags (not the
        // kernel variant: the gated and ungated kernels leave the same survivors)
        uint64_t plan_key = 1469598103934665603ull;
        for (uint64_t w : {(uint64_t)items.size(), (uint64_t)total, (uint64_t)flags}) {
            plan_key ^= w + 0x9e3779b97f4a7c15ull + (plan_key << 6) + (plan_key >> 2);
            plan_key *= 0xff51afd7ed558ccdull;
        }
        long long plan_widest = 0;
        {
            std::lock_guard<std::mutex> lock(P->ranges_mu);
            auto it = P->range_plans.find(plan_key);
            if (it != P->range_plans.end()) {
                plan = it->second.ranges;
                plan_widest = it->second.widest;
            }
        }
        if (!plan.empty() && plan_widest > scap) {  // replayed ranges: the buffer that plan's widest range needs
            scap = plan_widest;  // may exceed SURV_LIMIT: a single item with more survivors
            if (cudaError_t e = c->surv.grow(sizeof(int4) * (size_t)scap, c->stream))
                return cleanup(fail(RB_ERR_OOM, "survivor buffer of %lld entries: %s", scap, cudaGetErrorString(e)));
        }
        int retries = 0, next = 0;
        bool sync_next = false;  // the next range runs checked (an optimistic attempt of it did not fit)
        long long done_items = 0, done_surv = 0;
        for (;;) {
            if (ranges.empty()) {
                if (next >= n_items) break;
                if (replay < plan.size() && plan[replay].first == next) {
                    ranges.push_back(plan[replay++]);
                    next = ranges.back().second;
                    continue;
                }
                const double rate = done_items ? (double)done_surv / (double)done_items : P->surv_rate;
                long long size;
                if (rate < 0) {
                    size = std::max<long long>(grid, n_items / 64);  // probe
                } else {
                    const double budget = 0.8 * (double)SURV_LIMIT;
                    size = rate > 0 ? (long long)(budget / rate) : (long long)n_items;
                    const long long want = (long long)(rate * (double)std::min<long long>(size, n_items - next) * 1.25) + 4096;
                    if (want > scap) {  // grow ahead of the launch instead of after an overflow
                        scap = std::min(SURV_LIMIT, want);
                        if (cudaError_t e = c->surv.grow(sizeof(int4) * (size_t)scap, c->stream))
                            return cleanup(fail(RB_ERR_OOM, "survivor buffer of %lld entries: %s", scap,
                                                cudaGetErrorString(e)));
                    }
                }
                size = std::max<long long>(1, std::min<long long>(size, n_items - next));
                ranges.push_back({next, next + (int)size});
                next += (int)size;
            }
            const int lo = ranges.back().first, hi = ranges.back().second;
            ranges.pop_back();
            // Optimistic range: when the survivors seen so far say this range fits the
            // survivor buffer and the output, the verify kernel is queued right behind
            // the pair kernel and the host waits once.  Both kernels bound their writes
            // by the capacities and count past them, so a range that did not fit is
            // rolled back (counters restored) and re-run through the checked path.
            bool opt = false;
            {
                const double rate_now = done_items ? (double)done_surv / (double)done_items : P->surv_rate;
                if (!sync_next && rate_now >= 0) {
                    const char* env_margin = std::getenv("RB_OPT_MARGIN");  // tests: 0 forces roll-backs
                    const long long margin = env_margin ? std::max(0ll, std::atoll(env_margin)) : 4096;
                    const long long expect = (long long)(rate_now * (double)(hi - lo) * 1.25) + margin;
                    opt = expect <= scap && (long long)base[1] + expect * per_row <= cap;
                }
                sync_next = false;
            }
            CK(cudaMemsetAsync(&ctr[0], 0, sizeof(unsigned long long), c->stream));
            CK(cudaMemsetAsync(&ctr[SURV], 0, sizeof(unsigned long long), c->stream));
            R.items = (const Item*)c->items.p + lo;
            R.n_items = hi - lo;
            R.surv = (int4*)c->surv.p;
            R.surv_cap = scap;
            R.out_t = res->d_t;
            R.out_s = res->d_s;
            R.out_r = res->d_r;
            R.out_p = res->d_p;
            R.cap = cap;
            CK(cudaEventRecord(c->ev0, c->stream));
            cudaError_t e = launch_jit_kernel(J, *Fp, P->V, R, std::max(1, std::min(hi - lo, grid)), c->stream);
            if (e) return cleanup(fail(RB_ERR_CUDA, "pair kernel launch: %s", cudaGetErrorString(e)));
            CK(cudaEventRecord(c->ev_mid, c->stream));
            if (opt) {
                if ((e = launch_jit_verify(J, P->V, R, grid_v, c->stream)))
                    return cleanup(fail(RB_ERR_CUDA, "verify kernel launch: %s", cudaGetErrorString(e)));
                CK(cudaEventRecord(c->ev1, c->stream));
                CK(cudaMemcpyAsync(host_ctr, ctr, sizeof(unsigned long long) * n_counters, cudaMemcpyDeviceToHost,
                                   c->stream));
                if ((e = cudaStreamSynchronize(c->stream)))
                    return cleanup(fail(RB_ERR_CUDA, "pair + verify kernels: %s", cudaGetErrorString(e)));
                if (host_ctr[BAD]) return cleanup(bad_refs());
                const long long surv = (long long)host_ctr[SURV];
                if (surv > scap || (long long)host_ctr[1] > cap) {  // did not fit: roll back, re-run checked
                    retries++;
                    CK(cudaMemcpyAsync(ctr, base.data(), sizeof(unsigned long long) * n_counters,
                                       cudaMemcpyHostToDevice, c->stream));
                    ranges.push_back({lo, hi});
                    sync_next = true;
                    continue;
                }
                float pms = 0, vms = 0;
                cudaEventElapsedTime(&pms, c->ev0, c->ev_mid);
                cudaEventElapsedTime(&vms, c->ev_mid, c->ev1);
                res->stats.pair_ms += pms;
                res->stats.kernel_ms += pms + vms;
                res->stats.launches += 2;
                mark();  // [3] (first range) pair + verify done
                std::copy(host_ctr, host_ctr + n_counters, base.begin());
                P->last_surv = std::max(P->last_surv, surv);
                done_ranges.push_back({lo, hi});
                done_counts.push_back(surv);
                done_items += hi - lo;
                done_surv += surv;
                continue;
            }
            CK(cudaMemcpyAsync(host_ctr, ctr, sizeof(unsigned long long) * n_counters, cudaMemcpyDeviceToHost,
                               c->stream));
            if ((e = cudaStreamSynchronize(c->stream))) return cleanup(fail(RB_ERR_CUDA, "pair kernel: %s", cudaGetErrorString(e)));
            if (host_ctr[BAD]) return cleanup(bad_refs());
            float pms = 0;
            cudaEventElapsedTime(&pms, c->ev0, c->ev_mid);
            res->stats.pair_ms += pms;
            res->stats.kernel_ms += pms;
            res->stats.launches += 1;
            const long long surv = (long long)host_ctr[SURV];
            mark();  // [3] (first range) pair kernel done
            if (surv > scap) {  // roll this range back, then retry it with room or in halves
                retries++;
                CK(cudaMemcpyAsync(ctr, base.data(), sizeof(unsigned long long) * n_counters, cudaMemcpyHostToDevice,
                                   c->stream));
                if (surv <= SURV_LIMIT || hi - lo == 1) {
                    scap = surv;
                    if ((e = c->surv.grow(sizeof(int4) * (size_t)scap, c->stream)))
                        return cleanup(fail(RB_ERR_OOM, "survivor buffer of %lld entries: %s", scap,
                                            cudaGetErrorString(e)));
                    ranges.push_back({lo, hi});
                } else {
                    const int mid = lo + (hi - lo) / 2;
                    ranges.push_back({mid, hi});
                    ranges.push_back({lo, mid});
                }
                continue;
            }
            const long long need_rows = (long long)host_ctr[1] + surv * per_row;
            if (need_rows > cap) {  // grow the output, keeping the rows already written
                const long long ncap = std::max(need_rows, cap + cap / 2);
                const long long keep = (long long)host_ctr[1];
                int32_t* nb[4] = {nullptr, nullptr, nullptr, nullptr};
                int32_t* ob[4] = {res->d_t, res->d_s, res->d_r, res->d_p};
                for (int k = 0; k < 4; k++) {
                    if (!ob[k]) continue;
                    if ((e = dev_alloc((void**)&nb[k], sizeof(int32_t) * ncap, c->stream)))
                        return cleanup(fail(RB_ERR_OOM, "output buffer of %lld rows: %s", ncap, cudaGetErrorString(e)));
                    if (keep) CK(cudaMemcpyAsync(nb[k], ob[k], sizeof(int32_t) * keep, cudaMemcpyDeviceToDevice, c->stream));
                    dev_free(ob[k], c->stream);
                }
                res->d_t = nb[0];
                res->d_s = nb[1];
                res->d_r = nb[2];
                res->d_p = nb[3];
                cap = ncap;
                res->cap = cap;
                R.out_t = res->d_t;
                R.out_s = res->d_s;
                R.out_r = res->d_r;
                R.out_p = res->d_p;
                R.cap = cap;
            }
            CK(cudaEventRecord(c->ev0, c->stream));
            if ((e = launch_jit_verify(J, P->V, R, grid_v, c->stream)))
                return cleanup(fail(RB_ERR_CUDA, "verify kernel launch: %s", cudaGetErrorString(e)));
            CK(cudaEventRecord(c->ev1, c->stream));
            CK(cudaMemcpyAsync(host_ctr, ctr, sizeof(unsigned long long) * n_counters, cudaMemcpyDeviceToHost,
                               c->stream));
            if ((e = cudaStreamSynchronize(c->stream))) return cleanup(fail(RB_ERR_CUDA, "verify kernel: %s", cudaGetErrorString(e)));
            float vms = 0;
            cudaEventElapsedTime(&vms, c->ev0, c->ev1);
            res->stats.kernel_ms += vms;
            res->stats.launches += 1;
            std::copy(host_ctr, host_ctr + n_counters, base.begin());
            P->last_surv = std::max(P->last_surv, surv);
            done_ranges.push_back({lo, hi});
            done_counts.push_back(surv);
            done_items += hi - lo;
            done_surv += surv;
        }
        P->surv_rate = done_items ? (double)done_surv / (double)done_items : -1.0;
        // the plan for the next run: adjacent ranges merged while their survivors fit the
        // streaming budget (so a probe range or an over-cautious split is not replayed)
        std::vector<std::pair<int, int>> merged;
        long long acc = 0, widest = 0;
        for (size_t k = 0; k < done_ranges.size(); k++) {
            if (!merged.empty() && merged.back().second == done_ranges[k].first &&
                acc + done_counts[k] <= (long long)(0.8 * (double)SURV_LIMIT)) {
                merged.back().second = done_ranges[k].second;
                acc += done_counts[k];
            } else {
                merged.push_back(done_ranges[k]);
                acc = done_counts[k];
            }
            widest = std::max(widest, acc);  // survivors of the largest merged range: the buffer a replay needs
        }
        P->last_surv = widest;  // this run's own figure: a later run over other data re-adapts
        {
            std::lock_guard<std::mutex> lock(P->ranges_mu);
            if (P->range_plans.size() >= 8 && !P->range_plans.count(plan_key))
                P->range_plans.erase(P->range_plans.begin());
            RangePlan& rp = P->range_plans[plan_key];
            rp.ranges.swap(merged);
            rp.widest = widest;
        }
        // a gate that nearly every warp iteration passes only costs its vote:
        // later runs of this program use the ungated kernel
        if (Fp == &P->F && J.gated && base[GATE + 1] > 0 && (double)base[GATE] > 0.95 * (double)base[GATE + 1])
            P->gate_off = true;
        const long long rows = (long long)base[1];
        res->count = rows;
        res->stats.comparisons = (int64_t)base[2];
        res->stats.survivors = (int64_t)base[3];
        res->stats.emitted = rows;
        res->stats.retries = retries;
        res->stats.specialized = 1;
        res->stats.jit_compile_ms = J.compile_ms;
        P->last_rows = rows;
        {
            std::lock_guard<std::mutex> lock(P->ranges_mu);
            if (P->rows_by_items.size() >= 8 && !P->rows_by_items.count(n_items_now))
                P->rows_by_items.erase(P->rows_by_items.begin());
            P->rows_by_items[n_items_now] = rows;
        }
        for (int s = 0; s < RB_MAX_SLOTS; s++) res->stats.slot_evals[s] = (int64_t)base[4 + s];
        mark();  // verify done
        report();
        *out = res;
        return RB_OK;
    }

    // ---- the generic kernel (no NVRTC specialisation): survivors are
    // decided inside the pair kernel; an output overflow re-runs once with
    // the exact size
    for (int attempt = 0;; attempt++) {
        if (c->pool_take(cap, &res->d_t, &res->d_s, &res->d_r, &cap)) {  // reuse cached buffers
        } else {
            res->d_t = res->d_s = res->d_r = nullptr;
            cudaError_t e = dev_alloc((void**)&res->d_t, sizeof(int32_t) * cap, c->stream);
            if (!e) e = dev_alloc((void**)&res->d_s, sizeof(int32_t) * cap, c->stream);
            if (!e) e = dev_alloc((void**)&res->d_r, sizeof(int32_t) * cap, c->stream);
            if (e) return cleanup(fail(RB_ERR_OOM, "output buffer of %lld rows: %s", cap, cudaGetErrorString(e)));
        }
        res->cap = cap;
        cudaError_t e = cudaSuccess;
        if (want_parts) {
            e = dev_alloc((void**)&res->d_p, sizeof(int32_t) * cap, c->stream);
            if (e) return cleanup(fail(RB_ERR_OOM, "part buffer of %lld rows: %s", cap, cudaGetErrorString(e)));
        }
        CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * n_counters, c->stream));
        if (refs) {
            CK(launch_refs_check(d_refs, n, rel->n, &ctr[BAD], c->stream));
            res->stats.launches += 1;
        }

        RunParams R{};
        R.bad_refs = refs ? &ctr[BAD] : nullptr;
        R.refs = refs ? d_refs : nullptr;
        R.n = n;
        R.flags = flags;
        R.items = (const Item*)c->items.p;
        R.n_items = n_items;
        R.item_counter = (unsigned int*)&ctr[0];
        R.out_t = res->d_t;
        R.out_s = res->d_s;
        R.out_r = res->d_r;
        R.out_p = res->d_p;
        R.out_count = &ctr[1];
        R.cap = cap;
        R.stat_pairs = &ctr[2];
        R.stat_surv = &ctr[3];
        R.slot_evals = &ctr[4];
        R.scratch = (int32_t*)c->scratch.p;
        R.scratch_stride = stride;

        CK(cudaEventRecord(c->ev0, c->stream));
        e = J.ok ? launch_jit_kernel(J, *Fp, P->V, R, grid, c->stream)
                      : launch_pair_kernel(P->F, P->V, R, std::max(1, std::min(n_items, gridg)), c->stream);
        if (e) return cleanup(fail(RB_ERR_CUDA, "pair kernel launch: %s", cudaGetErrorString(e)));
        CK(cudaEventRecord(c->ev1, c->stream));
        CK(cudaMemcpyAsync(host_ctr, ctr, sizeof(unsigned long long) * n_counters, cudaMemcpyDeviceToHost, c->stream));
        e = cudaStreamSynchronize(c->stream);
        if (e) return cleanup(fail(RB_ERR_CUDA, "pair kernel: %s", cudaGetErrorString(e)));
        if (host_ctr[BAD]) return cleanup(bad_refs());
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev0, c->ev1);
        res->stats.kernel_ms += ms;
        res->stats.pair_ms += ms;
        res->stats.launches += 1;
        const long long rows = (long long)host_ctr[1];
        if (rows <= cap) {
            res->count = rows;
            res->stats.comparisons = (int64_t)host_ctr[2];
            res->stats.survivors = (int64_t)host_ctr[3];
            res->stats.emitted = rows;
            res->stats.retries = attempt;
            res->stats.specialized = J.ok ? 1 : 0;
            res->stats.jit_compile_ms = J.compile_ms;
            P->last_rows = rows;
            for (int s = 0; s < RB_MAX_SLOTS; s++) res->stats.slot_evals[s] = (int64_t)host_ctr[4 + s];
            break;
        }
        dev_free(res->d_t, c->stream);
        dev_free(res->d_s, c->stream);
        dev_free(res->d_r, c->stream);
        dev_free(res->d_p, c->stream);
        res->d_t = res->d_s = res->d_r = res->d_p = nullptr;
        cap = rows;
    }
    *out = res;
    return RB_OK;
}
}  // namespace

extern "C" {

int rb_run_partition(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, int64_t n, uint32_t flags,
                     rb_result** out) {
    return run(c, rel, P, refs, n, {Part{0, n, -1, 0}}, 0, n, flags, false, out);
}

int rb_run_partition_rows(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, int64_t n, int64_t row_lo,
                          int64_t row_hi, uint32_t flags, rb_result** out) {
    return run(c, rel, P, refs, n, {Part{0, n, -1, 0}}, row_lo, row_hi, flags, false, out);
}

int rb_run_cross(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* left, int64_t nl, const int32_t* right,
                 int64_t nr, uint32_t flags, rb_result** out) {
    if ((nl && !left) || (nr && !right) || nl < 0 || nr < 0) return fail(RB_ERR_INVALID, "rb_run_cross: bad refs");
    std::vector<int32_t> both((size_t)(nl + nr));
    if (nl) memcpy(both.data(), left, sizeof(int32_t) * nl);
    if (nr) memcpy(both.data() + nl, right, sizeof(int32_t) * nr);
    return run(c, rel, P, both.data(), nl + nr, {Part{0, nl + nr, nl, nl}}, 0, nl + nr, flags, false, out);
}

int rb_run_batch(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, const int64_t* offsets,
                 const int64_t* splits, int32_t n_parts, uint32_t flags, rb_result** out) {
    return rb_run_batch_implied(c, rel, P, refs, offsets, splits, n_parts, flags, 0, out);
}

int rb_run_batch_implied(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, const int64_t* offsets,
                         const int64_t* splits, int32_t n_parts, uint32_t flags, uint64_t implied_slots,
                         rb_result** out) {
    if (n_parts < 0 || (n_parts && (!offsets || !refs))) return fail(RB_ERR_INVALID, "rb_run_batch: bad arguments");
    if (P && implied_slots >> std::min(63, P->n_slots) && P->n_slots < 64)
        return fail(RB_ERR_INVALID, "rb_run_batch_implied: implied slots beyond the program's %d", P->n_slots);
    std::vector<Part> parts;
    parts.reserve(n_parts);
    if (n_parts && offsets[0] != 0) return fail(RB_ERR_INVALID, "rb_run_batch: offsets[0] must be 0");
    for (int32_t k = 0; k < n_parts; k++) {
        const int64_t len = offsets[k + 1] - offsets[k];
        if (len < 0) return fail(RB_ERR_INVALID, "rb_run_batch: offsets not monotone at %d", k);
        const int64_t sp = splits ? splits[k] : -1;
        if (sp > len) return fail(RB_ERR_INVALID, "rb_run_batch: split %lld beyond part %d", (long long)sp, k);
        parts.push_back(Part{offsets[k], len, sp, sp >= 0 ? offsets[k] + sp : 0});
    }
    const int64_t total = n_parts ? offsets[n_parts] : 0;
    const char* off = std::getenv("RB_IMPLIED_OFF");
    if (off && std::atoi(off) != 0) implied_slots = 0;
    return run_mixed(c, rel, P, refs, total, parts, flags, true, out, false, implied_slots);
}

int rb_result_copy_parts(const rb_result* r, int32_t* part) {
    if (!r) return fail(RB_ERR_INVALID, "rb_result_copy_parts: null result");
    if (r->count == 0) return RB_OK;
    if (!r->d_p) return fail(RB_ERR_INVALID, "rb_result_copy_parts: not a batched result");
    if (!part) return fail(RB_ERR_INVALID, "rb_result_copy_parts: null output array");
    CK(cudaMemcpyAsync(part, r->d_p, sizeof(int32_t) * r->count, cudaMemcpyDeviceToHost, r->stream));
    CK(cudaStreamSynchronize(r->stream));
    return RB_OK;
}

int rb_result_count(const rb_result* r, int64_t* rows) {
    if (!r || !rows) return fail(RB_ERR_INVALID, "rb_result_count: null argument");
    *rows = r->count;
    return RB_OK;
}

int rb_result_copy(const rb_result* r, int32_t* t, int32_t* s, int32_t* rule) {
    if (!r) return fail(RB_ERR_INVALID, "rb_result_copy: null result");
    if (r->count == 0) return RB_OK;
    if (!t || !s || !rule) return fail(RB_ERR_INVALID, "rb_result_copy: null output array");
    const size_t bytes = sizeof(int32_t) * r->count;
    CK(cudaMemcpyAsync(t, r->d_t, bytes, cudaMemcpyDeviceToHost, r->stream));
    CK(cudaMemcpyAsync(s, r->d_s, bytes, cudaMemcpyDeviceToHost, r->stream));
    CK(cudaMemcpyAsync(rule, r->d_r, bytes, cudaMemcpyDeviceToHost, r->stream));
    CK(cudaStreamSynchronize(r->stream));
    return RB_OK;
}

int rb_result_device(const rb_result* r, const int32_t** t, const int32_t** s, const int32_t** rule,
                     const int32_t** part) {
    if (!r || !t || !s || !rule) return fail(RB_ERR_INVALID, "rb_result_device: null argument");
    *t = r->d_t;
    *s = r->d_s;
    *rule = r->d_r;
    if (part) *part = r->d_p;
    return RB_OK;
}

int rb_result_stats(const rb_result* r, rb_stats* out) {
    if (!r || !out) return fail(RB_ERR_INVALID, "rb_result_stats: null argument");
    *out = r->stats;
    return RB_OK;
}

int rb_result_destroy(rb_result* r) {
    if (!r) return RB_OK;
    rb_ctx* c = r->ctx;
    std::unique_lock<std::mutex> lock;
    if (c) lock = std::unique_lock<std::mutex>(c->mu);  // the pool is context state
    if (c && r->d_t && r->d_s && r->d_r && r->cap > 0) {  // the rows' buffers go back to the context cache
        c->pool_give(r->d_t, r->d_s, r->d_r, r->cap, r->stream);
        r->d_t = r->d_s = r->d_r = nullptr;
    }
    dev_free(r->d_t, r->stream);
    dev_free(r->d_s, r->stream);
    dev_free(r->d_r, r->stream);
    dev_free(r->d_p, r->stream);
    delete r;
    return RB_OK;
}

}  // extern "C"
