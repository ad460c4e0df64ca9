// rb_state.cuh -- host-side state behind the C ABI handles (rb_ctx, rb_rel,
// rb_prog, rb_result) shared by rb_api.cu (relations, programs, runs) and
// rb_pipeline.cu (device partitioning and collect).  Not part of the ABI.
#pragma once
#include <map>
#include <unordered_map>

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "rb_internal.cuh"

namespace rb {

// records the message of the last failure on the calling thread (rb_last_error)
int fail(int code, const char* fmt, ...);

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(e_ == cudaErrorMemoryAllocation ? RB_ERR_OOM : RB_ERR_CUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
    } while (0)

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync
// with an unbounded release threshold): relations, programs and results are
// created and dropped per call on the e2e path, and plain cudaFree there
// costs tens to hundreds of milliseconds.
inline cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st) {
    return cudaMallocAsync(p, std::max(bytes, (size_t)16), st);
}
inline void dev_free(void* p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t grow(size_t need, cudaStream_t st) {
        if (need <= bytes) return cudaSuccess;
        dev_free(p, st);
        p = nullptr;
        bytes = 0;
        size_t want = std::max(need, (size_t)256);
        cudaError_t e = dev_alloc(&p, want, st);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
    void release(cudaStream_t st) {
        dev_free(p, st);
        p = nullptr;
        bytes = 0;
    }
};

// Growable array in pinned host memory: the work items are built straight
// into it and copied to the device asynchronously at full link speed (a
// batch of many small partitions has one item per partition).  Reused by
// every run on the context; a run synchronises its stream before returning,
// so the buffer is never overwritten under an in-flight copy.
template <typename T>
struct PinnedVec {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    bool failed = false;
    void clear() { n = 0; }
    void push_back(const T& v) {
        if (n == cap && !grow(cap ? 2 * cap : 4096)) return;
        p[n++] = v;
    }
    bool grow(size_t want) {
        T* q = nullptr;
        if (cudaMallocHost((void**)&q, sizeof(T) * want) != cudaSuccess) {
            failed = true;
            return false;
        }
        if (n) std::memcpy(q, p, sizeof(T) * n);
        if (p) cudaFreeHost(p);
        p = q;
        cap = want;
        return true;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = cap = 0;
    }
    size_t size() const { return n; }
    const T* data() const { return p; }
};

}  // namespace rb

using rb::DevBuf;
using rb::PinnedVec;
using rb::fail;
using rb::dev_alloc;
using rb::dev_free;
using rb::Item;
using rb::DevColumn;
using rb::FilterPlan;
using rb::VerifyProg;
using rb::JitKernel;

// What runs taught a program (variant, buffer sizes, survivor ranges), kept
// per context under the program's shape key: a new rb_prog for the same
// program over a relation of the same shape (the public API building its
// objects afresh on every call) starts from it instead of probing again.
// Only sizing hints: overflow handling keeps every run exact.
// item ranges that fit the survivor buffer in an earlier run over the same work
// items, and the survivors of the largest of them (the buffer a replay needs)
struct RangePlan {
    std::vector<std::pair<int, int>> ranges;
    long long widest = 0;
};

struct Learned {
    bool gate_off = false;
    long long last_rows = 0, last_surv = 0;
    std::map<int, long long> rows_by_items;
    double surv_rate = -1.0;
    std::map<uint64_t, RangePlan> range_plans;
};

struct rb_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int sm_count = 0;
    int blocks_per_sm = 1;
    size_t mem_total = 0;
    DevBuf items, refs, counters, scratch, surv, offs;
    // collect (rb_pipeline.cu): sort keys, flags, CUB temp and the collected
    // rows -- grown once and reused, so a step allocates nothing from the pool
    DevBuf col_k0, col_k1, col_flag, col_temp, col_r1, col_r2, col_cnt, col_out[3];
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_mid = nullptr;
    // output row buffers (t, s, rule) of destroyed results, reused best-fit by
    // later runs, merges and collects (at most 4 triples, the largest kept):
    // a step allocates no multi-GB buffers once the cache is warm
    struct PoolEntry {
        int32_t* d[3];
        long long cap;
    };
    std::vector<PoolEntry> pool;
    // the smallest cached triple holding `need` rows (removed from the cache), or false
    bool pool_take(long long need, int32_t** t, int32_t** s, int32_t** r, long long* cap) {
        int best = -1;
        for (size_t k = 0; k < pool.size(); k++)
            if (pool[k].cap >= need && (best < 0 || pool[k].cap < pool[(size_t)best].cap)) best = (int)k;
        if (best < 0) return false;
        *t = pool[(size_t)best].d[0];
        *s = pool[(size_t)best].d[1];
        *r = pool[(size_t)best].d[2];
        *cap = pool[(size_t)best].cap;
        pool.erase(pool.begin() + best);
        return true;
    }
    // cache a triple; the smallest is freed when more than 4 are held
    void pool_give(int32_t* t, int32_t* s, int32_t* r, long long cap, cudaStream_t st) {
        pool.push_back(PoolEntry{{t, s, r}, cap});
        if (pool.size() > 4) {
            size_t small = 0;
            for (size_t k = 1; k < pool.size(); k++)
                if (pool[k].cap < pool[small].cap) small = k;
            for (int q = 0; q < 3; q++) dev_free(pool[small].d[q], st);
            pool.erase(pool.begin() + (long)small);
        }
    }
    unsigned long long* host_ctr = nullptr;  // pinned: counters read back after each run
    PinnedVec<Item> host_items;              // the last run's work items
    PinnedVec<int32_t> host_offs;            // the last run's part starts / ends (packed items)
    std::mutex mu;                           // runs on one context are serialised (shared scratch)
    std::unordered_map<uint64_t, Learned> learned;  // by rb_prog::shape_key, guarded by mu
};

struct rb_rel {
    rb_ctx* ctx = nullptr;
    int64_t n = 0;
    std::vector<DevColumn> cols;
    std::vector<int64_t> max_len;
    std::vector<double> mean_len;
    std::vector<void*> allocs;
    void* d_cols = nullptr;
    bool cols_dirty = true;
};

struct rb_prog {
    rb_ctx* ctx = nullptr;
    rb_rel* rel = nullptr;
    FilterPlan F{};
    VerifyProg V{};
    int32_t n_slots = 0;
    int64_t lmax_edit = -1;  // longest string any edit slot reads (-1: no edit slot)
    std::vector<void*> allocs;
    JitKernel jit;
    JitKernel jit_small;  // 2-row variant for batches of small partitions (compiled on first use)
    bool jit_small_tried = false;
    // ungated variants, used once a run showed the stage-1 gate passing almost
    // every warp iteration (its tests never fail inside these partitions)
    JitKernel jit_nogate, jit_small_nogate;
    bool jit_nogate_tried = false, jit_small_nogate_tried = false;
    JitKernel jit_packed;  // 2-row variant taking packed items: batches of tiny partitions
    bool jit_packed_tried = false;
    bool gate_off = false;
    long long last_rows = 0;  // output size of the previous run: sizes the next buffer
    std::map<int, long long> rows_by_items;  // output size of the last run over that many items (guarded by ranges_mu)
    long long last_surv = 0;  // survivors of the previous run's largest range: sizes the deferred-verification buffer
    double surv_rate = -1.0;  // survivors per work item in the previous run (-1: none yet)
    // item ranges that fit the survivor buffer in earlier runs, keyed on a hash of the
    // run's work items, its tuple count and kernel variant: a run over the same items
    // (a repeated batch, or one of the size classes of a mixed batch) replays them
    // instead of re-learning where the survivors concentrate (each range that
    // overflows is re-run).  At most 8 plans are kept.
    std::map<uint64_t, RangePlan> range_plans;
    std::mutex ranges_mu;  // guards range_plans (a program may be run from several threads)
    uint64_t shape_key = 0;  // hash of the program arrays + relation shape (rb_ctx::learned)
    // the stage-1 gate's inputs (rb::choose_gate), kept for the runs that know
    // a slot holds for all their pairs (rb_run_parts: a branch's equality root)
    std::vector<uint64_t> gate_need;
    std::vector<int> gate_first_pos;
    std::vector<int> gate_cls;  // feature class of every slot (0 eq / const, 1 + f token, 1 + MAX_TOK + f string)
};



struct rb_result {
    rb_ctx* ctx = nullptr;
    long long cap = 0;
    int64_t count = 0;
    int32_t* d_t = nullptr;
    int32_t* d_s = nullptr;
    int32_t* d_r = nullptr;
    int32_t* d_p = nullptr;  // batched runs: partition index per row
    cudaStream_t stream = nullptr;
    rb_stats stats{};
};


namespace rb {

// one partition / cross block of a run.  split < 0: a partition over
// positions [base, base+n); else a cross block, left = [base, base+split),
// right = [rbase, rbase + n - split) (rbase = base + split when contiguous)
struct Part {
    int64_t base, n, split, rbase;
};

// the run orchestration (rb_api.cu): refs are host tuple ids, or device ids
// when refs_on_device; parts index positions of refs
int run(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, int64_t total, const std::vector<Part>& parts,
        int64_t row_lo, int64_t row_hi, uint32_t flags, bool want_parts, rb_result** out,
        bool refs_on_device = false, uint64_t implied = 0);
// one result from two (rows of `a`, then of `b`); part indices remapped
// through ia / ib when `want_parts`; consumes a and b
int merge_results(rb_ctx* c, rb_result* a, rb_result* b, bool want_parts, const std::vector<int32_t>& ia,
                  const std::vector<int32_t>& ib, rb_result** out);
// the stage-1 gate of a filter plan (rb_api.cu); `implied`: slots true for every pair of the run
void choose_gate(FilterPlan& F, const std::vector<uint64_t>& need, const std::vector<int>& first_pos, int n_slots,
                 uint64_t implied, const std::vector<int>* cls = nullptr);

// with RB_MIXED=1, a batch mixing large and small units runs as two runs --
// the units with a full item of rows on both sides on the large-partition
// kernel, the rest on the small / packed variant -- and one merged result
// (part indices global); otherwise one run
int run_mixed(rb_ctx* c, rb_rel* rel, rb_prog* P, const int32_t* refs, int64_t total, const std::vector<Part>& parts,
              uint32_t flags, bool want_parts, rb_result** out, bool refs_on_device = false, uint64_t implied = 0);

}  // namespace rb
