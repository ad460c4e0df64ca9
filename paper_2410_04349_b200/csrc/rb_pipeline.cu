// rb_pipeline.cu -- the callers on either side of the evaluation path, on the
// device: plan-derived partitioning and the collect step.
//
//   partitioning  pkg/src/ruleblock/partitioning.py:93-131 (iter_partitions)
//                 and 144-157 (sibling_pull_pairs)
//   collect       pkg/src/ruleblock/pipeline.py:407-421
//
// Partitioning a branch is a stable radix sort of (key, tid) -- equal keys
// become one group with its tuple ids ascending, groups in key order -- a
// run-length pass for the group sizes, and a round-robin deal of every
// oversize group into contiguous sibling ranges.  The sorted tuple ids stay
// in HBM as the refs of the batched run; only the group sizes come back to
// the host, which lays out the partition list (the run's work items are
// built from it as for rb_run_batch).  Collect sorts the rows on one 64-bit
// key ((t, s) then the rule index) and keeps the first row of every (t, s):
// the earliest rule in rule-set order, as the reference's lexsort + keep.
// All of it is HBM streaming (sort passes): no tensor-core work here.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <chrono>
#include <map>
#include <numeric>
#include <queue>
#include <thread>

#include "rb_state.cuh"

using namespace rb;

struct rb_parts {
    rb_ctx* ctx = nullptr;
    int64_t n = 0;            // tuples per branch
    int32_t n_branches = 0;
    int32_t* d_refs = nullptr;  // n_branches * n tuple ids, branch by branch
    // the partitions with more than one tuple (in iter_partitions order), then
    // the pulls; every other position of a branch is a single-tuple partition
    // (no pairs), implied by the gaps -- rb_parts_copy lists them too
    std::vector<Part> parts;
    std::vector<int32_t> branch, sibling;
    std::vector<uint8_t> first_group;  // per entry: the branch's first key group (may be the missing-value group)
    std::vector<int32_t> branch_ids;  // branch id of position range [b*n, (b+1)*n)
    std::vector<int32_t> root_slot;   // per branch position: path slot its key implies (rb_parts_set_roots), -1 none
    std::vector<uint8_t> first_missing;  // per branch position: its first key group may be the missing-value group
    bool keyed_on_codes = false;
    int64_t n_kept = 0;               // entries of parts that are partitions
    int64_t n_partitions = 0, n_pulls = 0, n_groups = 0;
};

namespace {

constexpr int PB = 256;  // threads per block of the streaming kernels

// The host lists of the last destroyed partition set, handed to the next one:
// a 10M-tuple step builds ~1.6M entries (60+ MB) and fresh vectors cost their
// first-touch page faults every step; recycled ones keep their capacity.
std::mutex g_spare_mu;
std::vector<Part> g_spare_parts;
std::vector<int32_t> g_spare_branch, g_spare_sibling;
std::vector<uint8_t> g_spare_first;

void spare_lists_take(rb_parts* P) {
    std::lock_guard<std::mutex> lock(g_spare_mu);
    P->parts.swap(g_spare_parts);
    P->branch.swap(g_spare_branch);
    P->sibling.swap(g_spare_sibling);
    P->first_group.swap(g_spare_first);
    P->parts.clear();
    P->branch.clear();
    P->sibling.clear();
    P->first_group.clear();
}

void spare_lists_put(rb_parts* P) {
    std::lock_guard<std::mutex> lock(g_spare_mu);
    if (P->parts.capacity() <= g_spare_parts.capacity()) return;  // keep the larger set
    P->parts.swap(g_spare_parts);
    P->branch.swap(g_spare_branch);
    P->sibling.swap(g_spare_sibling);
    P->first_group.swap(g_spare_first);
}

double host_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int grid_for(int64_t n, int sms) {
    const int64_t g = (n + PB - 1) / PB;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 8));
}

int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b)) b++;
    return b;
}

// key of tuple tid: codes (int32, < 0 = missing: one group, ordered first)
// or int64 keys shifted by their minimum; ids 0..n-1 as the sort values
__global__ void keys_from_codes(const int32_t* __restrict__ codes, int64_t n, uint64_t* __restrict__ key,
                                int32_t* __restrict__ tid) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = __ldg(codes + i);
        key[i] = c < 0 ? 0ull : (uint64_t)c + 1ull;
        tid[i] = (int32_t)i;
    }
}

__global__ void keys_from_int64(const int64_t* __restrict__ in, int64_t n, int64_t lo, uint64_t* __restrict__ key,
                                int32_t* __restrict__ tid) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = (uint64_t)(in[i] - lo);
        tid[i] = (int32_t)i;
    }
}

__global__ void minmax_int64(const int64_t* __restrict__ in, int64_t n, unsigned long long* out) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        lo = min(lo, (long long)in[i]);
        hi = max(hi, (long long)in[i]);
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        // order-preserving map of signed to unsigned for the atomics
        atomicMin(out, (unsigned long long)lo ^ 0x8000000000000000ull);
        atomicMax(out + 1, (unsigned long long)hi ^ 0x8000000000000000ull);
    }
}

// Deal every oversize group round-robin into k contiguous siblings:
// element i of the group goes to sibling i % k at index i / k
// (refs[sub::n_parts], partitioning.py:121-131).  One CTA per group.
struct Deal {
    int64_t start, m, k;
};
__global__ void deal_siblings(const Deal* __restrict__ deals, const int32_t* __restrict__ src, int32_t* __restrict__ dst) {
    const Deal d = deals[blockIdx.x];
    const int64_t q = d.m / d.k, r = d.m % d.k;
    for (int64_t i = threadIdx.x; i < d.m; i += blockDim.x) {
        const int64_t sub = i % d.k, idx = i / d.k;
        const int64_t pos = sub * q + (sub < r ? sub : r) + idx;
        dst[d.start + pos] = src[d.start + i];
    }
}

// groups of more than one tuple: (run index, start, size) of each, compacted
// in order; the exclusive scan of the run lengths gives the starts
__global__ void flag_multi(const int32_t* __restrict__ counts, const int64_t* __restrict__ runs,
                           uint8_t* __restrict__ flag) {
    const int64_t k = *runs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = counts[i] > 1;
}
__global__ void gather_groups(const int32_t* __restrict__ sel, const int64_t* __restrict__ n_sel,
                              const int32_t* __restrict__ counts, const int64_t* __restrict__ starts,
                              int4* __restrict__ out) {
    const int64_t k = *n_sel;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t g = sel[i];
        out[i] = make_int4(g, (int)starts[g], counts[g], 0);  // positions < n <= INT32_MAX
    }
}

// collect: rows -> one sortable key (t, s, rule) when it fits 64 bits
__global__ void pack_rows(const int32_t* __restrict__ t, const int32_t* __restrict__ s, const int32_t* __restrict__ r,
                          int64_t k, int sb, int rb, uint64_t* __restrict__ key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        key[i] = ((((uint64_t)(uint32_t)t[i] << sb) | (uint64_t)(uint32_t)s[i]) << rb) | (uint64_t)(uint32_t)r[i];
}

// first row of every (t, s) run of the sorted keys
__global__ void flag_firsts(const uint64_t* __restrict__ key, int64_t k, int rb, uint8_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || (key[i] >> rb) != (key[i - 1] >> rb)) ? 1 : 0;
}

__global__ void unpack_rows(const uint64_t* __restrict__ key, const int64_t* __restrict__ count, int sb, int rb,
                            int32_t* __restrict__ t, int32_t* __restrict__ s, int32_t* __restrict__ r) {
    const int64_t k = *count;
    const uint64_t smask = (sb >= 64) ? ~0ull : ((1ull << sb) - 1), rmask = rb ? ((1ull << rb) - 1) : 0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x = key[i];
        r[i] = (int32_t)(x & rmask);
        s[i] = (int32_t)((x >> rb) & smask);
        t[i] = (int32_t)(x >> (rb + sb));
    }
}

// wide keys: (t, s) sorted with the rule as value; the smallest rule per run
__global__ void pack_ts(const int32_t* __restrict__ t, const int32_t* __restrict__ s, int64_t k,
                        uint64_t* __restrict__ key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        key[i] = ((uint64_t)(uint32_t)t[i] << 32) | (uint64_t)(uint32_t)s[i];
}

__global__ void min_rule_runs(const uint64_t* __restrict__ key, const int32_t* __restrict__ rule, int64_t k,
                              uint64_t* __restrict__ out_key, int32_t* __restrict__ out_rule, uint8_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const bool first = i == 0 || key[i] != key[i - 1];
        flag[i] = first ? 1 : 0;
        if (!first) continue;
        int32_t m = rule[i];
        for (int64_t j = i + 1; j < k && key[j] == key[i]; j++) m = min(m, rule[j]);
        out_key[i] = key[i];
        out_rule[i] = m;
    }
}

__global__ void unpack_ts(const uint64_t* __restrict__ key, const int32_t* __restrict__ rule,
                          const int64_t* __restrict__ count, int32_t* __restrict__ t, int32_t* __restrict__ s,
                          int32_t* __restrict__ r) {
    const int64_t k = *count;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        t[i] = (int32_t)(key[i] >> 32);
        s[i] = (int32_t)(key[i] & 0xffffffffull);
        r[i] = rule[i];
    }
}

// scoped stream-ordered scratch
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    template <typename T>
    cudaError_t get(T** p, size_t count) {
        void* q = nullptr;
        cudaError_t e = dev_alloc(&q, sizeof(T) * std::max<size_t>(count, 1), st);
        if (e == cudaSuccess) ptrs.push_back(q);
        *p = (T*)q;
        return e;
    }
    ~Scratch() {
        for (void* p : ptrs) dev_free(p, st);
    }
};

#define CKS(call)                                                                                   \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(e_ == cudaErrorMemoryAllocation ? RB_ERR_OOM : RB_ERR_CUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
    } while (0)

// One branch: sort, run-length groups, deal oversize groups; appends the
// branch's partitions of more than one tuple to P (positions offset by
// `base`), returns the sibling ranges of every oversize group for the pulls.
// Only those groups come back to the host: the group sizes are scanned and
// compacted on the device (a 10M-tuple branch of mostly unique keys has
// millions of single-tuple groups, which evaluate no pairs).
int partition_branch(rb_parts* P, const uint64_t* d_key_in, int32_t* d_tid_in, int key_bits, int64_t base,
                     int32_t branch, int64_t maxp, int& sibling_counter,
                     std::vector<std::vector<std::pair<int64_t, int64_t>>>& sib_ranges, std::vector<uint8_t>& sib_first) {
    rb_ctx* c = P->ctx;
    cudaStream_t st = c->stream;
    const int64_t n = P->n;
    Scratch S(st);
    uint64_t *key_out, *uniq;
    int32_t *counts, *tid_out, *sel;
    int64_t *d_runs, *starts, *d_sel;
    uint8_t* flag;
    int4* groups;
    CKS(S.get(&key_out, n));
    CKS(S.get(&tid_out, n));
    CKS(S.get(&uniq, n));
    CKS(S.get(&counts, n));
    CKS(S.get(&starts, n));
    CKS(S.get(&flag, n));
    CKS(S.get(&sel, n));
    CKS(S.get(&d_runs, 1));
    CKS(S.get(&d_sel, 1));
    size_t tb1 = 0, tb2 = 0, tb3 = 0, tb4 = 0;
    CKS(cub::DeviceRadixSort::SortPairs(nullptr, tb1, d_key_in, key_out, d_tid_in, tid_out, n, 0,
                                        std::max(1, key_bits), st));
    CKS(cub::DeviceRunLengthEncode::Encode(nullptr, tb2, key_out, uniq, counts, d_runs, n, st));
    CKS(cub::DeviceScan::ExclusiveSum(nullptr, tb3, counts, starts, n, st));
    CKS(cub::DeviceSelect::Flagged(nullptr, tb4, thrust::counting_iterator<int32_t>(0), flag, sel, d_sel, n, st));
    const size_t tbm = std::max(std::max(tb1, tb2), std::max(tb3, tb4));
    void* temp;
    CKS(S.get((char**)&temp, tbm));
    size_t tb = tbm;
    CKS(cub::DeviceRadixSort::SortPairs(temp, tb, d_key_in, key_out, d_tid_in, tid_out, n, 0,
                                        std::max(1, key_bits), st));
    tb = tbm;
    CKS(cub::DeviceRunLengthEncode::Encode(temp, tb, key_out, uniq, counts, d_runs, n, st));
    int64_t runs = 0;
    CKS(cudaMemcpyAsync(&runs, d_runs, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CKS(cudaStreamSynchronize(st));
    const int grid = grid_for(std::max<int64_t>(runs, 1), c->sm_count);
    tb = tbm;
    CKS(cub::DeviceScan::ExclusiveSum(temp, tb, counts, starts, runs, st));
    flag_multi<<<grid, PB, 0, st>>>(counts, d_runs, flag);
    CKS(cudaGetLastError());
    tb = tbm;
    CKS(cub::DeviceSelect::Flagged(temp, tb, thrust::counting_iterator<int32_t>(0), flag, sel, d_sel, runs, st));
    int64_t n_multi = 0;
    uint64_t first_key = 1;
    if (runs) CKS(cudaMemcpyAsync(&first_key, uniq, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CKS(cudaMemcpyAsync(&n_multi, d_sel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CKS(cudaStreamSynchronize(st));
    CKS(S.get(&groups, n_multi));
    // pinned, grown as needed: the D2H of a branch's groups at link speed (1.35M groups
    // for a 10M-tuple phone branch), no zero-filled host vector
    static thread_local int4* pinned = nullptr;
    static thread_local size_t pinned_cap = 0;
    if ((size_t)n_multi > pinned_cap) {
        if (pinned) cudaFreeHost(pinned);
        pinned_cap = std::max<size_t>((size_t)n_multi, 2 * pinned_cap);
        if (cudaMallocHost((void**)&pinned, sizeof(int4) * pinned_cap) != cudaSuccess) {
            cudaGetLastError();
            pinned = nullptr;
            pinned_cap = 0;
            return fail(RB_ERR_OOM, "pinned group buffer of %lld entries", (long long)n_multi);
        }
    }
    int4* h_groups = pinned;
    if (n_multi) {
        gather_groups<<<grid_for(n_multi, c->sm_count), PB, 0, st>>>(sel, d_sel, counts, starts, groups);
        CKS(cudaGetLastError());
        CKS(cudaMemcpyAsync(h_groups, groups, sizeof(int4) * n_multi, cudaMemcpyDeviceToHost, st));
    }
    int32_t* dst = P->d_refs + base;
    CKS(cudaMemcpyAsync(dst, tid_out, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
    CKS(cudaStreamSynchronize(st));
    std::vector<Deal> deals;
    int64_t extra = 0;  // sibling sub-partitions beyond one per group: pids of the single-tuple gaps follow
    auto room = [&](auto& v) {  // geometric growth ahead of this branch's groups
        const size_t need = v.size() + (size_t)n_multi;
        if (v.capacity() < need) v.reserve(std::max(need, 2 * v.capacity()));
    };
    room(P->parts);
    room(P->branch);
    room(P->sibling);
    room(P->first_group);

    for (int64_t g = 0; g < n_multi; g++) {
        const int64_t start = h_groups[g].y, m = h_groups[g].z;
        const uint8_t first = h_groups[g].x == 0;
        if (m <= maxp) {
            P->parts.push_back(Part{base + start, m, -1, 0});
            P->branch.push_back(branch);
            P->sibling.push_back(0);
            P->first_group.push_back(first);
        } else {
            const int64_t k = (m + maxp - 1) / maxp, q = m / k, r = m % k;
            deals.push_back(Deal{start, m, k});  // positions relative to the branch
            sibling_counter++;
            extra += k - 1;
            std::vector<std::pair<int64_t, int64_t>> ranges;
            int64_t at = base + start;
            for (int64_t sub = 0; sub < k; sub++) {
                const int64_t sz = q + (sub < r ? 1 : 0);
                P->parts.push_back(Part{at, sz, -1, 0});
                P->branch.push_back(branch);
                P->sibling.push_back(sibling_counter);
                P->first_group.push_back(first);
                ranges.push_back({at, sz});
                at += sz;
            }
            sib_ranges.push_back(std::move(ranges));
            sib_first.push_back(first);
        }
    }
    P->n_groups += runs;
    P->n_partitions += runs + extra;
    // codes keys: missing values (code < 0) carry key 0, present ones code + 1;
    // int64 keys: the first group is the smallest key, which may be the missing key
    P->first_missing.push_back(P->keyed_on_codes ? (runs && first_key == 0) : 1);
    if (!deals.empty()) {
        // the deal reads the sorted ids (tid_out) and rewrites the oversize groups of dst
        Deal* d_deals;
        CKS(S.get(&d_deals, deals.size()));
        CKS(cudaMemcpyAsync(d_deals, deals.data(), sizeof(Deal) * deals.size(), cudaMemcpyHostToDevice, st));
        deal_siblings<<<(unsigned)deals.size(), 512, 0, st>>>(d_deals, tid_out, dst);
        CKS(cudaGetLastError());
        CKS(cudaStreamSynchronize(st));  // deals is a host vector
    }
    return RB_OK;
}

int finish_pulls(rb_parts* P, bool pulls, const std::vector<std::vector<std::pair<int64_t, int64_t>>>& sib_ranges,
                 const std::vector<int32_t>& sib_branch, const std::vector<uint8_t>& sib_first) {
    P->n_kept = (int64_t)P->parts.size();
    if (!pulls) return RB_OK;
    int gid = 0;
    for (size_t g = 0; g < sib_ranges.size(); g++) {
        const auto& rg = sib_ranges[g];
        gid++;
        for (size_t i = 0; i < rg.size(); i++)
            for (size_t j = i + 1; j < rg.size(); j++) {
                P->parts.push_back(Part{rg[i].first, rg[i].second + rg[j].second, rg[i].second, rg[j].first});
                P->branch.push_back(sib_branch[g]);
                P->sibling.push_back(gid);
                P->first_group.push_back(sib_first[g]);
                P->n_pulls++;
            }
    }
    return RB_OK;
}

int partition_impl(rb_ctx* c, rb_rel* rel, const int32_t* cols, const int64_t* keys, const int32_t* branch_ids,
                   int32_t nb, int64_t maxp, uint32_t flags, rb_parts** out) {
    if (!c || !rel || !out || nb < 1 || (!cols && !keys)) return fail(RB_ERR_INVALID, "rb_partition: bad arguments");
    if (rel->ctx->device != c->device) return fail(RB_ERR_INVALID, "rb_partition: relation lives on another device");
    if (rel->ctx != c) CKS(cudaStreamSynchronize(rel->ctx->stream));
    if (maxp < 1) return fail(RB_ERR_INVALID, "max_partition_size must be >= 1");
    const int64_t n = rel->n;
    if ((int64_t)nb * n > INT32_MAX) return fail(RB_ERR_LIMIT, "%d branches x %lld tuples exceed the run's position range", nb, (long long)n);
    if (cols)
        for (int b = 0; b < nb; b++)
            if (cols[b] < 0 || cols[b] >= (int)rel->cols.size() || rel->cols[cols[b]].kind != RB_COL_CODES)
                return fail(RB_ERR_INVALID, "rb_partition_codes: column %d is not a codes column", cols[b]);
    CKS(cudaSetDevice(c->device));
    std::lock_guard<std::mutex> lock(c->mu);
    rb_parts* P = new (std::nothrow) rb_parts();
    if (!P) return fail(RB_ERR_OOM, "host allocation failed");
    spare_lists_take(P);
    P->ctx = c;
    P->n = n;
    P->n_branches = nb;
    P->keyed_on_codes = cols != nullptr;
    cudaStream_t st = c->stream;
    auto bail = [&](int rc) {
        dev_free(P->d_refs, st);
        delete P;
        return rc;
    };
    if (cudaError_t e = dev_alloc((void**)&P->d_refs, sizeof(int32_t) * std::max<int64_t>(1, nb * n), st))
        return bail(fail(RB_ERR_OOM, "partition refs: %s", cudaGetErrorString(e)));
    int sibling_counter = 0;
    std::vector<std::vector<std::pair<int64_t, int64_t>>> sib_ranges;
    std::vector<int32_t> sib_branch;
    std::vector<uint8_t> sib_first;
    {
        Scratch S(st);
        uint64_t* key;
        int32_t* tid;
        int64_t* hkeys_dev = nullptr;
        unsigned long long* mm = nullptr;
        if (S.get(&key, n) || S.get(&tid, n) || S.get(&mm, 2) || (keys && !(flags & RB_PART_KEYS_DEVICE) && S.get(&hkeys_dev, n)))
            return bail(fail(RB_ERR_OOM, "partition scratch for %lld tuples", (long long)n));
        const int grid = grid_for(n, c->sm_count);
        for (int b = 0; b < nb && n > 0; b++) {
            const int32_t bid = branch_ids ? branch_ids[b] : b;
            P->branch_ids.push_back(bid);
            int key_bits;
            if (cols) {
                keys_from_codes<<<grid, PB, 0, st>>>(rel->cols[cols[b]].codes, n, key, tid);
                key_bits = 32;
            } else {
                const int64_t* kin = keys + (size_t)b * n;
                if (!(flags & RB_PART_KEYS_DEVICE)) {
                    if (cudaError_t e = cudaMemcpyAsync(hkeys_dev, kin, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st))
                        return bail(fail(RB_ERR_CUDA, "keys upload: %s", cudaGetErrorString(e)));
                    kin = hkeys_dev;
                }
                unsigned long long init[2] = {~0ull, 0ull};
                unsigned long long res[2];
                if (cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st) != cudaSuccess)
                    return bail(fail(RB_ERR_CUDA, "keys min/max"));
                minmax_int64<<<grid, PB, 0, st>>>(kin, n, mm);
                if (cudaMemcpyAsync(res, mm, sizeof res, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                    cudaStreamSynchronize(st) != cudaSuccess)
                    return bail(fail(RB_ERR_CUDA, "keys min/max: %s", cudaGetErrorString(cudaGetLastError())));
                const int64_t lo = (int64_t)(res[0] ^ 0x8000000000000000ull), hi = (int64_t)(res[1] ^ 0x8000000000000000ull);
                keys_from_int64<<<grid, PB, 0, st>>>(kin, n, lo, key, tid);
                key_bits = bits_for((uint64_t)hi - (uint64_t)lo);
            }
            if (cudaError_t e = cudaGetLastError()) return bail(fail(RB_ERR_CUDA, "partition keys: %s", cudaGetErrorString(e)));
            const size_t before = sib_ranges.size();
            static const bool timing = std::getenv("RB_HOST_TIMING") != nullptr;
            const double t0 = timing ? host_ms() : 0.0;
            if (int rc = partition_branch(P, key, tid, key_bits, (int64_t)b * n, bid, maxp, sibling_counter, sib_ranges,
                                          sib_first))
                return bail(rc);
            if (timing)
                fprintf(stderr, "rb partition: branch %d: %.3f ms, %zu entries\n", bid, host_ms() - t0, P->parts.size());
            for (size_t g = before; g < sib_ranges.size(); g++) sib_branch.push_back(bid);
        }
    }
    finish_pulls(P, (flags & RB_PART_PULLS) != 0, sib_ranges, sib_branch, sib_first);
    *out = P;
    return RB_OK;
}

// rows (t, s, r)[k] -> sorted unique (t, s) with the smallest rule, into out_*; count in *out_k
int collect_impl(rb_ctx* c, const int32_t* t, const int32_t* s, const int32_t* r, int64_t k, int64_t n_tuples,
                 int32_t n_rules, int32_t* ot, int32_t* os, int32_t* orr, int64_t* out_k) {
    cudaStream_t st = c->stream;
    *out_k = 0;
    if (k <= 0) return RB_OK;
    const int sb = std::max(1, bits_for((uint64_t)std::max<int64_t>(1, n_tuples - 1)));
    const int rb = bits_for((uint64_t)std::max(0, n_rules - 1));
    const int grid = grid_for(k, c->sm_count);
    // the context's collect scratch (grow-only)
    CKS(c->col_k0.grow(sizeof(uint64_t) * k, st));
    CKS(c->col_k1.grow(sizeof(uint64_t) * k, st));
    CKS(c->col_flag.grow(k, st));
    CKS(c->col_cnt.grow(sizeof(int64_t), st));
    uint64_t* k0 = (uint64_t*)c->col_k0.p;
    uint64_t* k1 = (uint64_t*)c->col_k1.p;
    uint8_t* flag = (uint8_t*)c->col_flag.p;
    int64_t* d_cnt = (int64_t*)c->col_cnt.p;
    if (2 * sb + rb <= 64) {
        pack_rows<<<grid, PB, 0, st>>>(t, s, r, k, sb, rb, k0);
        CKS(cudaGetLastError());
        size_t tb1 = 0, tb2 = 0;
        CKS(cub::DeviceRadixSort::SortKeys(nullptr, tb1, k0, k1, k, 0, 2 * sb + rb, st));
        CKS(cub::DeviceSelect::Flagged(nullptr, tb2, k1, flag, k0, d_cnt, k, st));
        const size_t tbm = std::max(tb1, tb2);
        CKS(c->col_temp.grow(tbm, st));
        void* temp = c->col_temp.p;
        size_t tb = tbm;
        CKS(cub::DeviceRadixSort::SortKeys(temp, tb, k0, k1, k, 0, 2 * sb + rb, st));
        flag_firsts<<<grid, PB, 0, st>>>(k1, k, rb, flag);
        CKS(cudaGetLastError());
        tb = tbm;
        CKS(cub::DeviceSelect::Flagged(temp, tb, k1, flag, k0, d_cnt, k, st));
        unpack_rows<<<grid, PB, 0, st>>>(k0, d_cnt, sb, rb, ot, os, orr);
        CKS(cudaGetLastError());
    } else {
        CKS(c->col_r1.grow(sizeof(int32_t) * k, st));
        CKS(c->col_r2.grow(sizeof(int32_t) * k, st));
        int32_t* r1 = (int32_t*)c->col_r1.p;
        int32_t* r2 = (int32_t*)c->col_r2.p;
        pack_ts<<<grid, PB, 0, st>>>(t, s, k, k0);
        CKS(cudaGetLastError());
        size_t tb1 = 0, tb2 = 0;
        CKS(cub::DeviceRadixSort::SortPairs(nullptr, tb1, k0, k1, r, r1, k, 0, 64, st));
        CKS(cub::DeviceSelect::Flagged(nullptr, tb2, k0, flag, k1, d_cnt, k, st));
        const size_t tbm = std::max(tb1, tb2);
        CKS(c->col_temp.grow(tbm, st));
        void* temp = c->col_temp.p;
        size_t tb = tbm;
        CKS(cub::DeviceRadixSort::SortPairs(temp, tb, k0, k1, r, r1, k, 0, 64, st));
        min_rule_runs<<<grid, PB, 0, st>>>(k1, r1, k, k0, r2, flag);
        CKS(cudaGetLastError());
        tb = tbm;
        CKS(cub::DeviceSelect::Flagged(temp, tb, k0, flag, k1, d_cnt, k, st));
        tb = tbm;
        CKS(cub::DeviceSelect::Flagged(temp, tb, r2, flag, r1, d_cnt, k, st));
        unpack_ts<<<grid, PB, 0, st>>>(k1, r1, d_cnt, ot, os, orr);
        CKS(cudaGetLastError());
    }
    CKS(cudaMemcpyAsync(out_k, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CKS(cudaStreamSynchronize(st));
    return RB_OK;
}

int64_t pair_count(const Part& p, bool symmetric) {
    if (p.split >= 0) return p.split * (p.n - p.split);
    return symmetric ? p.n * (p.n - 1) / 2 : p.n * (p.n - 1);
}

}  // namespace

extern "C" {

int rb_partition(rb_ctx* c, rb_rel* rel, const int64_t* keys, const int32_t* branch_ids, int32_t n_branches,
                 int64_t max_partition_size, uint32_t flags, rb_parts** out) {
    if (!keys) return fail(RB_ERR_INVALID, "rb_partition: keys is NULL");
    return partition_impl(c, rel, nullptr, keys, branch_ids, n_branches, max_partition_size, flags, out);
}

int rb_partition_codes(rb_ctx* c, rb_rel* rel, const int32_t* cols, const int32_t* branch_ids, int32_t n_branches,
                       int64_t max_partition_size, uint32_t flags, rb_parts** out) {
    if (!cols) return fail(RB_ERR_INVALID, "rb_partition_codes: cols is NULL");
    return partition_impl(c, rel, cols, nullptr, branch_ids, n_branches, max_partition_size, flags, out);
}

int rb_parts_info(const rb_parts* p, int64_t* n_partitions, int64_t* n_pulls, int64_t* n_refs, int64_t* n_groups) {
    if (!p) return fail(RB_ERR_INVALID, "rb_parts_info: null parts");
    if (n_partitions) *n_partitions = p->n_partitions;
    if (n_pulls) *n_pulls = p->n_pulls;
    if (n_refs) *n_refs = (int64_t)p->n_branches * p->n;
    if (n_groups) *n_groups = p->n_groups;
    return RB_OK;
}

int rb_parts_copy(const rb_parts* p, int32_t* refs, int64_t* base, int64_t* size, int64_t* split, int64_t* rbase,
                  int32_t* branch, int32_t* sibling) {
    if (!p) return fail(RB_ERR_INVALID, "rb_parts_copy: null parts");
    rb_ctx* c = p->ctx;
    CKS(cudaSetDevice(c->device));
    if (refs && p->n) {
        CKS(cudaMemcpyAsync(refs, p->d_refs, sizeof(int32_t) * p->n_branches * p->n, cudaMemcpyDeviceToHost, c->stream));
        CKS(cudaStreamSynchronize(c->stream));
    }
    int64_t out = 0;
    auto put = [&](int64_t b0, int64_t sz, int64_t sp, int64_t rb, int32_t br, int32_t sib) {
        if (base) base[out] = b0;
        if (size) size[out] = sz;
        if (split) split[out] = sp;
        if (rbase) rbase[out] = rb;
        if (branch) branch[out] = br;
        if (sibling) sibling[out] = sib;
        out++;
    };
    // partitions in pid order: the kept ones, every uncovered position of a
    // branch in between as a single-tuple partition
    size_t k = 0;
    for (int32_t b = 0; b < (int32_t)p->branch_ids.size(); b++) {
        const int64_t lo = (int64_t)b * p->n, hi = lo + p->n;
        int64_t at = lo;
        while (true) {
            const bool more = k < (size_t)p->n_kept && p->parts[k].base < hi;
            const int64_t next = more ? p->parts[k].base : hi;
            for (; at < next; at++) put(at, 1, -1, -1, p->branch_ids[(size_t)b], 0);
            if (!more) break;
            const Part& q = p->parts[k];
            put(q.base, q.n, -1, -1, p->branch[k], p->sibling[k]);
            at = q.base + q.n;
            k++;
        }
    }
    for (; k < p->parts.size(); k++) {
        const Part& q = p->parts[k];
        put(q.base, q.n, q.split, q.split >= 0 ? q.rbase : -1, p->branch[k], p->sibling[k]);
    }
    if (out != p->n_partitions + p->n_pulls)
        return fail(RB_ERR_INTERNAL, "rb_parts_copy: %lld entries for %lld partitions + %lld pulls", (long long)out,
                    (long long)p->n_partitions, (long long)p->n_pulls);
    return RB_OK;
}

int rb_parts_set_roots(rb_parts* p, const int32_t* root_slot, const uint8_t* first_missing, int32_t n_branches) {
    if (!p || (n_branches && !root_slot)) return fail(RB_ERR_INVALID, "rb_parts_set_roots: null argument");
    if (n_branches != (int32_t)p->branch_ids.size() && !(p->n == 0 && p->branch_ids.empty()))
        return fail(RB_ERR_INVALID, "rb_parts_set_roots: %d slots for %zu branches", n_branches, p->branch_ids.size());
    p->root_slot.assign(root_slot, root_slot + p->branch_ids.size());
    if (first_missing && !p->keyed_on_codes)  // int64 keys: the caller knows whether key 0 is the missing key
        for (size_t b = 0; b < p->branch_ids.size() && b < p->first_missing.size(); b++)
            p->first_missing[b] = first_missing[b] ? 1 : 0;
    for (int32_t s : p->root_slot)
        if (s >= RB_MAX_SLOTS) return fail(RB_ERR_INVALID, "rb_parts_set_roots: slot %d", s);
    return RB_OK;
}

int rb_parts_destroy(rb_parts* p) {
    if (!p) return RB_OK;
    cudaSetDevice(p->ctx->device);
    {
        std::lock_guard<std::mutex> lock(p->ctx->mu);
        dev_free(p->d_refs, p->ctx->stream);
        cudaStreamSynchronize(p->ctx->stream);
    }
    spare_lists_put(p);
    delete p;
    return RB_OK;
}

int rb_run_parts(rb_ctx* c, rb_rel* rel, rb_prog* P, const rb_parts* parts, int32_t rank, int32_t world,
                 uint32_t flags, rb_result** out) {
    if (!parts || !c || !out) return fail(RB_ERR_INVALID, "rb_run_parts: null argument");
    if (parts->ctx != c) return fail(RB_ERR_INVALID, "rb_run_parts: parts belong to another context");
    if (world < 1 || rank < 0 || rank >= world) return fail(RB_ERR_INVALID, "rb_run_parts: rank %d of %d", rank, world);
    const bool sym = (flags & RB_SYMMETRIC) != 0;
    static const bool timing = std::getenv("RB_HOST_TIMING") != nullptr;
    double tm[8] = {timing ? host_ms() : 0.0};
    int ntm = 1;
    auto mark = [&]() {
        if (timing && ntm < 8) tm[ntm++] = host_ms();
    };
    auto report = [&](const char* what) {
        if (!timing) return;
        fprintf(stderr, "rb run_parts (%s):", what);
        for (int k = 1; k < ntm; k++) fprintf(stderr, " %.3f", tm[k] - tm[k - 1]);
        fprintf(stderr, " ms\n");
    };
    // Host lists of the run, kept per thread between calls: fresh multi-MB
    // vectors cost ~80 ms of first-touch page faults per 10M-tuple step while
    // the GPU waits for the first launch (clear() keeps the capacity)
    struct Lists {
        std::vector<int64_t> units, sel;
        std::vector<Part> mine, pi, po;
        std::vector<int32_t> ii, io;
        std::vector<int> sel_bpos;
        std::vector<int64_t> cost;
        std::vector<size_t> idx;
        std::vector<int32_t> owner;
    };
    static thread_local Lists LS;
    // the evaluated units: partitions with pairs, and the pulls
    std::vector<int64_t>& units = LS.units;
    units.clear();
    std::vector<Part>& mine = LS.mine;
    std::vector<int64_t>& sel = LS.sel;  // entry index of every unit of `mine`
    mine.clear();
    sel.clear();
    // one rank whose every entry has pairs (the usual case: partitions of one
    // tuple are not entries): the entries themselves are the units, no copies
    bool alias = world == 1;
    for (size_t k = 0; k < parts->parts.size() && alias; k++) alias = pair_count(parts->parts[k], sym) > 0;
    if (!alias) {
        units.reserve(parts->parts.size());
        for (size_t k = 0; k < parts->parts.size(); k++)
            if (pair_count(parts->parts[k], sym) > 0) units.push_back((int64_t)k);
    }
    if (alias) {
    } else if (world == 1) {
        mine.reserve(units.size());
        sel.reserve(units.size());
        for (int64_t k : units) {
            mine.push_back(parts->parts[(size_t)k]);
            sel.push_back(k);
        }
    } else {
        // static placement on pair counts, the same on every rank, in O(n): the
        // largest units (at most 4096 per rank) longest-processing-time first
        // to the least-loaded rank, then the rest -- in entry order -- dealt as
        // contiguous runs that fill every rank up to the mean load
        // (water-filling over a prefix sum).  A full LPT sort of 1.6M units
        // cost ~150 ms of host time per rank at 10M tuples.
        const size_t nu = units.size();
        std::vector<int64_t>& cost = LS.cost;
        cost.resize(nu);
        int64_t all = 0;
        for (size_t q = 0; q < nu; q++) {
            cost[q] = pair_count(parts->parts[(size_t)units[q]], sym);
            all += cost[q];
        }
        const size_t kbig = std::min(nu, (size_t)4096 * (size_t)world);
        std::vector<size_t>& idx = LS.idx;
        idx.resize(nu);
        std::iota(idx.begin(), idx.end(), 0);
        if (kbig < nu)
            std::nth_element(idx.begin(), idx.begin() + (long)kbig, idx.end(), [&](size_t a, size_t b) {
                return cost[a] != cost[b] ? cost[a] > cost[b] : a < b;
            });
        std::sort(idx.begin(), idx.begin() + (long)kbig, [&](size_t a, size_t b) {
            return cost[a] != cost[b] ? cost[a] > cost[b] : a < b;
        });
        std::vector<int32_t>& owner = LS.owner;
        owner.assign(nu, -1);
        std::vector<int64_t> load((size_t)world, 0);
        for (size_t q = 0; q < kbig; q++) {
            int32_t best = 0;
            for (int32_t w = 1; w < world; w++)
                if (load[(size_t)w] < load[(size_t)best]) best = w;
            owner[idx[q]] = best;
            load[(size_t)best] += cost[idx[q]];
        }
        // the rest in entry order: rank w takes the next run until it reaches the mean
        const int64_t target = (all + world - 1) / world;
        int32_t w = 0;
        for (size_t q = 0; q < nu; q++) {
            if (owner[q] >= 0) continue;
            while (w < world - 1 && load[(size_t)w] >= target) w++;
            owner[q] = w;
            load[(size_t)w] += cost[q];
        }
        for (size_t q = 0; q < nu; q++)
            if (owner[q] == rank) {
                mine.push_back(parts->parts[(size_t)units[q]]);
                sel.push_back(units[q]);
            }
    }
    mark();  // [1] units selected and placed
    const std::vector<Part>& M = alias ? parts->parts : mine;  // the units
    const size_t nsel = M.size();
    auto S = [&](size_t q) -> size_t { return alias ? q : (size_t)sel[q]; };  // entry index of unit q
    std::vector<int>& sel_bpos = LS.sel_bpos;  // branch position of every unit
    sel_bpos.assign(nsel, -1);
    {
        std::map<int32_t, int> pos_of;
        for (size_t b = 0; b < parts->branch_ids.size(); b++) pos_of.emplace(parts->branch_ids[b], (int)b);
        int32_t last_id = INT32_MIN;
        int last_pos = -1;
        for (size_t q = 0; q < nsel; q++) {
            const int32_t id = parts->branch[S(q)];
            if (id != last_id) {  // units come branch by branch
                auto it = pos_of.find(id);
                last_pos = it == pos_of.end() ? -1 : it->second;
                last_id = id;
            }
            sel_bpos[q] = last_pos;
        }
    }
    const int64_t total = (int64_t)parts->n_branches * parts->n;
    // Units of a branch keyed on an equality root hold that slot for all their
    // pairs (except the first key group, which may be the missing-value
    // group): the branch holding most of this rank's pairs runs with the slot
    // implied (rb::choose_gate), the other units as usual, one merged result.
    int64_t best = 0;
    int32_t best_b = -1;
    const char* implied_off = std::getenv("RB_IMPLIED_OFF");
    if (!parts->root_slot.empty() && !(implied_off && std::atoi(implied_off) != 0)) {
        std::vector<int64_t> by_b(parts->branch_ids.size(), 0);
        int64_t all = 0;
        for (size_t q = 0; q < nsel; q++) {
            const int64_t pc = pair_count(M[q], sym);
            all += pc;
            const int bpos = sel_bpos[q];
            if (bpos >= 0 && parts->root_slot[(size_t)bpos] >= 0 &&
                !(parts->first_group[S(q)] && parts->first_missing[(size_t)bpos]))
                by_b[(size_t)bpos] += pc;
        }
        for (size_t b = 0; b < by_b.size(); b++)
            if (by_b[b] > best) {
                best = by_b[b];
                best_b = (int32_t)b;
            }
        if (best * 2 < all) best_b = -1;  // not worth a second run
    }
    mark();  // [2] branch totals
    if (best_b < 0) {
        const int rc0 = run_mixed(c, rel, P, parts->d_refs, total, M, flags, false, out, true);
        mark();
        report("one run: select, branches, run");
        return rc0;
    }
    std::vector<Part>&pi = LS.pi, &po = LS.po;
    std::vector<int32_t>&ii = LS.ii, &io = LS.io;
    pi.clear();
    po.clear();
    ii.clear();
    io.clear();
    auto implied_unit = [&](size_t q) {
        return sel_bpos[q] == best_b && !(parts->first_group[S(q)] && parts->first_missing[(size_t)best_b]);
    };
    // the implied units now; the others (most of the list) by a host thread
    // while the implied run is on the GPU
    for (size_t q = 0; q < nsel; q++)
        if (implied_unit(q)) {
            pi.push_back(M[q]);
            ii.push_back((int32_t)q);
        }
    std::thread plain_lists([&]() {
        po.reserve(nsel - pi.size());
        io.reserve(nsel - pi.size());
        for (size_t q = 0; q < nsel; q++)
            if (!implied_unit(q)) {
                po.push_back(M[q]);
                io.push_back((int32_t)q);
            }
    });
    const uint64_t implied = 1ull << parts->root_slot[(size_t)best_b];
    rb_result* ri = nullptr;
    mark();  // [3] implied / plain split
    int rc = run_mixed(c, rel, P, parts->d_refs, total, pi, flags, false, &ri, true, implied);
    plain_lists.join();
    mark();  // [4] implied run
    if (rc != RB_OK || po.empty()) {
        *out = ri;
        return rc;
    }
    rb_result* ro = nullptr;
    rc = run_mixed(c, rel, P, parts->d_refs, total, po, flags, false, &ro, true);
    mark();  // [5] plain run
    if (rc != RB_OK) {
        rb_result_destroy(ri);
        return rc;
    }
    rc = merge_results(c, ro, ri, false, io, ii, out);
    mark();  // [6] merged
    report("select, branches, split, implied run, plain run, merge");
    return rc;
}

int rb_result_collect(rb_result* res, int64_t n_tuples, int32_t n_rules) {
    if (!res) return fail(RB_ERR_INVALID, "rb_result_collect: null result");
    if (n_tuples < 0 || n_tuples > INT32_MAX || n_rules < 1) return fail(RB_ERR_INVALID, "rb_result_collect: bad sizes");
    if (res->count == 0) return RB_OK;
    rb_ctx* c = res->ctx;
    CKS(cudaSetDevice(c->device));
    std::lock_guard<std::mutex> lock(c->mu);
    const int64_t k = res->count;
    // the collected rows go to the context's spare row buffers, which then
    // swap owners with the result's (no allocation per collect)
    for (int q = 0; q < 3; q++)
        if (cudaError_t e = c->col_out[q].grow(sizeof(int32_t) * k, c->stream))
            return fail(RB_ERR_OOM, "collect output of %lld rows: %s", (long long)k, cudaGetErrorString(e));
    int32_t* t = (int32_t*)c->col_out[0].p;
    int32_t* s = (int32_t*)c->col_out[1].p;
    int32_t* r = (int32_t*)c->col_out[2].p;
    int64_t kept = 0;
    if (int rc = collect_impl(c, res->d_t, res->d_s, res->d_r, k, n_tuples, n_rules, t, s, r, &kept)) return rc;
    int32_t* old[3] = {res->d_t, res->d_s, res->d_r};
    const long long old_cap = res->cap;
    res->d_t = t;
    res->d_s = s;
    res->d_r = r;
    res->cap = (long long)(std::min(std::min(c->col_out[0].bytes, c->col_out[1].bytes), c->col_out[2].bytes) /
                           sizeof(int32_t));
    for (int q = 0; q < 3; q++) {
        c->col_out[q].p = old[q];
        c->col_out[q].bytes = old[q] ? sizeof(int32_t) * (size_t)old_cap : 0;
    }
    dev_free(res->d_p, c->stream);
    res->d_p = nullptr;
    res->count = kept;
    return RB_OK;
}

int rb_collect_device(rb_ctx* c, const int32_t* t, const int32_t* s, const int32_t* r, int64_t count, int64_t n_tuples,
                      int32_t n_rules, int32_t* out_t, int32_t* out_s, int32_t* out_r, int64_t* out_count) {
    if (!c || !out_count || (count > 0 && (!t || !s || !r || !out_t || !out_s || !out_r)))
        return fail(RB_ERR_INVALID, "rb_collect_device: null argument");
    if (n_tuples < 0 || n_tuples > INT32_MAX || n_rules < 1) return fail(RB_ERR_INVALID, "rb_collect_device: bad sizes");
    CKS(cudaSetDevice(c->device));
    std::lock_guard<std::mutex> lock(c->mu);
    return collect_impl(c, t, s, r, count, n_tuples, n_rules, out_t, out_s, out_r, out_count);
}

}  // extern "C"
