/*
 * rbgpu.h -- C ABI of the B200 rule-evaluation engine (librbgpu.so).
 *
 * Replaces the hot path of the reference package `ruleblock`:
 *   run_partition  pkg/src/ruleblock/engine.py:619-646
 *   run_cross      pkg/src/ruleblock/engine.py:649-681 (+ _bipartite_patch 684-719)
 * together with the per-slot evaluators they compile
 *   (pkg/src/ruleblock/encode.py:191-324) and the numba kernels they call
 *   (pkg/src/ruleblock/_kernels.py:29-83).
 *
 * Everything above this ABI (rule parsing, planning, text folding and
 * tokenising, dictionary encoding, exact threshold tables) stays on the
 * host in Python; everything below it runs on one sm_100a GPU.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Host buffers passed in are read during
 *    the call and never retained.
 *  - Every function returns RB_OK (0) or a negative status; the message of
 *    the last failure on the calling thread is rb_last_error().
 *  - Handles are owned by the library and freed with their *_destroy.
 *  - One rb_ctx per (host thread, device); calls on one ctx are serialised
 *    by the caller.  There is no CPU fallback: without a usable device every
 *    entry point that needs one fails with RB_ERR_CUDA.
 */
#ifndef RBGPU_H
#define RBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mapped by the Python shim: INVALID/LIMIT -> ConfigError,
 * CUDA/OOM/INTERNAL -> RuleBlockError; engine.py:53-59, 240-245) */
#define RB_OK 0
#define RB_ERR_INVALID (-1)
#define RB_ERR_CUDA (-2)
#define RB_ERR_OOM (-3)
#define RB_ERR_LIMIT (-4)
#define RB_ERR_INTERNAL (-5)

/* column kinds -- relation-wide encodings (encode.py:58-175) */
#define RB_COL_CODES 0  /* int32 dictionary codes, <0 = never equal      */
#define RB_COL_MASK 1   /* uint8 per tuple: t.attr = const holds          */
#define RB_COL_TOKENS 2 /* CSR of sorted unique int32 token ids + missing */
#define RB_COL_CHARS 3  /* CSR of folded codepoints (u8 or u32) + missing */

/* slot kinds -- one per distinct predicate of the path (encode.py:291-324) */
#define RB_SLOT_EQ_CODE 0  /* lhs[t] >= 0 && lhs[t] == rhs[s]           */
#define RB_SLOT_EQ_CONST 1 /* mask[t]  (depends on t only)               */
#define RB_SLOT_JACCARD 2  /* token-set Jaccard >= delta                 */
#define RB_SLOT_EXACT 3    /* token sets equal and not both empty        */
#define RB_SLOT_EDIT 4     /* 1 - lev/max(len) >= delta                  */

#define RB_SLOT_PREFILTER 1u /* engine form with the float length prefilter */

/* run flags (EngineConfig.symmetric_mode / enumerate_witnesses, engine.py:41-51) */
#define RB_SYMMETRIC 1u
#define RB_ENUMERATE 2u
#define RB_STATS 4u /* count per-slot exact evaluations */
/* slot_evals = first-touch evaluations of every slot over EVERY pair of the
 * run under evaluate_pair semantics (engine.py:93-132, 122-128; the counts
 * SURVEY 8d's E_s names), from a separate exact pass over all pairs -- not
 * only the survivors of the pair filter.  Slower: opt-in. */
#define RB_EXACT_STATS 8u

#define RB_MAX_SLOTS 64
#define RB_MAX_CHECKPOINTS 64

/* One predicate slot.  tab0/tab1 index the program's int32 table buffer:
 *   EDIT:    tab0 = maxgap[0..len0), tab1 = maxd[0..len1)
 *   JACCARD: tab0 = minsmall[0..len0), tab1 = mink[0..len1)
 * delta is the predicate threshold (used by the CPU oracle, not the GPU). */
typedef struct rb_slot {
    int32_t kind;
    int32_t lhs; /* column read on the t side */
    int32_t rhs; /* column read on the s side */
    int32_t flags;
    int64_t tab0;
    int64_t tab1;
    int32_t len0;
    int32_t len1;
    double delta;
} rb_slot;

typedef struct rb_stats {
    int64_t comparisons; /* pairs evaluated: BlockStats.comparisons (engine.py:486) */
    int64_t survivors;   /* pairs that needed the exact interpreter            */
    int64_t emitted;     /* rows produced                                       */
    double kernel_ms;    /* device time of the evaluation kernels (CUDA events) */
    int32_t launches;    /* kernels launched by the run                         */
    int32_t retries;     /* output-overflow re-runs                              */
    int64_t slot_evals[RB_MAX_SLOTS]; /* exact evaluations per slot (RB_STATS) */
    int32_t specialized;   /* 1: the NVRTC-specialised kernel ran, 0: the generic one */
    int32_t reserved;
    double jit_compile_ms; /* one-off specialisation cost of this program's kernel */
    double pair_ms;        /* device time of the pair (phase-1) kernel alone; kernel_ms adds
                              the deferred verification kernel                          */
} rb_stats;

typedef struct rb_ctx rb_ctx;
typedef struct rb_rel rb_rel;
typedef struct rb_prog rb_prog;
typedef struct rb_result rb_result;

const char* rb_last_error(void);
const char* rb_version(void);

/* context: device + stream.  rb_ctx_set_stream makes the engine launch on a
 * caller-owned cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream). */
int rb_ctx_create(int device, rb_ctx** out);
int rb_ctx_set_stream(rb_ctx* ctx, void* cuda_stream);
int rb_ctx_destroy(rb_ctx* ctx);

/* relation: uploaded once, shared by every program/partition over it
 * (the role of EncodedRelation shared copy-on-write, pipeline.py:273-307),
 * from any context of the same device (programs and partition sets of a
 * sibling context wait for its uploads; add no columns while they run) */
int rb_relation_create(rb_ctx* ctx, int64_t n_tuples, rb_rel** out);
int rb_relation_add_codes(rb_rel* rel, const int32_t* codes, int32_t* col);
int rb_relation_add_mask(rb_rel* rel, const uint8_t* mask, int32_t* col);
int rb_relation_add_tokens(rb_rel* rel, const int64_t* offsets, const int32_t* ids, const uint8_t* missing,
                           int32_t* col);
int rb_relation_add_chars(rb_rel* rel, const int64_t* offsets, const void* chars, int32_t width,
                          const uint8_t* missing, int32_t* col);
int rb_relation_destroy(rb_rel* rel);

/* program: the compiled ExecutionPath (planner/plan.py:232-300).
 * op[k] = 0 EvalPredicate(slot[k], fail[k]) | 1 Checkpoint(rule[k]),
 * rule[k] indexing path.rule_ids (rule-set order). */
int rb_program_create(rb_ctx* ctx, rb_rel* rel, const int32_t* op, const int32_t* slot, const int32_t* fail,
                      const int32_t* rule, int32_t n_ins, const rb_slot* slots, int32_t n_slots,
                      const int32_t* tables, int64_t n_tables, rb_prog** out);
int rb_program_destroy(rb_prog* prog);
/* how the pair kernel of this program was built: 1 specialised by NVRTC, 0
 * generic; *log receives the compiler log or why specialisation was skipped
 * (valid until the program is destroyed). */
int rb_program_kernel_info(const rb_prog* prog, int32_t* specialized, double* compile_ms, const char** log);

/* run_partition: all pairs of refs[0..n) (i<j symmetric, i!=j otherwise);
 * t = refs[i] (the lower position), s = refs[j].  refs == NULL means the
 * identity partition 0..n-1.  Rows are (t, s, rule) with t<s by tid in
 * symmetric mode.  rb_run_partition_rows restricts the outer position to
 * [row_lo, row_hi) -- the unit of multi-GPU sharding. */
int rb_run_partition(rb_ctx* ctx, rb_rel* rel, rb_prog* prog, const int32_t* refs, int64_t n, uint32_t flags,
                     rb_result** out);
int rb_run_partition_rows(rb_ctx* ctx, rb_rel* rel, rb_prog* prog, const int32_t* refs, int64_t n,
                          int64_t row_lo, int64_t row_hi, uint32_t flags, rb_result** out);
/* run_cross: every (t in left, s in right); t is always the left tuple. */
int rb_run_cross(rb_ctx* ctx, rb_rel* rel, rb_prog* prog, const int32_t* left, int64_t nl, const int32_t* right,
                 int64_t nr, uint32_t flags, rb_result** out);

/* batched run: n_parts partitions laid out back to back in refs, part k =
 * refs[offsets[k] .. offsets[k+1]); splits[k] < 0 (or splits == NULL)
 * evaluates part k as a partition (run_partition semantics), splits[k] >= 0
 * as a cross run with left = its first splits[k] refs.  One launch for the
 * whole batch; rb_result_copy_parts returns each row's part index.  This is
 * the many-small-partitions shape of the reference pipeline
 * (pipeline.py:177-209 running run_partition per task). */
int rb_run_batch(rb_ctx* ctx, rb_rel* rel, rb_prog* prog, const int32_t* refs, const int64_t* offsets,
                 const int64_t* splits, int32_t n_parts, uint32_t flags, rb_result** out);

/* rb_run_batch where the caller knows path slots that hold for every pair of
 * every part (bit s of implied_slots: e.g. the equality root every block of
 * a blocked run shares): the batch runs a filter plan regated without them
 * (their tests cannot fail there).  The filter only prunes, so results are
 * exact even if an implied slot were false for some pair. */
int rb_run_batch_implied(rb_ctx* ctx, rb_rel* rel, rb_prog* prog, const int32_t* refs, const int64_t* offsets,
                         const int64_t* splits, int32_t n_parts, uint32_t flags, uint64_t implied_slots,
                         rb_result** out);

int rb_result_count(const rb_result* res, int64_t* rows);
int rb_result_copy(const rb_result* res, int32_t* t, int32_t* s, int32_t* rule);
int rb_result_copy_parts(const rb_result* res, int32_t* part);
int rb_result_stats(const rb_result* res, rb_stats* out);
/* device pointers of the result rows (count rows each, on the result's
 * device, ordered on its stream), valid until rb_result_destroy: the rows
 * can be gathered across GPUs (NCCL) without a host round trip.  part is
 * NULL unless the result is batched. */
int rb_result_device(const rb_result* res, const int32_t** t, const int32_t** s, const int32_t** rule,
                     const int32_t** part);
int rb_result_destroy(rb_result* res);

/* ---- the callers either side of the path, on the device ------------------
 * Plan-derived partitioning (partitioning.py:93-131 iter_partitions,
 * 144-157 sibling_pull_pairs; the device half of pipeline_run,
 * pipeline.py:245-433).  Branch b keys tuple tid with keys[b*n + tid]
 * (int64): equal keys form one group, groups come in ascending key order,
 * tuple ids ascend inside a group -- the reference's sorted(groups) when the
 * keys are ranks of its key strings.  A group of more than
 * max_partition_size tuples is dealt round-robin into ceil(|g| / max)
 * sibling partitions (refs[sub::n_parts]); with RB_PART_PULLS every sibling
 * pair (i < j) also becomes a cross block, left = sibling i.  The sorted
 * tuple ids stay on the device as the refs of rb_run_parts.
 * rb_partition_codes keys branch b on the relation's CODES column cols[b]
 * (negative codes = missing: one group, ordered first), with no upload. */
#define RB_PART_PULLS 1u       /* PipelineConfig.enable_pulls               */
#define RB_PART_KEYS_DEVICE 2u /* keys is a device pointer                  */
typedef struct rb_parts rb_parts;
int rb_partition(rb_ctx* ctx, rb_rel* rel, const int64_t* keys, const int32_t* branch_ids, int32_t n_branches,
                 int64_t max_partition_size, uint32_t flags, rb_parts** out);
int rb_partition_codes(rb_ctx* ctx, rb_rel* rel, const int32_t* cols, const int32_t* branch_ids, int32_t n_branches,
                       int64_t max_partition_size, uint32_t flags, rb_parts** out);
int rb_parts_info(const rb_parts* parts, int64_t* n_partitions, int64_t* n_pulls, int64_t* n_refs, int64_t* n_groups);
/* host copies (any pointer may be NULL): refs[n_refs]; per partition, then
 * per pull: base position in refs, size, split (-1 partition, else |left|),
 * rbase (right side start of a pull, else -1), branch id, sibling group
 * (0 none, else 1-based in order of appearance) */
int rb_parts_copy(const rb_parts* parts, int32_t* refs, int64_t* base, int64_t* size, int64_t* split, int64_t* rbase,
                  int32_t* branch, int32_t* sibling);
/* The path slot each branch's key implies (root_slot[b], branch positions as
 * given to rb_partition; -1 for none): a branch keyed on the canonical value
 * of a same-attribute equality root holds that slot for every pair of its
 * groups except the missing-value group (rb_partition_codes: key 0;
 * rb_partition: the first group, unless first_missing[b] == 0 -- may be
 * NULL).  rb_run_parts then evaluates the branch holding most of the pairs
 * with a filter plan regated without that slot (its test cannot fail there). */
int rb_parts_set_roots(rb_parts* parts, const int32_t* root_slot, const uint8_t* first_missing, int32_t n_branches);
int rb_parts_destroy(rb_parts* parts);
/* One batched run over every partition with pairs and every pull of
 * `parts` that rank `rank` of `world` owns: static longest-processing-time
 * placement on pair counts, identical on every rank (world 1: all). */
int rb_run_parts(rb_ctx* ctx, rb_rel* rel, rb_prog* prog, const rb_parts* parts, int32_t rank, int32_t world,
                 uint32_t flags, rb_result** out);
/* Collect (pipeline.py:407-421): the rows sorted by (t, s), one row per
 * (t, s) carrying its smallest rule index (rule-set order), in place.  The
 * rows' part indices are dropped. */
int rb_result_collect(rb_result* res, int64_t n_tuples, int32_t n_rules);
/* the same over caller-owned device arrays (e.g. rows exchanged between
 * GPUs), ordered on the context's stream: out_* hold >= count rows */
int rb_collect_device(rb_ctx* ctx, const int32_t* t, const int32_t* s, const int32_t* rule, int64_t count,
                      int64_t n_tuples, int32_t n_rules, int32_t* out_t, int32_t* out_s, int32_t* out_rule,
                      int64_t* out_count);

#ifdef __cplusplus
}
#endif
#endif /* RBGPU_H */
