/* pbkv.h -- C ABI of the B200-native PBKV scoring / victim-selection hot path.
 *
 * Drop-in boundary for the reference policy interface in
 * /root/reference/proj/include/flowkv/ (a header-only C++20 library with no
 * virtual interface: policies are inline free functions chosen at the call
 * sites simulator.hpp:434, :464, :618, :635-637, :657).  Each entry point below
 * names the reference function it replaces.  The C++ shim that re-exposes the
 * exact reference signatures on top of this ABI is include/pbkv/flowkv_gpu.hpp;
 * INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *  - Every function returns a pbkv_status.  On failure, pbkv_last_error(ctx)
 *    (or pbkv_last_error(NULL) for functions without a ctx) returns the
 *    message.  PBKV_EINVAL carries exactly the reference's
 *    flowkv::ValidationError message (errors.hpp:24-26), so the C++ shim can
 *    rethrow it unchanged.
 *  - Plain pointers and sizes only; every array argument is HOST memory unless
 *    the function name ends in _dev.
 *  - A context owns one CUDA stream and all of its device memory; contexts
 *    share nothing (one per simulator instance, scenario.hpp:291-301).
 *  - No CPU fallback: when no sm_100 device is present, pbkv_ctx_create
 *    fails with PBKV_ECUDA.
 */
#ifndef PBKV_H_
#define PBKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBKV_ABI_VERSION 2

typedef enum pbkv_status {
    PBKV_OK = 0,
    PBKV_EINVAL = 1, /* flowkv::ValidationError (message preserved) */
    PBKV_ECUDA = 2,  /* CUDA runtime / device failure, or no sm_100 device */
    PBKV_ENOMEM = 3, /* device or host allocation failed */
    PBKV_EARG = 4,   /* bad pointer / size / capacity at the ABI level */
} pbkv_status;

/* cache.hpp:19  enum class Tier { Device, Host, Absent } */
enum { PBKV_TIER_DEVICE = 0, PBKV_TIER_HOST = 1, PBKV_TIER_ABSENT = 2 };

/* policies.hpp:19  enum class EvictionPolicy { Lru, Lae, Hierarchical, KvFlow } */
enum { PBKV_POLICY_LRU = 0, PBKV_POLICY_LAE = 1, PBKV_POLICY_HE = 2, PBKV_POLICY_KVFLOW = 3 };

/* Which score the HE key uses (SURVEY.md §7 hard part 5):
 *  CACHED    -- the mirrored CacheTree::Node::score (cache.hpp:61), exactly
 *               what select_victims_hierarchical reads (policies.hpp:113);
 *  RECOMPUTE -- Eq. 2 recomputed on the device from the resident forecasts
 *               for every node in the same launch sequence (the north_star
 *               "score all, then select" pipeline; equal to CACHED in the
 *               simulator). */
enum { PBKV_SCORE_CACHED = 0, PBKV_SCORE_RECOMPUTE = 1 };

typedef struct pbkv_ctx pbkv_ctx;   /* device-side mirror + forecasts + scratch */
typedef struct pbkv_tree pbkv_tree; /* host-side radix-tree mirror (RadixMirror) */

typedef struct pbkv_cfg {
    int device;        /* CUDA ordinal */
    int k;             /* ScoreParams::k      (scoring.hpp:17), >= 1 */
    double gamma;      /* ScoreParams::gamma  (scoring.hpp:18), in (0,1) */
    int num_agents;    /* A; forecasts have A+1 outcomes (forecast.hpp:46) */
} pbkv_cfg;

/* Struct-of-arrays view of a CacheTree (read-side fields, cache.hpp:54-69).
 * Node ids index every per-node array; id 0 is the root.  Access entries are
 * a CSR: node i owns entries [acc_off[i], acc_off[i+1]), sorted by ascending
 * WorkflowId (the std::map order of Node::access, cache.hpp:64). */
typedef struct pbkv_tree_soa {
    int64_t n_nodes;
    int64_t n_entries;
    int32_t* parent;          /* [n] -1 for the root */
    int32_t* len;             /* [n] tokens.size() */
    uint8_t* tier;            /* [n] PBKV_TIER_* */
    uint8_t* retired;         /* [n] 0/1 */
    uint64_t* last_access;    /* [n] < 2^63 */
    int32_t* ever_tagged;     /* [n] */
    double* score;            /* [n] cached score (may be NULL -> 0.0) */
    int32_t* device_children; /* [n] (export only; may be NULL) */
    int32_t* depth;           /* [n] root = 0 (may be NULL on input -> derived) */
    int64_t* acc_off;         /* [n+1] */
    int64_t* acc_wf;          /* [E] WorkflowId */
    uint64_t* acc_bits;       /* [E] agent bit set (bit a <-> agent a, cache.hpp:489) */
    int64_t device_capacity;  /* cache.hpp:81 */
    int64_t device_used;      /* cache.hpp:83 */
    int64_t retired_device_tokens; /* cache.hpp:87 */
    int64_t host_capacity;
    int64_t host_used;
} pbkv_tree_soa;

/* PrefetchPlan (policies.hpp:170-177) scalars; the candidate and selected
 * lists are returned through caller arrays. */
typedef struct pbkv_prefetch_plan {
    int64_t budget_space;        /* Sa = device_free + retired_device_tokens (policies.hpp:185) */
    int64_t budget_bw;           /* Sbw = bandwidth * step_duration (policies.hpp:186) */
    int64_t displacement_budget; /* aggressive only: (int64)(rho * capacity) (policies.hpp:233) */
    int64_t selected_tokens;
    int64_t n_candidates;        /* total candidates (may exceed the caller's capacity) */
    int64_t n_selected;
} pbkv_prefetch_plan;

/* Synthetic workload parameters (generator in
 * paper_2605_06472_b200/csrc/host/ops.hpp). */
typedef struct pbkv_synth_params {
    int64_t n_nodes, n_workflows;
    int agents, group_size, shared_len, group_len, alphabet, max_rand_len;
    double retired_frac;
    int host_every;
    uint64_t seed;
} pbkv_synth_params;

/* ---- library --------------------------------------------------------------- */
int pbkv_abi_version(void);
const char* pbkv_last_error(const pbkv_ctx* ctx); /* NULL ctx -> thread-local last error */
int pbkv_device_count(int* out);                   /* sm_100 devices visible */

/* ---- context --------------------------------------------------------------- */
int pbkv_ctx_create(pbkv_ctx** out, const pbkv_cfg* cfg); /* validates k/gamma like ScoreParams::validate (scoring.hpp:20-23) */
int pbkv_ctx_destroy(pbkv_ctx* ctx);
int pbkv_ctx_sync(pbkv_ctx* ctx);                          /* cudaStreamSynchronize on the ctx stream */
int pbkv_ctx_stream(pbkv_ctx* ctx, void** stream_out);     /* the ctx's cudaStream_t */
/* Per-stage device time of the most recent call, milliseconds (CUDA events on
 * the ctx stream): [0]=score [1]=keys+eff [2]=cut/sort [3]=prefetch [4]=total. */
int pbkv_ctx_timings(pbkv_ctx* ctx, float* ms5);
int pbkv_ctx_set_timing(pbkv_ctx* ctx, int enabled);
/* Device time of the dominant kernels of the most recent timed selection
 * (milliseconds, CUDA events on the ctx stream): [0] the light Eq. 2 + key
 * pass (score_light_kernel), [1] the persistent selection kernel. */
/* Orders the context's stream after all work enqueued so far on `stream` (a
 * cudaStream_t; NULL = the legacy default stream), without a host
 * synchronisation: callers that produce device inputs on their own stream
 * (e.g. PyTorch's current stream) call this before passing them. */
int pbkv_ctx_wait_stream(pbkv_ctx* ctx, void* stream);
int pbkv_ctx_kernel_timings(pbkv_ctx* ctx, float* ms2);
/* %globaltimer stamps (ns) taken by the selection kernel at its phase
 * boundaries during the most recent selection (diagnostics). */
int pbkv_ctx_phase_times(pbkv_ctx* ctx, uint64_t* ns, int cap, int* n);
/* Cumulative launch counts: pbkv's own kernels, and CUB library calls. */
int pbkv_ctx_launches(pbkv_ctx* ctx, int64_t* kernels, int64_t* lib_calls);
/* Heavy-node deferral in RECOMPUTE decisions: enable/disable,
 * and how many decisions took the fast path (placed from score intervals)
 * vs the exact-chain path.  Results are identical either way. */
int pbkv_ctx_set_defer(pbkv_ctx* ctx, int enabled);
int pbkv_ctx_defer_stats(pbkv_ctx* ctx, int64_t* fast, int64_t* slow);

/* ---- device mirror of the tree --------------------------------------------- */
/* Full upload of a CacheTree snapshot (SURVEY.md §8(b) pbkv_mirror_full). */
int pbkv_mirror_full(pbkv_ctx* ctx, const pbkv_tree_soa* soa);

/* One node of an incremental mirror update (SURVEY.md §8(b) pbkv_mirror_delta):
 * the node's CURRENT read-side fields (cache.hpp:54-69) after whatever
 * CacheTree mutation touched it -- match_prefix / insert_suffix / split
 * (cache.hpp:121-219, :531-569), on_workflow_terminated (:224-250),
 * demote / promote / drop (:254-301), set_score (:320-325).  Its access
 * entries are acc_wf / acc_bits[acc_begin, acc_end) of the batch, ascending
 * WorkflowId (the std::map order of Node::access, cache.hpp:64); they replace
 * the node's previous entries.  A record whose id equals the mirror's node
 * count appends a node (node ids stay dense, as CacheTree's do).
 * depth is the node's depth (root = 0).  split() moves a whole subtree one
 * level down: a batch that changes a node's depth must carry every node of
 * its subtree (include/pbkv/tracked_tree.hpp does this). */
typedef struct pbkv_node_delta {
    int32_t id;
    int32_t parent;      /* -1 only for the root */
    int32_t len;         /* tokens.size() */
    int32_t ever_tagged;
    int32_t depth;
    uint8_t tier;        /* PBKV_TIER_* */
    uint8_t retired;     /* 0/1 */
    uint8_t pad[2];
    uint64_t last_access; /* < 2^63 */
    double score;        /* cached score (cache.hpp:61) */
    int64_t acc_begin, acc_end;
} pbkv_node_delta;

/* CacheTree tier accounting (cache.hpp:81-87) after the batch. */
typedef struct pbkv_tree_totals {
    int64_t device_capacity, device_used, retired_device_tokens, host_capacity, host_used;
} pbkv_tree_totals;

/* Incremental upload: applies n node records in one pinned H2D copy and one
 * kernel on the context stream (asynchronous; later calls on the context are
 * ordered after it).  Records are applied in batch order; a node may appear
 * more than once (the last record wins).  totals may be NULL (unchanged). */
int pbkv_mirror_delta(pbkv_ctx* ctx, const pbkv_node_delta* nodes, int64_t n, const int64_t* acc_wf,
                      const uint64_t* acc_bits, const pbkv_tree_totals* totals);
/* Debug audit (the analogue of CacheTree::audit, cache.hpp:350-416): compares
 * every mirrored field of the device mirror against a full snapshot.
 * *mismatch = -1 when identical, else the smallest differing node id (or
 * n_nodes when only the node count / totals differ). */
int pbkv_mirror_verify(pbkv_ctx* ctx, const pbkv_tree_soa* soa, int64_t* mismatch);

/* Host trees (pbkv_tree: a flowkv::CacheTree with a change log,
 * include/pbkv/tracked_tree.hpp).  pbkv_mirror_tree uploads the whole tree;
 * pbkv_mirror_sync uploads only the nodes changed since this context last
 * mirrored the same tree (pbkv_mirror_delta), or the whole tree when the
 * context mirrors another tree or the change log no longer reaches back. */
int pbkv_mirror_tree(pbkv_ctx* ctx, pbkv_tree* tree);
int pbkv_mirror_sync(pbkv_ctx* ctx, pbkv_tree* tree);
/* Update the cached scores of `n` nodes (CacheTree::set_score, cache.hpp:320). */
int pbkv_mirror_set_scores(pbkv_ctx* ctx, const int32_t* ids, const double* scores, int64_t n);
int pbkv_mirror_node_count(pbkv_ctx* ctx, int64_t* n_nodes, int64_t* n_entries);

/* ---- forecasts (stage 1 output / stage 2 input) ---------------------------- */
/* Upload `n` Forecasts (forecast.hpp:19-42): p is n x horizon x outcomes
 * row-major.  Validated on the device exactly like the Forecast ctor
 * (entries >= -1e-12, each step sums to 1 within 1e-9); survival and the
 * gamma-weighted table gs[w][k] = gamma^k * s_w(k) are derived there.
 * Replaces the provider's std::map entry (simulator.hpp:433). */
int pbkv_forecast_put(pbkv_ctx* ctx, const int64_t* wf, int64_t n, int horizon, int outcomes,
                      const double* p);
/* pbkv_forecast_put without its synchronisation: the validation status
 * (forecast.hpp:25-34) is kept on the device and raised by the next call
 * that reads the status word (a score, select or plan call). */
int pbkv_forecast_put_async(pbkv_ctx* ctx, const int64_t* wf, int64_t n, int horizon, int outcomes, const double* p);
/* Drops forecasts (simulator.hpp:617 forecasts_.erase(w)). */
int pbkv_forecast_drop(pbkv_ctx* ctx, const int64_t* wf, int64_t n);
int pbkv_forecast_clear(pbkv_ctx* ctx);

/* ---- stage 1: the multi-step predictor ---------------
 * Replaces the predictor slot Simulator::predict (simulator.hpp:414-421): a
 * batched forward that emits K next-agent distributions over A agents + END
 * per workflow and stores them as that workflow's resident forecast (the
 * same rows pbkv_forecast_put writes; simulator.hpp:433).  The reference has
 * no code for this model; weights are the caller's.
 * Shapes: d must be 64 (one UMMA N tile), text_dim a multiple of 64. */
typedef struct pbkv_predictor_cfg {
    int num_agents; /* A, must equal the context's */
    int horizon;    /* K steps emitted per workflow (>= 1) */
    int dim;        /* d: agent embedding width (64) */
    int hidden;     /* h1: MLP hidden width (1..256) */
    int text_dim;   /* H: prefill hidden size (multiple of 64) */
    int max_prefix; /* longest accepted prefix (agents) */
} pbkv_predictor_cfg;

typedef struct pbkv_predictor_weights {
    const float* embed;      /* [A][d]     H^(0), learnable agent embeddings */
    const float* transition; /* [A][A]     row-normalised transition matrix */
    const float* sage1;      /* [d][2d]    W^(1) */
    const float* sage2;      /* [d][2d]    W^(2) */
    const float* query;      /* [d][d]     W_q */
    const uint16_t* text;    /* [d][H]     W_t (bf16 bit patterns) */
    const float* mlp1;       /* [h1][3d]   first MLP layer, input [h_cur|h_path|h_txt] */
    const float* mlp1_bias;  /* [h1] */
    const float* mlp2;       /* [K*(A+1)][h1] */
    const float* mlp2_bias;  /* [K*(A+1)] */
} pbkv_predictor_weights;

int pbkv_predictor_load(pbkv_ctx* ctx, const pbkv_predictor_cfg* cfg, const pbkv_predictor_weights* w);
/* Forward for n workflows: prefix CSR (prefix_off[n+1] into prefix; each
 * prefix is (v_1..v_t), t >= 1, current agent last), x = [n][H] bf16 post-norm
 * hidden states of the last prefill token (device memory when x_on_device,
 * else host).  probs_out (host, n x K x (A+1), nullable) receives the FP64
 * forecasts that were stored. */
int pbkv_predict(pbkv_ctx* ctx, const int64_t* wf, int64_t n, const int64_t* prefix_off, const int32_t* prefix,
                 const uint16_t* x, int x_on_device, double* probs_out);

/* ---- the reference predictors, batched and bit-exact ------------------------
 * CallGraph::true_kstep_marginals (callgraph.hpp:136-186), MarkovModel::predict
 * (predictor.hpp:79-118) and noisy_predict (predictor.hpp:25-35) propagate
 * alive mass over context states in std::map order.  The model is given as a
 * state table in that order (include/pbkv/flowkv_gpu.hpp builds it from a
 * CallGraph or a MarkovModel): rows[s] = the state's one-step distribution
 * over A agents + END, next[s][a] = the state reached by invoking agent a
 * (-1: none).  One thread per workflow replays the reference's loops in
 * binary64; the K-step forecasts become the workflows' resident forecasts. */
typedef struct pbkv_fmodel {
    int num_agents;       /* A, must equal the context's */
    int64_t n_states;
    const double* rows;   /* [n_states][A+1] */
    const int32_t* next;  /* [n_states][A] */
} pbkv_fmodel;

int pbkv_fmodel_load(pbkv_ctx* ctx, const pbkv_fmodel* model);
/* start_state[i]: table index of workflow i's current context; lambda < 0:
 * no noise, else noisy_predict(base, lambda).  probs_out (host, nullable):
 * n x horizon x (A+1). */
int pbkv_forecast_propagate(pbkv_ctx* ctx, const int64_t* wf, int64_t n, const int32_t* start_state, int horizon,
                            double lambda, double* probs_out);

/* ---- stage 2: Score(c), Eq. 2 ---------------------------------------------- */
/* multi_step_score(node_terms(...)) (scoring.hpp:49-75) for every node; nodes
 * without access entries score +0.0.  Raises EINVAL "missing forecast for
 * active workflow <w>" if any tagged workflow has no forecast.  scores_out
 * (host, n_nodes doubles) may be NULL: the scores then only stay resident. */
int pbkv_score_all(pbkv_ctx* ctx, double* scores_out);
/* refresh_nodes (scoring.hpp:95-101) without the write-back: Eq. 2 for the
 * listed node ids, results in `out` (host). */
int pbkv_score_nodes(pbkv_ctx* ctx, const int32_t* ids, int64_t n, double* out);
/* single_step_value (scoring.hpp:41-45), Eq. 1, for the listed node ids. */
int pbkv_value_nodes(pbkv_ctx* ctx, const int32_t* ids, int64_t n, double* out);

/* ---- stage 3: victim selection --------------------------------------------- */
/* select_victims / select_victims_{lru,lae,hierarchical}
 * (policies.hpp:88-115, :155-168): victims in eviction order, bit-identical
 * to the reference's greedy frontier (policies.hpp:50-83).  `locked` is the
 * image of std::set<int> (any order, duplicates allowed).  If `cap` is
 * smaller than the victim count, PBKV_EARG is returned and *n_victims holds
 * the required size. */
int pbkv_select(pbkv_ctx* ctx, int policy, int score_mode, int64_t needed, const int32_t* locked,
                int64_t n_locked, int32_t* victims, int64_t cap, int64_t* n_victims, int64_t* freed,
                int* shortfall);
/* Same, but `locked`/`victims` are device pointers and the three scalars are
 * written to a device int64[3] {n_victims, freed, shortfall}; no host
 * synchronisation beyond the ones the cut needs.  For benchmarking the
 * HBM-resident pipeline. */
int pbkv_select_dev(pbkv_ctx* ctx, int policy, int score_mode, int64_t needed, const int32_t* locked_dev,
                    int64_t n_locked, int32_t* victims_dev, int64_t cap, int64_t* result_dev);
/* KVFlow key (policies.hpp:117-153) needs the static remaining sequences:
 * seq_off[n_wf+1] CSR over seq (agent ids) for workflow ids wf[n_wf]. */
int pbkv_set_remaining(pbkv_ctx* ctx, const int64_t* wf, int64_t n_wf, const int64_t* seq_off,
                       const int32_t* seq);

/* ---- node-set sharding across GPUs (config 4) ---------------
 * One context per rank over the rank's shard: the subtrees it owns plus a copy
 * of the spine (ancestors whose subtrees span ranks), local ids increasing in
 * global id.  The global order is the merge of the ranks' local orders plus
 * the spine records; host code exchanges the records (paper_2605_06472_b200/
 * shard.py over torch.distributed / NCCL).  Order key of a record: (w0, w1,
 * eff_gid, d) = the chain head's CandidateKey (policies.hpp:40-48), then the
 * distance below the head. */
typedef struct pbkv_cand {
    uint64_t w0, w1; /* packed CandidateKey of the chain head (cls, rank, last_access) */
    int32_t eff_gid; /* global id of the chain head (the key's id component) */
    int32_t gid;     /* global id of the victim */
    int32_t d;       /* depth(head) - depth(victim) */
    int32_t len;     /* tokens freed */
} pbkv_cand;

typedef struct pbkv_spine_info {
    uint64_t w0, w1;   /* max key over the rank's device descendants of the spine node */
    int32_t eff_gid;   /* its global id (-1 when has_eff == 0) */
    int32_t eff_depth; /* its depth */
    int32_t has_eff;   /* the rank has device descendants below this spine node */
    int32_t sublock;   /* a locked node lies below (or is) this spine node on this rank */
} pbkv_spine_info;

/* Global ids of the local nodes ([n_nodes], increasing) and the local ids of
 * the spine copies.  Kept across pbkv_mirror_* calls. */
int pbkv_shard_set(pbkv_ctx* ctx, const int32_t* global_ids, const int32_t* spine, int64_t n_spine);
/* Local selection (spine excluded) -> records of the local cut in local
 * order (device array, cap entries) and one pbkv_spine_info per spine node
 * (device).  result_dev = int64[3] {n_cand, freed_local, shortfall_local}. */
int pbkv_shard_select(pbkv_ctx* ctx, int policy, int score_mode, int64_t needed, const int32_t* locked_dev,
                      int64_t n_locked, pbkv_cand* cand_dev, int64_t cap, pbkv_spine_info* spine_dev,
                      int64_t* result_dev);
/* Eq. 2 products of the spine nodes' local entries (node-major, WorkflowId
 * order, K per entry) into out_dev; counts[j] = entries(spine j) * K (host). */
int pbkv_shard_spine_products(pbkv_ctx* ctx, double* out_dev, int64_t* counts);
/* Exact serial FP64 chains: out[b] = RN-sum of x_dev[off[b], off[b+1]) in
 * order (off, out on the host). */
int pbkv_chain_sum(pbkv_ctx* ctx, const double* x_dev, const int64_t* off, int n_seg, double* out);
/* Any-order sums of x_dev over pieces: out[2j] = sum, out[2j+1] = sum of
 * magnitudes over the pieces [pieces[2q], pieces[2q+1]) for q in
 * [out_off[j], out_off[j+1]) (host arrays; one synchronisation).  The
 * sharded decision's interval test of the spine scores. */
int pbkv_interval_sums(pbkv_ctx* ctx, const double* x_dev, const int64_t* pieces, const int64_t* out_off, int n_out,
                       double* out);
/* Merge of exchanged record runs (each sorted) and the cut at `needed`:
 * victims_dev receives global ids in eviction order; result_dev = int64[3]
 * {n_victims, freed, shortfall}. */
int pbkv_merge_cut(pbkv_ctx* ctx, const pbkv_cand* runs_dev, const int64_t* run_start, const int64_t* run_len,
                   int n_runs, int64_t needed, int32_t* victims_dev, int64_t* result_dev);

/* ---- stage 4: prefetch candidate ranking ----------------------------------- */
/* plan_conservative_prefetch (rho < 0) / plan_aggressive_prefetch (rho in
 * [0,1]) (policies.hpp:181-235).  Candidates (id, Eq.1 value) sorted by value
 * desc then id asc, and the greedy-with-skip selection; arrays may be NULL
 * when their capacity is 0.  n_candidates/n_selected report full sizes. */
int pbkv_plan_prefetch(pbkv_ctx* ctx, int64_t bandwidth, int step_duration, double rho, int32_t* cand_ids,
                       double* cand_values, int64_t cand_cap, int32_t* selected, int64_t sel_cap,
                       pbkv_prefetch_plan* plan);
/* The arrays of the context's last plan (held in pinned host memory until
 * the next plan): callers that size their arrays from plan->n_candidates /
 * n_selected call pbkv_plan_prefetch with zero capacities, then this. */
int pbkv_plan_fetch(pbkv_ctx* ctx, int32_t* cand_ids, double* cand_values, int64_t cand_cap, int32_t* selected,
                    int64_t sel_cap);

/* One conservative prefetch round (simulator.hpp:632-681) as one device
 * decision: for the plan's selected candidates in order, promoted[i] = 1 when
 * the reference would admit candidate i, and its victims (demoted first, in
 * order) are victims[victim_end[i-1] .. victim_end[i]).  device_free is the
 * tree's free device space before the round.  The caller applies the
 * demotions / promotions to its tree (make_room_on_host etc. as the
 * reference). */
int pbkv_prefetch_round(pbkv_ctx* ctx, const int32_t* selected, int64_t n_sel, int64_t device_free, int32_t* promoted,
                        int64_t* victim_end, int32_t* victims, int64_t cap, int64_t* n_victims);

/* ---- host trees: the reference flowkv::CacheTree (cache.hpp) with a change
 * log for incremental device sync (include/pbkv/tracked_tree.hpp).  For the
 * tests, the bench and Python callers; C++ callers use the class directly. */
int pbkv_tree_create(pbkv_tree** out, int64_t device_capacity, int64_t host_capacity);
int pbkv_tree_destroy(pbkv_tree* tree);
/* Applies an op stream (paper_2605_06472_b200/csrc/host/ops.hpp). */
int pbkv_tree_apply_ops(pbkv_tree* tree, const int64_t* words, int64_t n_words);
int pbkv_tree_synth(pbkv_tree* tree, const pbkv_synth_params* params);
/* Sizes and tier scalars, written into soa (pointers untouched). */
int pbkv_tree_shape(pbkv_tree* tree, pbkv_tree_soa* soa);
/* Fills every non-NULL array of soa (sized from pbkv_tree_shape). */
int pbkv_tree_export(pbkv_tree* tree, pbkv_tree_soa* soa);
int pbkv_tree_touched(pbkv_tree* tree, int64_t wf, int32_t* ids, int64_t cap, int64_t* n);
/* Current change-log position, and the distinct nodes changed since `pos`
 * (ascending, up to cap ids; ids may be NULL): *n_changed = their count, or
 * -1 when the log no longer reaches back to pos. */
int pbkv_tree_log(pbkv_tree* tree, int64_t pos, int64_t* end, int32_t* ids, int64_t cap, int64_t* n_changed);

#ifdef __cplusplus
}
#endif

#endif /* PBKV_H_ */
