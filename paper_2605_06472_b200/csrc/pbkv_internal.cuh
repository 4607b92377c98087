// Internal definitions shared by the pbkv CUDA translation units.
//
// Device data layout.  Per node (SoA, index = node id):
//   parent i32, len i32, flags u8 (bits 0-1 tier, bit 2 retired),
//   last_access u64, ever_tagged i32, score f64 (cached, cache.hpp:61),
//   depth i32, acc_rng u32x2 ({begin, end} of the node's entries in the pool)
// Per access entry (CSR, WorkflowId-ascending within a node, cache.hpp:64):
//   slot i32 (forecast slot of the WorkflowId), bits u64
// Per forecast slot: P f64[V1][K] (agent-major: one agent's K steps contiguous),
//   gs f64[K] = gamma^k * s(k),
//   state u8 (0 missing, 1 ok, 2 horizon < K).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/pbkv.h"

namespace pbkv {

constexpr std::uint8_t kFlagTierMask = 0x3;
constexpr std::uint8_t kFlagRetired = 0x4;
// spine node of a sharded tree (shard.cu): never a local candidate, key zeroed
// so that eff() of a spine node is the maximum over its local descendants only
constexpr std::uint8_t kFlagExcluded = 0x8;
// heavy node whose exact Eq. 2 chain is deferred during a decision (DESIGN.md
// §3.2): handled like an excluded node, then placed from its score interval
constexpr std::uint8_t kFlagDeferred = 0x10;
constexpr std::uint8_t kFlagOutOfOrder = kFlagExcluded | kFlagDeferred;
constexpr int kMediumMaxChain = 256;  // entries*K above this -> heavy (CTA) path

// first-error-wins device status (kernels never throw)
struct DevStatus {
    int code;        // 0 ok, else PBKV_E*
    int kind;        // which check failed (kErr*)
    long long node;  // smallest offending node id (atomicMin)
    long long aux;   // extra info (e.g. last_access for host ordering)
};
enum : int {
    kErrNone = 0,
    kErrMissingForecast = 1,
    kErrShortHorizon = 2,
    kErrLastAccessRange = 3,
    kErrForecastNegative = 4,
    kErrForecastSum = 5,
    kErrKvflowMissing = 6,
    kErrModelState = 7,
};

struct ApiError : std::runtime_error {
    int status;
    ApiError(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define PBKV_CUDA(call)                                                                                  \
    do {                                                                                                 \
        cudaError_t pbkv_e_ = (call);                                                                    \
        if (pbkv_e_ != cudaSuccess)                                                                      \
            throw ::pbkv::ApiError(PBKV_ECUDA, std::string(#call) + ": " + cudaGetErrorString(pbkv_e_)); \
    } while (0)

template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t cap = 0;  // elements
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void reserve(std::size_t n) {
        if (n <= cap) return;
        std::size_t c = cap ? cap : 1024;
        while (c < n) c *= 2;
        T* np = nullptr;
        if (cudaMalloc(&np, c * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            throw ApiError(PBKV_ENOMEM, "device allocation failed");
        }
        if (p) cudaFree(p);
        p = np;
        cap = c;
    }
    // grow keeping the first `keep` elements
    void grow_keep(std::size_t n, std::size_t keep, cudaStream_t s) {
        if (n <= cap) return;
        std::size_t c = cap ? cap : 1024;
        while (c < n) c *= 2;
        T* np = nullptr;
        if (cudaMalloc(&np, c * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            throw ApiError(PBKV_ENOMEM, "device allocation failed");
        }
        if (p && keep) PBKV_CUDA(cudaMemcpyAsync(np, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
        if (p) {
            cudaStreamSynchronize(s);
            cudaFree(p);
        }
        p = np;
        cap = c;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

template <class T>
struct PinBuf {
    T* p = nullptr;
    std::size_t cap = 0;
    PinBuf() = default;
    PinBuf(const PinBuf&) = delete;
    PinBuf& operator=(const PinBuf&) = delete;
    ~PinBuf() { release(); }
    void reserve(std::size_t n) {
        if (n <= cap) return;
        std::size_t c = cap ? cap : 1024;
        while (c < n) c *= 2;
        T* np = nullptr;
        if (cudaMallocHost(&np, c * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            throw ApiError(PBKV_ENOMEM, "pinned allocation failed");
        }
        if (p) cudaFreeHost(p);
        p = np;
        cap = c;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

// 161-bit candidate key of policies.hpp:40-48 packed as (w0, w1) + node id:
//   w0 = cls << 63 | enc(rank) >> 1,  w1 = (enc(rank) & 1) << 63 | last_access
// enc() is the order-preserving map of a double onto uint64 (-0.0 folded
// into +0.0 because std::tie compares them equal).  Lexicographic
// (w0, w1, id) order == std::tie(cls, rank, last_access, id) order.
struct alignas(16) Key2 {
    unsigned long long w0, w1;
};

// 160-bit sort record of a head (fallback sort path)
struct HeadKey {
    unsigned long long w0, w1;
    unsigned int id;
    unsigned int pad;  // written (zero): the sort moves whole 8-byte words
};

// a prefetch plan in pinned host memory (prefetch.cu run_prefetch_plan):
// ctr = {n_candidates, n_selected, selected_tokens, error}
struct PrefetchOut {
    const long long* ctr;
    const int* cand;
    const double* val;
    const int* sel;
};

struct SelectCounts {
    std::int64_t n_victims = 0, freed = 0;
    int shortfall = 0;
};

struct PredictorState;  // predict.cu

struct Context {
    int device = 0;
    int K = 3;
    double gamma = 0.7;
    int A = 1;   // agents
    int V1 = 2;  // outcomes
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // heavy-node scoring, overlapped with the light pass
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::string err;

    // ---- mirror -------------------------------------------------------------
    std::int64_t n = 0, E = 0;
    DevBuf<int> parent, len, ever, depth;
    DevBuf<std::uint8_t> flags;
    DevBuf<unsigned long long> last;
    DevBuf<double> score;  // cached (mirrored) score
    // access entries live in a pool: node i owns [acc_rng[i].x, acc_rng[i].y),
    // WorkflowId-ascending, inside a segment of capacity h_acc_cap[i] that
    // starts at acc_rng[i].x.  An incremental update (pbkv_mirror_delta)
    // rewrites a node's segment in place, or moves it to the pool top when it
    // outgrows its capacity; the pool is repacked when dead space dominates.
    DevBuf<uint2> acc_rng;
    DevBuf<int> acc_slot;
    DevBuf<unsigned long long> acc_bits;
    std::vector<int> h_entries;  // entries per node (host copy, for id-list classification)
    std::vector<unsigned int> h_acc_beg, h_acc_cap;
    std::int64_t pool_top = 0;   // first unused pool position
    // host copies of the node fields the host-side planning reads (classes,
    // deferral placement, sharding)
    std::vector<int> h_depth;
    std::vector<int> h_len;  // token length of every node (host copy: the prefetch round's scan)
    std::vector<std::uint8_t> h_flags;
    std::vector<unsigned long long> h_last;
    // pinned staging + completion event of pbkv_mirror_delta's upload
    PinBuf<unsigned char> hdelta;
    DevBuf<unsigned char> ddelta;
    cudaEvent_t ev_delta = nullptr;
    bool delta_pending = false;
    // staging of the class tables (medium / heavy lists, products list,
    // heavy children): reused once ev_class has passed
    PinBuf<unsigned char> hclass;
    DevBuf<unsigned char> dclass;  // the class tables' upload blob (ClassStager)
    cudaEvent_t ev_class = nullptr;
    cudaEvent_t ev_caller = nullptr;  // pbkv_ctx_wait_stream
    bool class_pending = false;
    // mirror bookkeeping of pbkv_mirror_sync: which host tree this context
    // mirrors (TrackedCacheTree uid) and the change-log position it has applied
    std::uint64_t mirror_uid = 0;
    std::int64_t mirror_pos = 0;
    // node-indexed copy of the (at most two) access entries of every light
    // node, so the light pass reads them coalesced, without the acc_rng hop:
    // lslot = {slot0, slot1} (-1 none, -2 the node is not light), lbits = bits
    DevBuf<int2> lslot;
    DevBuf<ulonglong2> lbits;
    // node classes for Eq. 2
    DevBuf<int> medium;  // 2 < entries, entries*K <= kMediumMaxChain
    std::int64_t n_medium = 0;
    DevBuf<int> heavy;  // entries*K > kMediumMaxChain
    std::int64_t n_heavy = 0;
    DevBuf<unsigned int> hent;    // heavy entries, node-major
    DevBuf<int> hent_node;        // heavy index of each heavy entry
    DevBuf<long long> hstart;     // first product of each heavy node
    DevBuf<double> hxs;           // products of the heavy entries
    DevBuf<unsigned int> hmiss;   // per heavy node: missing (1) / short horizon (2)
    std::int64_t n_hent = 0;
    std::vector<int> h_heavy;                 // heavy node ids, ascending (host copy)
    std::vector<int> h_medium;                // medium node ids, ascending (host copy)
    std::vector<char> h_spine;                // sharded context: spine membership (not in the chain lists)
    // children of every heavy node, ascending ids: kept up to date by the
    // delta path (a parent change updates the two lists it touches)
    std::unordered_map<int, std::vector<int>> h_heavy_ch;
    std::vector<int> h_parent;                // parent of every node (host copy)
    // children of the out-of-order nodes (CSR in heavy / spine order): the
    // eff walk stops below them and their reports reduce over these lists
    DevBuf<int> hch_off, hch, sch_off, sch;
    std::vector<unsigned long long> h_heavy_last;
    std::vector<int> h_heavy_depth, h_heavy_parent;
    std::vector<std::uint8_t> h_heavy_flags;
    // place_deferred: heavy nodes deepest first, heavy children of each heavy node (CSR)
    std::vector<std::size_t> h_heavy_order;
    bool deferred_cleared = false;  // run_select already enqueued the deferral clear
    std::vector<int> h_heavy_kid_off, h_heavy_kids;
    DevBuf<double> happrox;                   // [2*n_heavy]: approximate Eq. 2 sum, sum of |terms|
    DevBuf<unsigned char> hreport;            // deferred-heavy reports + the tail record
    PinBuf<unsigned char> hreport_h;
    bool defer_heavy = true;                  // decision fast path enabled
    bool report_deferred = false;             // run_select also fetches the heavy reports
    long long defer_fast = 0, defer_slow = 0; // fast / slow path counts
    std::int64_t device_capacity = 0, device_used = 0, retired_device_tokens = 0, host_capacity = 0, host_used = 0;
    int max_depth = 0;
    std::vector<std::int64_t> h_slot_wf;  // slot -> WorkflowId
    std::unordered_map<std::int64_t, int> slot_of;
    std::vector<int> slot_dense;  // direct slot table for WorkflowIds < 2^24

    // ---- forecasts ----------------------------------------------------------
    DevBuf<double> P;   // [slots][V1][K] agent-major
    DevBuf<double> Pg;  // [slots][V1][K]: gs[k] * (0.0 + P[a][k]), the exact Eq. 2 term of a one-agent entry
    DevBuf<double> gs;  // [slots][K]
    DevBuf<std::uint8_t> fstate;
    std::int64_t n_slots = 0;
    DevBuf<double> fstage;  // staging for uploads (H rows)
    DevBuf<long long> fstage_slot;

    // ---- kvflow remaining sequences (per slot CSR) --------------------------
    DevBuf<int> rem_off;  // [slots+1]
    DevBuf<int> rem_seq;
    DevBuf<std::uint8_t> rem_has;  // per slot
    bool have_remaining = false;

    // ---- selection scratch ----------------------------------------------------
    DevBuf<double> score_rc;  // recomputed scores
    DevBuf<Key2> keys;
    DevBuf<int> eff;
    DevBuf<int> sublock;
    DevBuf<std::uint8_t> missing;
    DevBuf<unsigned long long> W;
    DevBuf<unsigned int> C;
    DevBuf<int> rank;
    DevBuf<int> heads, listB, listS, listS2;
    DevBuf<ulonglong2> listSK;
    DevBuf<unsigned int> listSC, listSC2;
    DevBuf<unsigned int> big;  // [2 * n]: (offset, count) of buckets sorted by rank counting
    // oversized-bucket refinement of the selection (select.cu refine_buckets)
    DevBuf<unsigned int> rf_u32;         // descriptors [2][2][cap] + histograms [2][cap][2048]
    DevBuf<unsigned long long> rf_orand; // [2][cap][6]
    DevBuf<unsigned int> rf_small;       // [2 * n]
    DevBuf<ulonglong2> rf_tmpk;          // [n]
    // small-cut path (select.cu): node sample, low list, histogram tables
    DevBuf<unsigned char> samp;
    DevBuf<int> low;
    DevBuf<long long> cut_partial;  // sharded merge: per-CTA token sums
    PinBuf<unsigned char> his;        // pbkv_interval_sums: pinned pieces, offsets and sums
    DevBuf<unsigned char> dis;
    DevBuf<unsigned long long> gbar;  // the persistent selection kernel's grid barrier
    int gbar_grid = 0;                // the grid size the counter is a multiple of (0: zero it first)
    DevBuf<unsigned int> small_u32;
    DevBuf<unsigned long long> small_u64;
    DevBuf<unsigned long long> hist_w, part_w;
    DevBuf<unsigned int> hist_c, part_c, seg_off, seg_cnt, cursor;
    std::vector<unsigned long long> phase_ns;  // select-kernel phase timestamps of the last call
    DevBuf<unsigned char> selstate;
    PinBuf<unsigned char> hselstate;
    DevBuf<unsigned long long> sortk_in, sortk_out;
    DevBuf<int> sorti_in, sorti_out;
    DevBuf<HeadKey> hk_in, hk_out;
    DevBuf<unsigned long long> cnt;
    DevBuf<int> vid_out;  // victims in eviction order
    DevBuf<int> locked;
    DevBuf<int> ids, ids2, ids3;
    DevBuf<double> vals;
    // stage 4 scratch (prefetch.cu)
    DevBuf<unsigned long long> pf_hi, pf_bkey, pf_bhi, pf_hlen, pf_shi;
    DevBuf<unsigned int> pf_id, pf_len, pf_bid, pf_blen, pf_hist, pf_big;
    DevBuf<int> pf_sid, pf_slen, pf_cmin;
    DevBuf<unsigned char> pf_state;
    PinBuf<unsigned char> hplan, hplan_init;
    PinBuf<int> hids;         // id lists in (score_ids_impl)
    PinBuf<double> hvals;     // values out (score_ids_impl)
    bool status_pending = false;  // an asynchronous forecast upload's status is still unread
    PrefetchOut plan_out{};  // the last plan (views into hplan)
    bool plan_valid = false;
    DevBuf<unsigned char> cub_tmp;
    DevBuf<long long> counters;  // small device scalars
    DevBuf<DevStatus> status;
    PinBuf<long long> hcounters;
    PinBuf<DevStatus> hstatus;
    PinBuf<int> hlocked, hvictims;  // pinned staging of the host-array select (pbkv_select)
    int* epi_vict = nullptr;  // pinned victims destination of the decision epilogue (pbkv_select)
    long long epi_cap = 0;
    bool epi_vict_valid = false;  // the last epilogue stored the victims there
    PinBuf<long long> hslots;       // pinned staging of the forecast slots (pbkv_forecast_put)
    PinBuf<double> hrows;           // pinned staging of pageable forecast rows (pbkv_forecast_put)
    cudaEvent_t ev_rows = nullptr;  // the staged rows' copy has completed
    PinBuf<unsigned char> hpred_blob;  // pinned staging of pbkv_predict's slots / offsets / prefix
    DevBuf<unsigned char> pred_blob;

    // ---- sharding (shard.cu) -------------------------------------------------------
    std::vector<int> spine;  // local ids of the spine copies
    DevBuf<int> spine_dev, gid;
    DevBuf<long long> spine_base, run_start, run_len;
    DevBuf<unsigned int> spine_miss;
    DevBuf<pbkv_cand> merged;

    // ---- forward-propagation forecaster (fmodel.cu) ----------------------------------
    DevBuf<double> fm_rows, fm_mass;
    DevBuf<int> fm_next, fm_start;
    std::int64_t fm_states = 0;

    // ---- stage-1 predictor (predict.cu) -----------------------------------------
    std::shared_ptr<PredictorState> pred;
    DevBuf<int> pre_off, pre;
    DevBuf<std::uint16_t> xstage;

    // launch accounting (pbkv kernels; CUB library calls counted separately)
    long long launches = 0, lib_calls = 0;

    // timing
    bool timing = false;
    cudaEvent_t ev[6] = {};
    float last_ms[5] = {0, 0, 0, 0, 0};
    // per-kernel events (timing mode): [0,1] around the light Eq. 2 pass,
    // [2,3] around the persistent selection kernel
    cudaEvent_t kev[4] = {};
    bool kev_light = false, kev_select = false;
    float kernel_ms[2] = {0, 0};
};

// ---- launchers (score.cu / select.cu / prefetch.cu) -------------------------------
void launch_forecast_prepare(Context& c, const double* stage, const long long* slots, std::int64_t n, int H);
void launch_score_all(Context& c, double* out, bool write_keys, int policy, bool report_missing);
void launch_score_ids(Context& c, const int* ids_dev, const int* h_ids, std::int64_t n, double* out, bool value_only);
void launch_chain_sum(Context& c, const double* x, const long long* off, int n_seg, double* out);
void launch_interval_sums(Context& c, const double* x, const long long* pieces, const long long* out_off, int n_out,
                          double* out_host);
void launch_gather_f64(Context& c, const double* src, const int* ids, std::int64_t n, double* dst);
void launch_keys_cached(Context& c, int policy);
void launch_score_decision(Context& c, int policy);  // Eq. 2 + keys with heavy chains deferred
void launch_set_deferred(Context& c, bool on, const int* skip_if = nullptr);
void launch_decision_prologue(Context& c, bool defer, cudaStream_t st);
void raise_status(Context& c, const DevStatus& s);
struct HeavyReport {  // one per heavy node, then one tail record (select.cu)
    unsigned long long w0, w1;  // key of eff(h) over its non-deferred descendants / of the tail head
    int eff;                    // node id (-1: none)
    int eff_depth;
    int sublock;
    int miss;                   // missing forecast on one of its entries (1/2)
    int depth_diff;             // tail record: depth(head) - depth(last victim)
    int pad;
};
void launch_heavy_report(Context& c, long long* result_dev, HeavyReport* out, double* approx_out);
SelectCounts run_select(Context& c, const int* locked_dev, std::int64_t n_locked, std::int64_t needed,
                        bool he_recompute, long long* result_dev);
std::size_t sel_state_bytes();
void run_prefetch_plan(Context& c, long long budget, PrefetchOut* out);
void predictor_load(Context& c, const pbkv_predictor_cfg& cfg, const pbkv_predictor_weights& w);
pbkv_predictor_cfg predictor_cfg(const Context& c);
void predictor_run(Context& c, std::int64_t n, const int* pre_off_dev, const int* pre_dev, const void* x_dev,
                   const long long* slots_dev, double* probs_dev);
void shard_apply_flags(Context& c);
void shard_records(Context& c, long long* result_dev, pbkv_cand* out, long long cap);
void shard_spine_report(Context& c, pbkv_spine_info* out);
void shard_spine_products(Context& c, const long long* base_dev, long long max_len, double* out, unsigned int* miss);
void shard_merge_cut(Context& c, const pbkv_cand* src, const long long* run_start_dev, const long long* run_len_dev,
                     int n_runs, long long max_run, long long total, pbkv_cand* merged, long long needed,
                     int* victims, long long* result);
void launch_propagate(Context& c, const int* start_dev, std::int64_t n, int H, double lambda);
void reset_status(Context& c);
void check_status(Context& c);  // syncs and throws on a device-side error

inline unsigned int grid_for(std::int64_t n, int block) {
    std::int64_t g = (n + block - 1) / block;
    return static_cast<unsigned int>(g < 1 ? 1 : g);
}

}  // namespace pbkv
