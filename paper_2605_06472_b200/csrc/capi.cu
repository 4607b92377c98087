// C ABI implementation (include/pbkv.h): context, device mirror, forecast
// store and the orchestration of the stage 2-4 kernels (kernels.cu).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <climits>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "host/internal_abi.h"
#include "pbkv_internal.cuh"

struct pbkv_ctx : pbkv::Context {};

namespace {

using namespace pbkv;

thread_local std::string g_last_error;

template <class F>
int api(pbkv_ctx* c, F&& f) {
    try {
        f();
        return PBKV_OK;
    } catch (const ApiError& e) {
        (c ? c->err : g_last_error) = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        (c ? c->err : g_last_error) = "host allocation failed";
        return PBKV_ENOMEM;
    } catch (const std::exception& e) {
        (c ? c->err : g_last_error) = e.what();
        return PBKV_EARG;
    }
}

void need(bool ok, const char* what) {
    if (!ok) throw ApiError(PBKV_EARG, what);
}

void invalid(const std::string& what) { throw ApiError(PBKV_EINVAL, what); }

void set_device(Context& c) { PBKV_CUDA(cudaSetDevice(c.device)); }

// ---- forecast slots ----------------------------------------------------------
// A slot without a usable forecast (missing, dropped, or horizon < K beyond
// its last step) holds NaN rows: the light Eq. 2 pass then needs no per-entry
// state lookup -- a NaN total marks a missing forecast (validated forecasts
// are finite), and the exact message comes from fstate on the error path.
std::size_t s_new_slot(const Context& c) { return static_cast<std::size_t>(c.n_slots); }

void poison_slot(Context& c, std::size_t slot) {
    const std::size_t row = static_cast<std::size_t>(c.K) * c.V1;
    PBKV_CUDA(cudaMemsetAsync(c.P.p + slot * row, 0xFF, row * sizeof(double), c.stream));
    PBKV_CUDA(cudaMemsetAsync(c.Pg.p + slot * row, 0xFF, row * sizeof(double), c.stream));
}

// zero a device buffer's elements [from, capacity)
template <class T>
void zero_tail(DevBuf<T>& b, std::size_t from, cudaStream_t st) {
    if (b.p && from < b.cap) PBKV_CUDA(cudaMemsetAsync(b.p + from, 0, (b.cap - from) * sizeof(T), st));
}

int slot_for(Context& c, std::int64_t wf) {
    // dense ids (the simulator allocates WorkflowIds monotonically) hit a
    // direct table; others fall back to the hash map
    if (wf >= 0 && wf < static_cast<std::int64_t>(c.slot_dense.size()) && c.slot_dense[static_cast<std::size_t>(wf)] >= 0)
        return c.slot_dense[static_cast<std::size_t>(wf)];
    auto it = c.slot_of.find(wf);
    if (it != c.slot_of.end()) return it->second;
    int s = static_cast<int>(c.n_slots);
    if (c.n_slots >= INT_MAX - 1) throw ApiError(PBKV_EARG, "too many workflows");
    std::size_t need_slots = static_cast<std::size_t>(c.n_slots + 1);
    std::size_t old = static_cast<std::size_t>(c.n_slots);
    c.P.grow_keep(need_slots * c.K * c.V1, old * c.K * c.V1, c.stream);
    c.Pg.grow_keep(need_slots * c.K * c.V1, old * c.K * c.V1, c.stream);
    poison_slot(c, s_new_slot(c));
    c.gs.grow_keep(need_slots * c.K, old * c.K, c.stream);
    // the new slot's gamma-weighted survival row (set by its first forecast)
    PBKV_CUDA(cudaMemsetAsync(c.gs.p + old * c.K, 0xFF, static_cast<std::size_t>(c.K) * sizeof(double), c.stream));
    std::size_t old_cap = c.fstate.cap;
    c.fstate.grow_keep(need_slots, old, c.stream);
    if (c.fstate.cap != old_cap)
        PBKV_CUDA(cudaMemsetAsync(c.fstate.p + old, 0, c.fstate.cap - old, c.stream));
    std::size_t old_rcap = c.rem_has.cap;
    c.rem_has.grow_keep(need_slots, old, c.stream);
    if (c.rem_has.cap != old_rcap)
        PBKV_CUDA(cudaMemsetAsync(c.rem_has.p + old, 0, c.rem_has.cap - old, c.stream));
    c.n_slots += 1;
    c.slot_of.emplace(wf, s);
    if (wf >= 0 && wf < (1ll << 24)) {
        if (static_cast<std::size_t>(wf) >= c.slot_dense.size())
            c.slot_dense.resize(std::max<std::size_t>(static_cast<std::size_t>(wf) + 1, 2 * c.slot_dense.size()), -1);
        c.slot_dense[static_cast<std::size_t>(wf)] = s;
    }
    c.h_slot_wf.push_back(wf);
    return s;
}

void ensure_scratch(Context& c) {
    std::size_t n = static_cast<std::size_t>(c.n) + 1;
    c.score_rc.reserve(n);
    c.keys.reserve(n);
    c.eff.reserve(n);
    c.sublock.reserve(n);
    c.missing.reserve(n);
    c.W.reserve(n);
    c.C.reserve(n);
    c.heads.reserve(n);
    c.listB.reserve(n);
    c.listS.reserve(n);
    c.listS2.reserve(n);
    c.listSK.reserve(n);
    c.listSC.reserve(n);
    c.listSC2.reserve(n);
    c.big.reserve(2 * n);
    c.rank.reserve(n);
    c.vid_out.reserve(n);
}

std::string missing_message(Context& c, long long node) {
    // first entry of `node` (WorkflowId order) lacking a forecast: node_terms
    // raises before multi_step_score checks horizons (scoring.hpp:66-75, :53)
    uint2 rg;
    PBKV_CUDA(cudaMemcpy(&rg, c.acc_rng.p + node, sizeof rg, cudaMemcpyDeviceToHost));
    std::vector<int> slots(rg.y - rg.x);
    if (!slots.empty())
        PBKV_CUDA(cudaMemcpy(slots.data(), c.acc_slot.p + rg.x, slots.size() * sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<std::uint8_t> st(static_cast<std::size_t>(c.n_slots));
    if (!st.empty()) PBKV_CUDA(cudaMemcpy(st.data(), c.fstate.p, st.size(), cudaMemcpyDeviceToHost));
    for (int s : slots)
        if (st[static_cast<std::size_t>(s)] == 0)
            return "missing forecast for active workflow " + std::to_string(c.h_slot_wf[static_cast<std::size_t>(s)]);
    for (int s : slots)
        if (st[static_cast<std::size_t>(s)] == 2) return "forecast horizon shorter than the scoring horizon";
    return "missing forecast";
}

std::string kvflow_message(Context& c, long long node) {
    uint2 rg;
    PBKV_CUDA(cudaMemcpy(&rg, c.acc_rng.p + node, sizeof rg, cudaMemcpyDeviceToHost));
    std::vector<int> slots(rg.y - rg.x);
    if (!slots.empty())
        PBKV_CUDA(cudaMemcpy(slots.data(), c.acc_slot.p + rg.x, slots.size() * sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<std::uint8_t> has(static_cast<std::size_t>(c.n_slots));
    if (!has.empty()) PBKV_CUDA(cudaMemcpy(has.data(), c.rem_has.p, has.size(), cudaMemcpyDeviceToHost));
    for (int s : slots)
        if (!has[static_cast<std::size_t>(s)])
            return "kvflow needs a static remaining sequence for workflow " +
                   std::to_string(c.h_slot_wf[static_cast<std::size_t>(s)]);
    return "kvflow needs a static remaining sequence";
}

}  // namespace

namespace pbkv {
void reset_status(Context& c) {
    if (c.status_pending) return;  // an asynchronous upload's status is still to be read
    DevStatus* h = c.hstatus.p;
    *h = DevStatus{0, 0, LLONG_MAX, LLONG_MAX};
    PBKV_CUDA(cudaMemcpyAsync(c.status.p, h, sizeof(DevStatus), cudaMemcpyHostToDevice, c.stream));
}

void check_status(Context& c) {
    PBKV_CUDA(cudaMemcpyAsync(c.hstatus.p, c.status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, c.stream));
    PBKV_CUDA(cudaStreamSynchronize(c.stream));
    c.status_pending = false;
    const DevStatus st = *c.hstatus.p;  // a copy: raising may reuse the pinned word
    raise_status(c, st);
}

// throws the API error a device status word describes (no-op when clear)
void raise_status(Context& c, const DevStatus& s) {
    c.status_pending = false;  // the word has been read
    if (s.code == 0) return;
    std::string msg;
    switch (s.kind) {
        case kErrMissingForecast:
        case kErrShortHorizon:
            msg = missing_message(c, s.node);
            break;
        case kErrLastAccessRange:
            msg = "pbkv: last_access >= 2^63 cannot be encoded in the candidate key";
            break;
        case kErrForecastNegative:
            msg = "negative forecast probability";
            break;
        case kErrForecastSum:
            msg = "forecast step does not sum to 1";
            break;
        case kErrKvflowMissing:
            msg = kvflow_message(c, s.node);
            break;
        case kErrModelState:
            msg = "prefix reaches a state with no kernel row";
            break;
        default:
            msg = "device-side validation failed";
    }
    reset_status(c);
    throw ApiError(s.code, msg);
}
}  // namespace pbkv

namespace {

void record(Context& c, int i) {
    if (c.timing) PBKV_CUDA(cudaEventRecord(c.ev[i], c.stream));
}

void finish_timing(Context& c, int last_ev) {
    if (!c.timing) return;
    PBKV_CUDA(cudaEventSynchronize(c.ev[last_ev]));
    c.kernel_ms[0] = c.kernel_ms[1] = 0.f;
    if (c.kev_light) cudaEventElapsedTime(&c.kernel_ms[0], c.kev[0], c.kev[1]);
    if (c.kev_select) cudaEventElapsedTime(&c.kernel_ms[1], c.kev[2], c.kev[3]);
    c.kev_light = c.kev_select = false;
    for (int i = 0; i < 5; ++i) c.last_ms[i] = 0.f;
    auto el = [&](int a, int b) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c.ev[a], c.ev[b]);
        return ms;
    };
    if (last_ev >= 1) c.last_ms[0] = el(0, 1);
    if (last_ev >= 2) c.last_ms[1] = el(1, 2);
    if (last_ev >= 3) c.last_ms[2] = el(2, 3);
    c.last_ms[4] = el(0, last_ev);
}

// children (ascending ids) of each of `nodes`: an O(n) scan of the host parents
std::vector<std::vector<int>> scan_children(const Context& c, const std::vector<int>& nodes) {
    std::unordered_map<int, int> idx;
    for (std::size_t j = 0; j < nodes.size(); ++j) idx[nodes[j]] = static_cast<int>(j);
    std::vector<std::vector<int>> lists(nodes.size());
    if (!nodes.empty())
        for (std::size_t i = 1; i < c.h_parent.size(); ++i) {
            auto it = idx.find(c.h_parent[i]);
            if (it != idx.end()) lists[static_cast<std::size_t>(it->second)].push_back(static_cast<int>(i));
        }
    return lists;
}

// children lists (CSR, in the order of `nodes`) of a few out-of-order nodes
// (the spine of a shard; set once per mirror)
void upload_children(Context& c, const std::vector<int>& nodes, DevBuf<int>& off_d, DevBuf<int>& ch_d) {
    const std::vector<std::vector<int>> lists = scan_children(c, nodes);
    std::vector<int> off{0}, ch;
    for (auto& l : lists) {
        ch.insert(ch.end(), l.begin(), l.end());
        off.push_back(static_cast<int>(ch.size()));
    }
    off_d.reserve(off.size());
    ch_d.reserve(ch.size() + 1);
    // pageable sources: the copies have read them when the calls return
    PBKV_CUDA(cudaMemcpyAsync(off_d.p, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
    if (!ch.empty())
        PBKV_CUDA(cudaMemcpyAsync(ch_d.p, ch.data(), ch.size() * sizeof(int), cudaMemcpyHostToDevice, c.stream));
}

// ---- mirror -----------------------------------------------------------------
// Eq. 2 class of a node with `ne` entries (score.cu): light <= 2 entries,
// medium chain <= kMediumMaxChain, heavy above
enum NodeClass : int { kLight = 0, kMedium = 1, kHeavy = 2 };
NodeClass class_of(const Context& c, std::int64_t ne) {
    if (ne * c.K > kMediumMaxChain) return kHeavy;
    return ne > 2 ? kMedium : kLight;
}

void insert_sorted(std::vector<int>& v, int x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it == v.end() || *it != x) v.insert(it, x);
}
void erase_sorted(std::vector<int>& v, int x) {
    auto it = std::lower_bound(v.begin(), v.end(), x);
    if (it != v.end() && *it == x) v.erase(it);
}

// Host arrays bound for device buffers, copied through one pinned staging
// buffer (c.hclass) with no host synchronisation: the next batch waits for
// ev_class before it rewrites the staging.
// byte ranges of one device blob copied into up to eight tables (one CTA each;
// 16-byte units: blob offsets are 16-byte aligned, table buffers 256-byte)
struct ScatterDesc {
    int n;
    unsigned char* dst[8];
    std::size_t off[8];
    std::size_t bytes[8];
};
__global__ void __launch_bounds__(256) scatter_blob_kernel(const unsigned char* blob, ScatterDesc d) {
    const int i = blockIdx.x;
    const unsigned char* src = blob + d.off[i];
    unsigned char* dst = d.dst[i];
    const std::size_t n16 = d.bytes[i] >> 4;
    for (std::size_t q = threadIdx.x; q < n16; q += blockDim.x)
        reinterpret_cast<uint4*>(dst)[q] = reinterpret_cast<const uint4*>(src)[q];
    for (std::size_t q = (n16 << 4) + threadIdx.x; q < d.bytes[i]; q += blockDim.x) dst[q] = src[q];
}

struct ClassStager {
    Context& c;
    struct Item {
        void* dst;
        const void* src;
        std::size_t bytes;
    };
    std::vector<Item> items;
    std::size_t total = 0;
    explicit ClassStager(Context& cc) : c(cc) {}
    template <class T>
    void add(DevBuf<T>& d, const std::vector<T>& v) {
        d.reserve(v.size() + 1);
        if (v.empty()) return;
        items.push_back(Item{d.p, v.data(), v.size() * sizeof(T)});
        total += (v.size() * sizeof(T) + 15) & ~std::size_t(15);
    }
    // one pinned blob, one H2D copy, one kernel scattering it into the
    // tables (seven copy calls cost ~25 us of host time per mirror delta)
    void flush() {
        if (c.class_pending) {
            PBKV_CUDA(cudaEventSynchronize(c.ev_class));
            c.class_pending = false;
        }
        if (items.empty()) return;
        c.hclass.reserve(total);
        c.dclass.reserve(total);
        ScatterDesc d{};
        std::size_t o = 0;
        for (const Item& it : items) {
            std::memcpy(c.hclass.p + o, it.src, it.bytes);
            d.dst[d.n] = static_cast<unsigned char*>(it.dst);
            d.off[d.n] = o;
            d.bytes[d.n] = it.bytes;
            ++d.n;
            o += (it.bytes + 15) & ~std::size_t(15);
        }
        PBKV_CUDA(cudaMemcpyAsync(c.dclass.p, c.hclass.p, o, cudaMemcpyHostToDevice, c.stream));
        PBKV_CUDA(cudaEventRecord(c.ev_class, c.stream));
        c.class_pending = true;
        scatter_blob_kernel<<<static_cast<unsigned int>(d.n), 256, 0, c.stream>>>(c.dclass.p, d);
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
};

// The class-derived device tables, from the host class lists (h_medium,
// h_heavy, h_heavy_ch) in O(medium + heavy entries): the medium / heavy
// lists, the products list of their entries (heavy first, then medium:
// combined index n_heavy + m, score.cu), the children lists of the heavy
// nodes and the deferral placement tables (place_deferred).
void refresh_heavy_tables(Context& c);
void upload_classes(Context& c) {
    const std::vector<int>& heavy = c.h_heavy;
    const std::vector<int>& medium = c.h_medium;
    std::vector<int> hent_node;
    std::vector<unsigned int> hent;
    std::vector<long long> hstart;
    auto add_entries = [&](int node, int idx) {
        hstart.push_back(static_cast<long long>(hent.size()) * c.K);
        const unsigned int b = c.h_acc_beg[static_cast<std::size_t>(node)];
        const int ne = c.h_entries[static_cast<std::size_t>(node)];
        for (int e = 0; e < ne; ++e) {
            hent.push_back(b + static_cast<unsigned int>(e));
            hent_node.push_back(idx);
        }
    };
    for (std::size_t j = 0; j < heavy.size(); ++j) add_entries(heavy[j], static_cast<int>(j));
    for (std::size_t m = 0; m < medium.size(); ++m) add_entries(medium[m], static_cast<int>(heavy.size() + m));
    std::vector<int> ch_off{0}, ch;
    for (int h : heavy) {
        const auto it = c.h_heavy_ch.find(h);
        if (it != c.h_heavy_ch.end()) ch.insert(ch.end(), it->second.begin(), it->second.end());
        ch_off.push_back(static_cast<int>(ch.size()));
    }
    ClassStager st(c);
    st.add(c.medium, medium);
    st.add(c.heavy, heavy);
    st.add(c.hent, hent);
    st.add(c.hent_node, hent_node);
    st.add(c.hstart, hstart);
    st.add(c.hch_off, ch_off);
    st.add(c.hch, ch);
    c.hmiss.reserve(heavy.size() + medium.size() + 1);
    c.hxs.reserve(hent.size() * static_cast<std::size_t>(c.K) + 1);
    st.flush();
    c.n_medium = static_cast<std::int64_t>(medium.size());
    c.n_heavy = static_cast<std::int64_t>(heavy.size());
    c.n_hent = static_cast<std::int64_t>(hent.size());
    refresh_heavy_tables(c);
}

// deferral placement tables of the heavy nodes (place_deferred), O(heavy)
void refresh_heavy_tables(Context& c) {
    const std::vector<int>& heavy = c.h_heavy;
    const std::size_t nh = heavy.size();
    c.h_heavy_last.resize(nh);
    c.h_heavy_parent.resize(nh);
    c.h_heavy_flags.resize(nh);
    c.h_heavy_depth.resize(nh);
    for (std::size_t j = 0; j < nh; ++j) {
        const std::size_t v = static_cast<std::size_t>(heavy[j]);
        c.h_heavy_last[j] = c.h_last[v];
        c.h_heavy_parent[j] = c.h_parent[v];
        c.h_heavy_flags[j] = c.h_flags[v];
        c.h_heavy_depth[j] = c.h_depth[v];
    }
    c.h_heavy_order.resize(nh);
    for (std::size_t j = 0; j < nh; ++j) c.h_heavy_order[j] = j;
    std::stable_sort(c.h_heavy_order.begin(), c.h_heavy_order.end(),
                     [&](std::size_t a, std::size_t b) { return c.h_heavy_depth[a] > c.h_heavy_depth[b]; });
    std::unordered_map<int, int> pos;
    for (std::size_t j = 0; j < nh; ++j) pos[heavy[j]] = static_cast<int>(j);
    std::vector<std::vector<int>> kids(nh);
    for (std::size_t q = 0; q < nh; ++q) {  // heavy children in index order
        const auto it = pos.find(c.h_heavy_parent[q]);
        if (it != pos.end()) kids[static_cast<std::size_t>(it->second)].push_back(static_cast<int>(q));
    }
    c.h_heavy_kid_off.assign(1, 0);
    c.h_heavy_kids.clear();
    for (std::size_t j = 0; j < nh; ++j) {
        c.h_heavy_kids.insert(c.h_heavy_kids.end(), kids[j].begin(), kids[j].end());
        c.h_heavy_kid_off.push_back(static_cast<int>(c.h_heavy_kids.size()));
    }
}

// Every node classified (O(n), full mirrors only), the heavy nodes'
// children by a scan, then the device tables.
void classify_all(Context& c) {
    c.h_medium.clear();
    c.h_heavy.clear();
    for (std::int64_t i = 0; i < c.n; ++i) {
        // a shard's spine nodes are scored from the exchanged products
        // (shard.py), not by the local medium / heavy chains
        if (static_cast<std::size_t>(i) < c.h_spine.size() && c.h_spine[static_cast<std::size_t>(i)]) continue;
        const NodeClass k = class_of(c, c.h_entries[static_cast<std::size_t>(i)]);
        if (k == kHeavy) c.h_heavy.push_back(static_cast<int>(i));
        else if (k == kMedium) c.h_medium.push_back(static_cast<int>(i));
    }
    const std::vector<std::vector<int>> lists = scan_children(c, c.h_heavy);
    c.h_heavy_ch.clear();
    for (std::size_t j = 0; j < c.h_heavy.size(); ++j) c.h_heavy_ch[c.h_heavy[j]] = lists[j];
    upload_classes(c);
}

void set_totals(Context& c, const pbkv_tree_totals& t) {
    c.device_capacity = t.device_capacity;
    c.device_used = t.device_used;
    c.retired_device_tokens = t.retired_device_tokens;
    c.host_capacity = t.host_capacity;
    c.host_used = t.host_used;
}

void mirror_full(Context& c, const pbkv_tree_soa& s) {
    need(s.n_nodes >= 1, "tree must contain the root");
    need(s.parent && s.len && s.tier && s.retired && s.last_access && s.ever_tagged && s.acc_off,
         "tree soa: missing required array");
    need(s.n_entries == 0 || (s.acc_wf && s.acc_bits), "tree soa: missing access arrays");
    need(s.n_nodes < INT_MAX, "tree too large for int32 node ids");
    need(s.n_entries < static_cast<std::int64_t>(UINT_MAX / 2), "too many access entries");
    const std::int64_t n = s.n_nodes, E = s.n_entries;
    const std::size_t nz = static_cast<std::size_t>(n);
    std::vector<uint2> rng(nz);
    std::vector<int> slot(static_cast<std::size_t>(E));
    std::vector<int2> lslot(nz);
    std::vector<ulonglong2> lbits(nz);
    c.h_entries.assign(nz, 0);
    c.h_acc_beg.assign(nz, 0);
    c.h_acc_cap.assign(nz, 0);
    c.h_flags.assign(nz, 0);
    c.h_last.assign(s.last_access, s.last_access + n);
    c.h_parent.assign(s.parent, s.parent + n);
    c.h_len.assign(s.len, s.len + n);
    for (std::int64_t i = 0; i < n; ++i) {
        const std::size_t iz = static_cast<std::size_t>(i);
        if (s.tier[i] > PBKV_TIER_ABSENT) invalid("tree soa: bad tier value");
        c.h_flags[iz] = static_cast<std::uint8_t>(s.tier[i] | (s.retired[i] ? kFlagRetired : 0));
        if (i > 0 && (s.parent[i] < 0 || s.parent[i] >= n)) invalid("tree soa: parent out of range");
        std::int64_t a = s.acc_off[i], b = s.acc_off[i + 1];
        if (a < 0 || b < a || b > E) invalid("tree soa: bad access offsets");
        for (std::int64_t e = a; e < b; ++e) {
            if (e > a && s.acc_wf[e] <= s.acc_wf[e - 1]) invalid("tree soa: access entries must ascend by workflow id");
            slot[static_cast<std::size_t>(e)] = slot_for(c, s.acc_wf[e]);
        }
        const std::int64_t ne = b - a;
        rng[iz] = make_uint2(static_cast<unsigned int>(a), static_cast<unsigned int>(b));
        c.h_entries[iz] = static_cast<int>(ne);
        c.h_acc_beg[iz] = static_cast<unsigned int>(a);
        c.h_acc_cap[iz] = static_cast<unsigned int>(ne);
        int2 ls{-1, -1};
        ulonglong2 lb{0ull, 0ull};
        if (ne > 2) {
            ls.x = ls.y = -2;
        } else {
            if (ne >= 1) {
                ls.x = slot[static_cast<std::size_t>(a)];
                lb.x = s.acc_bits[a];
            }
            if (ne == 2) {
                ls.y = slot[static_cast<std::size_t>(a + 1)];
                lb.y = s.acc_bits[a + 1];
            }
        }
        lslot[iz] = ls;
        lbits[iz] = lb;
    }
    if (s.depth) {
        c.h_depth.assign(s.depth, s.depth + n);
    } else {
        c.h_depth.assign(nz, -1);
        c.h_depth[0] = 0;
        std::vector<int> stack;
        for (std::int64_t i = 1; i < n; ++i) {
            int v = static_cast<int>(i);
            while (c.h_depth[static_cast<std::size_t>(v)] < 0) {
                stack.push_back(v);
                v = s.parent[v];
                if (stack.size() > nz) invalid("tree soa: parent cycle");
            }
            int d = c.h_depth[static_cast<std::size_t>(v)];
            while (!stack.empty()) {
                c.h_depth[static_cast<std::size_t>(stack.back())] = ++d;
                stack.pop_back();
            }
        }
    }
    int maxd = 0;
    for (int d : c.h_depth) maxd = std::max(maxd, d);
    if (maxd >= (1 << 24)) invalid("tree deeper than 2^24 levels");

    c.n = n;
    c.E = E;
    c.pool_top = E;
    c.parent.reserve(nz);
    c.len.reserve(nz);
    c.ever.reserve(nz);
    c.depth.reserve(nz);
    c.flags.reserve(nz);
    c.last.reserve(nz);
    c.score.reserve(nz);
    c.acc_rng.reserve(nz);
    c.lslot.reserve(nz);
    c.lbits.reserve(nz);
    c.acc_slot.reserve(static_cast<std::size_t>(E) + 1);
    c.acc_bits.reserve(static_cast<std::size_t>(E) + 1);
    cudaStream_t st = c.stream;
    // the pool above the packed entries (where deltas allocate) is defined:
    // the audit (pbkv_mirror_verify) copies the pool whole
    zero_tail(c.acc_slot, static_cast<std::size_t>(E), st);
    zero_tail(c.acc_bits, static_cast<std::size_t>(E), st);
    PBKV_CUDA(cudaMemcpyAsync(c.parent.p, s.parent, n * sizeof(int), cudaMemcpyHostToDevice, st));
    PBKV_CUDA(cudaMemcpyAsync(c.len.p, s.len, n * sizeof(int), cudaMemcpyHostToDevice, st));
    PBKV_CUDA(cudaMemcpyAsync(c.ever.p, s.ever_tagged, n * sizeof(int), cudaMemcpyHostToDevice, st));
    PBKV_CUDA(cudaMemcpyAsync(c.depth.p, c.h_depth.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    PBKV_CUDA(cudaMemcpyAsync(c.flags.p, c.h_flags.data(), n, cudaMemcpyHostToDevice, st));
    PBKV_CUDA(cudaMemcpyAsync(c.last.p, s.last_access, n * sizeof(std::uint64_t), cudaMemcpyHostToDevice, st));
    if (s.score)
        PBKV_CUDA(cudaMemcpyAsync(c.score.p, s.score, n * sizeof(double), cudaMemcpyHostToDevice, st));
    else
        PBKV_CUDA(cudaMemsetAsync(c.score.p, 0, n * sizeof(double), st));
    PBKV_CUDA(cudaMemcpyAsync(c.acc_rng.p, rng.data(), n * sizeof(uint2), cudaMemcpyHostToDevice, st));
    PBKV_CUDA(cudaMemcpyAsync(c.lslot.p, lslot.data(), n * sizeof(int2), cudaMemcpyHostToDevice, st));
    PBKV_CUDA(cudaMemcpyAsync(c.lbits.p, lbits.data(), n * sizeof(ulonglong2), cudaMemcpyHostToDevice, st));
    if (E > 0) {
        PBKV_CUDA(cudaMemcpyAsync(c.acc_slot.p, slot.data(), E * sizeof(int), cudaMemcpyHostToDevice, st));
        PBKV_CUDA(cudaMemcpyAsync(c.acc_bits.p, s.acc_bits, E * sizeof(std::uint64_t), cudaMemcpyHostToDevice, st));
    }
    classify_all(c);
    c.max_depth = maxd;
    set_totals(c, pbkv_tree_totals{s.device_capacity, s.device_used, s.retired_device_tokens, s.host_capacity,
                                   s.host_used});
    ensure_scratch(c);
    if (!c.spine.empty()) {
        for (int v : c.spine) need(v >= 0 && v < n, "shard spine id out of range for the mirrored tree");
        shard_apply_flags(c);
        upload_children(c, c.spine, c.sch_off, c.sch);
    }
    c.mirror_uid = 0;  // a snapshot of no tracked tree
    PBKV_CUDA(cudaStreamSynchronize(st));
}

// ---- incremental mirror (pbkv_mirror_delta) ----------------------------------
// Device record of one updated node: every mirrored field, the node's entry
// segment in the pool and its light-pass copies (lslot / lbits).
struct DeltaRec {
    int id, parent, len, ever, depth;
    unsigned int beg, cnt;
    int ls0, ls1;
    unsigned int flags;
    unsigned long long last, lb0, lb1;
    double score;
};

struct MirrorPtrs {
    int *parent, *len, *ever, *depth;
    std::uint8_t* flags;
    unsigned long long* last;
    double* score;
    uint2* rng;
    int2* lslot;
    ulonglong2* lbits;
    int* slot;
    unsigned long long* bits;
};

// records, then entries (dst position in the pool computed on the host),
// grid-stride: one launch per batch whatever its shape
__global__ void __launch_bounds__(256) mirror_delta_kernel(const DeltaRec* rec, long long n_rec,
                                                           const unsigned int* edst, const int* eslot,
                                                           const unsigned long long* ebits, long long n_ent,
                                                           MirrorPtrs m) {
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n_rec; i += stride) {
        const DeltaRec r = rec[i];
        m.parent[r.id] = r.parent;
        m.len[r.id] = r.len;
        m.ever[r.id] = r.ever;
        m.depth[r.id] = r.depth;
        m.flags[r.id] = static_cast<std::uint8_t>(r.flags);
        m.last[r.id] = r.last;
        m.score[r.id] = r.score;
        m.rng[r.id] = make_uint2(r.beg, r.beg + r.cnt);
        m.lslot[r.id] = make_int2(r.ls0, r.ls1);
        m.lbits[r.id] = make_ulonglong2(r.lb0, r.lb1);
    }
    for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < n_ent; j += stride) {
        const unsigned int d = edst[j];
        m.slot[d] = eslot[j];
        m.bits[d] = ebits[j];
    }
}

// pool repack: node i's entries move to new_beg[i] (dst buffers are fresh)
__global__ void __launch_bounds__(256) pool_repack_kernel(const uint2* rng_old, const unsigned int* new_beg,
                                                          long long n, const int* slot_old,
                                                          const unsigned long long* bits_old, int* slot_new,
                                                          unsigned long long* bits_new, uint2* rng_new) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const uint2 r = rng_old[i];
        const unsigned int b = new_beg[i];
        for (unsigned int e = r.x; e < r.y; ++e) {
            slot_new[b + (e - r.x)] = slot_old[e];
            bits_new[b + (e - r.x)] = bits_old[e];
        }
        rng_new[i] = make_uint2(b, b + (r.y - r.x));
    }
}

MirrorPtrs mirror_ptrs(Context& c) {
    return MirrorPtrs{c.parent.p, c.len.p,   c.ever.p,  c.depth.p, c.flags.p,    c.last.p,
                      c.score.p,  c.acc_rng.p, c.lslot.p, c.lbits.p, c.acc_slot.p, c.acc_bits.p};
}

// Dead pool space above half: pack every node's segment tightly (a device
// copy into fresh buffers; the host knows every segment's size).
void repack_pool(Context& c) {
    const std::size_t nz = static_cast<std::size_t>(c.n);
    std::vector<unsigned int> nb(nz);
    unsigned int top = 0;
    for (std::size_t i = 0; i < nz; ++i) {
        nb[i] = top;
        top += static_cast<unsigned int>(c.h_entries[i]);
    }
    DevBuf<int> slot_new;
    DevBuf<unsigned long long> bits_new;
    DevBuf<uint2> rng_new;
    DevBuf<unsigned int> nb_d;
    slot_new.reserve(std::max<std::size_t>(top, 1) + (top >> 2));
    bits_new.reserve(slot_new.cap);
    rng_new.reserve(std::max<std::size_t>(c.acc_rng.cap, nz));
    nb_d.reserve(nz);
    zero_tail(slot_new, top, c.stream);
    zero_tail(bits_new, top, c.stream);
    PBKV_CUDA(cudaMemcpyAsync(nb_d.p, nb.data(), nz * sizeof(unsigned int), cudaMemcpyHostToDevice, c.stream));
    pool_repack_kernel<<<grid_for(c.n, 256), 256, 0, c.stream>>>(c.acc_rng.p, nb_d.p, c.n, c.acc_slot.p,
                                                                c.acc_bits.p, slot_new.p, bits_new.p, rng_new.p);
    PBKV_CUDA(cudaGetLastError());
    ++c.launches;
    PBKV_CUDA(cudaStreamSynchronize(c.stream));
    std::swap(c.acc_slot.p, slot_new.p);
    std::swap(c.acc_slot.cap, slot_new.cap);
    std::swap(c.acc_bits.p, bits_new.p);
    std::swap(c.acc_bits.cap, bits_new.cap);
    std::swap(c.acc_rng.p, rng_new.p);
    std::swap(c.acc_rng.cap, rng_new.cap);
    for (std::size_t i = 0; i < nz; ++i) {
        c.h_acc_beg[i] = nb[i];
        c.h_acc_cap[i] = static_cast<unsigned int>(c.h_entries[i]);
    }
    c.pool_top = top;
}

void mirror_delta(Context& c, const pbkv_node_delta* d, std::int64_t n_rec, const std::int64_t* acc_wf,
                  const std::uint64_t* acc_bits, const pbkv_tree_totals* totals) {
    static const bool prof = std::getenv("PBKV_PROFILE_SYNC") != nullptr;
    auto prev = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!prof) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  [delta] %s %.1fus\n", what, std::chrono::duration<double, std::micro>(now - prev).count());
        prev = now;
    };
    if (prof) lap("start");
    need(c.n >= 1, "no tree mirrored");
    need(n_rec == 0 || d, "null delta records");
    int max_id = -1;
    bool ascending = true;  // the tracked tree's batches: distinct ids, ascending
    for (std::int64_t i = 0; i < n_rec; ++i) {
        const pbkv_node_delta& r = d[i];
        need(r.id >= 0 && r.id < INT_MAX - 1, "delta: node id out of range");
        if (r.tier > PBKV_TIER_ABSENT) invalid("tree delta: bad tier value");
        if (r.acc_begin < 0 || r.acc_end < r.acc_begin) invalid("tree delta: bad access range");
        need(r.acc_end == r.acc_begin || (acc_wf && acc_bits), "delta: null access arrays");
        for (std::int64_t e = r.acc_begin + 1; e < r.acc_end; ++e)
            if (acc_wf[e] <= acc_wf[e - 1]) invalid("tree delta: access entries must ascend by workflow id");
        if (r.depth < 0 || r.depth >= (1 << 24)) invalid("tree delta: bad depth");
        if (i > 0 && r.id <= d[i - 1].id) ascending = false;
        max_id = std::max(max_id, r.id);
    }
    // records ordered by id, the last record of a node winning
    std::vector<std::int64_t> order(static_cast<std::size_t>(n_rec));
    for (std::int64_t i = 0; i < n_rec; ++i) order[static_cast<std::size_t>(i)] = i;
    if (!ascending) {
        std::stable_sort(order.begin(), order.end(), [&](std::int64_t a, std::int64_t b) { return d[a].id < d[b].id; });
        std::size_t w = 0;
        for (std::size_t k = 0; k < order.size(); ++k) {
            if (k + 1 < order.size() && d[order[k + 1]].id == d[order[k]].id) continue;
            order[w++] = order[k];
        }
        order.resize(w);
    }
    const std::int64_t n_old = c.n;
    const std::int64_t n_new = std::max<std::int64_t>(n_old, static_cast<std::int64_t>(max_id) + 1);
    {  // distinct ids below n_new: the appended ones are dense iff there are n_new - n_old of them
        std::int64_t appended = 0;
        for (std::int64_t i : order) appended += d[i].id >= n_old ? 1 : 0;
        need(appended == n_new - n_old, "delta: appended node ids must be dense");
    }
    for (std::int64_t i : order) {
        const pbkv_node_delta& r = d[i];
        if (r.id == 0) {
            need(r.parent == -1, "delta: the root has no parent");
        } else if (r.parent < 0 || r.parent >= n_new) {
            invalid("tree delta: parent out of range");
        }
    }
    if (!c.spine.empty()) {  // sharded shards keep their global-id map: no structural updates
        need(n_new == n_old, "delta: sharded contexts cannot append nodes");
        for (std::int64_t i : order)
            need(d[i].parent == c.h_parent[static_cast<std::size_t>(d[i].id)], "delta: sharded contexts cannot move nodes");
    }

    lap("validate+order");
    // grow the mirror (keeping contents) and the host copies
    cudaStream_t st = c.stream;
    if (n_new > n_old) {
        const std::size_t nn = static_cast<std::size_t>(n_new), no = static_cast<std::size_t>(n_old);
        c.parent.grow_keep(nn, no, st);
        c.len.grow_keep(nn, no, st);
        c.ever.grow_keep(nn, no, st);
        c.depth.grow_keep(nn, no, st);
        c.flags.grow_keep(nn, no, st);
        c.last.grow_keep(nn, no, st);
        c.score.grow_keep(nn, no, st);
        c.acc_rng.grow_keep(nn, no, st);
        c.lslot.grow_keep(nn, no, st);
        c.lbits.grow_keep(nn, no, st);
        c.h_entries.resize(nn, 0);
        c.h_acc_beg.resize(nn, 0);
        c.h_acc_cap.resize(nn, 0);
        c.h_parent.resize(nn, -1);
        c.h_depth.resize(nn, 0);
        c.h_flags.resize(nn, 0);
        c.h_last.resize(nn, 0);
        c.h_len.resize(nn, 0);
    }
    // placement of every record's entries; class / structure bookkeeping
    std::int64_t n_ent = 0;
    for (std::int64_t i : order) n_ent += d[i].acc_end - d[i].acc_begin;
    std::vector<DeltaRec> recs(order.size());
    std::vector<unsigned int> edst(static_cast<std::size_t>(n_ent));
    std::vector<int> eslot(static_cast<std::size_t>(n_ent));
    std::vector<unsigned long long> ebits(static_cast<std::size_t>(n_ent));
    // class bookkeeping: `products` when the device class tables change (a
    // class transition, a medium / heavy segment moved or resized, a heavy
    // node's children), `tables` when only a heavy node's placement fields do
    bool products = false, tables = false;
    struct ClassMove {
        int id;
        NodeClass from, to;
    };
    std::vector<ClassMove> cls_moves;
    std::vector<std::pair<int, int>> reparented;  // (node, old parent) (-2: fresh)
    std::int64_t E = c.E, q = 0;
    for (std::size_t k = 0; k < order.size(); ++k) {
        if (k + 8 < order.size()) {  // sparse ids over 1M-entry host arrays: one miss per array per node
            const std::size_t f = static_cast<std::size_t>(d[order[k + 8]].id);
            if (f < c.h_entries.size()) {
                __builtin_prefetch(&c.h_entries[f], 1);
                __builtin_prefetch(&c.h_acc_beg[f], 1);
                __builtin_prefetch(&c.h_acc_cap[f], 1);
                __builtin_prefetch(&c.h_parent[f], 1);
                __builtin_prefetch(&c.h_depth[f], 1);
                __builtin_prefetch(&c.h_flags[f], 1);
                __builtin_prefetch(&c.h_last[f], 1);
                __builtin_prefetch(&c.h_len[f], 1);
            }
        }
        const pbkv_node_delta& r = d[order[k]];
        const std::size_t id = static_cast<std::size_t>(r.id);
        const bool fresh = r.id >= n_old;
        const std::int64_t ne = r.acc_end - r.acc_begin;
        need(ne < INT_MAX, "delta: too many entries on one node");
        const int ne_old = fresh ? 0 : c.h_entries[id];
        const NodeClass k_old = class_of(c, ne_old), k_new = class_of(c, ne);
        unsigned int beg = c.h_acc_beg[id];
        if (fresh || ne > static_cast<std::int64_t>(c.h_acc_cap[id])) {  // (re)allocate at the pool top
            const std::int64_t cap = fresh ? std::max<std::int64_t>(ne, 1) : std::max<std::int64_t>(2 * ne, 4);
            need(c.pool_top + cap < static_cast<std::int64_t>(UINT_MAX / 2), "too many access entries");
            beg = static_cast<unsigned int>(c.pool_top);
            c.pool_top += cap;
            c.h_acc_cap[id] = static_cast<unsigned int>(cap);
        }
        if (k_old != k_new) cls_moves.push_back(ClassMove{r.id, k_old, k_new});
        if (k_old != k_new || (k_new != kLight && (beg != c.h_acc_beg[id] || ne != ne_old))) products = true;
        if (k_new == kHeavy || k_old == kHeavy) tables = true;  // placement tables read its fields
        const int p_old = fresh ? -2 : c.h_parent[id];
        if (p_old != r.parent) reparented.emplace_back(r.id, p_old);
        E += ne - ne_old;
        c.h_entries[id] = static_cast<int>(ne);
        c.h_acc_beg[id] = beg;
        c.h_parent[id] = r.parent;
        c.h_depth[id] = r.depth;
        c.h_flags[id] = static_cast<std::uint8_t>(r.tier | (r.retired ? kFlagRetired : 0));
        c.h_last[id] = r.last_access;
        c.h_len[id] = r.len;
        c.max_depth = std::max(c.max_depth, static_cast<int>(r.depth));
        DeltaRec& o = recs[k];
        o.id = r.id;
        o.parent = r.parent;
        o.len = r.len;
        o.ever = r.ever_tagged;
        o.depth = r.depth;
        o.beg = beg;
        o.cnt = static_cast<unsigned int>(ne);
        o.flags = c.h_flags[id];
        o.last = r.last_access;
        o.score = r.score;
        o.ls0 = o.ls1 = ne > 2 ? -2 : -1;
        o.lb0 = o.lb1 = 0ull;
        for (std::int64_t e = 0; e < ne; ++e, ++q) {
            const int sl = slot_for(c, acc_wf[r.acc_begin + e]);
            const unsigned long long b = acc_bits[r.acc_begin + e];
            edst[static_cast<std::size_t>(q)] = beg + static_cast<unsigned int>(e);
            eslot[static_cast<std::size_t>(q)] = sl;
            ebits[static_cast<std::size_t>(q)] = b;
            if (ne <= 2 && e == 0) {
                o.ls0 = sl;
                o.lb0 = b;
            }
            if (ne == 2 && e == 1) {
                o.ls1 = sl;
                o.lb1 = b;
            }
        }
    }
    lap("records");
    c.n = n_new;
    c.E = E;
    if (c.pool_top > static_cast<std::int64_t>(c.acc_slot.cap)) {
        const std::size_t keep = c.acc_slot.cap;
        c.acc_slot.grow_keep(static_cast<std::size_t>(c.pool_top), keep, st);
        c.acc_bits.grow_keep(static_cast<std::size_t>(c.pool_top), keep, st);
        zero_tail(c.acc_slot, keep, st);  // segment slack stays defined
        zero_tail(c.acc_bits, keep, st);
    }
    // one pinned blob, one copy, one kernel
    auto align16 = [](std::size_t x) { return (x + 15) & ~std::size_t(15); };
    const std::size_t b_rec = align16(recs.size() * sizeof(DeltaRec));
    const std::size_t b_dst = align16(edst.size() * sizeof(unsigned int));
    const std::size_t b_slot = align16(eslot.size() * sizeof(int));
    const std::size_t b_bits = ebits.size() * sizeof(unsigned long long);
    const std::size_t blob = b_rec + b_dst + b_slot + b_bits;
    if (c.delta_pending) {  // the previous batch's copy still reads the pinned staging
        PBKV_CUDA(cudaEventSynchronize(c.ev_delta));
        c.delta_pending = false;
    }
    if (!recs.empty()) {
        c.hdelta.reserve(blob);
        c.ddelta.reserve(blob);
        unsigned char* h = c.hdelta.p;
        std::memcpy(h, recs.data(), recs.size() * sizeof(DeltaRec));
        if (!edst.empty()) {
            std::memcpy(h + b_rec, edst.data(), edst.size() * sizeof(unsigned int));
            std::memcpy(h + b_rec + b_dst, eslot.data(), eslot.size() * sizeof(int));
            std::memcpy(h + b_rec + b_dst + b_slot, ebits.data(), b_bits);
        }
        PBKV_CUDA(cudaMemcpyAsync(c.ddelta.p, h, blob, cudaMemcpyHostToDevice, st));
        PBKV_CUDA(cudaEventRecord(c.ev_delta, st));
        c.delta_pending = true;
        const unsigned char* dp = c.ddelta.p;
        const long long nr = static_cast<long long>(recs.size());
        mirror_delta_kernel<<<grid_for(std::max<long long>(nr, n_ent), 256), 256, 0, st>>>(
            reinterpret_cast<const DeltaRec*>(dp), nr, reinterpret_cast<const unsigned int*>(dp + b_rec),
            reinterpret_cast<const int*>(dp + b_rec + b_dst),
            reinterpret_cast<const unsigned long long*>(dp + b_rec + b_dst + b_slot), n_ent, mirror_ptrs(c));
        PBKV_CUDA(cudaGetLastError());
        ++c.launches;
    }
    lap("upload");
    if (totals) set_totals(c, *totals);
    if (n_new > n_old) ensure_scratch(c);
    lap("scratch");
    // class lists and heavy children, updated by the changed nodes only
    std::vector<int> newly_heavy;
    for (const ClassMove& m : cls_moves) {
        if (static_cast<std::size_t>(m.id) < c.h_spine.size() && c.h_spine[static_cast<std::size_t>(m.id)])
            continue;  // (classify_all)
        if (m.from == kMedium) erase_sorted(c.h_medium, m.id);
        if (m.from == kHeavy) {
            erase_sorted(c.h_heavy, m.id);
            c.h_heavy_ch.erase(m.id);
        }
        if (m.to == kMedium) insert_sorted(c.h_medium, m.id);
        if (m.to == kHeavy) {
            insert_sorted(c.h_heavy, m.id);
            newly_heavy.push_back(m.id);
        }
    }
    if (!newly_heavy.empty()) {  // rare (a node crossing the heavy threshold): one O(n) scan
        const std::vector<std::vector<int>> lists = scan_children(c, newly_heavy);
        for (std::size_t j = 0; j < newly_heavy.size(); ++j) c.h_heavy_ch[newly_heavy[j]] = lists[j];
    }
    for (const auto& [id, p_old] : reparented) {
        auto is_new = [&](int p) { return std::find(newly_heavy.begin(), newly_heavy.end(), p) != newly_heavy.end(); };
        if (p_old >= 0 && !is_new(p_old)) {
            const auto it = c.h_heavy_ch.find(p_old);
            if (it != c.h_heavy_ch.end()) {
                erase_sorted(it->second, id);
                products = true;
            }
        }
        const int p_new = c.h_parent[static_cast<std::size_t>(id)];
        if (p_new >= 0 && !is_new(p_new)) {
            const auto it = c.h_heavy_ch.find(p_new);
            if (it != c.h_heavy_ch.end()) {
                insert_sorted(it->second, id);
                products = true;
            }
        }
    }
    lap("class lists");
    if (products)
        upload_classes(c);
    else if (tables)
        refresh_heavy_tables(c);
    lap(products ? "upload_classes" : "heavy tables");
    if (!c.spine.empty()) shard_apply_flags(c);
    // dead space above half of the pool: repack (rare; amortised O(1) per entry)
    if (c.pool_top > 2 * c.E + (1 << 16)) repack_pool(c);
}

// device mirror vs a full snapshot, field by field (pbkv_mirror_verify)
std::int64_t mirror_verify(Context& c, const pbkv_tree_soa& s) {
    need(s.parent && s.len && s.tier && s.retired && s.last_access && s.ever_tagged && s.acc_off,
         "tree soa: missing required array");
    PBKV_CUDA(cudaStreamSynchronize(c.stream));
    const std::int64_t n = std::min<std::int64_t>(c.n, s.n_nodes);
    const std::size_t nz = static_cast<std::size_t>(c.n);
    std::vector<int> parent(nz), len(nz), ever(nz), depth(nz);
    std::vector<std::uint8_t> flags(nz);
    std::vector<unsigned long long> last(nz);
    std::vector<double> score(nz);
    std::vector<uint2> rng(nz);
    std::vector<int2> lslot(nz);
    std::vector<ulonglong2> lbits(nz);
    std::vector<int> slot(static_cast<std::size_t>(c.pool_top) + 1);
    std::vector<unsigned long long> bits(static_cast<std::size_t>(c.pool_top) + 1);
    auto get = [&](void* dst, const void* src, std::size_t bytes) {
        if (bytes) PBKV_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    };
    get(parent.data(), c.parent.p, nz * sizeof(int));
    get(len.data(), c.len.p, nz * sizeof(int));
    get(ever.data(), c.ever.p, nz * sizeof(int));
    get(depth.data(), c.depth.p, nz * sizeof(int));
    get(flags.data(), c.flags.p, nz);
    get(last.data(), c.last.p, nz * sizeof(unsigned long long));
    get(score.data(), c.score.p, nz * sizeof(double));
    get(rng.data(), c.acc_rng.p, nz * sizeof(uint2));
    get(lslot.data(), c.lslot.p, nz * sizeof(int2));
    get(lbits.data(), c.lbits.p, nz * sizeof(ulonglong2));
    get(slot.data(), c.acc_slot.p, static_cast<std::size_t>(c.pool_top) * sizeof(int));
    get(bits.data(), c.acc_bits.p, static_cast<std::size_t>(c.pool_top) * sizeof(unsigned long long));
    for (std::int64_t i = 0; i < n; ++i) {
        const std::size_t iz = static_cast<std::size_t>(i);
        const std::uint8_t f = static_cast<std::uint8_t>(s.tier[i] | (s.retired[i] ? kFlagRetired : 0));
        bool ok = parent[iz] == s.parent[i] && len[iz] == s.len[i] && ever[iz] == s.ever_tagged[i] &&
                  (flags[iz] & (kFlagTierMask | kFlagRetired)) == f && last[iz] == s.last_access[i] &&
                  (!s.depth || depth[iz] == s.depth[i]) && c.h_depth[iz] == depth[iz] &&
                  (!s.score || std::memcmp(&score[iz], &s.score[i], sizeof(double)) == 0);
        const std::int64_t a = s.acc_off[i], b = s.acc_off[i + 1];
        ok = ok && static_cast<std::int64_t>(rng[iz].y) - rng[iz].x == b - a && c.h_entries[iz] == b - a &&
             rng[iz].x == c.h_acc_beg[iz] && rng[iz].y <= static_cast<unsigned int>(c.pool_top);
        for (std::int64_t e = 0; ok && e < b - a; ++e) {
            const std::size_t pe = rng[iz].x + static_cast<std::size_t>(e);
            const int sl = slot[pe];
            ok = sl >= 0 && sl < c.n_slots && c.h_slot_wf[static_cast<std::size_t>(sl)] == s.acc_wf[a + e] &&
                 bits[pe] == s.acc_bits[a + e];
        }
        if (ok) {  // the light pass's node-indexed copies
            const std::int64_t ne = b - a;
            if (ne > 2) {
                ok = lslot[iz].x == -2 && lslot[iz].y == -2;
            } else {
                ok = lslot[iz].x == (ne >= 1 ? slot[rng[iz].x] : -1) && lslot[iz].y == (ne == 2 ? slot[rng[iz].x + 1] : -1) &&
                     lbits[iz].x == (ne >= 1 ? s.acc_bits[a] : 0ull) && lbits[iz].y == (ne == 2 ? s.acc_bits[a + 1] : 0ull);
            }
        }
        if (!ok) return i;
    }
    if (c.n != s.n_nodes || c.device_used != s.device_used || c.retired_device_tokens != s.retired_device_tokens ||
        c.device_capacity != s.device_capacity || c.host_used != s.host_used || c.host_capacity != s.host_capacity)
        return n;
    return -1;
}

// ---- stage 3 ------------------------------------------------------------------
// Keys (from the recomputed or the cached score), lock marks, subtree max,
// then the weighted cut and the victim order (select.cu).  Victims land in
// c.vid_out[0..n_victims).
// ---- deferred heavy nodes ------------------------------------
// CandidateKey packing (common.cuh make_key) on the host
unsigned long long host_enc_rank(double r) {
    if (r == 0.0) r = 0.0;
    unsigned long long b;
    std::memcpy(&b, &r, sizeof b);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct HKey {  // (w0, w1, id) of policies.hpp:40-48
    unsigned long long w0 = 0, w1 = 0;
    int id = -1;
};

bool hkey_less(const HKey& a, const HKey& b) {
    if (a.w0 != b.w0) return a.w0 < b.w0;
    if (a.w1 != b.w1) return a.w1 < b.w1;
    return a.id < b.id;
}

HKey make_hkey(int cls, double rank, unsigned long long last, int id) {
    const unsigned long long e = host_enc_rank(rank);
    HKey k;
    k.w0 = (static_cast<unsigned long long>(cls) << 63) | (e >> 1);
    k.w1 = ((e & 1ull) << 63) | last;
    k.id = id;
    return k;
}

// The selection ran with heavy nodes out of the order (zero keys, not
// candidates).  Their exact scores lie in [A - B, A + B] (A the approximate
// sum, B = L * ulp(sum |x|)), so each one's (eff, d) record is either known
// exactly (a descendant's key beats its whole interval), or is its own key
// with a known interval.  If every eligible heavy node's record is provably
// after the last victim's, the cut is exact as computed.  Returns false when
// that cannot be proved (the caller then runs the exact chains).
bool place_deferred(Context& c, long long* result_dev, const SelectCounts& o, std::int64_t needed) {
    if (o.shortfall || o.n_victims == 0) return false;
    (void)result_dev;  // the reports were fetched with the selection's readback (run_select)
    const std::size_t nh = static_cast<std::size_t>(c.n_heavy);
    const std::size_t bytes = (nh + 1) * sizeof(HeavyReport);
    const HeavyReport* rep = reinterpret_cast<const HeavyReport*>(c.hreport_h.p);
    const double* ap = reinterpret_cast<const double*>(c.hreport_h.p + bytes);
    const HeavyReport& tail = rep[nh];
    if (tail.eff < 0) return false;
    HKey tkey;
    tkey.w0 = tail.w0;
    tkey.w1 = tail.w1;
    tkey.id = tail.eff;
    // record order (key, d) of the tail
    auto after_tail = [&](const HKey& k, int d) {
        if (hkey_less(tkey, k)) return true;
        if (hkey_less(k, tkey)) return false;
        return d > tail.depth_diff;
    };
    // heavy nodes deepest first (eff of a heavy node may come from a heavy
    // descendant); order and heavy-children lists are built at mirror time
    const std::vector<std::size_t>& order = c.h_heavy_order;
    struct Eff {
        HKey lo, hi;   // exact when lo == hi
        int depth = -1;
        bool any = false;
    };
    std::vector<Eff> eff(nh);
    std::vector<char> sub(nh, 0);
    for (std::size_t j : order) {
        const HeavyReport& r = rep[j];
        const int h = c.h_heavy[j];
        const int d = c.h_heavy_depth[j];
        const bool device = (c.h_heavy_flags[j] & kFlagTierMask) == PBKV_TIER_DEVICE;
        Eff best;
        if (r.eff >= 0) {
            best.lo.w0 = best.hi.w0 = r.w0;
            best.lo.w1 = best.hi.w1 = r.w1;
            best.lo.id = best.hi.id = r.eff;
            best.depth = r.eff_depth;
            best.any = true;
        }
        sub[j] = sub[j] || r.sublock;
        // heavy children already resolved (their eff covers their subtrees)
        for (int kq = c.h_heavy_kid_off[j]; kq < c.h_heavy_kid_off[j + 1]; ++kq) {
            const std::size_t q = static_cast<std::size_t>(c.h_heavy_kids[static_cast<std::size_t>(kq)]);
            if (!eff[q].any) continue;
            sub[j] = sub[j] || sub[q];
            if (!best.any || hkey_less(best.hi, eff[q].lo)) {
                best = eff[q];
            } else if (!hkey_less(eff[q].hi, best.lo)) {
                return false;  // overlapping intervals: order unknown
            }
        }
        if (device && h != 0) {
            const double A = ap[2 * j], S = ap[2 * j + 1];
            int ex = 0;
            std::frexp(S, &ex);
            const double L = static_cast<double>(c.h_entries[static_cast<std::size_t>(h)]) * c.K;
            const double B = S > 0.0 ? 2.0 * L * std::ldexp(1.0, ex - 53) : 0.0;
            if (!(std::isfinite(A) && std::isfinite(B))) return false;
            const bool retired = (c.h_heavy_flags[j] & kFlagRetired) != 0;
            if (retired) return false;  // not expected for a node with entries
            Eff own;
            own.lo = make_hkey(1, A - B, c.h_heavy_last[j], h);
            own.hi = make_hkey(1, A + B, c.h_heavy_last[j], h);
            own.depth = d;
            own.any = true;
            if (!best.any || hkey_less(best.hi, own.lo)) {
                best = own;
            } else if (!hkey_less(own.hi, best.lo)) {
                return false;  // own interval straddles the descendants' maximum
            }
        }
        eff[j] = best;
        if (!device || h == 0 || sub[j] || !best.any) continue;
        if (r.miss) return false;  // eligible with a missing forecast: the exact path raises
        if (!after_tail(best.lo, best.depth - d)) return false;
    }
    (void)needed;
    return true;
}

SelectCounts select_core(Context& c, int policy, int score_mode, std::int64_t needed, const int* locked_dev,
                         std::int64_t n_locked, long long* result_dev) {
    if (needed <= 0) invalid("eviction request must free a positive amount");
    if (policy < PBKV_POLICY_LRU || policy > PBKV_POLICY_KVFLOW) invalid("unknown eviction policy");
    if (policy == PBKV_POLICY_KVFLOW && !c.have_remaining) invalid("kvflow selected without static sequences");
    if (score_mode != PBKV_SCORE_CACHED && score_mode != PBKV_SCORE_RECOMPUTE)
        throw ApiError(PBKV_EARG, "bad score mode");
    need(c.n >= 1, "no tree mirrored");
    record(c, 0);
    const bool recompute = score_mode == PBKV_SCORE_RECOMPUTE && policy == PBKV_POLICY_HE;
    const bool defer = recompute && c.defer_heavy && c.n_heavy > 0 && c.spine.empty();
    if (defer) {
        launch_score_decision(c, policy);  // (its prologue: status reset + the deferral)
    } else if (recompute) {
        launch_decision_prologue(c, false, c.stream);  // status reset
        launch_score_all(c, c.score_rc.p, true, policy, false);
    } else {
        launch_decision_prologue(c, false, c.stream);
        launch_keys_cached(c, policy);
    }
    record(c, 1);
    c.report_deferred = defer;
    SelectCounts o = run_select(c, locked_dev, n_locked, needed, recompute, result_dev);
    c.report_deferred = false;
    if (defer) {
        const bool placed = place_deferred(c, result_dev ? result_dev : c.counters.p + 8, o, needed);
        if (!c.deferred_cleared) launch_set_deferred(c, false);
        c.deferred_cleared = false;
        if (placed) {
            ++c.defer_fast;
        } else {  // slow path: exact chains, full selection
            ++c.defer_slow;
            reset_status(c);
            launch_score_all(c, c.score_rc.p, true, policy, false);
            o = run_select(c, locked_dev, n_locked, needed, recompute, result_dev);
        }
    }
    record(c, 2);
    finish_timing(c, 2);
    static const bool dbg_t = std::getenv("PBKV_DEBUG_TIMING") != nullptr;
    if (dbg_t && c.timing) {
        float a = 0, b = 0, d = 0, e = 0;
        cudaEventElapsedTime(&a, c.ev[0], c.kev[0]);   // decision start -> light start
        cudaEventElapsedTime(&b, c.kev[1], c.kev[2]);  // light end -> select kernel start
        cudaEventElapsedTime(&d, c.kev[3], c.ev[2]);   // select kernel end -> decision end
        cudaEventElapsedTime(&e, c.ev[0], c.ev[2]);
        std::fprintf(stderr, "[pbkv timing] start->light %.1f us, light->select %.1f us, select->end %.1f us, total %.1f us\n",
                     a * 1e3, b * 1e3, d * 1e3, e * 1e3);
    }
    return o;
}

}  // namespace

// =============================================================================
extern "C" {

int pbkv_abi_version(void) { return PBKV_ABI_VERSION; }

const char* pbkv_last_error(const pbkv_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int pbkv_device_count(int* out) {
    return api(nullptr, [&] {
        need(out != nullptr, "null out");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        int good = 0;
        for (int d = 0; d < n; ++d) {
            cudaDeviceProp p{};
            if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++good;
        }
        *out = good;
    });
}

int pbkv_ctx_create(pbkv_ctx** out, const pbkv_cfg* cfg) {
    return api(nullptr, [&] {
        need(out && cfg, "null argument");
        *out = nullptr;
        if (cfg->k < 1) invalid("lookahead horizon must be >= 1");
        if (!(cfg->gamma > 0.0 && cfg->gamma < 1.0)) invalid("gamma must be in (0, 1)");
        if (cfg->k > 32) throw ApiError(PBKV_EARG, "pbkv supports lookahead horizons up to 32");
        if (cfg->num_agents < 1 || cfg->num_agents > 63) invalid("agent count must be in [1, 63]");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw ApiError(PBKV_ECUDA, "no CUDA device visible (pbkv has no CPU fallback)");
        }
        need(cfg->device >= 0 && cfg->device < n, "device ordinal out of range");
        cudaDeviceProp prop{};
        PBKV_CUDA(cudaGetDeviceProperties(&prop, cfg->device));
        if (prop.major != 10)
            throw ApiError(PBKV_ECUDA, "pbkv is built for sm_100a (B200); device " + std::string(prop.name) +
                                           " is not compute capability 10.x");
        auto c = std::make_unique<pbkv_ctx>();
        c->device = cfg->device;
        c->K = cfg->k;
        c->gamma = cfg->gamma;
        c->A = cfg->num_agents;
        c->V1 = cfg->num_agents + 1;
        PBKV_CUDA(cudaSetDevice(c->device));
        PBKV_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        {  // the side stream (medium / heavy chains) outranks the light pass for
           // free SM slots, so it finishes inside the light pass even when
           // enqueued after it (launch_score_decision)
            int lo = 0, hi = 0;
            PBKV_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            PBKV_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
        }
        for (auto& e : c->ev) PBKV_CUDA(cudaEventCreate(&e));
        for (auto& e : c->kev) PBKV_CUDA(cudaEventCreate(&e));
        PBKV_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        PBKV_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        PBKV_CUDA(cudaEventCreateWithFlags(&c->ev_delta, cudaEventDisableTiming));
        PBKV_CUDA(cudaEventCreateWithFlags(&c->ev_class, cudaEventDisableTiming));
        PBKV_CUDA(cudaEventCreateWithFlags(&c->ev_caller, cudaEventDisableTiming));
        PBKV_CUDA(cudaEventCreateWithFlags(&c->ev_rows, cudaEventDisableTiming));
        c->selstate.reserve(sel_state_bytes());
        c->hselstate.reserve(2 * sel_state_bytes());  // [0] readback, [1] initial-state template
        c->counters.reserve(16);
        c->status.reserve(1);
        c->hcounters.reserve(16);
        c->hstatus.reserve(1);
        c->P.reserve(64);
        c->gs.reserve(64);
        c->fstate.reserve(64);
        c->rem_has.reserve(64);
        reset_status(*c);
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
        *out = c.release();
    });
}

int pbkv_ctx_destroy(pbkv_ctx* c) {
    if (!c) return PBKV_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->side) cudaStreamSynchronize(c->side);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->kev)
        if (e) cudaEventDestroy(e);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_delta) cudaEventDestroy(c->ev_delta);
    if (c->ev_class) cudaEventDestroy(c->ev_class);
    if (c->ev_caller) cudaEventDestroy(c->ev_caller);
    if (c->ev_rows) cudaEventDestroy(c->ev_rows);
    cudaStream_t s = c->stream, side = c->side;
    delete c;  // DevBuf / PinBuf destructors free the device and pinned memory
    cudaStreamDestroy(s);
    if (side) cudaStreamDestroy(side);
    return PBKV_OK;
}

int pbkv_ctx_sync(pbkv_ctx* c) {
    return api(c, [&] {
        need(c, "null ctx");
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int pbkv_ctx_stream(pbkv_ctx* c, void** s) {
    return api(c, [&] {
        need(c && s, "null argument");
        *s = c->stream;
    });
}

int pbkv_ctx_timings(pbkv_ctx* c, float* ms5) {
    return api(c, [&] {
        need(c && ms5, "null argument");
        for (int i = 0; i < 5; ++i) ms5[i] = c->last_ms[i];
    });
}

int pbkv_ctx_set_timing(pbkv_ctx* c, int enabled) {
    return api(c, [&] {
        need(c, "null ctx");
        c->timing = enabled != 0;
    });
}

int pbkv_ctx_phase_times(pbkv_ctx* c, uint64_t* ns, int cap, int* n) {
    return api(c, [&] {
        need(c && n, "null argument");
        *n = static_cast<int>(c->phase_ns.size());
        for (int i = 0; i < *n && i < cap; ++i) ns[i] = c->phase_ns[static_cast<std::size_t>(i)];
    });
}

int pbkv_ctx_launches(pbkv_ctx* c, int64_t* kernels, int64_t* lib_calls) {
    return api(c, [&] {
        need(c, "null ctx");
        if (kernels) *kernels = c->launches;
        if (lib_calls) *lib_calls = c->lib_calls;
    });
}

int pbkv_ctx_wait_stream(pbkv_ctx* c, void* stream) {
    return api(c, [&] {
        need(c, "null ctx");
        set_device(*c);
        PBKV_CUDA(cudaEventRecord(c->ev_caller, static_cast<cudaStream_t>(stream)));
        PBKV_CUDA(cudaStreamWaitEvent(c->stream, c->ev_caller, 0));
    });
}

int pbkv_ctx_kernel_timings(pbkv_ctx* c, float* ms2) {
    return api(c, [&] {
        need(c && ms2, "null argument");
        ms2[0] = c->kernel_ms[0];
        ms2[1] = c->kernel_ms[1];
    });
}

int pbkv_ctx_set_defer(pbkv_ctx* c, int enabled) {
    return api(c, [&] {
        need(c, "null ctx");
        c->defer_heavy = enabled != 0;
    });
}

int pbkv_ctx_defer_stats(pbkv_ctx* c, int64_t* fast, int64_t* slow) {
    return api(c, [&] {
        need(c, "null ctx");
        if (fast) *fast = c->defer_fast;
        if (slow) *slow = c->defer_slow;
    });
}

int pbkv_mirror_full(pbkv_ctx* c, const pbkv_tree_soa* soa) {
    return api(c, [&] {
        need(c && soa, "null argument");
        set_device(*c);
        mirror_full(*c, *soa);
    });
}

int pbkv_mirror_delta(pbkv_ctx* c, const pbkv_node_delta* nodes, int64_t n, const int64_t* acc_wf,
                      const uint64_t* acc_bits, const pbkv_tree_totals* totals) {
    return api(c, [&] {
        need(c != nullptr, "null ctx");
        need(n >= 0, "negative record count");
        set_device(*c);
        mirror_delta(*c, nodes, n, acc_wf, acc_bits, totals);
    });
}

int pbkv_mirror_verify(pbkv_ctx* c, const pbkv_tree_soa* soa, int64_t* mismatch) {
    return api(c, [&] {
        need(c && soa && mismatch, "null argument");
        need(c->n >= 1, "no tree mirrored");
        set_device(*c);
        *mismatch = mirror_verify(*c, *soa);
    });
}

int pbkv_mirror_set_scores(pbkv_ctx* c, const int32_t* ids, const double* scores, int64_t n) {
    return api(c, [&] {
        need(c && (n == 0 || (ids && scores)), "null argument");
        set_device(*c);
        for (int64_t i = 0; i < n; ++i) need(ids[i] >= 0 && ids[i] < c->n, "node id out of range");
        // small batches: individual copies are fine (the simulator refreshes a handful of nodes)
        for (int64_t i = 0; i < n; ++i)
            PBKV_CUDA(cudaMemcpyAsync(c->score.p + ids[i], scores + i, sizeof(double), cudaMemcpyHostToDevice,
                                      c->stream));
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int pbkv_mirror_node_count(pbkv_ctx* c, int64_t* n_nodes, int64_t* n_entries) {
    return api(c, [&] {
        need(c, "null ctx");
        if (n_nodes) *n_nodes = c->n;
        if (n_entries) *n_entries = c->E;
    });
}

static int forecast_put_impl(pbkv_ctx* c, const int64_t* wf, int64_t n, int horizon, int outcomes, const double* p,
                             bool async) {
    return api(c, [&] {
        need(c && (n == 0 || (wf && p)), "null argument");
        if (horizon < 1) invalid("forecast horizon must be >= 1");
        if (outcomes < 2) invalid("forecast needs at least one agent plus END");
        if (outcomes != c->V1) invalid("forecast outcomes do not match the context's agent count");
        if (n == 0) return;
        set_device(*c);
        c->hslots.reserve(static_cast<std::size_t>(n));  // pinned: the H2D below stays asynchronous
        long long* slots = c->hslots.p;
        for (int64_t i = 0; i < n; ++i) slots[i] = slot_for(*c, wf[i]);
        const std::size_t per = static_cast<std::size_t>(horizon) * static_cast<std::size_t>(outcomes);
        c->fstage.reserve(static_cast<std::size_t>(n) * per);
        c->fstage_slot.reserve(static_cast<std::size_t>(n));
        if (!c->status_pending) reset_status(*c);
        if (async) c->status_pending = true;  // checked by the next call that reads the status word
        // pageable rows go through pinned staging, so the copy stays
        // asynchronous; pinned (or registered) caller memory is copied directly
        const std::size_t bytes = static_cast<std::size_t>(n) * per * sizeof(double);
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        const double* src = p;
        if (!pinned) {
            PBKV_CUDA(cudaEventSynchronize(c->ev_rows));  // the previous staged copy has drained
            c->hrows.reserve(static_cast<std::size_t>(n) * per);
            std::memcpy(c->hrows.p, p, bytes);
            src = c->hrows.p;
        }
        PBKV_CUDA(cudaMemcpyAsync(c->fstage.p, src, bytes, cudaMemcpyHostToDevice, c->stream));
        if (!pinned) PBKV_CUDA(cudaEventRecord(c->ev_rows, c->stream));
        PBKV_CUDA(cudaMemcpyAsync(c->fstage_slot.p, slots, static_cast<std::size_t>(n) * sizeof(long long),
                                  cudaMemcpyHostToDevice, c->stream));
        launch_forecast_prepare(*c, c->fstage.p, c->fstage_slot.p, n, horizon);
        if (!async) check_status(*c);
    });
}

int pbkv_forecast_put(pbkv_ctx* c, const int64_t* wf, int64_t n, int horizon, int outcomes, const double* p) {
    return forecast_put_impl(c, wf, n, horizon, outcomes, p, false);
}

int pbkv_forecast_put_async(pbkv_ctx* c, const int64_t* wf, int64_t n, int horizon, int outcomes, const double* p) {
    return forecast_put_impl(c, wf, n, horizon, outcomes, p, true);
}

int pbkv_forecast_drop(pbkv_ctx* c, const int64_t* wf, int64_t n) {
    return api(c, [&] {
        need(c && (n == 0 || wf), "null argument");
        set_device(*c);
        for (int64_t i = 0; i < n; ++i) {
            auto it = c->slot_of.find(wf[i]);
            if (it == c->slot_of.end()) continue;
            PBKV_CUDA(cudaMemsetAsync(c->fstate.p + it->second, 0, 1, c->stream));
            poison_slot(*c, static_cast<std::size_t>(it->second));
        }
        // stream-ordered: every later call on the context sees the drop
    });
}

int pbkv_forecast_clear(pbkv_ctx* c) {
    return api(c, [&] {
        need(c, "null ctx");
        set_device(*c);
        if (c->n_slots > 0) {
            const std::size_t rows = static_cast<std::size_t>(c->n_slots) * c->K * c->V1;
            PBKV_CUDA(cudaMemsetAsync(c->fstate.p, 0, static_cast<std::size_t>(c->n_slots), c->stream));
            PBKV_CUDA(cudaMemsetAsync(c->P.p, 0xFF, rows * sizeof(double), c->stream));
            PBKV_CUDA(cudaMemsetAsync(c->Pg.p, 0xFF, rows * sizeof(double), c->stream));
        }
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int pbkv_score_all(pbkv_ctx* c, double* scores_out) {
    return api(c, [&] {
        need(c, "null ctx");
        need(c->n >= 1, "no tree mirrored");
        set_device(*c);
        reset_status(*c);
        record(*c, 0);
        launch_score_all(*c, c->score_rc.p, false, PBKV_POLICY_HE, true);
        record(*c, 1);
        check_status(*c);
        finish_timing(*c, 1);
        if (scores_out)
            PBKV_CUDA(cudaMemcpy(scores_out, c->score_rc.p, static_cast<std::size_t>(c->n) * sizeof(double),
                                 cudaMemcpyDeviceToHost));
    });
}

static int score_ids_impl(pbkv_ctx* c, const int32_t* ids, int64_t n, double* out, bool value_only) {
    return api(c, [&] {
        need(c && (n == 0 || (ids && out)), "null argument");
        if (n == 0) return;
        set_device(*c);
        for (int64_t i = 0; i < n; ++i) need(ids[i] >= 0 && ids[i] < c->n, "node id out of range");
        c->ids.reserve(static_cast<std::size_t>(n));
        c->vals.reserve(static_cast<std::size_t>(n));
        reset_status(*c);
        // ids in and values + status out through pinned staging: one synchronisation
        c->hids.reserve(static_cast<std::size_t>(n));
        c->hvals.reserve(static_cast<std::size_t>(n));
        std::memcpy(c->hids.p, ids, static_cast<std::size_t>(n) * sizeof(int));
        PBKV_CUDA(cudaMemcpyAsync(c->ids.p, c->hids.p, n * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        launch_score_ids(*c, c->ids.p, ids, n, c->score_rc.p, value_only);
        launch_gather_f64(*c, c->score_rc.p, c->ids.p, n, c->vals.p);
        PBKV_CUDA(cudaMemcpyAsync(c->hvals.p, c->vals.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        PBKV_CUDA(cudaMemcpyAsync(c->hstatus.p, c->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, c->stream));
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
        const DevStatus st = *c->hstatus.p;
        raise_status(*c, st);
        std::memcpy(out, c->hvals.p, static_cast<std::size_t>(n) * sizeof(double));
    });
}

int pbkv_score_nodes(pbkv_ctx* c, const int32_t* ids, int64_t n, double* out) {
    return score_ids_impl(c, ids, n, out, false);
}

int pbkv_value_nodes(pbkv_ctx* c, const int32_t* ids, int64_t n, double* out) {
    return score_ids_impl(c, ids, n, out, true);
}

int pbkv_select(pbkv_ctx* c, int policy, int score_mode, int64_t needed, const int32_t* locked, int64_t n_locked,
                int32_t* victims, int64_t cap, int64_t* n_victims, int64_t* freed, int* shortfall) {
    return api(c, [&] {
        need(c && n_victims && freed && shortfall, "null argument");
        need(n_locked == 0 || locked, "null locked array");
        set_device(*c);
        c->locked.reserve(static_cast<std::size_t>(n_locked) + 1);
        if (n_locked > 0) {
            // through pinned staging: a pageable source would make the copy
            // (and every launch behind it) wait for the driver's staging
            c->hlocked.reserve(static_cast<std::size_t>(n_locked));
            std::memcpy(c->hlocked.p, locked, static_cast<std::size_t>(n_locked) * sizeof(int));
            PBKV_CUDA(cudaMemcpyAsync(c->locked.p, c->hlocked.p, n_locked * sizeof(int), cudaMemcpyHostToDevice,
                                      c->stream));
        }
        // the decision's epilogue kernel stores up to kEpiVictims victim ids
        // straight into pinned memory, so the common cut needs no copy after
        // the decision's synchronisation
        constexpr long long kEpiVictims = 1 << 16;
        c->hvictims.reserve(static_cast<std::size_t>(kEpiVictims));
        c->epi_vict = c->hvictims.p;
        c->epi_cap = std::min<long long>(kEpiVictims, cap);
        SelectCounts o;
        try {
            o = select_core(*c, policy, score_mode, needed, c->locked.p, n_locked, nullptr);
        } catch (...) {
            c->epi_vict = nullptr;
            throw;
        }
        c->epi_vict = nullptr;
        *n_victims = o.n_victims;
        *freed = o.freed;
        *shortfall = o.shortfall;
        if (o.n_victims > cap) throw ApiError(PBKV_EARG, "victim capacity too small");
        if (o.n_victims > 0) {
            need(victims != nullptr, "null victims array");
            if (o.n_victims > c->epi_cap || !c->epi_vict_valid) {
                c->hvictims.reserve(static_cast<std::size_t>(o.n_victims));
                PBKV_CUDA(cudaMemcpyAsync(c->hvictims.p, c->vid_out.p, o.n_victims * sizeof(int),
                                          cudaMemcpyDeviceToHost, c->stream));
                PBKV_CUDA(cudaStreamSynchronize(c->stream));
            }
            std::memcpy(victims, c->hvictims.p, static_cast<std::size_t>(o.n_victims) * sizeof(int));
        }
    });
}

int pbkv_select_dev(pbkv_ctx* c, int policy, int score_mode, int64_t needed, const int32_t* locked_dev,
                    int64_t n_locked, int32_t* victims_dev, int64_t cap, int64_t* result_dev) {
    return api(c, [&] {
        need(c && result_dev, "null argument");
        need(n_locked == 0 || locked_dev, "null locked array");
        set_device(*c);
        SelectCounts o = select_core(*c, policy, score_mode, needed, locked_dev, n_locked,
                                     reinterpret_cast<long long*>(result_dev));
        if (o.n_victims > cap) throw ApiError(PBKV_EARG, "victim capacity too small");
        if (o.n_victims > 0) {
            need(victims_dev != nullptr, "null victims array");
            PBKV_CUDA(cudaMemcpyAsync(victims_dev, c->vid_out.p, o.n_victims * sizeof(int), cudaMemcpyDeviceToDevice,
                                      c->stream));
        }
    });
}

int pbkv_set_remaining(pbkv_ctx* c, const int64_t* wf, int64_t n_wf, const int64_t* seq_off, const int32_t* seq) {
    return api(c, [&] {
        need(c && (n_wf == 0 || (wf && seq_off)), "null argument");
        set_device(*c);
        std::vector<int> slots(static_cast<std::size_t>(n_wf));
        for (int64_t i = 0; i < n_wf; ++i) slots[static_cast<std::size_t>(i)] = slot_for(*c, wf[i]);
        // per-slot CSR (slots without a sequence get an empty range + has=0)
        const std::size_t ns = static_cast<std::size_t>(c->n_slots);
        std::vector<int> off(ns + 1, 0), cnt(ns, 0);
        std::vector<std::uint8_t> has(ns, 0);
        for (int64_t i = 0; i < n_wf; ++i) {
            std::size_t s = static_cast<std::size_t>(slots[static_cast<std::size_t>(i)]);
            cnt[s] = static_cast<int>(seq_off[i + 1] - seq_off[i]);
            has[s] = 1;
        }
        for (std::size_t s = 0; s < ns; ++s) off[s + 1] = off[s] + cnt[s];
        std::vector<int> flat(static_cast<std::size_t>(off[ns]) + 1);
        for (int64_t i = 0; i < n_wf; ++i) {
            std::size_t s = static_cast<std::size_t>(slots[static_cast<std::size_t>(i)]);
            for (int64_t k = seq_off[i]; k < seq_off[i + 1]; ++k)
                flat[static_cast<std::size_t>(off[s] + (k - seq_off[i]))] = seq[k];
        }
        c->rem_off.reserve(ns + 1);
        c->rem_seq.reserve(flat.size());
        PBKV_CUDA(cudaMemcpyAsync(c->rem_off.p, off.data(), (ns + 1) * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        PBKV_CUDA(cudaMemcpyAsync(c->rem_seq.p, flat.data(), flat.size() * sizeof(int), cudaMemcpyHostToDevice,
                                  c->stream));
        if (ns) PBKV_CUDA(cudaMemcpyAsync(c->rem_has.p, has.data(), ns, cudaMemcpyHostToDevice, c->stream));
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
        c->have_remaining = true;
    });
}

namespace {
// the last plan's arrays (pinned host memory) into the caller's
void copy_plan(const Context& c, int32_t* cand_ids, double* cand_values, int64_t cand_cap, int32_t* selected,
               int64_t sel_cap) {
    const PrefetchOut& o = c.plan_out;
    const std::int64_t mc = std::min<std::int64_t>(cand_cap, o.ctr[0]);
    if (mc > 0 && cand_ids) std::memcpy(cand_ids, o.cand, static_cast<std::size_t>(mc) * sizeof(int32_t));
    if (mc > 0 && cand_values) std::memcpy(cand_values, o.val, static_cast<std::size_t>(mc) * sizeof(double));
    const std::int64_t ms = std::min<std::int64_t>(sel_cap, o.ctr[1]);
    if (ms > 0 && selected) std::memcpy(selected, o.sel, static_cast<std::size_t>(ms) * sizeof(int32_t));
}
}  // namespace

int pbkv_plan_prefetch(pbkv_ctx* c, int64_t bandwidth, int step_duration, double rho, int32_t* cand_ids,
                       double* cand_values, int64_t cand_cap, int32_t* selected, int64_t sel_cap,
                       pbkv_prefetch_plan* plan) {
    return api(c, [&] {
        need(c && plan, "null argument");
        need(c->n >= 1, "no tree mirrored");
        std::int64_t extra = 0;
        if (!(rho < 0.0)) {
            if (rho < 0.0 || rho > 1.0 || rho != rho) invalid("rho must be in [0, 1]");
            extra = static_cast<std::int64_t>(rho * static_cast<double>(c->device_capacity));
        }
        set_device(*c);
        std::memset(plan, 0, sizeof *plan);
        plan->budget_space = (c->device_capacity - c->device_used) + c->retired_device_tokens;
        plan->budget_bw = bandwidth * static_cast<std::int64_t>(step_duration);
        plan->displacement_budget = extra;
        const long long budget = std::min(plan->budget_space + extra, plan->budget_bw);
        record(*c, 0);
        reset_status(*c);
        c->plan_valid = false;
        PrefetchOut o;
        run_prefetch_plan(*c, budget, &o);  // one synchronisation
        record(*c, 1);
        finish_timing(*c, 1);
        const std::int64_t nc = o.ctr[0];
        plan->n_candidates = nc;
        plan->n_selected = o.ctr[1];
        plan->selected_tokens = o.ctr[2];
        c->plan_out = o;
        c->plan_valid = true;
        copy_plan(*c, cand_ids, cand_values, cand_cap, selected, sel_cap);
    });
}

int pbkv_plan_fetch(pbkv_ctx* c, int32_t* cand_ids, double* cand_values, int64_t cand_cap, int32_t* selected,
                    int64_t sel_cap) {
    return api(c, [&] {
        need(c != nullptr, "null ctx");
        need(c->plan_valid, "no prefetch plan to fetch");
        copy_plan(*c, cand_ids, cand_values, cand_cap, selected, sel_cap);
    });
}

// ---- the prefetch round (simulator.hpp:632-681), conservative mode -------------------
// The reference admits the plan's candidates one by one: when candidate i does
// not fit in free device space it runs select_victims_hierarchical(need_i)
// under locks on the remaining candidates' ancestry and the pinned paths, and
// takes that order's retired prefix (a conservative round never displaces
// active cache); short of need_i the candidate is skipped.  Every lock is
// active (a candidate has value > 0, so its parent and ancestors carry active
// access tags; pinned paths belong to decoding workflows), a lock only makes
// ancestors ineligible, and retired subtrees hold only retired nodes -- so the
// retired nodes' order is the same under every candidate's lock set, and a
// promoted candidate (active) never enters it.  The greedy frontier resumes
// where a demoted prefix ended.  Hence the whole round is ONE hierarchical
// decision for the round's total length followed by a scan that hands each
// candidate the next retired victims (device_free bookkeeping as the
// reference: demotions add, promotions subtract).
int pbkv_prefetch_round(pbkv_ctx* c, const int32_t* selected, int64_t n_sel, int64_t device_free, int32_t* promoted,
                        int64_t* victim_end, int32_t* victims, int64_t cap, int64_t* n_victims) {
    return api(c, [&] {
        need(c && n_victims && (n_sel == 0 || (selected && promoted && victim_end)), "null argument");
        need(c->n >= 1, "no tree mirrored");
        set_device(*c);
        *n_victims = 0;
        std::int64_t total = 0;
        for (int64_t i = 0; i < n_sel; ++i) {
            need(selected[i] > 0 && selected[i] < c->n, "prefetch round: candidate id out of range");
            total += c->h_len[static_cast<std::size_t>(selected[i])];
        }
        std::vector<int> order;  // the hierarchical victim order for the round's total length
        if (total > 0) {
            constexpr long long kEpiVictims = 1 << 16;
            c->hvictims.reserve(static_cast<std::size_t>(kEpiVictims));
            c->epi_vict = c->hvictims.p;
            c->epi_cap = kEpiVictims;
            SelectCounts o;
            try {
                o = select_core(*c, PBKV_POLICY_HE, PBKV_SCORE_CACHED, total, nullptr, 0, nullptr);
            } catch (...) {
                c->epi_vict = nullptr;
                throw;
            }
            c->epi_vict = nullptr;
            if (o.n_victims > c->epi_cap || !c->epi_vict_valid) {
                c->hvictims.reserve(static_cast<std::size_t>(o.n_victims));
                PBKV_CUDA(cudaMemcpyAsync(c->hvictims.p, c->vid_out.p, o.n_victims * sizeof(int), cudaMemcpyDeviceToHost,
                                          c->stream));
                PBKV_CUDA(cudaStreamSynchronize(c->stream));
            }
            order.assign(c->hvictims.p, c->hvictims.p + o.n_victims);
        }
        // the reference's per-candidate loop over the one order
        std::size_t at = 0;
        std::int64_t out = 0, free_tok = device_free;
        for (int64_t i = 0; i < n_sel; ++i) {
            const std::size_t id = static_cast<std::size_t>(selected[i]);
            promoted[i] = 0;
            const bool host = (c->h_flags[id] & kFlagTierMask) == PBKV_TIER_HOST;
            const int p = c->h_parent[id];
            const bool dev_parent = p >= 0 && (c->h_flags[static_cast<std::size_t>(p)] & kFlagTierMask) == PBKV_TIER_DEVICE;
            if (host && dev_parent) {  // simulator.hpp:647-648
                const std::int64_t len = c->h_len[id];
                const std::int64_t needt = len - free_tok;
                bool admit = true;
                if (needt > 0) {  // :650-671: the retired prefix of the order from `at`
                    std::size_t q = at;
                    std::int64_t freed = 0;
                    while (q < order.size() && freed < needt &&
                           (c->h_flags[static_cast<std::size_t>(order[q])] & kFlagRetired)) {
                        freed += c->h_len[static_cast<std::size_t>(order[q])];
                        ++q;
                    }
                    if (freed < needt) {
                        admit = false;  // :671 cannot admit this candidate safely
                    } else {
                        if (out + static_cast<std::int64_t>(q - at) > cap) throw ApiError(PBKV_EARG, "victim capacity too small");
                        if (q > at) std::memcpy(victims + out, order.data() + at, (q - at) * sizeof(int32_t));
                        out += static_cast<std::int64_t>(q - at);
                        at = q;
                        free_tok += freed;
                    }
                }
                if (admit) {
                    promoted[i] = 1;
                    free_tok -= len;
                }
            }
            victim_end[i] = out;
        }
        *n_victims = out;
    });
}

// ---- sharding ---------------------------------------------------------------------
int pbkv_shard_set(pbkv_ctx* c, const int32_t* global_ids, const int32_t* spine, int64_t n_spine) {
    return api(c, [&] {
        need(c && global_ids && (n_spine == 0 || spine), "null argument");
        need(c->n >= 1, "no tree mirrored");
        set_device(*c);
        c->spine.assign(spine, spine + n_spine);
        std::vector<char> is_sp(static_cast<std::size_t>(c->n), 0);
        for (int v : c->spine) {
            need(v >= 0 && v < c->n, "shard spine id out of range");
            is_sp[static_cast<std::size_t>(v)] = 1;
        }
        // local tie-breaks (node id) must agree with global ones among the
        // nodes that can be candidates: global ids increase with local ids
        long long prev = LLONG_MIN;
        for (int64_t i = 1; i < c->n; ++i) {
            if (is_sp[static_cast<std::size_t>(i)]) continue;
            need(global_ids[i] > prev, "shard global ids must increase with local ids (non-spine nodes)");
            prev = global_ids[i];
        }
        c->gid.reserve(static_cast<std::size_t>(c->n));
        PBKV_CUDA(cudaMemcpyAsync(c->gid.p, global_ids, static_cast<std::size_t>(c->n) * sizeof(int),
                                  cudaMemcpyHostToDevice, c->stream));
        shard_apply_flags(*c);
        upload_children(*c, c->spine, c->sch_off, c->sch);
        c->h_spine.assign(is_sp.begin(), is_sp.end());
        classify_all(*c);  // the spine leaves the local medium / heavy chains
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int pbkv_shard_select(pbkv_ctx* c, int policy, int score_mode, int64_t needed, const int32_t* locked_dev,
                      int64_t n_locked, pbkv_cand* cand_dev, int64_t cap, pbkv_spine_info* spine_dev,
                      int64_t* result_dev) {
    return api(c, [&] {
        need(c && cand_dev && result_dev, "null argument");
        need(c->gid.p != nullptr, "pbkv_shard_set not called");
        need(n_locked == 0 || locked_dev, "null locked array");
        need(c->spine.empty() || spine_dev, "null spine output");
        if (policy == PBKV_POLICY_KVFLOW) throw ApiError(PBKV_EARG, "kvflow is not supported on a sharded tree");
        set_device(*c);
        long long* res = reinterpret_cast<long long*>(result_dev);
        SelectCounts o = select_core(*c, policy, score_mode, needed, locked_dev, n_locked, res);
        if (o.n_victims > cap) throw ApiError(PBKV_EARG, "candidate capacity too small");
        shard_records(*c, res, cand_dev, cap);
        shard_spine_report(*c, spine_dev);
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int pbkv_shard_spine_products(pbkv_ctx* c, double* out_dev, int64_t* counts) {
    return api(c, [&] {
        need(c && counts, "null argument");
        set_device(*c);
        const std::size_t ns = c->spine.size();
        std::vector<long long> base(ns + 1, 0);
        long long mx = 0;
        for (std::size_t j = 0; j < ns; ++j) {
            const long long L = static_cast<long long>(c->h_entries[static_cast<std::size_t>(c->spine[j])]) * c->K;
            counts[j] = L;
            base[j + 1] = base[j] + L;
            mx = std::max(mx, L);
        }
        if (ns == 0 || base[ns] == 0) return;
        need(out_dev != nullptr, "null products array");
        c->spine_base.reserve(ns + 1);
        c->spine_miss.reserve(1);
        PBKV_CUDA(cudaMemcpyAsync(c->spine_base.p, base.data(), (ns + 1) * sizeof(long long), cudaMemcpyHostToDevice,
                                  c->stream));
        PBKV_CUDA(cudaMemsetAsync(c->spine_miss.p, 0, sizeof(unsigned int), c->stream));
        shard_spine_products(*c, c->spine_base.p, mx, out_dev, c->spine_miss.p);
        unsigned int miss = 0;
        PBKV_CUDA(cudaMemcpyAsync(&miss, c->spine_miss.p, sizeof miss, cudaMemcpyDeviceToHost, c->stream));
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
        if (miss) invalid("missing forecast for a workflow tagged on a spine node");
    });
}

int pbkv_chain_sum(pbkv_ctx* c, const double* x_dev, const int64_t* off, int n_seg, double* out) {
    return api(c, [&] {
        need(c && off && out && n_seg >= 0, "null argument");
        if (n_seg == 0) return;
        need(x_dev || off[n_seg] == 0, "null products array");
        for (int b = 0; b < n_seg; ++b) need(off[b + 1] >= off[b], "chain offsets must not decrease");
        set_device(*c);
        c->run_start.reserve(static_cast<std::size_t>(n_seg) + 1);
        c->vals.reserve(static_cast<std::size_t>(n_seg));
        PBKV_CUDA(cudaMemcpyAsync(c->run_start.p, off, (static_cast<std::size_t>(n_seg) + 1) * sizeof(long long),
                                  cudaMemcpyHostToDevice, c->stream));
        launch_chain_sum(*c, x_dev, c->run_start.p, n_seg, c->vals.p);
        PBKV_CUDA(cudaMemcpyAsync(out, c->vals.p, static_cast<std::size_t>(n_seg) * sizeof(double),
                                  cudaMemcpyDeviceToHost, c->stream));
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int pbkv_interval_sums(pbkv_ctx* c, const double* x_dev, const int64_t* pieces, const int64_t* out_off, int n_out,
                       double* out) {
    return api(c, [&] {
        need(c && pieces && out_off && out && n_out >= 0, "null argument");
        if (n_out == 0) return;
        need(out_off[0] == 0, "out_off must start at 0");
        const int64_t np = out_off[n_out];
        for (int j = 0; j < n_out; ++j) need(out_off[j + 1] >= out_off[j], "out_off must not decrease");
        for (int64_t q = 0; q < np; ++q) need(pieces[2 * q] >= 0 && pieces[2 * q + 1] >= pieces[2 * q], "bad piece");
        need(np == 0 || x_dev, "null array");
        set_device(*c);
        // pieces and offsets through one pinned staging blob; sums straight into pinned memory
        const std::size_t b_p = static_cast<std::size_t>(2 * np) * sizeof(long long);
        const std::size_t b_o = (static_cast<std::size_t>(n_out) + 1) * sizeof(long long);
        const std::size_t b_r = static_cast<std::size_t>(2 * n_out) * sizeof(double);
        c->his.reserve(b_p + b_o + b_r);
        c->dis.reserve(b_p + b_o + 8);
        unsigned char* h = c->his.p;
        if (b_p) std::memcpy(h, pieces, b_p);
        std::memcpy(h + b_p, out_off, b_o);
        PBKV_CUDA(cudaMemcpyAsync(c->dis.p, h, b_p + b_o, cudaMemcpyHostToDevice, c->stream));
        double* res = reinterpret_cast<double*>(h + b_p + b_o);
        launch_interval_sums(*c, x_dev, reinterpret_cast<const long long*>(c->dis.p),
                             reinterpret_cast<const long long*>(c->dis.p + b_p), n_out, res);
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
        std::memcpy(out, res, b_r);
    });
}

int pbkv_merge_cut(pbkv_ctx* c, const pbkv_cand* runs_dev, const int64_t* run_start, const int64_t* run_len,
                   int n_runs, int64_t needed, int32_t* victims_dev, int64_t* result_dev) {
    return api(c, [&] {
        need(c && run_start && run_len && victims_dev && result_dev && n_runs >= 0, "null argument");
        if (needed <= 0) invalid("eviction request must free a positive amount");
        set_device(*c);
        long long total = 0, mx = 0;
        for (int r = 0; r < n_runs; ++r) {
            need(run_len[r] >= 0 && run_start[r] >= 0, "bad run extent");
            total += run_len[r];
            mx = std::max<long long>(mx, run_len[r]);
        }
        need(total == 0 || runs_dev, "null runs array");
        c->merged.reserve(static_cast<std::size_t>(total) + 1);
        c->run_start.reserve(static_cast<std::size_t>(n_runs) + 1);
        c->run_len.reserve(static_cast<std::size_t>(n_runs) + 1);
        if (n_runs > 0) {
            PBKV_CUDA(cudaMemcpyAsync(c->run_start.p, run_start, n_runs * sizeof(long long), cudaMemcpyHostToDevice,
                                      c->stream));
            PBKV_CUDA(cudaMemcpyAsync(c->run_len.p, run_len, n_runs * sizeof(long long), cudaMemcpyHostToDevice,
                                      c->stream));
        }
        shard_merge_cut(*c, runs_dev, c->run_start.p, c->run_len.p, n_runs, mx, total, c->merged.p, needed,
                        victims_dev, reinterpret_cast<long long*>(result_dev));
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// ---- reference forecasters (oracle / Markov / noisy) --------------------------------
int pbkv_fmodel_load(pbkv_ctx* c, const pbkv_fmodel* m) {
    return api(c, [&] {
        need(c && m, "null argument");
        if (m->num_agents != c->A) invalid("model agent count does not match the context's");
        need(m->n_states >= 1 && m->n_states < (1ll << 24), "model state count out of range");
        need(m->rows && m->next, "model arrays missing");
        const std::size_t S = static_cast<std::size_t>(m->n_states), V1 = static_cast<std::size_t>(c->V1);
        for (std::size_t i = 0; i < S * static_cast<std::size_t>(c->A); ++i)
            need(m->next[i] >= -1 && m->next[i] < m->n_states, "model next-state index out of range");
        set_device(*c);
        c->fm_rows.reserve(S * V1);
        c->fm_next.reserve(S * static_cast<std::size_t>(c->A));
        PBKV_CUDA(cudaMemcpyAsync(c->fm_rows.p, m->rows, S * V1 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        PBKV_CUDA(cudaMemcpyAsync(c->fm_next.p, m->next, S * c->A * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        PBKV_CUDA(cudaStreamSynchronize(c->stream));
        c->fm_states = m->n_states;
    });
}

int pbkv_forecast_propagate(pbkv_ctx* c, const int64_t* wf, int64_t n, const int32_t* start_state, int horizon,
                            double lambda, double* probs_out) {
    return api(c, [&] {
        need(c, "null ctx");
        if (c->fm_states < 1) throw ApiError(PBKV_EARG, "no forecaster model loaded (pbkv_fmodel_load)");
        if (horizon < 1) invalid("horizon must be >= 1");
        if (lambda >= 0.0 && lambda > 1.0) invalid("noise level must be in [0, 1]");
        if (n == 0) return;
        need(wf && start_state, "null argument");
        set_device(*c);
        std::vector<long long> slots(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) slots[static_cast<std::size_t>(i)] = slot_for(*c, wf[i]);
        const std::size_t per = static_cast<std::size_t>(horizon) * c->V1;
        c->fstage.reserve(static_cast<std::size_t>(n) * per);
        c->fstage_slot.reserve(static_cast<std::size_t>(n));
        c->fm_start.reserve(static_cast<std::size_t>(n));
        cudaStream_t st = c->stream;
        PBKV_CUDA(cudaMemcpyAsync(c->fstage_slot.p, slots.data(), slots.size() * sizeof(long long),
                                  cudaMemcpyHostToDevice, st));
        PBKV_CUDA(cudaMemcpyAsync(c->fm_start.p, start_state, static_cast<std::size_t>(n) * sizeof(int),
                                  cudaMemcpyHostToDevice, st));
        reset_status(*c);
        launch_propagate(*c, c->fm_start.p, n, horizon, lambda < 0.0 ? -1.0 : lambda);
        check_status(*c);  // a propagation error precedes the Forecast checks
        launch_forecast_prepare(*c, c->fstage.p, c->fstage_slot.p, n, horizon);
        if (probs_out)
            PBKV_CUDA(cudaMemcpyAsync(probs_out, c->fstage.p, static_cast<std::size_t>(n) * per * sizeof(double),
                                      cudaMemcpyDeviceToHost, st));
        check_status(*c);
    });
}

// ---- stage 1: predictor ----------------------------------------------------------
int pbkv_predictor_load(pbkv_ctx* c, const pbkv_predictor_cfg* cfg, const pbkv_predictor_weights* w) {
    return api(c, [&] {
        need(c && cfg && w, "null argument");
        need(w->embed && w->transition && w->sage1 && w->sage2 && w->query && w->text && w->mlp1 && w->mlp1_bias &&
                 w->mlp2 && w->mlp2_bias,
             "predictor weights: missing array");
        if (cfg->num_agents != c->A) invalid("predictor agent count does not match the context's");
        if (cfg->horizon < 1) invalid("forecast horizon must be >= 1");
        need(cfg->dim == 64, "predictor dim must be 64 (one UMMA N tile)");
        need(cfg->text_dim >= 64 && cfg->text_dim % 64 == 0, "predictor text_dim must be a positive multiple of 64");
        need(cfg->hidden >= 1 && cfg->hidden <= 256, "predictor hidden width must be in [1, 256]");
        need(cfg->max_prefix >= 1, "predictor max_prefix must be >= 1");
        need(cfg->horizon * (cfg->num_agents + 1) <= 1024, "predictor K*(A+1) must be <= 1024");
        set_device(*c);
        predictor_load(*c, *cfg, *w);
    });
}

int pbkv_predict(pbkv_ctx* c, const int64_t* wf, int64_t n, const int64_t* prefix_off, const int32_t* prefix,
                 const uint16_t* x, int x_on_device, double* probs_out) {
    return api(c, [&] {
        need(c, "null ctx");
        if (!c->pred) throw ApiError(PBKV_EARG, "no predictor loaded (pbkv_predictor_load)");
        if (n == 0) return;
        need(wf && prefix_off && prefix && x, "null argument");
        set_device(*c);
        const pbkv_predictor_cfg cfg = predictor_cfg(*c);
        need(prefix_off[0] == 0, "prefix offsets must start at 0");
        const int64_t np = prefix_off[n];
        // one pinned blob -> one asynchronous upload: [slots (i64) | offsets (i32) | prefix (i32)]
        const std::size_t b_slots = static_cast<std::size_t>(n) * sizeof(long long);
        const std::size_t b_off = (static_cast<std::size_t>(n) + 1) * sizeof(int);
        const std::size_t b_pre = static_cast<std::size_t>(np > 0 ? np : 1) * sizeof(int);
        const std::size_t blob = b_slots + b_off + b_pre;
        c->hpred_blob.reserve(blob);
        long long* slots = reinterpret_cast<long long*>(c->hpred_blob.p);
        int* off = reinterpret_cast<int*>(c->hpred_blob.p + b_slots);
        int* pre = reinterpret_cast<int*>(c->hpred_blob.p + b_slots + b_off);
        for (int64_t i = 0; i < n; ++i) {
            const int64_t t = prefix_off[i + 1] - prefix_off[i];
            if (t < 1) invalid("predictor needs a non-empty prefix (current agent last)");
            if (t > cfg.max_prefix) invalid("prefix longer than the predictor's max_prefix");
            off[i] = static_cast<int>(prefix_off[i]);
        }
        off[n] = static_cast<int>(np);
        if (np > 0) {  // copy, then one vectorisable range reduction
            std::memcpy(pre, prefix, static_cast<std::size_t>(np) * sizeof(int));
            int lo = pre[0], hi = pre[0];
            for (int64_t j = 1; j < np; ++j) {
                lo = std::min(lo, pre[j]);
                hi = std::max(hi, pre[j]);
            }
            if (lo < 0 || hi >= cfg.num_agents) invalid("prefix agent out of range");
        }
        for (int64_t i = 0; i < n; ++i) slots[i] = slot_for(*c, wf[i]);
        const std::size_t per = static_cast<std::size_t>(cfg.horizon) * (cfg.num_agents + 1);
        c->fstage.reserve(static_cast<std::size_t>(n) * per);
        c->pred_blob.reserve(blob);
        cudaStream_t st = c->stream;
        PBKV_CUDA(cudaMemcpyAsync(c->pred_blob.p, c->hpred_blob.p, blob, cudaMemcpyHostToDevice, st));
        const long long* slots_d = reinterpret_cast<const long long*>(c->pred_blob.p);
        const int* off_d = reinterpret_cast<const int*>(c->pred_blob.p + b_slots);
        const int* pre_d = reinterpret_cast<const int*>(c->pred_blob.p + b_slots + b_off);
        const void* xd = x;
        if (!x_on_device) {
            const std::size_t xb = static_cast<std::size_t>(n) * cfg.text_dim;
            c->xstage.reserve(xb);
            PBKV_CUDA(cudaMemcpyAsync(c->xstage.p, x, xb * sizeof(uint16_t), cudaMemcpyHostToDevice, st));
            xd = c->xstage.p;
        }
        reset_status(*c);
        record(*c, 0);
        predictor_run(*c, n, off_d, pre_d, xd, slots_d, probs_out ? c->fstage.p : nullptr);
        record(*c, 1);
        if (probs_out)
            PBKV_CUDA(cudaMemcpyAsync(probs_out, c->fstage.p, static_cast<std::size_t>(n) * per * sizeof(double),
                                      cudaMemcpyDeviceToHost, st));
        check_status(*c);
        finish_timing(*c, 1);
    });
}

// ---- internal (host_tree.cpp): the tracked-tree tag of pbkv_mirror_sync ---------
void pbkv_internal_set_error(const char* msg) { g_last_error = msg ? msg : ""; }

int pbkv_internal_mirror_tag(pbkv_ctx* c, uint64_t** uid, int64_t** pos) {
    if (!c) return PBKV_EARG;
    *uid = &c->mirror_uid;
    *pos = &c->mirror_pos;
    return PBKV_OK;
}

}  // extern "C"
