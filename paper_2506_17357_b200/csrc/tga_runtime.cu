// tga_runtime.cu -- host runtime behind the tga_* C ABI (include/tga.h).
//
// Owns instance / solution state, the physical slot layout, device memory,
// the TMA descriptor of the position-ordered distance matrix, the tile plan
// (and its row shards), the NCCL communicator, and the host side of the
// update step (route-list splice + span re-upload, P:241 step 5).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <limits>
#include <new>
#include <string>
#include <vector>

#include "tga.h"
#include "tga_launch.h"

using namespace tga;

// ============================================================== errors
static thread_local std::string g_err;
static int32_t fail(int32_t code, const std::string &msg) {
    g_err = msg;
    return code;
}
#define TGA_CUDA(x)                                                                            \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            return fail(e_ == cudaErrorMemoryAllocation ? TGA_ERR_OOM : TGA_ERR_CUDA,          \
                        std::string(#x) + ": " + cudaGetErrorString(e_));                      \
        }                                                                                      \
    } while (0)

// ============================================================== NCCL (dlopen'd)
namespace {
typedef struct ncclComm *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclUint64 = 5, kNcclMin = 3;
struct Nccl {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*errStr)(ncclResult_t) = nullptr;
    bool load() {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        getUniqueId = reinterpret_cast<decltype(getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        commInitRank = reinterpret_cast<decltype(commInitRank)>(dlsym(h, "ncclCommInitRank"));
        allReduce = reinterpret_cast<decltype(allReduce)>(dlsym(h, "ncclAllReduce"));
        commDestroy = reinterpret_cast<decltype(commDestroy)>(dlsym(h, "ncclCommDestroy"));
        errStr = reinterpret_cast<decltype(errStr)>(dlsym(h, "ncclGetErrorString"));
        return getUniqueId && commInitRank && allReduce && commDestroy;
    }
};
Nccl g_nccl;

// ============================================================== TMA descriptor
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// variant -> segment lengths (0 = n/a)
void variant_lengths(int v, int *n1, int *n2) {
    *n1 = *n2 = 0;
    if (v >= TGA_V_RELOCATE1 && v <= TGA_V_OROPT3) { *n1 = v - TGA_V_RELOCATE1 + 1; return; }
    static const int sw[6][2] = {{1, 1}, {1, 2}, {1, 3}, {2, 2}, {2, 3}, {3, 3}};
    if (v >= TGA_V_SWAP11 && v <= TGA_V_CROSS33) { *n1 = sw[v - 5][0]; *n2 = sw[v - 5][1]; return; }
    if (v >= TGA_V_IRELOCATE1 && v <= TGA_V_IRELOCATE3) { *n1 = v - TGA_V_IRELOCATE1 + 1; return; }
    if (v >= TGA_V_ISWAP11 && v <= TGA_V_ISWAP33) { *n1 = (v - 14) / 3 + 1; *n2 = (v - 14) % 3 + 1; return; }
    if (v == TGA_V_OROPT2R || v == TGA_V_OROPT3R) { *n1 = v - TGA_V_OROPT2R + 2; return; }
    if (v == TGA_V_CROSS22R || v == TGA_V_CROSS33R) { *n1 = *n2 = v - TGA_V_CROSS22R + 2; }
}
}  // namespace

// ============================================================== objects
struct tga_instance {
    int n = 0, dtype = TGA_I32, Q = 0, device = 0;
    bool tw = false;
    tga_options opt{};
    void *dC = nullptr;
    int32_t *dDemand = nullptr;
    int32_t *dPickup = nullptr;    // VRPSPDTW pickup demands (tga_instance_set_pickup); null = none
    int live_solutions = 0;        // pickups may only be set before any solution is loaded
    TwRec *dNodeTw = nullptr;
    std::vector<int32_t> hDemand;
    std::vector<float> hTw;
    int max_c_abs = 0;
    bool fast_ok = false;  // loads small enough for the poisoned-load fast path
    bool fast_pen_ok = false;  // ... and penalised scores small enough for its 32-bit running minima
    // edge-based neighbourhood (ETGA): unordered customer pairs of the edge mask
    int theta = 0;
    int n_gpairs = 0;
    int2 *dGpairs = nullptr;
};

// Edge mask of the granular neighbourhood (reading 21): NN(i) = the
// theta customers j != i with the smallest (c_ij, j); M_ij = 1 iff j in NN(i) or
// i in NN(j) (pairs with the depot are always kept and are not listed here).
// Returns the unordered customer pairs (i < j) with M_ij = 1.
template <class T>
static std::vector<int2> granular_pairs(const T *dist, int n, int theta) {
    std::vector<uint64_t> pk;
    pk.reserve(static_cast<size_t>(n) * theta);
    std::vector<std::pair<double, int>> cand;
    for (int i = 1; i < n; ++i) {
        cand.clear();
        for (int j = 1; j < n; ++j)
            if (j != i) cand.emplace_back(static_cast<double>(dist[static_cast<size_t>(i) * n + j]), j);
        const int k = std::min<int>(theta, static_cast<int>(cand.size()));
        std::partial_sort(cand.begin(), cand.begin() + k, cand.end());
        for (int q = 0; q < k; ++q) {
            const int j = cand[q].second;
            const uint32_t a = static_cast<uint32_t>(std::min(i, j)), b = static_cast<uint32_t>(std::max(i, j));
            pk.push_back((static_cast<uint64_t>(a) << 32) | b);
        }
    }
    std::sort(pk.begin(), pk.end());
    pk.erase(std::unique(pk.begin(), pk.end()), pk.end());
    std::vector<int2> out(pk.size());
    for (size_t q = 0; q < pk.size(); ++q)
        out[q] = make_int2(static_cast<int>(pk[q] >> 32), static_cast<int>(pk[q] & 0xFFFFFFFFu));
    return out;
}

struct tga_solution {
    tga_instance *inst = nullptr;
    uint64_t gen = 1;
    std::vector<std::vector<int32_t>> routes;
    int R = 0, N = 0, Qc = 0, Qp = 0, pitch = 0, cap = 0;
    std::vector<int32_t> rbase, cbase, rcap;            // host: physical base / canonical base / slot capacity
    int slack = 2;                                      // spare slots per route (full relayout)
    // device arena
    void *arena = nullptr;
    int32_t *node = nullptr, *route = nullptr, *pos = nullptr, *rlen = nullptr, *canon = nullptr;
    int32_t *fwdL = nullptr, *bwdL = nullptr;
    void *enext = nullptr, *fwdD = nullptr, *bwdD = nullptr, *br1 = nullptr, *br2 = nullptr, *br3 = nullptr;
    TwRec *fwdT = nullptr, *bwdT = nullptr, *seg2T = nullptr, *seg3T = nullptr;
    int32_t *d_rbase = nullptr, *d_rlenR = nullptr, *d_cbase = nullptr, *d_rW = nullptr;
    // device-resident step
    DevState *d_ds = nullptr;      // this solution's DevState (device copy)
    void *d_sa = nullptr;          // ScanArgs<DT> (device copy)
    int32_t *d_desc = nullptr, *d_scratch = nullptr;
    unsigned long long *d_acc = nullptr;
    bool host_stale = false;       // host route lists lag behind device-resident steps
    int32_t *slot_of = nullptr;    // ETGA: node -> physical slot
    bool slot_of_fresh = false;    // ... current (device steps keep it so; host layout uploads do not)
    bool keys_clean = false;       // keys are all ~0 (a device step consumed them) ...
    unsigned long long clean_cap = 0;  // ... as of capture sequence clean_cap (0 = executed work)
    float *d_rTV = nullptr;
    void *d_rD = nullptr;
    void *Dp = nullptr;
    uint64_t *keys = nullptr;
    uint32_t *d_tiles = nullptr;
    int n_tiles = 0;
    CUtensorMap tmap{};
    bool tmap_ok = false;
    // CVRP fast path: per-slot records, its own tile plan and TMA box
    SlotRec *rec = nullptr;
    SlotTW *rectw = nullptr;       // VRPTW (TW-I) fast path
    uint32_t *d_ftiles = nullptr;
    int n_ftiles = 0;
    CUtensorMap fmap{};
    CUtensorMap nsmap{};           // Dp with the north-star sweep's box (tga_ns.cu)
    bool ns_ok = false;            // CVRP feasible-only int32 with |c| < 2^20: the NS sweep kernel applies
    int ns_rw = 8;                 // its rows per warp (ns_rows_per_warp)
    uint64_t ns_eval_gen = ~0ull;  // generation / stream of the last evaluation that ended in the NS sweep
    cudaStream_t ns_eval_stream = nullptr;
    int32_t *nsc = nullptr;        // its column-term planes [kNscF][pitch] (written by the scans)
    LoadRec *fwdP = nullptr, *bwdP = nullptr;   // VRPSPDTW prefix / suffix load records (Eq. 3a-d)
    bool fast = false;
    int fastU = 16;                // rows per fast-path tile (8 for small neighbourhoods)
    uint64_t *h_keys = nullptr;                         // pinned
    int32_t *h_stage = nullptr;                         // pinned staging: 5 rows of lay_pitch bytes
    int32_t *h_rstage = nullptr;                        // pinned staging: 2 rows of route_pitch bytes
    size_t lay_pitch = 0, route_pitch = 0;              // arena pitch of the slot / route arrays
    cudaStream_t stream = nullptr;                     // current stream (own or user's)
    cudaStream_t own_stream = nullptr;
    cudaStream_t side = nullptr;                       // fork for a concurrent intra-route kernel
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int shard = 0, n_shards = 1;
    ncclComm_t comm = nullptr;
    int sm_count = 148;
    uint64_t eval_gen = 0;
    uint32_t eval_mask = 0;
    bool drained = false;  // the stream was synchronised after the last enqueued work
    // live timing of the inter-route launch (ring of event pairs)
    bool timing = false;
    std::vector<cudaEvent_t> tev;
    int tev_n = 0;
};

// ============================================================== helpers
static bool is_intra_variant(int v) { return v == TGA_V_2OPT || (v >= TGA_V_IRELOCATE1 && v <= TGA_V_ISWAP33); }

// make `later` wait for everything already enqueued on `earlier`
static cudaError_t order_after(cudaStream_t later, cudaStream_t earlier) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(ev, earlier);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(later, ev, 0);
    cudaEventDestroy(ev);
    return e;
}

static int32_t set_device(const tga_instance *inst) {
    TGA_CUDA(cudaSetDevice(inst->device));
    (void)cudaGetLastError();  // drop non-sticky errors left by other code on this thread
    return TGA_OK;
}

// Physical layout: route r owns slots rbase[r] .. rbase[r]+cap[r]-1: start depot,
// customers, end depot, then cap - L - 2 spare "hole" slots (canonical id -1,
// route -1).  cap = L + 2 + slack is assigned by a full relayout; a move whose
// changed routes still fit keeps every base, so only those routes' slots, Dp rows
// and columns are refreshed.  Canonical id of (r, p), p <= L, is cbase[r] + p
// (SURVEY §8(c)); it is the host's business (keys index physical slots).
static void compute_cbase(tga_solution *s) {
    s->cbase.resize(s->R + 1);
    int cb = 0;
    for (int r = 0; r < s->R; ++r) {
        s->cbase[r] = cb;
        cb += static_cast<int>(s->routes[r].size()) + 1;
    }
    s->cbase[s->R] = cb;
}

static void relayout_full(tga_solution *s) {
    s->rbase.resize(s->R + 1);
    s->rcap.resize(s->R);
    int pb = 0;
    for (int r = 0; r < s->R; ++r) {
        s->rbase[r] = pb;
        s->rcap[r] = static_cast<int>(s->routes[r].size()) + 2 + s->slack;
        pb += s->rcap[r];
    }
    s->rbase[s->R] = pb;  // == Qp, constant
    compute_cbase(s);
}

static bool route_fits(const tga_solution *s, int r) {
    return static_cast<int>(s->routes[r].size()) + 2 <= s->rcap[r];
}

// Stage the 5 layout arrays (node, route, pos, rlen, canon) of route r's whole
// slot range into the pinned staging rows at column offset `off`.
static void stage_route(tga_solution *s, int r, int off) {
    const size_t rp = s->lay_pitch / 4;
    int32_t *nd = s->h_stage, *rt = nd + rp, *ps = rt + rp, *rl = ps + rp, *cn = rl + rp;
    const int L = static_cast<int>(s->routes[r].size());
    for (int p = 0; p < s->rcap[r]; ++p) {
        const int i = off + p;
        if (p <= L + 1) {
            nd[i] = (p == 0 || p == L + 1) ? 0 : s->routes[r][p - 1];
            rt[i] = r;
            ps[i] = p;
            rl[i] = L;
            cn[i] = (p <= L) ? s->cbase[r] + p : -1;
        } else {  // hole
            nd[i] = 0; rt[i] = -1; ps[i] = 0; rl[i] = -1; cn[i] = -1;
        }
    }
}

static void stage_route_arrays(tga_solution *s) {
    const size_t rq = s->route_pitch / 4;
    int32_t *rb = s->h_rstage, *rn = rb + rq, *rc = rn + rq;
    for (int r = 0; r <= s->R; ++r) {
        rb[r] = s->rbase[r];
        rn[r] = r < s->R ? static_cast<int32_t>(s->routes[r].size()) : 0;
        rc[r] = s->cbase[r];
    }
}

// Asynchronous 2-D copies from pinned staging (no host synchronisation: the
// staging buffers are reused only after the stream has drained).
//   routes = {ra, rb} (rb may be -1) : just those routes' slot ranges
//   full                            : every slot
static int32_t upload_layout(tga_solution *s, bool full, int ra = -1, int rb = -1) {
    s->slot_of_fresh = false;  // the ETGA node -> slot map is rebuilt before the next edge-based eval
    if (full) {
        int off = 0;
        for (int r = 0; r < s->R; ++r) { stage_route(s, r, off); off += s->rcap[r]; }
        TGA_CUDA(cudaMemcpy2DAsync(s->node, s->lay_pitch, s->h_stage, s->lay_pitch, sizeof(int32_t) * off, 5,
                                   cudaMemcpyHostToDevice, s->stream));
    } else {
        int off = 0;
        for (int k = 0; k < 2; ++k) {
            const int r = k == 0 ? ra : rb;
            if (r < 0 || (k == 1 && rb == ra)) continue;
            stage_route(s, r, off);
            TGA_CUDA(cudaMemcpy2DAsync(s->node + s->rbase[r], s->lay_pitch, s->h_stage + off, s->lay_pitch,
                                       sizeof(int32_t) * s->rcap[r], 5, cudaMemcpyHostToDevice, s->stream));
            off += s->rcap[r];
        }
    }
    stage_route_arrays(s);
    TGA_CUDA(cudaMemcpy2DAsync(s->d_rbase, s->route_pitch, s->h_rstage, s->route_pitch, sizeof(int32_t) * (s->R + 1),
                               3, cudaMemcpyHostToDevice, s->stream));
    return TGA_OK;
}

template <class DT>
static ScanArgs<DT> scan_args(tga_solution *s) {
    ScanArgs<DT> a;
    a.n_nodes = s->inst->n;
    a.C = static_cast<const DT *>(s->inst->dC);
    a.demand = s->inst->dDemand;
    a.node_tw = s->inst->dNodeTw;
    a.node = s->node;
    a.rbase = s->d_rbase;
    a.rlenR = s->d_rlenR;
    a.fwdL = s->fwdL;
    a.bwdL = s->bwdL;
    a.enext = static_cast<DT *>(s->enext);
    a.fwdD = static_cast<DT *>(s->fwdD);
    a.bwdD = static_cast<DT *>(s->bwdD);
    a.bridge1 = static_cast<DT *>(s->br1);
    a.bridge2 = static_cast<DT *>(s->br2);
    a.bridge3 = static_cast<DT *>(s->br3);
    a.fwdT = s->fwdT;
    a.bwdT = s->bwdT;
    a.seg2T = s->seg2T;
    a.seg3T = s->seg3T;
    a.rW = s->d_rW;
    a.rTV = s->d_rTV;
    a.rD = static_cast<DT *>(s->d_rD);
    a.canon = s->canon;
    a.capacity = s->inst->Q;
    a.pen_wQ = s->inst->opt.score_mode == TGA_SCORE_PENALISED ? s->inst->opt.w_load : 0;
    a.rec = s->rec;
    a.rectw = s->rectw;
    a.nsc = s->nsc;
    a.nsc_pitch = s->pitch;
    a.pickup = s->inst->dPickup;
    a.fwdP = s->fwdP;
    a.bwdP = s->bwdP;
    return a;
}

template <class DT>
static SolView<DT> sol_view(const tga_solution *s) {
    SolView<DT> v;
    v.node = s->node;
    v.route = s->route;
    v.pos = s->pos;
    v.rlen = s->rlen;
    v.canon = s->canon;
    v.fwdL = s->fwdL;
    v.bwdL = s->bwdL;
    v.enext = static_cast<const DT *>(s->enext);
    v.bridge1 = static_cast<const DT *>(s->br1);
    v.bridge2 = static_cast<const DT *>(s->br2);
    v.bridge3 = static_cast<const DT *>(s->br3);
    v.fwdT = s->fwdT;
    v.bwdT = s->bwdT;
    v.seg2T = s->seg2T;
    v.seg3T = s->seg3T;
    v.node_tw = s->inst->dNodeTw;
    v.dem = s->inst->dDemand;
    v.pick = s->inst->dPickup;
    v.fwdP = s->fwdP;
    v.bwdP = s->bwdP;
    v.rW = s->d_rW;
    v.rTV = s->d_rTV;
    v.Dp = static_cast<const DT *>(s->Dp);
    v.pitch = s->pitch;
    v.Qp = s->Qp;
    v.Qc = static_cast<uint32_t>(s->pitch);  // keys index physical slots
    v.tiles = s->d_tiles;
    return v;
}

static DevState make_devstate(const tga_solution *s, uint64_t *keys) {
    DevState d;
    d.node = s->node; d.route = s->route; d.pos = s->pos; d.rlen = s->rlen; d.canon = s->canon;
    d.rbase = s->d_rbase; d.rlenR = s->d_rlenR; d.cbase = s->d_cbase;
    d.scratch = s->d_scratch; d.keys = keys; d.desc = s->d_desc; d.acc = s->d_acc; d.Dp = s->Dp;
    d.slot_of = s->slot_of;
    d.R = s->R; d.Qc = s->pitch; d.Qp = s->Qp; d.pitch = s->pitch; d.slack = s->slack;
    return d;
}

// Device-resident steps changed the routes on the device only: rebuild the host
// route lists (node ids + route lengths, one D2H each) before any host-side use.
static int32_t sync_host(tga_solution *s) {
    if (!s->host_stale) return TGA_OK;
    TGA_CUDA(cudaStreamSynchronize(s->stream));
    std::vector<int32_t> nd(s->Qp), L(s->R), B(s->R + 1);
    TGA_CUDA(cudaMemcpy(nd.data(), s->node, 4 * s->Qp, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(L.data(), s->d_rlenR, 4 * s->R, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(B.data(), s->d_rbase, 4 * (s->R + 1), cudaMemcpyDeviceToHost));
    for (int r = 0; r < s->R; ++r) {
        s->routes[r].assign(nd.begin() + B[r] + 1, nd.begin() + B[r] + 1 + L[r]);
        s->rbase[r] = B[r];
        s->rcap[r] = B[r + 1] - B[r];
    }
    s->rbase[s->R] = B[s->R];
    compute_cbase(s);
    s->host_stale = false;
    s->drained = true;
    return TGA_OK;
}

// Device state of the current layout: full (load / reload / relayout) or just
// the slot ranges, Dp rows / columns and records of routes ra, rb.
static int32_t refresh(tga_solution *s, bool full, int ra = -1, int rb = -1) {
    const tga_instance *I = s->inst;
    cudaError_t e;
    if (!full) {  // update step of one applied move: one launch (Dp rows + columns + re-scan)
        UpdateSpec u{};
        u.lo1 = s->rbase[ra]; u.hi1 = s->rbase[ra] + s->rcap[ra]; u.r1 = ra;
        if (rb >= 0 && rb != ra) { u.lo2 = s->rbase[rb]; u.hi2 = s->rbase[rb] + s->rcap[rb]; u.r2 = rb; }
        else { u.lo2 = u.hi2 = 0; u.r2 = -1; }
        u.full = 0;
        if (I->dtype == TGA_I32)
            e = launch_update<int32_t>(scan_args<int32_t>(s), I->tw, static_cast<int32_t *>(s->Dp), s->pitch, s->Qp,
                                       s->R, u, s->stream);
        else
            e = launch_update<float>(scan_args<float>(s), I->tw, static_cast<float *>(s->Dp), s->pitch, s->Qp, s->R,
                                     u, s->stream);
        if (e != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("update: ") + cudaGetErrorString(e));
        return TGA_OK;
    }
    if (I->dtype == TGA_I32) {
        e = launch_dp<int32_t>(static_cast<int32_t *>(s->Dp), s->pitch, s->node, static_cast<const int32_t *>(I->dC),
                               I->n, s->Qp, 0, s->pitch, true, s->stream);
        if (e == cudaSuccess) e = launch_scan<int32_t>(scan_args<int32_t>(s), I->tw, 0, s->R, s->stream);
    } else {
        e = launch_dp<float>(static_cast<float *>(s->Dp), s->pitch, s->node, static_cast<const float *>(I->dC), I->n,
                             s->Qp, 0, s->pitch, true, s->stream);
        if (e == cudaSuccess) e = launch_scan<float>(scan_args<float>(s), I->tw, 0, s->R, s->stream);
    }
    if (e != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("refresh: ") + cudaGetErrorString(e));
    return TGA_OK;
}

// fast-path plan: fastU x kFastTV tiles (I << 16 | J) of the upper triangle, in the
// order the tile kernel decodes arithmetically (fast_tile_of, tga_inter_fast.cu):
// the diagonal tiles first (one per row band, the lightest: with one tile per CTA the
// intra-route units, which ride with the first CTAs, land on them), then the full
// tiles column by column (with several tiles per CTA the grid-stride walk gives every
// CTA a similar share).  The population batch keeps the table.
static std::vector<uint32_t> fast_plan(const tga_solution *s) {
    const int U = s->fastU, R = kFastTV / U;
    const int nI = (s->Qp + U - 1) / U, nJ = (s->Qp + kFastTV - 1) / kFastTV;
    std::vector<uint32_t> f;
    for (int I = 0; I < nI; ++I) f.push_back((static_cast<uint32_t>(I) << 16) | static_cast<uint32_t>(I / R));
    for (int J = 1; J < nJ; ++J)
        for (int I = 0; I < R * J; ++I) f.push_back((static_cast<uint32_t>(I) << 16) | static_cast<uint32_t>(J));
    return f;
}

// Tile plans, uploaded on the solution's stream: the arena they live in was
// initialised by stream-ordered memsets (a legacy-stream copy would not be
// ordered after them); the host vectors are pageable locals, so the stream is
// drained before they go out of scope.
static cudaError_t build_tiles(tga_solution *s) {
    std::vector<uint32_t> t;
    const int nI = s->pitch / kTileU, nJ = s->pitch / kTileV;
    for (int I = 0; I < nI; ++I) {
        if (I * kTileU >= s->Qp) break;
        for (int J = 0; J < nJ; ++J) {
            if (J * kTileV >= s->Qp) break;
            if (I * kTileU < J * kTileV + kTileV - 1) t.push_back((static_cast<uint32_t>(I) << 16) | J);
        }
    }
    s->n_tiles = static_cast<int>(t.size());
    cudaError_t e = cudaMemcpyAsync(s->d_tiles, t.data(), sizeof(uint32_t) * t.size(), cudaMemcpyHostToDevice, s->stream);
    // fast-path plan: fastU x kFastTV tiles of the upper triangle
    const std::vector<uint32_t> f = fast_plan(s);
    s->n_ftiles = static_cast<int>(f.size());
    if (e == cudaSuccess && s->d_ftiles)
        e = cudaMemcpyAsync(s->d_ftiles, f.data(), sizeof(uint32_t) * f.size(), cudaMemcpyHostToDevice, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    return e;
}

static void free_solution(tga_solution *s) {
    if (!s) return;
    if (s->inst) cudaSetDevice(s->inst->device);
    // work still queued on the solution's streams must not outlive its memory
    if (s->stream) cudaStreamSynchronize(s->stream);
    if (s->own_stream && s->own_stream != s->stream) cudaStreamSynchronize(s->own_stream);
    if (s->side) cudaStreamSynchronize(s->side);
    (void)cudaGetLastError();
    if (s->comm && g_nccl.commDestroy) g_nccl.commDestroy(s->comm);
    if (s->inst) --s->inst->live_solutions;
    if (s->arena) cudaFree(s->arena);
    if (s->Dp) cudaFree(s->Dp);
    if (s->h_keys) cudaFreeHost(s->h_keys);
    if (s->h_stage) cudaFreeHost(s->h_stage);
    if (s->h_rstage) cudaFreeHost(s->h_rstage);
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    if (s->side) cudaStreamDestroy(s->side);
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    for (auto e : s->tev) cudaEventDestroy(e);
    delete s;
}

// ============================================================== ABI: instance
extern "C" int32_t tga_instance_create(int32_t n, const void *dist, int32_t dtype, const void *time,
                                       const int32_t *demand, const float *tw, int32_t capacity,
                                       const tga_options *opt, tga_instance **out) {
    if (!out) return fail(TGA_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (n < 2 || !dist || !demand) return fail(TGA_ERR_INVALID_ARGUMENT, "n_nodes < 2 or NULL dist/demand");
    if (n > 65535) return fail(TGA_ERR_INVALID_ARGUMENT, "n_nodes > 65535 (flat index is 32-bit)");
    if (dtype != TGA_I32 && dtype != TGA_F32) return fail(TGA_ERR_INVALID_ARGUMENT, "dist_dtype");
    if (time) return fail(TGA_ERR_UNSUPPORTED, "separate travel-time matrix (T != C) not supported");
    if (capacity <= 0) return fail(TGA_ERR_INVALID_ARGUMENT, "capacity <= 0");
    if (demand[0] != 0) return fail(TGA_ERR_INVALID_ARGUMENT, "depot demand must be 0");
    for (int i = 0; i < n; ++i)
        if (demand[i] < 0) return fail(TGA_ERR_INVALID_ARGUMENT, "negative demand");
    // matrix checks: zero diagonal, non-negative, symmetric (inter-route kernels)
    int max_abs = 0;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            double a, b;
            if (dtype == TGA_I32) {
                a = static_cast<const int32_t *>(dist)[static_cast<size_t>(i) * n + j];
                b = static_cast<const int32_t *>(dist)[static_cast<size_t>(j) * n + i];
            } else {
                a = static_cast<const float *>(dist)[static_cast<size_t>(i) * n + j];
                b = static_cast<const float *>(dist)[static_cast<size_t>(j) * n + i];
            }
            if (!(a >= 0) || (i == j && a != 0)) return fail(TGA_ERR_INVALID_ARGUMENT, "negative distance or non-zero diagonal");
            if (a != b) return fail(TGA_ERR_UNSUPPORTED, "asymmetric distance matrix");
            max_abs = std::max(max_abs, static_cast<int>(std::min(a, 2.0e9)));
        }
    }
    if (tw) {
        for (int i = 0; i < n; ++i) {
            const float e = tw[3 * i], l = tw[3 * i + 1], s = tw[3 * i + 2];
            if (!(e <= l) || !(s >= 0)) return fail(TGA_ERR_INVALID_ARGUMENT, "time window e > l or s < 0");
        }
    }
    auto *I = new (std::nothrow) tga_instance();
    if (!I) return fail(TGA_ERR_OOM, "host allocation");
    I->n = n;
    I->dtype = dtype;
    I->Q = capacity;
    I->tw = tw != nullptr;
    I->max_c_abs = max_abs;
    {
        int64_t tot = 0;
        for (int i = 0; i < n; ++i) tot += demand[i];
        // poisoned loads stay below 2^31; |delta| <= 8 max c < 2^25 fits the packed 32-bit keys
        I->fast_ok = tot < (kPoison >> 2) && capacity < (kPoison >> 2) && max_abs < (1 << 21);
        I->fast_pen_ok = false;   // set below once the options are known
    }
    if (opt) I->opt = *opt;
    else { I->opt.score_mode = TGA_SCORE_FEASIBLE; I->opt.w_load = 10; I->opt.w_tw = 10; I->opt.device = -1; }
    if (I->opt.score_mode != TGA_SCORE_FEASIBLE && I->opt.score_mode != TGA_SCORE_PENALISED) {
        delete I;
        return fail(TGA_ERR_INVALID_ARGUMENT, "score_mode");
    }
    if (dtype == TGA_I32) {
        // integer scores are packed as 32-bit order-preserving images: bound |score| of any
        // candidate.  dD sums at most 8 distances (Eq. 2); penalised mode adds
        // w_load * dL_V with |dL_V| <= 2 x total demand and w_tw * dT_V with |dT_V| <= the
        // warp two routes can hold, each stop at most max l + max s + max c (Eq. 4).
        double bound = 8.0 * max_abs;
        if (I->opt.score_mode == TGA_SCORE_PENALISED) {
            double tot = 0;
            for (int i = 0; i < n; ++i) tot += demand[i];
            bound += std::fabs(static_cast<double>(I->opt.w_load)) * 2.0 * tot;
            if (tw) {
                double ml = 0, ms = 0;
                for (int i = 0; i < n; ++i) { ml = std::max(ml, static_cast<double>(tw[3 * i + 1])); ms = std::max(ms, static_cast<double>(tw[3 * i + 2])); }
                bound += std::fabs(static_cast<double>(I->opt.w_tw)) * (n + 1.0) * (ml + ms + max_abs);
            }
        }
        if (bound >= 2147483647.0) {
            delete I;
            return fail(TGA_ERR_INVALID_ARGUMENT, "integer score range exceeds int32 (distances, demands or "
                                                  "penalty weights too large; use TGA_F32)");
        }
        // penalised CVRP on the fast path: |score| <= 8 max c + w_load x 2 x total demand < 2^25
        // (the packed 32-bit running minima of the tile body), non-negative weight
        if (I->opt.score_mode == TGA_SCORE_PENALISED && !tw && I->opt.w_load >= 0) {
            double tot = 0;
            for (int i = 0; i < n; ++i) tot += demand[i];
            I->fast_pen_ok = I->fast_ok && 8.0 * max_abs + 2.0 * I->opt.w_load * tot < 33554432.0;
        }
    }
    if (I->opt.device < 0) cudaGetDevice(&I->device);
    else I->device = I->opt.device;
    I->hDemand.assign(demand, demand + n);
    std::vector<TwRec> ntw(n);
    if (tw) {
        I->hTw.assign(tw, tw + 3 * static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) ntw[i] = tw_single(tw[3 * i], tw[3 * i + 1], tw[3 * i + 2]);
    } else {
        for (int i = 0; i < n; ++i) ntw[i] = tw_single(0.f, 3.0e38f, 0.f);
    }
    auto cleanup = [&](int32_t code) {
        if (I->dC) cudaFree(I->dC);
        if (I->dDemand) cudaFree(I->dDemand);
        if (I->dNodeTw) cudaFree(I->dNodeTw);
        if (I->dGpairs) cudaFree(I->dGpairs);
        delete I;
        return code;
    };
    if (cudaSetDevice(I->device) != cudaSuccess) return cleanup(fail(TGA_ERR_CUDA, "cudaSetDevice"));
    (void)cudaGetLastError();
    const size_t nn = static_cast<size_t>(n) * n;
    cudaError_t e = cudaMalloc(&I->dC, nn * 4);
    if (e == cudaSuccess) e = cudaMalloc(&I->dDemand, sizeof(int32_t) * n);
    if (e == cudaSuccess) e = cudaMalloc(&I->dNodeTw, sizeof(TwRec) * n);
    if (e == cudaSuccess) e = cudaMemcpy(I->dC, dist, nn * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(I->dDemand, demand, sizeof(int32_t) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(I->dNodeTw, ntw.data(), sizeof(TwRec) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && I->opt.granular_theta > 0) {
        I->theta = I->opt.granular_theta;
        const std::vector<int2> gp = dtype == TGA_I32
            ? granular_pairs(static_cast<const int32_t *>(dist), n, I->theta)
            : granular_pairs(static_cast<const float *>(dist), n, I->theta);
        I->n_gpairs = static_cast<int>(gp.size());
        e = cudaMalloc(&I->dGpairs, sizeof(int2) * std::max<size_t>(1, gp.size()));
        if (e == cudaSuccess && !gp.empty())
            e = cudaMemcpy(I->dGpairs, gp.data(), sizeof(int2) * gp.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess)
        return cleanup(fail(e == cudaErrorMemoryAllocation ? TGA_ERR_OOM : TGA_ERR_CUDA,
                            std::string("instance upload: ") + cudaGetErrorString(e)));
    *out = I;
    return TGA_OK;
}

extern "C" int32_t tga_instance_info(const tga_instance *I, int32_t *n_nodes, int32_t *theta, int64_t *n_pairs) {
    if (!I) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL instance");
    if (n_nodes) *n_nodes = I->n;
    if (theta) *theta = I->theta;
    if (n_pairs) *n_pairs = I->n_gpairs;
    return TGA_OK;
}

extern "C" int32_t tga_instance_destroy(tga_instance *I) {
    if (!I) return TGA_OK;
    cudaSetDevice(I->device);
    cudaDeviceSynchronize();   // no solution's queued work may still read C / demand / windows
    (void)cudaGetLastError();
    cudaFree(I->dC);
    cudaFree(I->dDemand);
    if (I->dPickup) cudaFree(I->dPickup);
    cudaFree(I->dNodeTw);
    if (I->dGpairs) cudaFree(I->dGpairs);
    delete I;
    return TGA_OK;
}

extern "C" int32_t tga_instance_set_pickup(tga_instance *I, const int32_t *pickup) {
    if (!I || !pickup) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (I->live_solutions > 0) return fail(TGA_ERR_INVALID_ARGUMENT, "pickups must be set before any solution is loaded");
    if (pickup[0] != 0) return fail(TGA_ERR_INVALID_ARGUMENT, "depot pickup p_0 != 0");
    int64_t tot = 0;
    for (int i = 0; i < I->n; ++i) {
        if (pickup[i] < 0) return fail(TGA_ERR_INVALID_ARGUMENT, "pickup demand < 0");
        tot += pickup[i];
    }
    if (tot >= (int64_t(1) << 30)) return fail(TGA_ERR_INVALID_ARGUMENT, "pickup sum exceeds the int32 load range");
    if (set_device(I) != TGA_OK) return TGA_ERR_CUDA;
    if (!I->dPickup) TGA_CUDA(cudaMalloc(&I->dPickup, sizeof(int32_t) * I->n));
    TGA_CUDA(cudaMemcpy(I->dPickup, pickup, sizeof(int32_t) * I->n, cudaMemcpyHostToDevice));
    // the capacity test becomes one on the largest load carried (Eq. 3a-d): the generic
    // kernels concatenate (L_I, L_O, L_M) records; the fast paths assume delivery sums
    I->fast_ok = false;
    I->fast_pen_ok = false;
    return TGA_OK;
}

// ============================================================== ABI: solution
extern "C" int32_t tga_solution_load(tga_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                                     tga_solution **out) {
    if (!out || !I || !ptr || (R > 0 && !cust && ptr[R] > 0))
        return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    *out = nullptr;
    if (R < 1) return fail(TGA_ERR_INVALID_ARGUMENT, "n_routes < 1");
    if (ptr[0] != 0) return fail(TGA_ERR_STRUCTURE, "route_ptr[0] != 0");
    std::vector<char> seen(I->n, 0);
    for (int r = 0; r < R; ++r) {
        if (ptr[r + 1] < ptr[r]) return fail(TGA_ERR_STRUCTURE, "route_ptr not non-decreasing");
        for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
            const int c = cust[k];
            if (c <= 0 || c >= I->n) return fail(TGA_ERR_STRUCTURE, "customer id out of range");
            if (seen[c]) return fail(TGA_ERR_STRUCTURE, "customer visited twice");
            seen[c] = 1;
        }
    }
    if (ptr[R] != I->n - 1) return fail(TGA_ERR_STRUCTURE, "not every customer is visited");
    if (set_device(I) != TGA_OK) return TGA_ERR_CUDA;

    auto *s = new (std::nothrow) tga_solution();
    if (!s) return fail(TGA_ERR_OOM, "host allocation");
    s->inst = I;
    ++I->live_solutions;   // (free_solution counts it back out, also on a failed load)
    s->R = R;
    s->routes.resize(R);
    for (int r = 0; r < R; ++r) s->routes[r].assign(cust + ptr[r], cust + ptr[r + 1]);
    s->N = ptr[R];
    s->Qc = s->N + R;
    s->slack = I->opt.slack > 0 ? I->opt.slack : (I->opt.slack < 0 ? 0 : 2);
    s->Qp = s->N + (2 + s->slack) * R;
    s->pitch = static_cast<int>(align_up(static_cast<size_t>(s->Qp) + 4, kPitchAlign));
    s->cap = s->pitch + 2 * kGuard;
    // keys pack the flat index over PHYSICAL slots, u * pitch + v < pitch^2, in 32 bits
    // (pitch >= Q_p > Q = N + R, so this also bounds the canonical index)
    if (static_cast<uint64_t>(s->pitch) * static_cast<uint64_t>(s->pitch) > 0x100000000ull) {
        delete s;
        return fail(TGA_ERR_INVALID_ARGUMENT, "physical slot pitch^2 exceeds the 32-bit flat index "
                                              "(too many customers + routes x (2 + slack))");
    }
    relayout_full(s);
    int32_t rc = TGA_OK;
    auto bail = [&](int32_t code) { free_solution(s); return code; };
    {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, I->device) == cudaSuccess) s->sm_count = prop.multiProcessorCount;
    }
    if (cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(TGA_ERR_CUDA, "stream create"));
    s->stream = s->own_stream;
    if (cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(TGA_ERR_CUDA, "side stream"));
    // ---- device arena: slot arrays (with guards), per-route arrays, keys, tiles
    const size_t cap = s->cap, Rr = static_cast<size_t>(R) + 1;
    struct Item { void **p; size_t bytes; };
    const size_t tiles_max = static_cast<size_t>(s->pitch / kTileU) * (s->pitch / kTileV) + 1;
    void *v_node, *v_route, *v_pos, *v_rlen, *v_canon, *v_fwdL, *v_bwdL, *v_en, *v_fD, *v_bD, *v_b1, *v_b2, *v_b3;
    void *v_fT, *v_bT, *v_s2, *v_s3, *v_rbase, *v_rlenR, *v_cbase, *v_rW, *v_rTV, *v_rD, *v_keys, *v_tiles;
    void *v_ds, *v_sa, *v_desc, *v_scr, *v_acc;
    void *v_rec = nullptr, *v_ftiles = nullptr, *v_rectw = nullptr, *v_slot_of = nullptr, *v_nsc = nullptr;
    void *v_fP = nullptr, *v_bP = nullptr;
    s->fastU = 16;  // U = 8 measured no better at n = 1000 (more tiles, more per-tile overhead)
    if (const char *ev = std::getenv("TGA_FAST_U")) s->fastU = std::atoi(ev) == 8 ? 8 : 16;  // tuning override
    if (I->opt.score_mode == TGA_SCORE_PENALISED) s->fastU = 16;   // the penalised tile body is built for U = 16
    const size_t ftiles_max = static_cast<size_t>(s->pitch / s->fastU) * (s->pitch / kFastTV) + 1;
    // fast path: integer distances (CVRP, or VRPTW TW-I), feasible-only scoring
    // fast path: integer distances; feasible-only (CVRP or VRPTW TW-I) or penalised CVRP
    const bool want_fast = I->dtype == TGA_I32 && I->fast_ok &&
                           (I->opt.score_mode == TGA_SCORE_FEASIBLE || I->fast_pen_ok);
    // the north-star sweep kernel (tga_ns.cu): CVRP, feasible-only, |c| < 2^20
    const bool want_ns = want_fast && !I->tw && I->opt.score_mode == TGA_SCORE_FEASIBLE && I->max_c_abs < (1 << 20);
    Item items[] = {
        {&v_node, cap * 4}, {&v_route, cap * 4}, {&v_pos, cap * 4}, {&v_rlen, cap * 4}, {&v_canon, cap * 4},
        {&v_fwdL, cap * 4}, {&v_bwdL, cap * 4}, {&v_en, cap * 4}, {&v_fD, cap * 4}, {&v_bD, cap * 4},
        {&v_b1, cap * 4}, {&v_b2, cap * 4}, {&v_b3, cap * 4},
        {&v_fT, cap * 16}, {&v_bT, cap * 16}, {&v_s2, cap * 16}, {&v_s3, cap * 16},
        {&v_rbase, Rr * 4}, {&v_rlenR, Rr * 4}, {&v_cbase, Rr * 4}, {&v_rW, Rr * 4}, {&v_rTV, Rr * 4},
        {&v_rD, Rr * 4}, {&v_ds, sizeof(DevState)}, {&v_sa, sizeof(ScanArgs<int32_t>)}, {&v_desc, 16 * 4},
        {&v_scr, cap * 4}, {&v_acc, kAccWords * 8},
        {&v_keys, TGA_N_VARIANTS * 8}, {&v_tiles, tiles_max * 4},
        {&v_rec, want_fast ? cap * sizeof(SlotRec) : 0}, {&v_ftiles, want_fast ? ftiles_max * 4 : 0},
        {&v_rectw, want_fast && I->tw ? cap * sizeof(SlotTW) : 0},
        {&v_slot_of, I->theta > 0 ? static_cast<size_t>(I->n) * 4 : 0},
        {&v_nsc, want_ns ? static_cast<size_t>(kNscF) * s->pitch * 4 : 0},
        {&v_fP, I->dPickup ? cap * sizeof(LoadRec) : 0}, {&v_bP, I->dPickup ? cap * sizeof(LoadRec) : 0}};
    size_t total = 0;
    for (auto &it : items) total += align_up(it.bytes, 256);
    if (cudaMalloc(&s->arena, total) != cudaSuccess) return bail(fail(TGA_ERR_OOM, "device arena"));
    {
        size_t off = 0;
        for (auto &it : items) {
            *it.p = static_cast<char *>(s->arena) + off;
            off += align_up(it.bytes, 256);
        }
    }
    // guards: ints -> -1 (route/pos/rlen/canon invalid), node -> 0 (a valid node id)
    // every initialisation is ordered on the solution's (non-blocking) stream: a
    // legacy-stream cudaMemset would not be ordered before the layout upload
    if (cudaMemsetAsync(s->arena, 0xFF, total, s->stream) != cudaSuccess) return bail(fail(TGA_ERR_CUDA, "memset"));
    if (cudaMemsetAsync(v_node, 0, cap * 4, s->stream) != cudaSuccess) return bail(fail(TGA_ERR_CUDA, "memset"));
    auto g32 = [&](void *p) { return static_cast<int32_t *>(p) + kGuard; };
    auto g128 = [&](void *p) { return static_cast<TwRec *>(p) + kGuard; };
    s->node = g32(v_node); s->route = g32(v_route); s->pos = g32(v_pos); s->rlen = g32(v_rlen);
    s->canon = g32(v_canon); s->fwdL = g32(v_fwdL); s->bwdL = g32(v_bwdL);
    s->enext = g32(v_en); s->fwdD = g32(v_fD); s->bwdD = g32(v_bD);
    s->br1 = g32(v_b1); s->br2 = g32(v_b2); s->br3 = g32(v_b3);
    s->fwdT = g128(v_fT); s->bwdT = g128(v_bT); s->seg2T = g128(v_s2); s->seg3T = g128(v_s3);
    s->d_rbase = static_cast<int32_t *>(v_rbase); s->d_rlenR = static_cast<int32_t *>(v_rlenR);
    s->d_rW = static_cast<int32_t *>(v_rW); s->d_rTV = static_cast<float *>(v_rTV); s->d_rD = v_rD;
    s->d_cbase = static_cast<int32_t *>(v_cbase);
    s->d_ds = static_cast<DevState *>(v_ds); s->d_sa = v_sa;
    s->d_desc = static_cast<int32_t *>(v_desc); s->d_scratch = static_cast<int32_t *>(v_scr);
    s->d_acc = static_cast<unsigned long long *>(v_acc);
    s->slot_of = I->theta > 0 ? static_cast<int32_t *>(v_slot_of) : nullptr;  // zero-size items point past the arena
    s->keys = static_cast<uint64_t *>(v_keys);
    if (I->dPickup) {   // VRPSPDTW prefix / suffix load records (guards included, like the other slot arrays)
        s->fwdP = static_cast<LoadRec *>(v_fP) + kGuard;
        s->bwdP = static_cast<LoadRec *>(v_bP) + kGuard;
        if (cudaMemsetAsync(v_fP, 0, cap * sizeof(LoadRec), s->stream) != cudaSuccess ||
            cudaMemsetAsync(v_bP, 0, cap * sizeof(LoadRec), s->stream) != cudaSuccess)
            return bail(fail(TGA_ERR_CUDA, "memset"));
    }
    if (want_ns) {   // column-term planes: route -1 (no canonical slot) until the scan writes a slot
        s->nsc = static_cast<int32_t *>(v_nsc);
        if (cudaMemsetAsync(s->nsc, 0xFF, static_cast<size_t>(s->pitch) * 4, s->stream) != cudaSuccess ||
            cudaMemsetAsync(s->nsc + s->pitch, 0, static_cast<size_t>(kNscF - 1) * s->pitch * 4, s->stream) != cudaSuccess)
            return bail(fail(TGA_ERR_CUDA, "memset"));
    }
    s->d_tiles = static_cast<uint32_t *>(v_tiles);
    if (want_fast) {
        s->fast = true;
        s->rec = static_cast<SlotRec *>(v_rec) + kGuard;
        s->d_ftiles = static_cast<uint32_t *>(v_ftiles);
        // every record starts poisoned (padding, guards); the scan overwrites route slots
        SlotRec p{};
        p.r = -1; p.fL = p.bL1 = p.W = kPoison;
        for (int k = 0; k < 3; ++k) { p.so[k] = kPoison; p.sA[k] = kPoison; }
        std::vector<SlotRec> init(cap, p);
        if (I->tw) {
            s->rectw = static_cast<SlotTW *>(v_rectw) + kGuard;
            SlotTW pt{};
            pt.EF = pt.EFm = kTwBig;
            for (int k = 0; k < 3; ++k) { pt.LBN[k] = -kTwBig; pt.sTL[k] = -kTwBig; }
            std::vector<SlotTW> tinit(cap, pt);
            if (cudaMemcpyAsync(v_rectw, tinit.data(), cap * sizeof(SlotTW), cudaMemcpyHostToDevice, s->stream) !=
                    cudaSuccess ||
                cudaStreamSynchronize(s->stream) != cudaSuccess)
                return bail(fail(TGA_ERR_CUDA, "record init"));
        }
        if (cudaMemcpyAsync(v_rec, init.data(), cap * sizeof(SlotRec), cudaMemcpyHostToDevice, s->stream) !=
                cudaSuccess ||
            cudaStreamSynchronize(s->stream) != cudaSuccess)  // `init` is pageable and local
            return bail(fail(TGA_ERR_CUDA, "record init"));
    }
    // numeric per-slot arrays start at 0 (guards are only read by masked-out lanes)
    for (void *p : {v_fwdL, v_bwdL, v_en, v_fD, v_bD, v_b1, v_b2, v_b3})
        if (cudaMemsetAsync(p, 0, cap * 4, s->stream) != cudaSuccess) return bail(fail(TGA_ERR_CUDA, "memset"));
    for (void *p : {v_fT, v_bT, v_s2, v_s3})
        if (cudaMemsetAsync(p, 0, cap * 16, s->stream) != cudaSuccess) return bail(fail(TGA_ERR_CUDA, "memset"));
    // ---- position-ordered distance matrix
    const size_t dp_bytes = static_cast<size_t>(s->pitch) * s->pitch * 4;
    if (cudaMalloc(&s->Dp, dp_bytes) != cudaSuccess) return bail(fail(TGA_ERR_OOM, "Dp allocation"));
    s->lay_pitch = align_up(cap * 4, 256);
    s->route_pitch = align_up(Rr * 4, 256);
    if (cudaMallocHost(&s->h_keys, TGA_N_VARIANTS * 8) != cudaSuccess ||
        cudaMallocHost(&s->h_stage, 5 * s->lay_pitch) != cudaSuccess ||
        cudaMallocHost(&s->h_rstage, 3 * s->route_pitch) != cudaSuccess)
        return bail(fail(TGA_ERR_OOM, "pinned host allocation"));
    // ---- layout upload, Dp build, scan
    if ((rc = upload_layout(s, true)) != TGA_OK) return bail(rc);
    if ((rc = refresh(s, true)) != TGA_OK) return bail(rc);
    if (build_tiles(s) != cudaSuccess) return bail(fail(TGA_ERR_CUDA, "tile plan upload"));
    // ---- TMA descriptor over Dp: dims {pitch cols, pitch rows}, box {kBoxW, kBoxH}
    if (auto enc = get_encode()) {
        // the tensor spans the Qp physical slots only: box parts past them (the pitch padding of
        // the last row / column band) are zero-filled by the TMA unit instead of read from HBM --
        // they only feed candidates of padding slots, which are invalid
        cuuint64_t gdim[2] = {static_cast<cuuint64_t>(s->Qp), static_cast<cuuint64_t>(s->Qp)};
        cuuint64_t gstride[1] = {static_cast<cuuint64_t>(s->pitch) * 4};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(kBoxW), static_cast<cuuint32_t>(kBoxH)};
        cuuint32_t estr[2] = {1, 1};
        CUresult cr = enc(&s->tmap, I->dtype == TGA_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                          2, s->Dp, gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        s->tmap_ok = (cr == CUDA_SUCCESS);
    }
    if (!s->tmap_ok) return bail(fail(TGA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable or failed"));
    if (s->fast) {
        auto enc = get_encode();
        cuuint64_t gdim[2] = {static_cast<cuuint64_t>(s->Qp), static_cast<cuuint64_t>(s->Qp)};
        cuuint64_t gstride[1] = {static_cast<cuuint64_t>(s->pitch) * 4};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(kFastTV + 8), static_cast<cuuint32_t>(s->fastU + 4)};
        cuuint32_t estr[2] = {1, 1};
        CUresult cr = enc(&s->fmap, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, s->Dp, gdim, gstride, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return bail(fail(TGA_ERR_CUDA, "fast-path tensor map"));
        if (s->nsc) {
            s->ns_rw = ns_rows_per_warp(s->Qp, s->sm_count);
            cuuint32_t nbox[2] = {static_cast<cuuint32_t>(ns_box_cols()), static_cast<cuuint32_t>(ns_box_rows(s->ns_rw))};
            cr = enc(&s->nsmap, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, s->Dp, gdim, gstride, nbox, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) return bail(fail(TGA_ERR_CUDA, "north-star sweep tensor map"));
            s->ns_ok = true;
        }
    }
    {   // device-resident step state
        DevState ds = make_devstate(s, s->keys);
        if (cudaMemcpyAsync(s->d_ds, &ds, sizeof(ds), cudaMemcpyHostToDevice, s->stream) != cudaSuccess ||
            cudaMemsetAsync(s->d_acc, 0, kAccWords * 8, s->stream) != cudaSuccess ||

            cudaMemsetAsync(s->d_desc, 0, 16 * 4, s->stream) != cudaSuccess)
            return bail(fail(TGA_ERR_CUDA, "device step state"));
        cudaError_t e2;
        if (I->dtype == TGA_I32) { auto a = scan_args<int32_t>(s); e2 = cudaMemcpyAsync(s->d_sa, &a, sizeof(a), cudaMemcpyHostToDevice, s->stream);
                                   if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(s->stream); }
        else { auto a = scan_args<float>(s); e2 = cudaMemcpyAsync(s->d_sa, &a, sizeof(a), cudaMemcpyHostToDevice, s->stream);
               if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(s->stream); }
        if (e2 != cudaSuccess) return bail(fail(TGA_ERR_CUDA, "device step state"));
    }
    if (cudaStreamSynchronize(s->stream) != cudaSuccess)
        return bail(fail(TGA_ERR_CUDA, std::string("load: ") + cudaGetErrorString(cudaGetLastError())));
    *out = s;
    return TGA_OK;
}

extern "C" int32_t tga_solution_destroy(tga_solution *s) {
    free_solution(s);
    return TGA_OK;
}

extern "C" int32_t tga_shard_range(int64_t n, int32_t shard, int32_t n_shards, int64_t *lo, int64_t *hi) {
    if (!lo || !hi || n < 0 || n_shards < 1 || shard < 0 || shard >= n_shards)
        return fail(TGA_ERR_INVALID_ARGUMENT, "shard range");
    *lo = n * shard / n_shards;
    *hi = n * (shard + 1) / n_shards;
    return TGA_OK;
}

extern "C" int32_t tga_solution_set_stream(tga_solution *s, void *stream) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->own_stream;
    if (st != s->stream) {
        // order the new stream after everything queued on the old one
        cudaEvent_t ev;
        TGA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        TGA_CUDA(cudaEventRecord(ev, s->stream));
        TGA_CUDA(cudaStreamWaitEvent(st, ev, 0));
        cudaEventDestroy(ev);
    }
    s->stream = st;
    return TGA_OK;
}

extern "C" int32_t tga_solution_set_shard(tga_solution *s, int32_t shard, int32_t n_shards) {
    if (!s || n_shards < 1 || shard < 0 || shard >= n_shards) return fail(TGA_ERR_INVALID_ARGUMENT, "shard plan");
    s->shard = shard;
    s->n_shards = n_shards;
    return TGA_OK;
}

extern "C" int32_t tga_shard_range(int64_t n, int32_t shard, int32_t n_shards, int64_t *lo, int64_t *hi);

// ============================================================== ABI: evaluation
// id of the capture sequence `st` is recording into (0 when not capturing)
static unsigned long long capture_id(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    unsigned long long id = 0;
    if (cudaStreamGetCaptureInfo(st, &cs, &id) != cudaSuccess || cs != cudaStreamCaptureStatusActive) return 0;
    return id;
}

// the north-star sweep kernel takes an evaluation whose inter-route part is exactly
// {2-opt*, relocate, swap (1,1)} (TGA_NO_NS=1: the all-variant tile kernel instead)
static bool ns_path(const tga_solution *s, uint32_t mask) {
    static const bool off = std::getenv("TGA_NO_NS") != nullptr;
    constexpr uint32_t NS = TGA_OP_2OPT_STAR | (1u << 2) | (1u << 5);
    return s->ns_ok && !off && s->inst->theta <= 0 && (mask & TGA_OP_INTER) == NS;
}

extern "C" int32_t tga_eval(tga_solution *s, uint32_t mask, void *stream) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    const tga_instance *I = s->inst;
    const bool accumulate = (mask & TGA_EVAL_ACCUMULATE) && s->eval_gen == s->gen;
    mask &= TGA_OP_ALL;
    if ((mask & TGA_OP_2OPT) && I->tw)
        return fail(TGA_ERR_UNSUPPORTED, "2-opt is only defined without time windows (P:148)");
    if ((mask & TGA_OP_2OPT) && I->dPickup)
        return fail(TGA_ERR_UNSUPPORTED, "2-opt is applied to the CVRP only (P:510), not with pickups");
    if (set_device(I) != TGA_OK) return TGA_ERR_CUDA;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
    if (st != s->stream) TGA_CUDA(order_after(st, s->stream));  // see the latest applied move
    // a device step leaves the keys reset (consumed), so the next eval needs no memset node --
    // unless that step belongs to another capture sequence (a graph replayed later)
    const bool ns = ns_path(s, mask);
    bool reset = false;
    if (!accumulate && !(s->keys_clean && s->clean_cap == capture_id(st))) {
        // before the north-star sweep the reset is a programmatic dependent of its predecessor;
        // when that is the sweep of the same, unchanged solution on this stream (an evaluation
        // loop) the next sweep may start before the previous one ends (k_fill_u64)
        const bool early = ns && s->ns_eval_gen == s->gen && s->ns_eval_stream == st;
        TGA_CUDA(launch_fill_u64(s->keys, TGA_N_VARIANTS, ~0ull, st, ns, early));
        reset = true;
    }
    s->ns_eval_gen = ns ? s->gen : ~0ull;
    s->ns_eval_stream = st;
    s->keys_clean = false;
    ScoreParams sp{I->Q, I->opt.score_mode, I->opt.w_load, I->opt.w_tw};
    // row shard of the tile list and of the intra slot range
    int64_t a, b;
    tga_shard_range(s->n_tiles, s->shard, s->n_shards, &a, &b);
    const int t_lo = static_cast<int>(a), t_hi = static_cast<int>(b);
    tga_shard_range(s->Qp, s->shard, s->n_shards, &a, &b);
    const int x_lo = static_cast<int>(a), x_hi = static_cast<int>(b);
    const int grid = std::max(1, std::min(t_hi - t_lo, s->sm_count * 4));
    cudaError_t e;
    bool fused_intra = false;
    const bool timed = s->timing && (mask & TGA_OP_INTER) && s->tev_n + 2 <= static_cast<int>(s->tev.size());
    // inside a captured graph (tga_descent) the records must be external event nodes
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (timed) TGA_CUDA(cudaStreamIsCapturing(st, &cst));
    const unsigned rec_flags = cst == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
    // VRPTW: the intra-route kernel is latency-bound and independent of the inter-route one;
    // TGA_FORK_INTRA=1 runs it on a forked stream beside it.  Off by default: measured 2-3 %
    // faster steps (cfg3 40.4 -> 39.2 us) but the inter kernel then shares the SMs, so its own
    // duration (the roofline's) grows 23 -> 32 us.
    static const bool fork_env = std::getenv("TGA_FORK_INTRA") && std::atoi(std::getenv("TGA_FORK_INTRA")) == 1;
    // VRPTW intra kernel: the warp-parallel one (warp scans of Eq. 4 records) for long routes, the
    // thread-per-(slot, variant) walk for short ones -- measured: cfg3 R1 (mean route 11 slots)
    // 35.9 vs 38.8 us/step with the walk, R2 (50 slots) 54.0 vs 76.2 with the warp kernel; the
    // same mean-length threshold as the population batch.  TGA_WARP_TW=0/1 forces one (A/B).
    static const int force_warp = std::getenv("TGA_WARP_TW") ? std::atoi(std::getenv("TGA_WARP_TW")) : -1;
    // (the warp-scan kernel has no pickup-and-delivery load records: VRPSPDTW takes the walk)
    const bool warp_tw = !I->dPickup && (force_warp >= 0 ? force_warp != 0 : s->N >= 16 * s->R);
    const bool fork_intra = fork_env && I->tw && (mask & TGA_OP_INTER) && (mask & TGA_OP_INTRA) && x_hi > x_lo;
    if (fork_intra) {
        TGA_CUDA(cudaEventRecord(s->ev_fork, st));
        TGA_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
        const cudaError_t ei = I->dtype == TGA_I32
            ? launch_intra<int32_t>(mask, true, sol_view<int32_t>(s), sp, x_lo, x_hi, s->keys, s->side, false, warp_tw)
            : launch_intra<float>(mask, true, sol_view<float>(s), sp, x_lo, x_hi, s->keys, s->side, false, warp_tw);
        if (ei != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("intra launch: ") + cudaGetErrorString(ei));
        TGA_CUDA(cudaEventRecord(s->ev_join, s->side));
    }
    if (timed) TGA_CUDA(cudaEventRecordWithFlags(s->tev[s->tev_n], st, rec_flags));
    const bool etga = I->theta > 0;
    if (etga && !(I->dtype == TGA_I32 && s->fast && I->opt.score_mode == TGA_SCORE_FEASIBLE))
        return fail(TGA_ERR_UNSUPPORTED, "edge-based neighbourhood: integer feasible-only fast path only");
    if (etga && (mask & TGA_OP_REVERSED))
        return fail(TGA_ERR_UNSUPPORTED, "edge-based neighbourhood: reversed-segment variants");
    if (etga) {
        // ETGA: node -> slot map, then the cells the edge mask keeps; the
        // evaluated inter-route candidates are counted exactly on the device
        const int n_cust = I->n - 1;
        const int64_t cells = static_cast<int64_t>(I->n_gpairs) + static_cast<int64_t>(n_cust) * s->R +
                              static_cast<int64_t>(s->R) * s->R;
        tga_shard_range(cells, s->shard, s->n_shards, &a, &b);
        EtgaArgs ea{s->rec, s->rectw, static_cast<const int32_t *>(s->Dp), s->pitch, static_cast<uint32_t>(s->pitch),
                    s->node, s->pos, s->rlen, s->d_rbase, s->slot_of, I->dGpairs, I->n_gpairs, n_cust, s->R, s->Qp,
                    I->Q, s->keys, s->d_acc, static_cast<int>(a), static_cast<int>(b), s->sm_count};
        e = launch_etga(mask, I->tw, ea, st, !s->slot_of_fresh);
        s->slot_of_fresh = true;
    } else if (ns) {
        // the north-star sweep (2-opt* + relocate + swap (1,1)) has its own kernel;
        // intra-route variants, if any, follow in their own launch
        tga_shard_range(ns_tile_count(s->Qp, s->ns_rw), s->shard, s->n_shards, &a, &b);
        e = launch_ns_sweep(s->ns_rw, s->rec, s->nsc, s->pitch, s->nsmap, s->Qp, static_cast<int>(a), static_cast<int>(b),
                            static_cast<uint32_t>(s->pitch), I->Q, s->keys, reset && !timed, st, nullptr);
    } else if (I->dtype == TGA_I32 && s->fast) {
        tga_shard_range(s->n_ftiles, s->shard, s->n_shards, &a, &b);
        const int f_lo = static_cast<int>(a), f_hi = static_cast<int>(b);
        // fused: inter tiles + the intra-route CVRP work in one launch (when there is inter work)
        static const bool no_fuse = std::getenv("TGA_NO_FUSE") != nullptr;  // tuning override
        fused_intra = (mask & TGA_OP_INTER) && !I->tw && I->max_c_abs < (1 << 21) && !no_fuse;
        const uint32_t imask = fused_intra ? (mask & TGA_OP_INTRA) : 0u;
        e = launch_inter_fast(s->fastU, mask, s->rec, s->rectw, s->fmap, s->d_ftiles, f_lo, f_hi,
                              static_cast<uint32_t>(s->pitch), I->Q, s->keys, s->sm_count * 4, st,
                              sol_view<int32_t>(s), sp, imask, x_lo, x_hi);
    } else if (I->dtype == TGA_I32) {
        e = launch_inter<int32_t>(mask, I->tw, sol_view<int32_t>(s), s->tmap, s->d_tiles, t_lo, t_hi, sp, s->keys,
                                  grid, st);
    } else {
        e = launch_inter<float>(mask, I->tw, sol_view<float>(s), s->tmap, s->d_tiles, t_lo, t_hi, sp, s->keys, grid,
                                st);
    }
    if (timed) {
        TGA_CUDA(cudaEventRecordWithFlags(s->tev[s->tev_n + 1], st, rec_flags));
        s->tev_n += 2;
    }
    if (fork_intra && e == cudaSuccess) TGA_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));  // join
    if (e == cudaSuccess && !fused_intra && !fork_intra) {
        if (I->dtype == TGA_I32)
            e = launch_intra<int32_t>(mask, I->tw, sol_view<int32_t>(s), sp, x_lo, x_hi, s->keys, st,
                                      I->max_c_abs < (1 << 21) && !I->dPickup, warp_tw);
        else
            e = launch_intra<float>(mask, I->tw, sol_view<float>(s), sp, x_lo, x_hi, s->keys, st, false, warp_tw);
    }
    // reversed-segment variants beside a fast-path / north-star sweep: the generic
    // tile kernel (the generic branch above already covered them in its own launch)
    const bool generic_branch = !etga && !ns && !(I->dtype == TGA_I32 && s->fast);
    if (e == cudaSuccess && (mask & TGA_OP_REVERSED) && !generic_branch)
        e = launch_inter<int32_t>(mask & TGA_OP_REVERSED, I->tw, sol_view<int32_t>(s), s->tmap, s->d_tiles, t_lo, t_hi, sp,
                                  s->keys, grid, st);
    if (e != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("eval launch: ") + cudaGetErrorString(e));
    if (s->comm) {
        const ncclResult_t r = g_nccl.allReduce(s->keys, s->keys, TGA_N_VARIANTS, kNcclUint64, kNcclMin, s->comm, st);
        if (r != 0) return fail(TGA_ERR_NCCL, std::string("ncclAllReduce: ") + (g_nccl.errStr ? g_nccl.errStr(r) : "?"));
    }
    if (st != s->stream) TGA_CUDA(order_after(s->stream, st));  // later calls use the solution's stream
    s->eval_mask = accumulate ? (s->eval_mask | mask) : mask;
    s->eval_gen = s->gen;
    s->drained = false;
    return TGA_OK;
}

static uint64_t key_to_canonical(const tga_solution *s, uint64_t k);

// Test-only: one evaluation with the DUMP instantiations of the same kernels and launch
// decisions as tga_eval (no shards, no NCCL); every evaluated candidate's packed key
// is returned per variant over CANONICAL slots (see tga.h).
extern "C" int32_t tga_debug_eval_dump(tga_solution *s, uint32_t mask, int32_t flags, uint64_t *out, int64_t out_len) {
    if (!s || !out) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    const tga_instance *I = s->inst;
    mask &= TGA_OP_ALL;
    const int64_t Q = s->Qc;
    if (out_len < static_cast<int64_t>(TGA_N_VARIANTS) * Q * Q) return fail(TGA_ERR_INVALID_ARGUMENT, "out too small");
    if ((mask & TGA_OP_2OPT) && I->tw) return fail(TGA_ERR_UNSUPPORTED, "2-opt is only defined without time windows (P:148)");
    if (I->theta > 0) return fail(TGA_ERR_UNSUPPORTED, "dump of the edge-based neighbourhood");
    if (set_device(I) != TGA_OK) return TGA_ERR_CUDA;
    if (sync_host(s) != TGA_OK) return TGA_ERR_CUDA;
    const size_t plane = static_cast<size_t>(s->pitch) * s->pitch;
    unsigned long long *dump = nullptr;
    TGA_CUDA(cudaMalloc(&dump, plane * TGA_N_VARIANTS * 8));
    std::vector<unsigned long long> h(plane * TGA_N_VARIANTS);
    cudaStream_t st = s->stream;
    cudaError_t e = cudaMemsetAsync(dump, 0, plane * TGA_N_VARIANTS * 8, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(s->keys, 0xFF, TGA_N_VARIANTS * 8, st);
    const ScoreParams sp{I->Q, I->opt.score_mode, I->opt.w_load, I->opt.w_tw};
    const bool warp_tw = !I->dPickup && ((flags & 1) ? true : ((flags & 2) ? false : s->N >= 16 * s->R));
    const bool small = I->max_c_abs < (1 << 21) && !I->dPickup;
    const int grid = std::max(1, std::min(s->n_tiles, s->sm_count * 4));
    if (e == cudaSuccess) {
        if (ns_path(s, mask)) {   // the north-star sweep kernel, as tga_eval launches it
            e = launch_ns_sweep(s->ns_rw, s->rec, s->nsc, s->pitch, s->nsmap, s->Qp, 0, ns_tile_count(s->Qp, s->ns_rw),
                                static_cast<uint32_t>(s->pitch), I->Q,
                                s->keys, false, st, dump);
            if (e == cudaSuccess && (mask & TGA_OP_INTRA))
                e = launch_eval_dump<int32_t>(mask, I->tw, sol_view<int32_t>(s), s->tmap, s->d_tiles, 0, 0, sp, s->keys,
                                              grid, 0, s->Qp, false, small, warp_tw, st, dump);
        } else if (I->dtype == TGA_I32 && s->fast) {
            const bool fused = (mask & TGA_OP_INTER) && !I->tw && small;
            const uint32_t imask = fused ? (mask & TGA_OP_INTRA) : 0u;
            if (mask & TGA_OP_INTER)
                e = launch_inter_fast_dump(I->tw, s->rec, s->rectw, s->fmap, s->d_ftiles, 0, s->n_ftiles,
                                           static_cast<uint32_t>(s->pitch), I->Q, s->keys, st, sol_view<int32_t>(s),
                                           sp, imask, 0, s->Qp, dump);
            if (e == cudaSuccess && !fused)
                e = launch_eval_dump<int32_t>(mask, I->tw, sol_view<int32_t>(s), s->tmap, s->d_tiles, 0, 0, sp, s->keys,
                                              grid, 0, s->Qp, false, small, warp_tw, st, dump);
        }
        if ((ns_path(s, mask) || (I->dtype == TGA_I32 && s->fast)) && e == cudaSuccess && (mask & TGA_OP_REVERSED)) {
            // reversed-segment variants beside the fast paths: the generic tile kernel, as tga_eval
            e = launch_eval_dump<int32_t>(mask & TGA_OP_REVERSED, I->tw, sol_view<int32_t>(s), s->tmap, s->d_tiles, 0,
                                          s->n_tiles, sp, s->keys, grid, 0, s->Qp, false, small, warp_tw, st, dump);
        } else if (ns_path(s, mask) || (I->dtype == TGA_I32 && s->fast)) {
        } else if (I->dtype == TGA_I32) {
            e = launch_eval_dump<int32_t>(mask, I->tw, sol_view<int32_t>(s), s->tmap, s->d_tiles, 0, s->n_tiles, sp,
                                          s->keys, grid, 0, s->Qp, true, small, warp_tw, st, dump);
        } else {
            e = launch_eval_dump<float>(mask, I->tw, sol_view<float>(s), s->tmap, s->d_tiles, 0, s->n_tiles, sp,
                                        s->keys, grid, 0, s->Qp, true, false, warp_tw, st, dump);
        }
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), dump, plane * TGA_N_VARIANTS * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dump);
    if (e != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("eval dump: ") + cudaGetErrorString(e));
    // physical slot -> canonical id (-1: end depot, spare or padding)
    std::vector<int> can(s->pitch, -1);
    for (int r = 0; r < s->R; ++r)
        for (int p = 0; p <= static_cast<int>(s->routes[r].size()); ++p) can[s->rbase[r] + p] = s->cbase[r] + p;
    std::fill(out, out + TGA_N_VARIANTS * Q * Q, 0ull);
    for (int v = 0; v < TGA_N_VARIANTS; ++v) {
        if (!(mask & (1u << v))) continue;
        for (int a = 0; a < s->pitch; ++a) {
            if (can[a] < 0) continue;
            for (int b = 0; b < s->pitch; ++b) {
                const unsigned long long k = h[v * plane + static_cast<size_t>(a) * s->pitch + b];
                if (!k || can[b] < 0) continue;
                const uint64_t ci = static_cast<uint64_t>(can[a]) * Q + can[b];
                out[v * Q * Q + ci] = k == ~0ull ? ~0ull : ((k & 0xFFFFFFFF00000000ull) | ci);
            }
        }
    }
    s->eval_gen = s->gen;
    s->eval_mask = mask;
    s->keys_clean = false;
    s->drained = true;
    return TGA_OK;
}

extern "C" int32_t tga_solution_keys(tga_solution *s, uint64_t *keys) {
    if (!s || !keys) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (sync_host(s) != TGA_OK) return TGA_ERR_CUDA;
    TGA_CUDA(cudaMemcpyAsync(s->h_keys, s->keys, TGA_N_VARIANTS * 8, cudaMemcpyDeviceToHost, s->stream));
    TGA_CUDA(cudaStreamSynchronize(s->stream));
    for (int v = 0; v < TGA_N_VARIANTS; ++v) keys[v] = key_to_canonical(s, s->h_keys[v]);
    return TGA_OK;
}

static double decode_score(uint32_t ord, bool integer, int64_t *as_int) {
    if (integer) {
        const int32_t v = static_cast<int32_t>(ord ^ 0x80000000u);
        *as_int = v;
        return static_cast<double>(v);
    }
    const uint32_t u = (ord & 0x80000000u) ? (ord ^ 0x80000000u) : ~ord;
    float f;
    std::memcpy(&f, &u, 4);
    *as_int = static_cast<int64_t>(std::llround(static_cast<double>(f)));
    return static_cast<double>(f);
}

// physical slot -> (route, position): largest route with rbase <= x
static void phys_to_rp(const tga_solution *s, int x, int *r, int *p) {
    const auto it = std::upper_bound(s->rbase.begin(), s->rbase.begin() + s->R, x);
    *r = static_cast<int>(it - s->rbase.begin()) - 1;
    *p = x - s->rbase[*r];
}

// a key over physical slots -> the same key over canonical slots (u * Q + v)
static uint64_t key_to_canonical(const tga_solution *s, uint64_t k) {
    if (k == ~0ull) return k;
    const uint32_t idx = static_cast<uint32_t>(k & 0xFFFFFFFFu);
    int ra, pa, rb, pb;
    phys_to_rp(s, static_cast<int>(idx / static_cast<uint32_t>(s->pitch)), &ra, &pa);
    phys_to_rp(s, static_cast<int>(idx % static_cast<uint32_t>(s->pitch)), &rb, &pb);
    const uint64_t c = static_cast<uint64_t>(s->cbase[ra] + pa) * static_cast<uint32_t>(s->Qc) + (s->cbase[rb] + pb);
    return (k & 0xFFFFFFFF00000000ull) | c;
}

static void canon_to_rp(const tga_solution *s, int c, int *r, int *p) {
    // largest route with cbase <= c
    const auto it = std::upper_bound(s->cbase.begin(), s->cbase.begin() + s->R, c);
    *r = static_cast<int>(it - s->cbase.begin()) - 1;
    *p = c - s->cbase[*r];
}

static int32_t decode_best(const tga_solution *s, const uint64_t *keys, uint32_t mask, tga_move *out);

extern "C" int32_t tga_best_move(tga_solution *s, uint32_t mask, tga_move *out) {
    if (!s || !out) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (s->eval_gen != s->gen) return fail(TGA_ERR_STALE, "no evaluation for the current generation");
    if (sync_host(s) != TGA_OK) return TGA_ERR_CUDA;
    TGA_CUDA(cudaMemcpyAsync(s->h_keys, s->keys, TGA_N_VARIANTS * 8, cudaMemcpyDeviceToHost, s->stream));
    TGA_CUDA(cudaStreamSynchronize(s->stream));
    s->drained = true;
    mask &= s->eval_mask;
    return decode_best(s, s->h_keys, mask, out);
}

// lowest (score, variant rank, flat index) over the keys of `mask` -> tga_move
static int32_t decode_best(const tga_solution *s, const uint64_t *keys, uint32_t mask, tga_move *out) {
    int bv = -1;
    uint64_t bk = ~0ull;
    for (int v = 0; v < TGA_N_VARIANTS; ++v) {
        if (!(mask & (1u << v))) continue;
        const uint64_t k = keys[v];
        if (k == ~0ull) continue;
        // variants visited in rank order: a later variant wins only with a strictly lower score
        if (bv < 0 || (k >> 32) < (bk >> 32)) { bv = v; bk = k; }
    }
    std::memset(out, 0, sizeof(*out));
    out->key = ~0ull;
    out->generation = s->gen;
    out->variant = -1;
    if (bv < 0) return TGA_NO_IMPROVING_MOVE;
    const uint32_t idx = static_cast<uint32_t>(bk & 0xFFFFFFFFu);
    const int xu = static_cast<int>(idx / static_cast<uint32_t>(s->pitch));  // physical slots
    const int xv = static_cast<int>(idx % static_cast<uint32_t>(s->pitch));
    out->variant = bv;
    variant_lengths(bv, &out->n1, &out->n2);
    phys_to_rp(s, xu, &out->route_a, &out->pos_a);
    phys_to_rp(s, xv, &out->route_b, &out->pos_b);
    out->u = s->cbase[out->route_a] + out->pos_a;  // canonical ids
    out->v = s->cbase[out->route_b] + out->pos_b;
    bk = (bk & 0xFFFFFFFF00000000ull) | (static_cast<uint64_t>(out->u) * static_cast<uint32_t>(s->Qc) + out->v);
    out->delta_f = decode_score(static_cast<uint32_t>(bk >> 32), s->inst->dtype == TGA_I32, &out->delta_i);
    out->feasible = 1;
    if (s->inst->opt.score_mode == TGA_SCORE_PENALISED) out->feasible = -1;  // not tracked in penalised mode
    out->key = bk;
    return out->delta_f < 0 ? TGA_OK : TGA_NO_IMPROVING_MOVE;
}

// ============================================================== ABI: update
// Splice the host route lists (Fig. `operators` P:107-146) -- the update of S
// (Alg. A2 line 7) -- then synchronise the device state of the changed
// span only.
static bool splice(std::vector<std::vector<int32_t>> &routes, const tga_move *m) {
    const int v = m->variant, ra = m->route_a, rb = m->route_b, pa = m->pos_a, pb = m->pos_b;
    const int R = static_cast<int>(routes.size());
    if (ra < 0 || ra >= R || rb < 0 || rb >= R) return false;
    std::vector<int32_t> &a = routes[ra];
    std::vector<int32_t> &b = routes[rb];
    const int La = static_cast<int>(a.size()), Lb = static_cast<int>(b.size());
    int n1, n2;
    variant_lengths(v, &n1, &n2);
    typedef std::vector<int32_t> V;
    auto sl = [](const V &x, int i, int j) { return V(x.begin() + i, x.begin() + j); };  // [i, j)
    auto cat = [](std::initializer_list<V> parts) {
        V r;
        for (auto &p : parts) r.insert(r.end(), p.begin(), p.end());
        return r;
    };
    if (v == TGA_V_2OPT_STAR) {
        if (ra == rb || pa < 0 || pa > La || pb < 0 || pb > Lb) return false;
        V na = cat({sl(a, 0, pa), sl(b, pb, Lb)}), nb = cat({sl(b, 0, pb), sl(a, pa, La)});
        a.swap(na); b.swap(nb);
    } else if (v >= TGA_V_RELOCATE1 && v <= TGA_V_OROPT3) {
        if (ra == rb || pa < 1 || pa + n1 - 1 > La || pb < 0 || pb > Lb) return false;
        V seg = sl(a, pa - 1, pa - 1 + n1);
        V na = cat({sl(a, 0, pa - 1), sl(a, pa - 1 + n1, La)}), nb = cat({sl(b, 0, pb), seg, sl(b, pb, Lb)});
        a.swap(na); b.swap(nb);
    } else if (v >= TGA_V_SWAP11 && v <= TGA_V_CROSS33) {
        if (ra == rb || pa < 1 || pa + n1 - 1 > La || pb < 1 || pb + n2 - 1 > Lb) return false;
        V sa = sl(a, pa - 1, pa - 1 + n1), sb = sl(b, pb - 1, pb - 1 + n2);
        V na = cat({sl(a, 0, pa - 1), sb, sl(a, pa - 1 + n1, La)});
        V nb = cat({sl(b, 0, pb - 1), sa, sl(b, pb - 1 + n2, Lb)});
        a.swap(na); b.swap(nb);
    } else if (v == TGA_V_2OPT) {
        if (ra != rb || pa < 1 || pb <= pa || pb > La) return false;
        std::reverse(a.begin() + (pa - 1), a.begin() + pb);
    } else if (v >= TGA_V_IRELOCATE1 && v <= TGA_V_IRELOCATE3) {
        if (ra != rb || pa < 1 || pa + n1 - 1 > La || pb < 0 || pb > La) return false;
        if (pb >= pa - 1 && pb <= pa + n1 - 1) return false;
        V seg = sl(a, pa - 1, pa - 1 + n1), na;
        if (pb > pa) na = cat({sl(a, 0, pa - 1), sl(a, pa - 1 + n1, pb), seg, sl(a, pb, La)});
        else na = cat({sl(a, 0, pb), seg, sl(a, pb, pa - 1), sl(a, pa - 1 + n1, La)});
        a.swap(na);
    } else if (v >= TGA_V_ISWAP11 && v <= TGA_V_ISWAP33) {
        if (ra != rb || pa < 1 || pa + n1 > pb || pb + n2 - 1 > La) return false;
        V na = cat({sl(a, 0, pa - 1), sl(a, pb - 1, pb - 1 + n2), sl(a, pa - 1 + n1, pb - 1), sl(a, pa - 1, pa - 1 + n1),
                    sl(a, pb - 1 + n2, La)});
        a.swap(na);
    } else if (v == TGA_V_OROPT2R || v == TGA_V_OROPT3R) {   // the segment inserted reversed
        if (ra == rb || pa < 1 || pa + n1 - 1 > La || pb < 0 || pb > Lb) return false;
        V seg = sl(a, pa - 1, pa - 1 + n1);
        std::reverse(seg.begin(), seg.end());
        V na = cat({sl(a, 0, pa - 1), sl(a, pa - 1 + n1, La)}), nb = cat({sl(b, 0, pb), seg, sl(b, pb, Lb)});
        a.swap(na); b.swap(nb);
    } else if (v == TGA_V_CROSS22R || v == TGA_V_CROSS33R) {   // both segments reversed
        if (ra == rb || pa < 1 || pa + n1 - 1 > La || pb < 1 || pb + n2 - 1 > Lb) return false;
        V sa = sl(a, pa - 1, pa - 1 + n1), sb = sl(b, pb - 1, pb - 1 + n2);
        std::reverse(sa.begin(), sa.end());
        std::reverse(sb.begin(), sb.end());
        V na = cat({sl(a, 0, pa - 1), sb, sl(a, pa - 1 + n1, La)});
        V nb = cat({sl(b, 0, pb - 1), sa, sl(b, pb - 1 + n2, Lb)});
        a.swap(na); b.swap(nb);
    } else {
        return false;
    }
    return true;
}

extern "C" int32_t tga_apply_move(tga_solution *s, const tga_move *m) {
    if (!s || !m) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (m->generation != s->gen) return fail(TGA_ERR_STALE, "move generation does not match the solution");
    if (m->variant < 0 || m->variant >= TGA_N_VARIANTS) return fail(TGA_ERR_INVALID_ARGUMENT, "variant");
    if (set_device(s->inst) != TGA_OK) return TGA_ERR_CUDA;
    if (sync_host(s) != TGA_OK) return TGA_ERR_CUDA;
    if (!s->drained) TGA_CUDA(cudaStreamSynchronize(s->stream));  // staging buffers may still be in flight
    s->drained = false;
    if (!splice(s->routes, m)) return fail(TGA_ERR_INVALID_ARGUMENT, "move positions out of range for its variant");
    const int ra = m->route_a, rb = m->route_b;
    int32_t rc;
    if (route_fits(s, ra) && route_fits(s, rb)) {  // bases unchanged: refresh the two routes only
        compute_cbase(s);
        if ((rc = upload_layout(s, false, ra, rb)) != TGA_OK) return rc;
        if ((rc = refresh(s, false, ra, rb)) != TGA_OK) return rc;
    } else {                                        // a route outgrew its slots: full relayout
        relayout_full(s);
        if ((rc = upload_layout(s, true)) != TGA_OK) return rc;
        if ((rc = refresh(s, true)) != TGA_OK) return rc;
    }
    ++s->gen;
    return TGA_OK;
}

// ============================================================== ABI: queries
extern "C" int32_t tga_solution_counts(const tga_solution *cs, uint64_t *c) {
    if (!cs || !c) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    tga_solution *s = const_cast<tga_solution *>(cs);  // refreshing the host cache only
    if (sync_host(s) != TGA_OK) return TGA_ERR_CUDA;
    std::memset(c, 0, sizeof(uint64_t) * TGA_N_VARIANTS);
    const int R = s->R;
    std::vector<int64_t> L(R);
    for (int r = 0; r < R; ++r) L[r] = static_cast<int64_t>(s->routes[r].size());
    auto pos = [](int64_t x) { return x > 0 ? x : 0; };
    int64_t sumL1 = 0;
    for (int r = 0; r < R; ++r) sumL1 += L[r] + 1;
    // 2-opt*: sum_{a<b} (La+1)(Lb+1)
    {
        int64_t acc = 0, pre = 0;
        for (int r = 0; r < R; ++r) { acc += pre * (L[r] + 1); pre += L[r] + 1; }
        c[TGA_V_2OPT_STAR] = acc;
    }
    for (int N = 1; N <= 3; ++N) {  // relocate: sum_a max(La-N+1,0) * (sum_{b != a} (Lb+1))
        int64_t acc = 0;
        for (int r = 0; r < R; ++r) acc += pos(L[r] - N + 1) * (sumL1 - (L[r] + 1));
        c[TGA_V_RELOCATE1 + N - 1] = acc;
    }
    static const int sw[6][2] = {{1, 1}, {1, 2}, {1, 3}, {2, 2}, {2, 3}, {3, 3}};
    for (int k = 0; k < 6; ++k) {
        const int n1 = sw[k][0], n2 = sw[k][1];
        int64_t s1 = 0, s2 = 0, diag = 0;
        for (int r = 0; r < R; ++r) { s1 += pos(L[r] - n1 + 1); s2 += pos(L[r] - n2 + 1); diag += pos(L[r] - n1 + 1) * pos(L[r] - n2 + 1); }
        const int64_t ordered = s1 * s2 - diag;
        c[TGA_V_SWAP11 + k] = (n1 == n2) ? ordered / 2 : ordered;
    }
    for (int r = 0; r < R; ++r) {
        c[TGA_V_2OPT] += L[r] * (L[r] - 1) / 2;
        for (int N = 1; N <= 3; ++N) c[TGA_V_IRELOCATE1 + N - 1] += pos(L[r] - N + 1) * pos(L[r] - N);
        for (int a = 1; a <= 3; ++a)
            for (int b = 1; b <= 3; ++b) {
                const int64_t M = L[r] - a - b + 1;
                c[TGA_V_ISWAP11 + 3 * (a - 1) + (b - 1)] += M >= 1 ? M * (M + 1) / 2 : 0;
            }
    }
    // reversed segments: the candidate spaces of or-opt N and cross (N, N)
    c[TGA_V_OROPT2R] = c[TGA_V_OROPT2];
    c[TGA_V_OROPT3R] = c[TGA_V_OROPT3];
    c[TGA_V_CROSS22R] = c[TGA_V_CROSS22];
    c[TGA_V_CROSS33R] = c[TGA_V_CROSS33];
    return TGA_OK;
}

extern "C" int32_t tga_solution_info(const tga_solution *s, int32_t *R, int32_t *N, int32_t *Q, uint64_t *gen) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    if (R) *R = s->R;
    if (N) *N = s->N;
    if (Q) *Q = s->Qc;
    if (gen) *gen = s->gen;
    return TGA_OK;
}

extern "C" int32_t tga_solution_routes(const tga_solution *cs, int32_t *ptr, int32_t *cust) {
    if (!cs || !ptr || !cust) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    tga_solution *s = const_cast<tga_solution *>(cs);  // refreshing the host cache only
    if (sync_host(s) != TGA_OK) return TGA_ERR_CUDA;
    int q = 0;
    ptr[0] = 0;
    for (int r = 0; r < s->R; ++r) {
        for (int32_t c : s->routes[r]) cust[q++] = c;
        ptr[r + 1] = q;
    }
    return TGA_OK;
}

extern "C" int32_t tga_solution_cost(tga_solution *s, int64_t *dist_i, double *dist_f, int64_t *lex, double *tex) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    TGA_CUDA(cudaStreamSynchronize(s->stream));
    std::vector<int32_t> W(s->R), Draw(s->R);
    std::vector<float> TV(s->R);
    TGA_CUDA(cudaMemcpy(W.data(), s->d_rW, 4 * s->R, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(Draw.data(), s->d_rD, 4 * s->R, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(TV.data(), s->d_rTV, 4 * s->R, cudaMemcpyDeviceToHost));
    int64_t di = 0, le = 0;
    double df = 0, te = 0;
    for (int r = 0; r < s->R; ++r) {
        if (s->inst->dtype == TGA_I32) { di += Draw[r]; df += Draw[r]; }
        else { float f; std::memcpy(&f, &Draw[r], 4); df += f; di = static_cast<int64_t>(std::llround(df)); }
        le += std::max<int64_t>(W[r] - s->inst->Q, 0);
        if (s->inst->tw) te += TV[r];
    }
    if (dist_i) *dist_i = di;
    if (dist_f) *dist_f = df;
    if (lex) *lex = le;
    if (tex) *tex = te;
    return TGA_OK;
}

extern "C" int32_t tga_solution_attributes(tga_solution *s, int64_t *pre_L, int64_t *suf_L, double *pre_D,
                                           double *suf_D, double *pre_TV, double *suf_TV, double *start) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    if (sync_host(s) != TGA_OK) return TGA_ERR_CUDA;
    TGA_CUDA(cudaStreamSynchronize(s->stream));
    const int Qp = s->Qp;
    std::vector<int32_t> fL(Qp), bL(Qp), fD(Qp), bD(Qp), nd(Qp);
    std::vector<TwRec> fT(Qp), bT(Qp);
    TGA_CUDA(cudaMemcpy(fL.data(), s->fwdL, 4 * Qp, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(bL.data(), s->bwdL, 4 * Qp, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(fD.data(), s->fwdD, 4 * Qp, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(bD.data(), s->bwdD, 4 * Qp, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(nd.data(), s->node, 4 * Qp, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(fT.data(), s->fwdT, 16 * Qp, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(bT.data(), s->bwdT, 16 * Qp, cudaMemcpyDeviceToHost));
    auto asd = [&](int32_t raw) -> double {
        if (s->inst->dtype == TGA_I32) return raw;
        float f;
        std::memcpy(&f, &raw, 4);
        return f;
    };
    for (int r = 0; r < s->R; ++r) {
        const int L = static_cast<int>(s->routes[r].size());
        for (int p = 0; p <= L; ++p) {
            const int x = s->rbase[r] + p, c = s->cbase[r] + p;
            if (pre_L) pre_L[c] = fL[x];
            if (suf_L) suf_L[c] = bL[x];
            if (pre_D) pre_D[c] = asd(fD[x]);
            if (suf_D) suf_D[c] = asd(bD[x]);
            if (pre_TV) pre_TV[c] = s->inst->tw ? fT[x].w : 0.0;
            if (suf_TV) suf_TV[c] = s->inst->tw ? bT[x].w : 0.0;
            if (start) {
                // service start at p from the prefix record: T_E + T_D - T_V - s
                start[c] = s->inst->tw
                               ? static_cast<double>(fT[x].y) + fT[x].x - fT[x].w - s->inst->hTw[3 * nd[x] + 2]
                               : 0.0;
            }
        }
    }
    return TGA_OK;
}

extern "C" int32_t tga_solution_load_records(tga_solution *s, int32_t *pre, int32_t *suf) {
    if (!s || !pre || !suf) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!s->fwdP) return fail(TGA_ERR_UNSUPPORTED, "no pickups: the instance has no load records");
    if (sync_host(s) != TGA_OK) return TGA_ERR_CUDA;
    TGA_CUDA(cudaStreamSynchronize(s->stream));
    std::vector<LoadRec> fP(s->Qp), bP(s->Qp);
    TGA_CUDA(cudaMemcpy(fP.data(), s->fwdP, sizeof(LoadRec) * s->Qp, cudaMemcpyDeviceToHost));
    TGA_CUDA(cudaMemcpy(bP.data(), s->bwdP, sizeof(LoadRec) * s->Qp, cudaMemcpyDeviceToHost));
    for (int r = 0; r < s->R; ++r) {
        const int L = static_cast<int>(s->routes[r].size());
        for (int p = 0; p <= L; ++p) {
            const int x = s->rbase[r] + p, c = s->cbase[r] + p;
            pre[3 * c] = fP[x].x; pre[3 * c + 1] = fP[x].y; pre[3 * c + 2] = fP[x].z;
            suf[3 * c] = bP[x].x; suf[3 * c + 1] = bP[x].y; suf[3 * c + 2] = bP[x].z;
        }
    }
    return TGA_OK;
}

// ============================================================== ABI: multi-GPU
extern "C" int32_t tga_nccl_unique_id(void *out) {
    if (!out) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!g_nccl.load()) return fail(TGA_ERR_NCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    const ncclResult_t r = g_nccl.getUniqueId(&id);
    if (r != 0) return fail(TGA_ERR_NCCL, "ncclGetUniqueId failed");
    std::memcpy(out, &id, sizeof(id));
    return TGA_OK;
}

extern "C" int32_t tga_comm_init(tga_solution *s, int32_t rank, int32_t world, const void *uid) {
    if (!s || !uid || world < 1 || rank < 0 || rank >= world) return fail(TGA_ERR_INVALID_ARGUMENT, "comm args");
    if (!g_nccl.load()) return fail(TGA_ERR_NCCL, "libnccl.so.2 not loadable");
    if (set_device(s->inst) != TGA_OK) return TGA_ERR_CUDA;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    ncclComm_t c = nullptr;
    const ncclResult_t r = g_nccl.commInitRank(&c, world, id, rank);
    if (r != 0) return fail(TGA_ERR_NCCL, std::string("ncclCommInitRank: ") + (g_nccl.errStr ? g_nccl.errStr(r) : "?"));
    if (s->comm) g_nccl.commDestroy(s->comm);
    s->comm = c;
    s->shard = rank;
    s->n_shards = world;
    return TGA_OK;
}

// ============================================================== ABI: step / reload / timing
extern "C" int32_t tga_step(tga_solution *s, uint32_t mask, tga_move *out) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    int32_t rc = tga_eval(s, mask, nullptr);
    if (rc != TGA_OK) return rc;
    tga_move m;
    rc = tga_best_move(s, mask, &m);
    if (out) *out = m;
    if (rc != TGA_OK) return rc;  // TGA_NO_IMPROVING_MOVE or an error
    return tga_apply_move(s, &m);
}

extern "C" int32_t tga_solution_reload(tga_solution *s, int32_t R, const int32_t *ptr, const int32_t *cust) {
    if (!s || !ptr || !cust) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    const tga_instance *I = s->inst;
    if (R != s->R) return fail(TGA_ERR_INVALID_ARGUMENT, "reload needs the same route count");
    if (ptr[0] != 0 || ptr[R] != I->n - 1) return fail(TGA_ERR_STRUCTURE, "route_ptr does not cover the customers");
    std::vector<char> seen(I->n, 0);
    for (int r = 0; r < R; ++r) {
        if (ptr[r + 1] < ptr[r]) return fail(TGA_ERR_STRUCTURE, "route_ptr not non-decreasing");
        for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
            const int c = cust[k];
            if (c <= 0 || c >= I->n || seen[c]) return fail(TGA_ERR_STRUCTURE, "customer out of range or repeated");
            seen[c] = 1;
        }
    }
    if (set_device(I) != TGA_OK) return TGA_ERR_CUDA;
    TGA_CUDA(cudaStreamSynchronize(s->stream));  // staging buffers may still be in flight
    s->host_stale = false;
    for (int r = 0; r < R; ++r) s->routes[r].assign(cust + ptr[r], cust + ptr[r + 1]);
    relayout_full(s);
    int32_t rc;
    if ((rc = upload_layout(s, true)) != TGA_OK) return rc;
    if ((rc = refresh(s, true)) != TGA_OK) return rc;
    ++s->gen;
    s->drained = false;
    return TGA_OK;
}

extern "C" int32_t tga_solution_enable_timing(tga_solution *s, int32_t enable) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    if (enable && s->tev.empty()) {
        s->tev.resize(8192);
        for (auto &e : s->tev) TGA_CUDA(cudaEventCreate(&e));
    }
    s->timing = enable != 0;
    s->tev_n = 0;
    return TGA_OK;
}

extern "C" int32_t tga_solution_timings(tga_solution *s, float *ms, int32_t max_n, int32_t *n_out) {
    if (!s || !n_out) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    int n = 0;
    for (int i = 0; i + 1 < s->tev_n && n < max_n; i += 2) {
        TGA_CUDA(cudaEventSynchronize(s->tev[i + 1]));
        float t = 0.f;
        TGA_CUDA(cudaEventElapsedTime(&t, s->tev[i], s->tev[i + 1]));
        if (ms) ms[n] = t;
        ++n;
    }
    s->tev_n = 0;
    *n_out = n;
    return TGA_OK;
}

// ============================================================== ABI: device-resident step
extern "C" int32_t tga_step_async(tga_solution *s, uint32_t mask) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    int32_t rc = tga_eval(s, mask, nullptr);
    if (rc != TGA_OK) return rc;
    const tga_instance *I = s->inst;
    // pick + splice + update in one launch: one block per SM at most (grid barrier)
    // ETGA counts its (masked) inter-route candidates in the eval kernel; the closed forms cover the rest
    const uint32_t cmask = I->theta > 0 ? (s->eval_mask & TGA_OP_INTRA) : s->eval_mask;
    // the state by value (kernel parameters): the chain's first loads are data, not the state
    const DevState hs = make_devstate(s, s->keys);
    const auto hsi = I->dtype == TGA_I32 ? scan_args<int32_t>(s) : ScanArgs<int32_t>{};
    const auto hsf = I->dtype == TGA_I32 ? ScanArgs<float>{} : scan_args<float>(s);
    const void *hsa = I->dtype == TGA_I32 ? static_cast<const void *>(&hsi) : static_cast<const void *>(&hsf);
    cudaError_t e = launch_pick_update(s->d_ds, s->d_sa, 1, I->tw, I->dtype == TGA_I32, s->eval_mask, cmask, s->R,
                                       s->N + 2 + s->slack,  // upper bound of any route's slot capacity
                                       s->sm_count, s->stream, &hs, hsa);
    if (e != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("device step: ") + cudaGetErrorString(e));
    s->keys_clean = true;
    s->clean_cap = capture_id(s->stream);
    ++s->gen;
    s->host_stale = true;
    s->drained = false;
    return TGA_OK;
}

// The whole descent is captured once into a CUDA graph (memsets, kernels and the
// per-step event records as external event nodes) and launched as one unit:
// no per-kernel CPU launch cost and short inter-kernel gaps.
extern "C" int32_t tga_descent(tga_solution *s, uint32_t mask, int32_t n_steps, void *l2_flush, uint64_t flush_bytes,
                               float *step_ms) {
    if (!s || n_steps < 0) return fail(TGA_ERR_INVALID_ARGUMENT, "descent arguments");
    if (n_steps == 0) return TGA_OK;
    if (set_device(s->inst) != TGA_OK) return TGA_ERR_CUDA;
    std::vector<cudaEvent_t> ev;
    if (step_ms) {
        ev.resize(2 * static_cast<size_t>(n_steps));
        for (auto &e : ev) TGA_CUDA(cudaEventCreate(&e));
    }
    // capture on a private stream forked from the solution's stream
    cudaStream_t cap;
    TGA_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaStream_t saved = s->stream;
    int32_t rc = TGA_OK;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = order_after(cap, saved);
    if (e == cudaSuccess) e = cudaStreamSynchronize(saved);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        s->stream = cap;
        for (int k = 0; k < n_steps && rc == TGA_OK && e == cudaSuccess; ++k) {
            if (l2_flush && flush_bytes) e = cudaMemsetAsync(l2_flush, k & 0xFF, flush_bytes, cap);
            if (e == cudaSuccess && step_ms) e = cudaEventRecordWithFlags(ev[2 * k], cap, cudaEventRecordExternal);
            if (e == cudaSuccess) rc = tga_step_async(s, mask);
            if (e == cudaSuccess && rc == TGA_OK && step_ms)
                e = cudaEventRecordWithFlags(ev[2 * k + 1], cap, cudaEventRecordExternal);
        }
        const cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
        if (e == cudaSuccess) e = e2;
        s->stream = saved;
    }
    if (e == cudaSuccess && rc == TGA_OK) e = cudaGraphInstantiate(&exec, graph, 0);
    if (e == cudaSuccess && rc == TGA_OK) e = cudaGraphLaunch(exec, saved);
    if (e == cudaSuccess && rc == TGA_OK) e = cudaStreamSynchronize(saved);
    if (e == cudaSuccess && rc == TGA_OK) s->clean_cap = 0;  // the captured steps have executed
    else s->keys_clean = false;
    if (e == cudaSuccess && rc == TGA_OK && step_ms)
        for (int k = 0; k < n_steps && e == cudaSuccess; ++k) e = cudaEventElapsedTime(&step_ms[k], ev[2 * k], ev[2 * k + 1]);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    for (auto x : ev) cudaEventDestroy(x);
    if (rc != TGA_OK) return rc;
    if (e != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("descent graph: ") + cudaGetErrorString(e));
    return TGA_OK;
}

extern "C" int32_t tga_solution_debug_probe(tga_solution *s, int32_t enable, uint64_t *out) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    if (set_device(s->inst) != TGA_OK) return TGA_ERR_CUDA;
    if (out) {
        TGA_CUDA(cudaMemcpyAsync(out, s->d_acc + 32, 16 * 8, cudaMemcpyDeviceToHost, s->stream));
        TGA_CUDA(cudaMemcpyAsync(out + 16, s->d_acc + kTimeline, 2 * kTimelineBlocks * 8, cudaMemcpyDeviceToHost, s->stream));
        TGA_CUDA(cudaStreamSynchronize(s->stream));
    }
    const unsigned long long flag = enable ? 1ull : 0ull;
    TGA_CUDA(cudaMemcpyAsync(s->d_acc + 31, &flag, 8, cudaMemcpyHostToDevice, s->stream));
    TGA_CUDA(cudaStreamSynchronize(s->stream));
    return TGA_OK;
}

extern "C" int32_t tga_solution_device_stats(tga_solution *s, uint64_t *counts, uint64_t *applied) {
    if (!s) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL solution");
    unsigned long long acc[48];
    TGA_CUDA(cudaMemcpyAsync(acc, s->d_acc, sizeof(acc), cudaMemcpyDeviceToHost, s->stream));
    TGA_CUDA(cudaStreamSynchronize(s->stream));
    TGA_CUDA(cudaMemsetAsync(s->d_acc, 0, (kAccApplied + 1) * 8, s->stream));  // counts + applied (not the probe)
    if (counts) for (int v = 0; v < TGA_N_VARIANTS; ++v) counts[v] = acc[v];
    if (applied) *applied = acc[kAccApplied];
    return TGA_OK;
}

// ============================================================== ABI: population batch
struct tga_batch {
    tga_instance *inst = nullptr;
    std::vector<tga_solution *> sols;
    cudaStream_t stream = nullptr;
    void *d_views = nullptr;        // SolView<DT>[n]
    CUtensorMap *d_maps = nullptr;  // [n]
    uint32_t *d_work = nullptr;     // (solution << 20 | tile) work items
    uint64_t *d_keys = nullptr;     // [n][23]
    uint64_t *h_keys = nullptr;     // pinned [n][23]
    int n_work = 0, max_qp = 0, sm_count = 148;
    uint32_t eval_mask = 0;
    std::vector<uint64_t> eval_gen;
    cudaStream_t own_stream = nullptr;
    DevState *d_states = nullptr;   // per solution, keys pointing into d_keys
    void *d_scans = nullptr;        // ScanArgs<DT> per solution
    // fast path (integer, feasible-only): per-solution records, fast TMA maps, (k, I, J) items
    bool fast = false;
    FastSol *d_fsols = nullptr;
    CUtensorMap *d_fmaps = nullptr;
    uint32_t *d_fwork = nullptr;
    int n_fwork = 0;
};

static void free_batch(tga_batch *b) {
    if (!b) return;
    for (auto *s : b->sols) free_solution(s);
    if (b->d_views) cudaFree(b->d_views);
    if (b->d_maps) cudaFree(b->d_maps);
    if (b->d_fsols) cudaFree(b->d_fsols);
    if (b->d_fmaps) cudaFree(b->d_fmaps);
    if (b->d_fwork) cudaFree(b->d_fwork);
    if (b->d_work) cudaFree(b->d_work);
    if (b->d_keys) cudaFree(b->d_keys);
    if (b->h_keys) cudaFreeHost(b->h_keys);
    if (b->d_states) cudaFree(b->d_states);
    if (b->d_scans) cudaFree(b->d_scans);
    if (b->own_stream) cudaStreamDestroy(b->own_stream);
    delete b;
}

extern "C" int32_t tga_batch_load(tga_instance *I, int32_t n_sol, const int32_t *n_routes, const int32_t *route_ptr,
                                  const int32_t *customers, tga_batch **out) {
    if (!I || !n_routes || !route_ptr || !customers || !out || n_sol < 1 || n_sol > 4096)
        return fail(TGA_ERR_INVALID_ARGUMENT, "batch arguments");
    *out = nullptr;
    if (set_device(I) != TGA_OK) return TGA_ERR_CUDA;
    auto *b = new (std::nothrow) tga_batch();
    if (!b) return fail(TGA_ERR_OOM, "host allocation");
    b->inst = I;
    auto bail = [&](int32_t code) { free_batch(b); return code; };
    if (cudaStreamCreateWithFlags(&b->own_stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(TGA_ERR_CUDA, "stream"));
    b->stream = b->own_stream;
    size_t rp = 0;
    const int ncust = I->n - 1;
    std::vector<uint32_t> work;
    for (int k = 0; k < n_sol; ++k) {
        tga_solution *s = nullptr;
        int32_t rc = tga_solution_load(I, n_routes[k], route_ptr + rp, customers + static_cast<size_t>(k) * ncust, &s);
        if (rc != TGA_OK) return bail(rc);
        b->sols.push_back(s);
        tga_solution_set_stream(s, b->stream);
        rp += static_cast<size_t>(n_routes[k]) + 1;
        b->max_qp = std::max(b->max_qp, s->Qp);
        if (s->n_tiles >= (1 << 20)) return bail(fail(TGA_ERR_INVALID_ARGUMENT, "too many tiles per solution"));
        for (int t = 0; t < s->n_tiles; ++t) work.push_back((static_cast<uint32_t>(k) << 20) | static_cast<uint32_t>(t));
    }
    b->n_work = static_cast<int>(work.size());
    b->eval_gen.assign(n_sol, 0);
    {
        cudaDeviceProp prop;
        if (cudaGetDeviceProperties(&prop, I->device) == cudaSuccess) b->sm_count = prop.multiProcessorCount;
    }
    const size_t vsz = I->dtype == TGA_I32 ? sizeof(SolView<int32_t>) : sizeof(SolView<float>);
    std::vector<unsigned char> views(vsz * n_sol);
    std::vector<CUtensorMap> maps(n_sol);
    for (int k = 0; k < n_sol; ++k) {
        if (I->dtype == TGA_I32) { auto v = sol_view<int32_t>(b->sols[k]); std::memcpy(&views[vsz * k], &v, vsz); }
        else { auto v = sol_view<float>(b->sols[k]); std::memcpy(&views[vsz * k], &v, vsz); }
        maps[k] = b->sols[k]->tmap;
    }
    if (cudaMalloc(&b->d_views, views.size()) != cudaSuccess ||
        cudaMalloc(&b->d_maps, sizeof(CUtensorMap) * n_sol) != cudaSuccess ||
        cudaMalloc(&b->d_work, sizeof(uint32_t) * std::max<size_t>(1, work.size())) != cudaSuccess ||
        cudaMalloc(&b->d_keys, sizeof(uint64_t) * TGA_N_VARIANTS * n_sol) != cudaSuccess ||
        cudaMallocHost(&b->h_keys, sizeof(uint64_t) * TGA_N_VARIANTS * n_sol) != cudaSuccess)
        return bail(fail(TGA_ERR_OOM, "batch allocation"));
    {
        std::vector<DevState> ds(n_sol);
        const size_t ssz = I->dtype == TGA_I32 ? sizeof(ScanArgs<int32_t>) : sizeof(ScanArgs<float>);
        std::vector<unsigned char> sa(ssz * n_sol);
        for (int k = 0; k < n_sol; ++k) {
            ds[k] = make_devstate(b->sols[k], b->d_keys + static_cast<size_t>(k) * TGA_N_VARIANTS);
            if (I->dtype == TGA_I32) { auto a = scan_args<int32_t>(b->sols[k]); std::memcpy(&sa[ssz * k], &a, ssz); }
            else { auto a = scan_args<float>(b->sols[k]); std::memcpy(&sa[ssz * k], &a, ssz); }
        }
        if (cudaMalloc(&b->d_states, sizeof(DevState) * n_sol) != cudaSuccess ||
            cudaMalloc(&b->d_scans, sa.size()) != cudaSuccess ||
            cudaMemcpy(b->d_states, ds.data(), sizeof(DevState) * n_sol, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(b->d_scans, sa.data(), sa.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            return bail(fail(TGA_ERR_OOM, "batch step state"));
    }
    if (cudaMemcpy(b->d_views, views.data(), views.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(b->d_maps, maps.data(), sizeof(CUtensorMap) * n_sol, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(b->d_work, work.data(), sizeof(uint32_t) * work.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(fail(TGA_ERR_CUDA, "batch upload"));
    {   // fast path: every solution has its records and fast map; items (k << 20 | I << 10 | J)
        bool ok = true;
        std::vector<FastSol> fs(n_sol);
        std::vector<CUtensorMap> fm(n_sol);
        std::vector<uint32_t> fw;
        for (int k = 0; k < n_sol && ok; ++k) {
            tga_solution *s = b->sols[k];
            ok = s->fast && s->rec && (!I->tw || s->rectw) && s->fastU == 16 && s->pitch / 16 < 1024 &&
                 I->opt.score_mode == TGA_SCORE_FEASIBLE;   // the batch tile body is feasible-only
            if (!ok) break;
            fs[k] = FastSol{s->rec, s->rectw, b->d_keys + static_cast<size_t>(k) * TGA_N_VARIANTS,
                            static_cast<uint32_t>(s->pitch), 0};
            fm[k] = s->fmap;
            // a solution's tiles by column band, then row band: a CTA's run of items reuses the
            // column records a stage already holds (fast_body) -- cfg5 traffic 3.3x -> ~1.4x the Dp
            std::vector<uint32_t> plan = fast_plan(s);
            std::stable_sort(plan.begin(), plan.end(), [](uint32_t x, uint32_t y) {
                return (x & 0xFFFFu) != (y & 0xFFFFu) ? (x & 0xFFFFu) < (y & 0xFFFFu) : (x >> 16) < (y >> 16);
            });
            for (uint32_t ij : plan)
                fw.push_back((static_cast<uint32_t>(k) << 20) | ((ij >> 16) << 10) | (ij & 0xFFFFu));
        }
        if (ok && !fw.empty()) {
            if (cudaMalloc(&b->d_fsols, sizeof(FastSol) * n_sol) != cudaSuccess ||
                cudaMalloc(&b->d_fmaps, sizeof(CUtensorMap) * n_sol) != cudaSuccess ||
                cudaMalloc(&b->d_fwork, sizeof(uint32_t) * fw.size()) != cudaSuccess ||
                cudaMemcpy(b->d_fsols, fs.data(), sizeof(FastSol) * n_sol, cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(b->d_fmaps, fm.data(), sizeof(CUtensorMap) * n_sol, cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(b->d_fwork, fw.data(), sizeof(uint32_t) * fw.size(), cudaMemcpyHostToDevice) != cudaSuccess)
                return bail(fail(TGA_ERR_OOM, "batch fast path"));
            b->n_fwork = static_cast<int>(fw.size());
            b->fast = true;
        }
    }
    *out = b;
    return TGA_OK;
}

extern "C" int32_t tga_batch_destroy(tga_batch *b) {
    free_batch(b);
    return TGA_OK;
}

extern "C" int32_t tga_batch_size(const tga_batch *b, int32_t *n_sol) {
    if (!b || !n_sol) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    *n_sol = static_cast<int32_t>(b->sols.size());
    return TGA_OK;
}

extern "C" int32_t tga_batch_solution(tga_batch *b, int32_t i, tga_solution **out) {
    if (!b || !out || i < 0 || i >= static_cast<int>(b->sols.size())) return fail(TGA_ERR_INVALID_ARGUMENT, "index");
    *out = b->sols[i];
    return TGA_OK;
}

extern "C" int32_t tga_batch_eval(tga_batch *b, uint32_t mask, void *stream) {
    if (!b) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL batch");
    const tga_instance *I = b->inst;
    mask &= TGA_OP_ALL;
    if ((mask & TGA_OP_2OPT) && I->tw) return fail(TGA_ERR_UNSUPPORTED, "2-opt with time windows (P:148)");
    if ((mask & TGA_OP_2OPT) && I->dPickup) return fail(TGA_ERR_UNSUPPORTED, "2-opt with pickups (P:510)");
    if (set_device(I) != TGA_OK) return TGA_ERR_CUDA;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : b->stream;
    if (st != b->stream) TGA_CUDA(order_after(st, b->stream));
    const int n = static_cast<int>(b->sols.size());
    TGA_CUDA(launch_fill_u64(b->d_keys, static_cast<size_t>(TGA_N_VARIANTS) * n, ~0ull, st));
    ScoreParams sp{I->Q, I->opt.score_mode, I->opt.w_load, I->opt.w_tw};
    const int grid = std::max(1, std::min(b->n_work, b->sm_count * 4));
    static const int force_warp = std::getenv("TGA_WARP_TW_BATCH") ? std::atoi(std::getenv("TGA_WARP_TW_BATCH")) : -1;
    const bool warp_tw = !I->dPickup && (force_warp >= 0 ? force_warp != 0 : b->sols[0]->N >= 16 * b->sols[0]->R);
    static const bool no_fast = std::getenv("TGA_BATCH_GENERIC") != nullptr;  // A/B override
    uint32_t rest = mask;
    if (b->fast && !no_fast && (mask & TGA_OP_INTER)) {
        const cudaError_t ef = launch_inter_fast_batch(16, I->tw, mask & TGA_OP_INTER, b->d_fsols,
                                                       b->d_fmaps, b->d_fwork, b->n_fwork, I->Q, sp,
                                                       b->sm_count * 4, st);
        if (ef != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("batch fast eval: ") + cudaGetErrorString(ef));
        rest &= ~TGA_OP_INTER;
    }
    cudaError_t e = I->dtype == TGA_I32
        ? launch_batch<int32_t>(rest, I->tw, static_cast<const SolView<int32_t> *>(b->d_views), b->d_maps, b->d_work,
                                b->n_work, n, b->max_qp, sp, b->d_keys, grid, st, warp_tw)
        : launch_batch<float>(rest, I->tw, static_cast<const SolView<float> *>(b->d_views), b->d_maps, b->d_work,
                              b->n_work, n, b->max_qp, sp, b->d_keys, grid, st, warp_tw);
    if (e != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("batch eval: ") + cudaGetErrorString(e));
    if (st != b->stream) TGA_CUDA(order_after(b->stream, st));
    b->eval_mask = mask;
    for (int k = 0; k < n; ++k) {
        b->eval_gen[k] = b->sols[k]->gen;
        b->sols[k]->drained = false;
    }
    return TGA_OK;
}

extern "C" int32_t tga_batch_keys(tga_batch *b, uint64_t *keys) {
    if (!b || !keys) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    const size_t bytes = sizeof(uint64_t) * TGA_N_VARIANTS * b->sols.size();
    TGA_CUDA(cudaMemcpyAsync(b->h_keys, b->d_keys, bytes, cudaMemcpyDeviceToHost, b->stream));
    TGA_CUDA(cudaStreamSynchronize(b->stream));
    for (size_t k = 0; k < b->sols.size(); ++k) {
        if (sync_host(b->sols[k]) != TGA_OK) return TGA_ERR_CUDA;
        for (int v = 0; v < TGA_N_VARIANTS; ++v)
            keys[k * TGA_N_VARIANTS + v] = key_to_canonical(b->sols[k], b->h_keys[k * TGA_N_VARIANTS + v]);
    }
    return TGA_OK;
}

extern "C" int32_t tga_batch_best_moves(tga_batch *b, uint32_t mask, tga_move *out, int32_t *status) {
    if (!b || !out) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    const int n = static_cast<int>(b->sols.size());
    TGA_CUDA(cudaMemcpyAsync(b->h_keys, b->d_keys, sizeof(uint64_t) * TGA_N_VARIANTS * n, cudaMemcpyDeviceToHost,
                             b->stream));
    TGA_CUDA(cudaStreamSynchronize(b->stream));
    mask &= b->eval_mask;
    for (int k = 0; k < n; ++k) {
        tga_solution *s = b->sols[k];
        s->drained = true;
        if (b->eval_gen[k] != s->gen) return fail(TGA_ERR_STALE, "batch evaluation is stale");
        const int32_t rc = decode_best(s, b->h_keys + static_cast<size_t>(k) * TGA_N_VARIANTS, mask, &out[k]);
        if (status) status[k] = rc;
    }
    return TGA_OK;
}

extern "C" int32_t tga_batch_apply_moves(tga_batch *b, const tga_move *moves, const int32_t *apply) {
    if (!b || !moves) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL argument");
    for (size_t k = 0; k < b->sols.size(); ++k) {
        if (apply && !apply[k]) continue;
        if (moves[k].variant < 0) continue;
        const int32_t rc = tga_apply_move(b->sols[k], &moves[k]);
        if (rc != TGA_OK) return rc;
    }
    return TGA_OK;
}

extern "C" int32_t tga_batch_set_stream(tga_batch *b, void *stream) {
    if (!b) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL batch");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : b->own_stream;
    if (st != b->stream) TGA_CUDA(order_after(st, b->stream));
    b->stream = st;
    for (auto *s : b->sols) s->stream = st;
    return TGA_OK;
}

extern "C" int32_t tga_batch_step_async(tga_batch *b, uint32_t mask) {
    if (!b) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL batch");
    int32_t rc = tga_batch_eval(b, mask, nullptr);
    if (rc != TGA_OK) return rc;
    const tga_instance *I = b->inst;
    const int n = static_cast<int>(b->sols.size());
    int max_r = 0;
    for (auto *s : b->sols) max_r = std::max(max_r, s->R);
    // blocks per solution so that the whole grid is co-resident (grid barrier)
    cudaError_t e = launch_pick_update(b->d_states, b->d_scans, n, I->tw, I->dtype == TGA_I32, b->eval_mask,
                                       b->eval_mask, max_r,
                                       b->sols[0]->N + 2 + b->sols[0]->slack,
                                       std::max(1, b->sm_count * 2 / n), b->stream);
    if (e != cudaSuccess) return fail(TGA_ERR_CUDA, std::string("batch device step: ") + cudaGetErrorString(e));
    for (auto *s : b->sols) {
        ++s->gen;
        s->host_stale = true;
        s->drained = false;
    }
    return TGA_OK;
}

extern "C" int32_t tga_batch_device_stats(tga_batch *b, uint64_t *counts, uint64_t *applied) {
    if (!b) return fail(TGA_ERR_INVALID_ARGUMENT, "NULL batch");
    TGA_CUDA(cudaStreamSynchronize(b->stream));
    uint64_t tot[TGA_N_VARIANTS] = {0}, app = 0;
    for (auto *s : b->sols) {
        uint64_t c[TGA_N_VARIANTS], a = 0;
        const int32_t rc = tga_solution_device_stats(s, c, &a);
        if (rc != TGA_OK) return rc;
        for (int v = 0; v < TGA_N_VARIANTS; ++v) tot[v] += c[v];
        app += a;
    }
    if (counts) std::memcpy(counts, tot, sizeof(tot));
    if (applied) *applied = app;
    return TGA_OK;
}

// ============================================================== ABI: misc
extern "C" const char *tga_last_error(void) { return g_err.c_str(); }
extern "C" const char *tga_version(void) { return "tga-b200 0.1 (sm_100a)"; }
extern "C" uint64_t tga_launch_count(void) { return tga::launch_count(); }
