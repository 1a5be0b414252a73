// tga_device.cuh -- device-side building blocks of the TGA hot path (sm_100a).
//
// Attribute records and the concatenation algebra of PAPER.md §4.3:
//   Eq. 2   D(s1 + s2)   = D(s1) + c_jk + D(s2)
//   Eq. 3ef L_M(s1 + s2) = L_M(s1) + L_M(s2)   (no pickups)
//   Eq. 4   time-warp record {T_D, T_E, T_L, T_V}, T_W == 0 reading
// and the packed (score, canonical index) key of the fused argmin
// (Eq. 16c; deterministic lowest-index tie-break, reading 5).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tga {

// PDL controls (see launch_pdl in tga_launch.h)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


// ------------------------------------------------------------------ records
// A time-window record of a subsequence: x = T_D (duration incl.
// waiting), y = T_E (earliest start), z = T_L (latest start), w = T_V (warp).
using TwRec = float4;

// Eq. 4b-4h with T_W(s1) == 0 (reading 1).  `t` is t_jk, the travel
// time from the last node of a to the first node of b.  In TW-I mode every
// operand is an integer-valued float below 2^24, so the result is exact.
__host__ __device__ __forceinline__ TwRec tw_cat(const TwRec a, const TwRec b, const float t) {
    const float dt = a.x + t - a.w;                  // Eq. 4b  Delta_t
    const float dw = fmaxf(b.y - dt - a.z, 0.0f);    // Eq. 4c  Delta_w
    const float dv = fmaxf(a.y + dt - b.z, 0.0f);    // Eq. 4d  Delta_v
    TwRec r;
    r.x = a.x + t + dw + b.x;                        // Eq. 4e  T_D
    r.y = fmaxf(a.y, b.y - dt) - dw;                 // Eq. 4f  T_E
    r.z = fminf(a.z, b.z - dt) + dv;                 // Eq. 4g  T_L
    r.w = a.w + dv + b.w;                            // Eq. 4h  T_V
    return r;
}

// Eq. 4a: a single node k: T_D = s_k, T_E = e_k, T_L = l_k, T_V = 0.
__host__ __device__ __forceinline__ TwRec tw_single(float e, float l, float s) {
    return make_float4(s, e, l, 0.0f);
}

// ------------------------------------------------------------------ pickup and delivery loads
// Eq. 3a-d: a subsequence's incoming load L_I (its deliveries), outgoing
// load L_O (its pickups) and largest load L_M; x = L_I, y = L_O, z = L_M, w unused.
using LoadRec = int4;
__host__ __device__ __forceinline__ LoadRec ld_single(int32_t d, int32_t p) {   // Eq. 3a
    return make_int4(d, p, d > p ? d : p, 0);
}
__host__ __device__ __forceinline__ LoadRec ld_cat(const LoadRec a, const LoadRec b) {   // Eq. 3b-d
    const int32_t m1 = a.z + b.x, m2 = a.y + b.z;
    return make_int4(a.x + b.x, a.y + b.y, m1 > m2 ? m1 : m2, 0);
}

// ------------------------------------------------------------------ keys
// Order-preserving 32-bit images of a score.
__device__ __forceinline__ uint32_t ord_score(int32_t s) { return static_cast<uint32_t>(s) ^ 0x80000000u; }
__device__ __forceinline__ uint32_t ord_score(float s) {
    const uint32_t u = __float_as_uint(s);
    return u ^ ((u & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u);
}
constexpr uint64_t kNoKey = ~0ull;
// variant count (include/tga.h TGA_N_VARIANTS): 23 standard + 4 reversed-segment variants;
// a solution's accumulator words: [0, kNV) candidate counts, [kAccApplied] applied moves
constexpr int kNV = 27;
constexpr int kAccApplied = 27;
constexpr uint32_t kRevMask = 0xFu << 23;   // the reversed-segment inter variants

__device__ __forceinline__ uint64_t pack_key(uint32_t ord, uint32_t idx) {
    return (static_cast<uint64_t>(ord) << 32) | idx;
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// 64-bit warp minimum with two REDUX.MIN (high words, then low words among the lanes holding the high minimum)
__device__ __forceinline__ uint64_t warp_min64(uint64_t k) {
    const uint32_t hi = static_cast<uint32_t>(k >> 32), lo = static_cast<uint32_t>(k);
    const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xFFFFFFFFu);
    return (static_cast<uint64_t>(mh) << 32) | ml;
}

// ------------------------------------------------------------------ scoring
// Score of a candidate (Eq. 16a; modes = DESIGN.md reading 4).
//   feasible-only : dD if every new route has L <= Q and T_V == 0, else no key
//   penalised     : dD + wQ * dL_V + wT * dT_V
struct ScoreParams {
    int32_t capacity;
    int32_t mode;      // 0 feasible-only, 1 penalised
    int32_t wQ, wT;
};

template <class DT> struct ScoreT;
template <> struct ScoreT<int32_t> {
    __device__ __forceinline__ static int32_t tv(float x) { return __float2int_rn(x); }
};
template <> struct ScoreT<float> {
    __device__ __forceinline__ static float tv(float x) { return x; }
};

// dLV / dTV are differences of new-minus-old excess (old values per route).
template <class DT, bool TW>
__device__ __forceinline__ uint64_t score_key(const ScoreParams &sp, bool valid, DT dD,
                                              int32_t la, int32_t lb, int32_t la0, int32_t lb0,
                                              float tva, float tvb, float tva0, float tvb0,
                                              uint32_t idx) {
    const int32_t Q = sp.capacity;
    if (sp.mode == 0) {
        bool feas = valid && (la <= Q) && (lb <= Q);
        if (TW) feas = feas && (tva == 0.0f) && (tvb == 0.0f);
        return feas ? pack_key(ord_score(dD), idx) : kNoKey;
    }
    const int32_t dlv = max(la - Q, 0) + max(lb - Q, 0) - max(la0 - Q, 0) - max(lb0 - Q, 0);
    DT s = dD + static_cast<DT>(sp.wQ * dlv);
    if (TW) s += static_cast<DT>(sp.wT) * ScoreT<DT>::tv((tva + tvb) - (tva0 + tvb0));
    return valid ? pack_key(ord_score(s), idx) : kNoKey;
}

// ------------------------------------------------------------------ test-only candidate dump
// DUMP instantiations of the evaluation kernels (tga_debug_eval_dump) also store the
// packed key of EVERY candidate they evaluate -- kNoKey when it is infeasible or
// structurally invalid -- at dump[variant * stride + physical flat index]; the host
// pre-fills 0 (= not evaluated).  Production instantiations never touch it.
__device__ __forceinline__ void dump_put(unsigned long long *dump, uint32_t stride, int var, uint32_t idx, uint64_t k) {
    dump[static_cast<size_t>(var) * stride + idx] = k;
}

// ------------------------------------------------------------------ per-slot record (CVRP fast path)
// Everything the fused inter-route kernel needs about one slot x in one
// 80-byte record, so a tile row is one bulk copy and a lane's column is five
// 16-byte loads.  Validity is folded into the load terms: an invalid role
// carries kPoison in a load that is compared against the capacity, so the
// candidate fails the capacity test without a branch (feasible-only mode).
constexpr int32_t kPoison = 1 << 28;
struct __align__(16) SlotRec {
    int32_t r;       // route id; -1 for an end depot, a spare slot or padding (not a canonical slot)
    int32_t fL;      // prefix load of [0..x]               (2-opt* head),  +P if r < 0
    int32_t bL1;     // suffix load of [x+1..L+1]            (2-opt* tail),  +P if r < 0
    int32_t ne;      // -e(x), e(x) = c(x, x+1)                               [- w_Q ex, penalised]
    int32_t W;       // route load (insertion target),       +P if r < 0
    int32_t so[3];   // relocate-out load s_N of x..x+N-1,   +P if the segment is invalid or (feasible-only
                     //                                         records) W - s_N > Q
    int32_t rem[3];  // relocate-out distance c(x-1, x+N) - e(x-1) - e(x+N-1)  (Eq. 2)  [- w_Q ex]
    int32_t sA[3];   // swap: W - s_N,                       +P if the segment is invalid
    int32_t sS[3];   // swap: s_N
    int32_t sE[3];   // swap: -e(x-1) - e(x+N-1)                              [- w_Q ex]
};
// Penalised records (score = dD + w_Q dL_V, Eq. 16a with reading 4): every candidate
// changes exactly two routes and its distance formula uses exactly one of {ne, rem[N],
// sE[N]} of each, so the old excess ex = max(W - Q, 0) of the slot's route enters those
// three fields as -w_Q ex; a candidate then adds w_Q (max(L_a' - Q, 0) + max(L_b' - Q, 0)).
static_assert(sizeof(SlotRec) == 80, "SlotRec layout: five 16-byte shared loads per column");

// Time-window part of the fast-path record (VRPTW "TW-I", feasible-only mode).
// With T_V = 0 on both sides, T_V(s1 + s2) == 0  <=>  T_E(s1)+T_D(s1)+t <= T_L(s2)
// (Eq. 4b/4d/4h with T_W = 0), and the earliest completion of s1 + seg is
// max(T_E(s1)+T_D(s1)+t, T_E(seg)) + T_D(seg) (Eq. 4e/4f): every concatenation
// of a candidate becomes one add, one max and one compare.  Infeasible parts
// carry +-kTwBig.  All values are integer-valued floats (< 2^24: exact).
constexpr float kTwBig = 1.0e30f;
struct __align__(16) SlotTW {
    float EF;        // earliest completion of the prefix [0..x] (T_E + T_D), +BIG if T_V > 0
    float EFm;       // the same for [0..x-1]
    float LBN[3];    // latest start of the suffix [x+N..L+1] (T_L), -BIG if T_V > 0 or absent
    float sTE[3];    // segment x..x+N-1: earliest start
    float sTL[3];    //                   latest start, -BIG if the segment warps or is invalid
    float sTD[3];    //                   duration
    float pad[2];
};
static_assert(sizeof(SlotTW) == 64, "SlotTW layout");

// ------------------------------------------------------------------ launch-side views
// Device view of one solution (all arrays indexed by physical slot unless noted).
template <class DT>
struct SolView {
    // layout
    const int32_t *node, *route, *pos, *rlen, *canon;
    // loads: prefix [0..x] and suffix [x..L+1]
    const int32_t *fwdL, *bwdL;
    // distances: edge x -> x+1, and bridge_N[x] = c(x-1, x+N) (N = 1..3)
    const DT *enext;
    const DT *bridge1, *bridge2, *bridge3;
    // time-window records: prefix, suffix, segments of 2 and 3 starting at x
    const TwRec *fwdT, *bwdT, *seg2T, *seg3T;
    const TwRec *node_tw;     // per node: (s, e, l, 0)
    // VRPSPDTW (null without pickups): node demands d_i / p_i, prefix / suffix Eq. 3 load records
    const int32_t *dem, *pick;
    const LoadRec *fwdP, *bwdP;
    // per route
    const int32_t *rW;        // load (the largest load carried, L_M, with pickups)
    const float *rTV;         // time warp
    // position-ordered distance matrix Dp[a][b] = c(node(a), node(b))
    const DT *Dp;
    int32_t pitch;            // elements per Dp row
    int32_t Qp;               // physical slots (rows of Dp)
    uint32_t Qc;              // flat-index multiplier (= pitch): key index = u * Qc + v over PHYSICAL slots
    const uint32_t *tiles;    // generic inter-route tile plan (batch kernels)
};

// ------------------------------------------------------------------ intra-route CVRP (warp per u slot)
__device__ __forceinline__ uint32_t intra_k32(bool ok, int32_t dD, int lane) {
    // dD is bounded by 8 * max c < 2^25 (host-checked: max c < 2^21)
    return ok ? ((static_cast<uint32_t>(dD + (1 << 25)) << 5) | static_cast<uint32_t>(lane)) : 0xFFFFFFFFu;
}
// wred: this warp's private row of per-variant minima in shared memory (plain
// read-min-write by lane 0: a 64-bit shared atomicMin compiles to a CAS spin loop)
__device__ __forceinline__ void warp_keep(unsigned long long *wred, int var, uint32_t k32, uint32_t idx_base, int lane) {
    const uint32_t m = __reduce_min_sync(0xffffffffu, k32);
    if (lane == 0 && m != 0xFFFFFFFFu) {
        const int32_t s = static_cast<int32_t>(m >> 5) - (1 << 25);
        const unsigned long long k = pack_key(ord_score(s), idx_base + (m & 31u));
        if (k < wred[var]) wred[var] = k;
    }
}

// One warp evaluates every intra-route CVRP variant of u slot x (lane <-> v);
// the per-variant warp minima are MIN-combined into red[23], the calling warp's
// private row of shared memory.
template <bool DUMP = false>
__device__ __forceinline__ void intra_cvrp_warp(const SolView<int32_t> &S, const ScoreParams &sp, uint32_t vmask,
                                                int x, unsigned long long *red, unsigned long long *pslot = nullptr,
                                                unsigned long long *dump = nullptr) {
    const int lane = threadIdx.x & 31;
    auto stamp = [&](int k) {
        if (pslot && lane == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            pslot[k] = t;
        }
    };
    stamp(0);
    // two dependent rounds of global loads: (1) everything indexed by x alone,
    // (2) the route load and the Dp / edge values of the lanes' v (needs the
    // route base) -- the loads of each round are issued together
    const int32_t cx = S.canon[x], p = S.pos[x], L = S.rlen[x], r = S.route[x];
    const int32_t em = S.enext[x - 1];
    int32_t eo[3], br[3];
#pragma unroll
    for (int N = 1; N <= 3; ++N) eo[N - 1] = S.enext[x + N - 1];  // past the route end: only in masked candidates
    br[0] = S.bridge1[x]; br[1] = S.bridge2[x]; br[2] = S.bridge3[x];
    if (!(cx >= 0 && p >= 1)) return;   // warp-uniform
    stamp(1);
    const int base = x - p;
    int32_t rem[3];
#pragma unroll
    for (int N = 1; N <= 3; ++N) rem[N - 1] = br[N - 1] - em - eo[N - 1];
    const int32_t Wr = S.rW[max(r, 0)];
    for (int qb = 0; qb <= L; qb += 32) {
        const int q = qb + lane;
        const bool in = q <= L;
        const int v = base + min(q, L);
        const int vm1 = max(v - 1, base);          // masked lanes (q = 0) must still read a valid row
        const uint32_t ib = static_cast<uint32_t>(x) * S.Qc + static_cast<uint32_t>(base + qb);  // physical
        const int32_t ev = S.enext[v], evm = (q >= 1 && in) ? S.enext[v - 1] : 0;
        int32_t ev2[3];
#pragma unroll
        for (int b = 1; b <= 3; ++b) ev2[b - 1] = S.enext[min(v + b - 1, base + L + 1)];
        const bool ok_route = sp.mode == 1 || Wr <= sp.capacity;
        // every Dp value any variant reads, loaded up front and unconditionally so
        // that they are one round trip (inside the variant branches they were one
        // round trip per variant): row x-1 at v; rows x..x+3 at v..v+3; row x at vm1
        int32_t d[5][4];
        const int32_t *dr = S.Dp + static_cast<size_t>(x - 1) * S.pitch + v;
        const int32_t dm1 = __ldg(dr), dxm = __ldg(S.Dp + static_cast<size_t>(x) * S.pitch + vm1);
#pragma unroll
        for (int i = 1; i < 5; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) d[i][j] = (i == 4 && j == 3) ? 0 : __ldg(dr + i * S.pitch + j);
        auto D = [&](int i, int j) -> int32_t { return i < 0 ? dm1 : d[i + 1][j]; };  // Dp(x + i, v + j)
        uint32_t k[23];
#pragma unroll
        for (int i = 0; i < 23; ++i) k[i] = 0xFFFFFFFFu;
        if (vmask & 1u)   // 2-opt: reverse u..v
            k[0] = intra_k32(ok_route && in && q > p, D(-1, 0) + D(0, 1) - em - ev, lane);
#pragma unroll
        for (int N = 1; N <= 3; ++N) {  // intra relocate / or-opt
            if (!(vmask & (1u << (10 + N)))) continue;
            const bool ok = ok_route && in && p + N - 1 <= L && (q < p - 1 || q > p + N - 1);
            // c is symmetric (host-checked): every Dp read is row x.. with lanes along columns
            k[10 + N] = intra_k32(ok, rem[N - 1] + D(0, 0) + D(N - 1, 1) - ev, lane);
        }
#pragma unroll
        for (int a = 1; a <= 3; ++a) {   // intra swap (N1 = a at u, N2 = b at v), u + N1 <= v
#pragma unroll
            for (int b = 1; b <= 3; ++b) {
                const int var = 14 + 3 * (a - 1) + (b - 1);
                if (!(vmask & (1u << var))) continue;
                const bool ok = ok_route && in && q >= p + a && q + b - 1 <= L;
                const int32_t adj = D(-1, 0) + D(0, b - 1) + D(a - 1, b) - em - evm - ev2[b - 1];
                const int32_t gap = D(-1, 0) + D(a, b - 1) + dxm + D(a - 1, b) - em - eo[a - 1] - evm - ev2[b - 1];
                k[var] = intra_k32(ok, q == p + a ? adj : gap, lane);
            }
        }
        if constexpr (DUMP) {
            const uint32_t stride = static_cast<uint32_t>(S.pitch) * static_cast<uint32_t>(S.pitch);
#pragma unroll
            for (int i = 0; i < 23; ++i) {
                if (!((i == 0 || i >= 11) && (vmask & (1u << i))) || !in) continue;
                const uint64_t kk = k[i] == 0xFFFFFFFFu ? kNoKey
                                    : pack_key(ord_score(static_cast<int32_t>(k[i] >> 5) - (1 << 25)), ib + lane);
                dump_put(dump, stride, i, ib + lane, kk);
            }
        }
        // phase 2: one REDUX.MIN per variant, all issued before lane 0 merges them
        // into the warp's private row (independent read-min-writes)
        if (qb == 0) stamp(2);
        uint32_t m[23];
#pragma unroll
        for (int i = 0; i < 23; ++i)
            m[i] = ((i == 0 || i >= 11) && (vmask & (1u << i))) ? __reduce_min_sync(0xffffffffu, k[i]) : 0xFFFFFFFFu;
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < 23; ++i) {
                if (!(i == 0 || i >= 11) || m[i] == 0xFFFFFFFFu) continue;
                const int32_t sc = static_cast<int32_t>(m[i] >> 5) - (1 << 25);
                const unsigned long long key = pack_key(ord_score(sc), ib + (m[i] & 31u));
                if (key < red[i]) red[i] = key;
            }
        }
    }
    stamp(3);
}

}  // namespace tga
