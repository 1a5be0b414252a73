// tga_kernels.cu -- hand-written sm_100a kernels of the TGA hot path.
//
//   k_dp_rows / k_dp_cols   position-ordered distance matrix Dp[a][b] = c(node a, node b)
//                           (build, and the row/column refresh of the update step)
//   k_scan                  attribute rebuild: per-route segmented prefix/suffix scans with
//                           warp shuffles of the Eq. 2 / 3e-f / 4 records
//   k_inter<DT,TW,MASK>     inter-route candidates (2-opt*, relocate/or-opt, swap/cross),
//                           TMA-staged Dp tiles, branch-free feasibility, fused argmin
//                           (P:241 steps 1-4; Eq. 16)
//   k_intra<DT,TW>          intra-route candidates (2-opt, intra relocate, intra swap) with
//                           incremental middle-segment composition
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

#include "tga_device.cuh"
#include "tga_launch.h"
#include "tga_pick.cuh"

namespace tga {

// ============================================================== Dp build / refresh
__device__ __forceinline__ int bits(int32_t v) { return v; }
__device__ __forceinline__ int bits(float v) { return __float_as_int(v); }

template <class DT>
__global__ void __launch_bounds__(256) k_dp_rows(DT *__restrict__ Dp, int pitch,
                                                 const int32_t *__restrict__ node,
                                                 const DT *__restrict__ C, int n, int lo, int hi) {
    const int a = lo + blockIdx.y;
    if (a >= hi) return;
    const DT *crow = C + static_cast<size_t>(node[a]) * n;
    DT *drow = Dp + static_cast<size_t>(a) * pitch;
    for (int b = 4 * (blockIdx.x * blockDim.x + threadIdx.x); b < pitch; b += 4 * gridDim.x * blockDim.x) {
        const int4 nd = *reinterpret_cast<const int4 *>(node + b);
        const DT v0 = __ldg(crow + nd.x), v1 = __ldg(crow + nd.y), v2 = __ldg(crow + nd.z), v3 = __ldg(crow + nd.w);
        *reinterpret_cast<int4 *>(drow + b) = make_int4(bits(v0), bits(v1), bits(v2), bits(v3));
    }
}

// columns b in [lo, hi) of every row (the transpose half of a refresh)
template <class DT>
__global__ void __launch_bounds__(256) k_dp_cols(DT *__restrict__ Dp, int pitch,
                                                 const int32_t *__restrict__ node,
                                                 const DT *__restrict__ C, int n, int rows, int lo, int hi) {
    const int b = lo + blockIdx.x * 32 + threadIdx.x;
    const int a = blockIdx.y * 8 + threadIdx.y;
    if (b >= hi || a >= rows) return;
    Dp[static_cast<size_t>(a) * pitch + b] = __ldg(C + static_cast<size_t>(node[a]) * n + node[b]);
}

// ============================================================== attribute rebuild scan
// One warp per route; chunks of 32 positions with carries.  Positions
// k = 0..L+1 of route r live at physical slots base..base+L+1.
// NodeF(x) / CanonF(x): node id / canonical-validity of slot x of this route
// (global arrays for a plain rebuild; the decoded new route in the device step,
// whose slot arrays are rewritten concurrently).  base, L, cap: the route's first
// physical slot, customer count and slot capacity.
// NodeF(x) / CanonF(x): node id / canonical-validity of slot x of this route
// (global arrays for a plain rebuild; the decoded new route in the device step,
// whose slot arrays are rewritten concurrently).  base, L, cap: the route's first
// physical slot, customer count and slot capacity.  The rebuild is three passes:
// forward (prefix records), backward (suffix records), per-slot records; a warp
// runs them one after the other (scan_route_g), a block can run the first two in
// two warps at once and the third over all its threads (scan_route_block).
template <class DT, bool TW>
__device__ __forceinline__ void scan_spare(const ScanArgs<DT> &A, const int k0, const int kstep, const int base,
                                           const int L, const int cap) {
    const int len = L + 2;
    if constexpr (std::is_same<DT, int32_t>::value) {
        // spare (hole) slots of the route carry poisoned fast-path records
        for (int k = len + k0; k < cap; k += kstep) {
            if (A.rec) {
                SlotRec q{};
                q.r = -1; q.fL = q.bL1 = q.W = kPoison;
                for (int j = 0; j < 3; ++j) { q.so[j] = kPoison; q.sA[j] = kPoison; }
                A.rec[base + k] = q;
            }
            if (A.nsc) A.nsc[base + k] = -1;   // route plane: not a canonical slot
            if (TW && A.rectw) {
                SlotTW w{};
                w.EF = w.EFm = kTwBig;
                for (int j = 0; j < 3; ++j) { w.LBN[j] = -kTwBig; w.sTL[j] = -kTwBig; }
                A.rectw[base + k] = w;
            }
        }
    }

}

template <class DT, bool TW, class NodeF>
__device__ __forceinline__ int scan_fwd_pass(const ScanArgs<DT> &A, const int r, const int lane, const int base,
                                             const int L, NodeF nodeAt, int32_t *sfL = nullptr, DT *sen = nullptr,
                                             TwRec *sfT = nullptr) {
    const int len = L + 2;
    const int n = A.n_nodes;
    // ---------------- forward pass: prefix loads, prefix distance, prefix TW records
    int carryL = 0;
    LoadRec carryP = make_int4(0, 0, 0, 0);   // VRPSPDTW prefix record of the chunks so far
    DT carryD = DT(0);
    TwRec carryT = make_float4(0.f, 0.f, 0.f, 0.f);
    DT carryE = DT(0);  // edge into the first position of the chunk
    for (int c0 = 0; c0 < len; c0 += 32) {
        const int k = c0 + lane;
        const bool in = k < len;
        const int x = base + k;
        const int nd = in ? nodeAt(x) : 0;
        const bool has_next = in && (k + 1 < len);
        const int nn = has_next ? nodeAt(x + 1) : 0;
        const DT e = has_next ? A.C[static_cast<size_t>(nd) * n + nn] : DT(0);
        // loads (Eq. 3e-f): inclusive prefix sum
        int sL = in ? A.demand[nd] : 0;
        DT sD = e;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int oL = __shfl_up_sync(0xffffffffu, sL, off);
            const DT oD = __shfl_up_sync(0xffffffffu, sD, off);
            if (lane >= off) { sL += oL; sD += oD; }
        }
        const int fL = carryL + sL;
        const DT fD = carryD + sD - e;  // exclusive: distance of [0..k] (Eq. 2)
        TwRec fT = make_float4(0.f, 0.f, 0.f, 0.f);
        if (TW) {
            const TwRec nt = A.node_tw[nd];
            TwRec rec = nt;
            // link into this position = edge (k-1 -> k)
            const DT ein_lane = __shfl_up_sync(0xffffffffu, e, 1);
            float inl = (lane == 0) ? static_cast<float>(carryE) : static_cast<float>(ein_lane);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                TwRec o;
                o.x = __shfl_up_sync(0xffffffffu, rec.x, off);
                o.y = __shfl_up_sync(0xffffffffu, rec.y, off);
                o.z = __shfl_up_sync(0xffffffffu, rec.z, off);
                o.w = __shfl_up_sync(0xffffffffu, rec.w, off);
                const float oin = __shfl_up_sync(0xffffffffu, inl, off);
                if (lane >= off) { rec = tw_cat(o, rec, inl); inl = oin; }
            }
            fT = (c0 > 0) ? tw_cat(carryT, rec, inl) : rec;
        }
        if (A.pickup) {   // VRPSPDTW: inclusive prefix scan of the Eq. 3a-d load records (warp-uniform branch)
            LoadRec pr = in ? ld_single(A.demand[nd], A.pickup[nd]) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                LoadRec o;
                o.x = __shfl_up_sync(0xffffffffu, pr.x, off);
                o.y = __shfl_up_sync(0xffffffffu, pr.y, off);
                o.z = __shfl_up_sync(0xffffffffu, pr.z, off);
                o.w = 0;
                if (lane >= off) pr = ld_cat(o, pr);
            }
            if (c0 > 0) pr = ld_cat(carryP, pr);
            if (in) A.fwdP[x] = pr;
            const int lst = min(31, len - 1 - c0);
            carryP.x = __shfl_sync(0xffffffffu, pr.x, lst);
            carryP.y = __shfl_sync(0xffffffffu, pr.y, lst);
            carryP.z = __shfl_sync(0xffffffffu, pr.z, lst);
        }
        if (in) {
            A.fwdL[x] = fL;
            A.fwdD[x] = fD;
            A.enext[x] = e;
            if (TW) A.fwdT[x] = fT;
            if (sfL) {   // the block rebuild's shared mirror (position k of the route)
                sfL[k] = fL;
                sen[k] = e;
                if (TW) sfT[k] = fT;
            }
        }
        const int last = min(31, len - 1 - c0);
        carryL = __shfl_sync(0xffffffffu, fL, last);
        carryD = __shfl_sync(0xffffffffu, fD + e, last);
        carryE = __shfl_sync(0xffffffffu, e, last);
        if (TW) {
            carryT.x = __shfl_sync(0xffffffffu, fT.x, last);
            carryT.y = __shfl_sync(0xffffffffu, fT.y, last);
            carryT.z = __shfl_sync(0xffffffffu, fT.z, last);
            carryT.w = __shfl_sync(0xffffffffu, fT.w, last);
        }
    }
    // the route's load: the delivery sum (Eq. 3e-f), or with pickups the largest load
    // carried, L_M of the whole route (Eq. 3a-d) -- what the capacity constraint bounds
    const int Wr = A.pickup ? carryP.z : carryL;
    if (lane == 0) {
        A.rW[r] = Wr;
        if (TW) A.rTV[r] = carryT.w;
    }

    return Wr;
}

template <class DT, bool TW, class NodeF>
__device__ __forceinline__ void scan_bwd_pass(const ScanArgs<DT> &A, const int r, const int lane, const int base,
                                              const int L, NodeF nodeAt, const bool e_from_C,
                                              int32_t *sbL = nullptr, TwRec *sbT = nullptr) {
    const int len = L + 2;
    const int n = A.n_nodes;
    // ---------------- backward pass: suffix loads, suffix distance, suffix TW records
    int bcarryL = 0;
    LoadRec bcarryP = make_int4(0, 0, 0, 0);
    DT bcarryD = DT(0);
    TwRec bcarryT = make_float4(0.f, 0.f, 0.f, 0.f);
    const int nchunks = (len + 31) / 32;
    for (int ci = nchunks - 1; ci >= 0; --ci) {
        const int c0 = ci * 32;
        const int nvalid = min(32, len - c0);
        const int k = c0 + lane;
        const bool in = lane < nvalid;
        const int x = base + k;
        const int nd = in ? nodeAt(x) : 0;
        // the edge out of position k: written by the forward pass (same warp), or
        // gathered again when the two passes run in different warps
        const DT e = !in ? DT(0) : (e_from_C ? ((k + 1 < len) ? A.C[static_cast<size_t>(nd) * n + nodeAt(x + 1)] : DT(0))
                                              : A.enext[x]);
        int sL = in ? A.demand[nd] : 0;
        DT sD = e;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int oL = __shfl_down_sync(0xffffffffu, sL, off);
            const DT oD = __shfl_down_sync(0xffffffffu, sD, off);
            if (lane + off < nvalid) { sL += oL; sD += oD; }
        }
        const int bL = bcarryL + sL;
        const DT bD = bcarryD + sD;
        TwRec bT = make_float4(0.f, 0.f, 0.f, 0.f);
        if (TW) {
            TwRec rec = A.node_tw[nd];
            float outl = static_cast<float>(e);  // edge out of the record's last position
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                TwRec o;
                o.x = __shfl_down_sync(0xffffffffu, rec.x, off);
                o.y = __shfl_down_sync(0xffffffffu, rec.y, off);
                o.z = __shfl_down_sync(0xffffffffu, rec.z, off);
                o.w = __shfl_down_sync(0xffffffffu, rec.w, off);
                const float oout = __shfl_down_sync(0xffffffffu, outl, off);
                if (lane + off < nvalid) { rec = tw_cat(rec, o, outl); outl = oout; }
            }
            bT = (ci < nchunks - 1) ? tw_cat(rec, bcarryT, outl) : rec;
        }
        if (A.pickup) {   // VRPSPDTW: inclusive suffix scan of the Eq. 3a-d load records
            LoadRec pr = in ? ld_single(A.demand[nd], A.pickup[nd]) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                LoadRec o;
                o.x = __shfl_down_sync(0xffffffffu, pr.x, off);
                o.y = __shfl_down_sync(0xffffffffu, pr.y, off);
                o.z = __shfl_down_sync(0xffffffffu, pr.z, off);
                o.w = 0;
                if (lane + off < nvalid) pr = ld_cat(pr, o);
            }
            if (ci < nchunks - 1) pr = ld_cat(pr, bcarryP);
            if (in) A.bwdP[x] = pr;
            bcarryP.x = __shfl_sync(0xffffffffu, pr.x, 0);
            bcarryP.y = __shfl_sync(0xffffffffu, pr.y, 0);
            bcarryP.z = __shfl_sync(0xffffffffu, pr.z, 0);
        }
        if (in) {
            A.bwdL[x] = bL;
            A.bwdD[x] = bD;
            if (TW) A.bwdT[x] = bT;
            if (sbL) {
                sbL[k] = bL;
                if (TW) sbT[k] = bT;
            }
        }
        bcarryL = __shfl_sync(0xffffffffu, bL, 0);
        bcarryD = __shfl_sync(0xffffffffu, bD, 0);
        if (TW) {
            bcarryT.x = __shfl_sync(0xffffffffu, bT.x, 0);
            bcarryT.y = __shfl_sync(0xffffffffu, bT.y, 0);
            bcarryT.z = __shfl_sync(0xffffffffu, bT.z, 0);
            bcarryT.w = __shfl_sync(0xffffffffu, bT.w, 0);
        }
    }
    if (lane == 0) A.rD[r] = bcarryD;
}

// bridge_N[x] = c(x-1, x+N): the edge that closes the gap left by removing the segment
// x..x+N-1 (relocate / or-opt removal, Eq. 2); k = position of slot x in its route
template <class DT, class NodeF>
__device__ __forceinline__ void scan_bridges(const ScanArgs<DT> &A, const int k, const int x, const int len,
                                             NodeF nodeAt, DT &b1, DT &b2, DT &b3) {
    const int n = A.n_nodes;
    const int np = (k >= 1) ? nodeAt(x - 1) : 0;
    b1 = b2 = b3 = DT(0);
    if (k >= 1 && k + 1 <= len - 1) b1 = A.C[static_cast<size_t>(np) * n + nodeAt(x + 1)];
    if (k >= 1 && k + 2 <= len - 1) b2 = A.C[static_cast<size_t>(np) * n + nodeAt(x + 2)];
    if (k >= 1 && k + 3 <= len - 1) b3 = A.C[static_cast<size_t>(np) * n + nodeAt(x + 3)];
}
// Where the record pass reads the passes' results: the global arrays (a warp's rebuild),
// or the shared mirror a block rebuild keeps of one route (position k = x - base)
template <class DT>
struct ScanSrcGlobal {
    const ScanArgs<DT> &A;
    __device__ __forceinline__ int32_t fL(int x, int) const { return A.fwdL[x]; }
    __device__ __forceinline__ int32_t bL(int x, int) const { return A.bwdL[x]; }
    __device__ __forceinline__ DT en(int x, int) const { return A.enext[x]; }
    __device__ __forceinline__ TwRec fT(int x, int) const { return A.fwdT[x]; }
    __device__ __forceinline__ TwRec bT(int x, int) const { return A.bwdT[x]; }
    __device__ __forceinline__ TwRec nt(int node, int) const { return A.node_tw[node]; }
    template <class NodeF>
    __device__ __forceinline__ void br(int k, int x, int len, NodeF nodeAt, DT &b1, DT &b2, DT &b3) const {
        scan_bridges<DT>(A, k, x, len, nodeAt, b1, b2, b3);
    }
};
#ifndef TGA_SCAN_SHARED
#define TGA_SCAN_SHARED 1
#endif
constexpr int kScanShared = 256;   // route positions a block rebuild mirrors in shared memory
template <class DT, bool TW>
struct ScanSrcShared {
    const int32_t *sfL, *sbL;
    const DT *sen, *sbr;           // sbr[3][kScanShared]
    const TwRec *sfT, *sbT, *snt;  // snt: node_tw of the route's positions
    __device__ __forceinline__ int32_t fL(int, int k) const { return sfL[k]; }
    __device__ __forceinline__ int32_t bL(int, int k) const { return sbL[k]; }
    __device__ __forceinline__ DT en(int, int k) const { return sen[k]; }
    __device__ __forceinline__ TwRec fT(int, int k) const { return sfT[k]; }
    __device__ __forceinline__ TwRec bT(int, int k) const { return sbT[k]; }
    __device__ __forceinline__ TwRec nt(int, int k) const { return snt[k]; }
    template <class NodeF>
    __device__ __forceinline__ void br(int k, int, int, NodeF, DT &b1, DT &b2, DT &b3) const {
        b1 = sbr[k]; b2 = sbr[kScanShared + k]; b3 = sbr[2 * kScanShared + k];
    }
};

template <class DT, bool TW, class NodeF, class CanonF, class Src>
__device__ __forceinline__ void scan_rec_pass(const ScanArgs<DT> &A, const int r, const int k0, const int kstep,
                                              const int base, const int L, const int Wr, NodeF nodeAt,
                                              CanonF canonAt, const Src &src) {
    const int len = L + 2;
    // ---------------- per-position segment records and bridges (N = 1..3)
    for (int k = k0; k < len; k += kstep) {
        const int x = base + k;
        DT b1, b2, b3;
        src.br(k, x, len, nodeAt, b1, b2, b3);
        A.bridge1[x] = b1;
        A.bridge2[x] = b2;
        A.bridge3[x] = b3;
        TwRec seg2v = make_float4(0.f, 0.f, 0.f, 0.f), seg3v = seg2v;   // kept for the SlotTW below
        if (TW) {
            const TwRec s1 = src.nt(nodeAt(x), k);
            TwRec s2 = s1, s3 = s1;
            if (k + 1 < len) {
                s2 = tw_cat(s1, src.nt(nodeAt(x + 1), k + 1), static_cast<float>(src.en(x, k)));
                s3 = s2;
                if (k + 2 < len) s3 = tw_cat(s2, src.nt(nodeAt(x + 2), k + 2), static_cast<float>(src.en(x + 1, k + 1)));
            }
            A.seg2T[x] = s2;
            A.seg3T[x] = s3;
            seg2v = s2;
            seg3v = s3;
        }
        if constexpr (std::is_same<DT, int32_t>::value) {
            if (A.rec) {
                SlotRec q;
                const bool slot = k <= L;  // canonical slot (not the end depot)
                const int32_t e_x = src.en(x, k), e_prev = (k >= 1) ? src.en(x - 1, k - 1) : 0;
                const int32_t fl_prev = (k >= 1) ? src.fL(x - 1, k - 1) : 0;
                q.r = (slot && canonAt(x) >= 0) ? r : -1;
                q.fL = slot ? src.fL(x, k) : kPoison;
                q.bL1 = (slot && k + 1 < len) ? src.bL(x + 1, k + 1) : kPoison;
                q.ne = -e_x;
                q.W = slot ? Wr : kPoison;
                const DT br[3] = {b1, b2, b3};
                // time-window part (TW-I): earliest completions / latest starts
                SlotTW w{};
                auto EFof = [&](int y) { const TwRec f = src.fT(y, y - base); return f.w == 0.f ? f.y + f.x : kTwBig; };
                auto LBof = [&](int y) { const TwRec b = src.bT(y, y - base); return b.w == 0.f ? b.z : -kTwBig; };
                if (TW && A.rectw) {
                    w.EF = EFof(x);
                    w.EFm = (k >= 1) ? EFof(x - 1) : kTwBig;
                    const TwRec s1 = src.nt(nodeAt(x), k);
                    const TwRec sg[3] = {s1, seg2v, seg3v};
#pragma unroll
                    for (int N = 1; N <= 3; ++N) {
                        const bool segok = (k >= 1) && (k + N - 1 <= L);
                        w.LBN[N - 1] = (k + N < len) ? LBof(x + N) : -kTwBig;
                        w.sTE[N - 1] = sg[N - 1].y;
                        w.sTL[N - 1] = (segok && sg[N - 1].w == 0.f) ? sg[N - 1].z : -kTwBig;
                        w.sTD[N - 1] = sg[N - 1].x;
                    }
                    w.pad[0] = w.pad[1] = 0.f;
                    A.rectw[x] = w;
                }
                // penalised records: the route's old load excess, weighted (SlotRec)
                const int32_t pex = A.pen_wQ * max(Wr - A.capacity, 0);
                q.ne -= pex;
#pragma unroll
                for (int N = 1; N <= 3; ++N) {
                    const bool segok = (k >= 1) && (k + N - 1 <= L);
                    const int32_t sN = segok ? src.fL(x + N - 1, k + N - 1) - fl_prev : 0;
                    const int32_t eout = segok ? src.en(x + N - 1, k + N - 1) : 0;
                    // route a after removing the segment: F(x-1) + B(x+N) must stay feasible
                    // (feasible-only records; penalised records price the excess instead)
                    bool rem_ok = segok && (A.pen_wQ || Wr - sN <= A.capacity);
                    if (TW && A.rectw && segok)
                        rem_ok = rem_ok && (w.EFm + static_cast<float>(br[N - 1]) <= LBof(x + N));
                    q.so[N - 1] = rem_ok ? sN : kPoison;
                    q.rem[N - 1] = segok ? br[N - 1] - e_prev - eout - pex : 0;
                    q.sA[N - 1] = segok ? Wr - sN : kPoison;
                    q.sS[N - 1] = sN;
                    q.sE[N - 1] = segok ? -e_prev - eout - pex : 0;
                }
                A.rec[x] = q;
                if (A.nsc) {   // the north-star sweep's column terms, one plane per term
                    int32_t *c = A.nsc + x;
                    const size_t P = static_cast<size_t>(A.nsc_pitch);
                    c[0] = q.r; c[P] = q.ne; c[2 * P] = q.rem[0]; c[3 * P] = q.sE[0];
                    c[4 * P] = A.capacity - q.bL1; c[5 * P] = A.capacity - q.fL; c[6 * P] = A.capacity - q.W;
                    c[7 * P] = A.capacity - q.sS[0]; c[8 * P] = q.so[0]; c[9 * P] = q.sA[0];
                }
            }
        }
    }
}

template <class DT, bool TW, class NodeF, class CanonF>
__device__ __forceinline__ void scan_route_g(const ScanArgs<DT> &A, const int r, const int lane, const int base,
                                             const int L, const int cap, NodeF nodeAt, CanonF canonAt) {
    scan_spare<DT, TW>(A, lane, 32, base, L, cap);
    const int Wr = scan_fwd_pass<DT, TW>(A, r, lane, base, L, nodeAt);
    scan_bwd_pass<DT, TW>(A, r, lane, base, L, nodeAt, false);
    __syncwarp();   // fwdL / bwdL / enext of this route are visible to the whole warp
    scan_rec_pass<DT, TW>(A, r, lane, 32, base, L, Wr, nodeAt, canonAt, ScanSrcGlobal<DT>{A});
}

// The same rebuild by a whole block (every thread must call it): forward and
// backward passes in warps 0 and 1 at once, then the per-slot records over all
// threads -- the critical path of the device step's update for long routes.
__device__ __forceinline__ unsigned long long scan_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
template <class DT, bool TW, class NodeF, class CanonF>
__device__ __forceinline__ void scan_route_block(const ScanArgs<DT> &A, const int r, const int base, const int L,
                                                 const int cap, NodeF nodeAt, CanonF canonAt,
                                                 unsigned long long *stamp = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (stamp && tid == 0) stamp[0] = scan_gtime();   // diagnostics: start / passes done / records done
    // routes of up to kScanShared positions: the passes mirror their results in shared memory
    // and the other warps gather the bridges (and node windows) meanwhile, so the record
    // pass reads no global memory (one round trip less on the update's critical path)
    __shared__ int32_t s_fL[kScanShared], s_bL[kScanShared], s_W;
    __shared__ DT s_en[kScanShared], s_br[3 * kScanShared];
    __shared__ TwRec s_fT[TW ? kScanShared : 1], s_bT[TW ? kScanShared : 1], s_nt[TW ? kScanShared : 1];
    const int len = L + 2;
    const bool sh = TGA_SCAN_SHARED && len <= kScanShared && blockDim.x > 64;
    scan_spare<DT, TW>(A, tid, blockDim.x, base, L, cap);
    if (warp == 0) {
        const int W = scan_fwd_pass<DT, TW>(A, r, lane, base, L, nodeAt, sh ? s_fL : nullptr, sh ? s_en : nullptr,
                                            sh ? s_fT : nullptr);
        if (lane == 0) s_W = W;
    } else if (warp == 1) {
        scan_bwd_pass<DT, TW>(A, r, lane, base, L, nodeAt, true, sh ? s_bL : nullptr, sh ? s_bT : nullptr);
    } else if (sh) {
        for (int k = tid - 64; k < len; k += blockDim.x - 64) {
            DT b1, b2, b3;
            scan_bridges<DT>(A, k, base + k, len, nodeAt, b1, b2, b3);
            s_br[k] = b1; s_br[kScanShared + k] = b2; s_br[2 * kScanShared + k] = b3;
            if (TW) s_nt[k] = A.node_tw[nodeAt(base + k)];
        }
    }
    __syncthreads();   // prefix / suffix records and rW[r] of this route are visible to the block
    if (stamp && tid == 0) stamp[1] = scan_gtime();
    if (sh)
        scan_rec_pass<DT, TW>(A, r, tid, blockDim.x, base, L, s_W, nodeAt, canonAt,
                              ScanSrcShared<DT, TW>{s_fL, s_bL, s_en, s_br, s_fT, s_bT, s_nt});
    else
        scan_rec_pass<DT, TW>(A, r, tid, blockDim.x, base, L, A.rW[r], nodeAt, canonAt, ScanSrcGlobal<DT>{A});
    if (stamp) {
        __syncthreads();
        if (tid == 0) stamp[2] = scan_gtime();
    }
}

template <class DT, bool TW>
__device__ __forceinline__ void scan_route(const ScanArgs<DT> &A, const int r, const int lane) {
    const int base = A.rbase[r];
    scan_route_g<DT, TW>(A, r, lane, base, A.rlenR[r], A.rbase[r + 1] - base,
                         [&](int x) { return A.node[x]; }, [&](int x) { return A.canon[x]; });
}

template <class DT, bool TW>
__global__ void __launch_bounds__(256) k_scan(ScanArgs<DT> A, int r_lo, int r_hi) {
    const int lane = threadIdx.x & 31;
    const int r = r_lo + static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (r >= r_hi) return;
    scan_route<DT, TW>(A, r, lane);
}

// The update step of an applied move, phase 1: one unit per Dp row of
// the changed slot ranges (a full C row gather each) and one unit per 8 routes
// to re-scan (a full relayout refreshes every row and re-scans every route).
// The scan reads node ids and C, never Dp: both roles run together.
template <class DT, bool TW>
__device__ __forceinline__ void update_rows(const ScanArgs<DT> &A, DT *__restrict__ Dp, int pitch, int R,
                                            const UpdateSpec u, int unit0, int ustride) {
    const DT *__restrict__ C = A.C;
    const int n = A.n_nodes;
    const int n1 = u.hi1 - u.lo1, n2 = u.hi2 - u.lo2;
    const int nb_rows = n1 + n2;
    const int n_routes = u.full ? R : (u.r1 >= 0) + (u.r2 >= 0);
    const int total = nb_rows + (n_routes + 7) / 8;
    // rows: a block takes its units RG at a time -- the RG row node ids in one round, then
    // per column chunk one (L1-resident) load of the column node ids and RG x 4 gathers in
    // flight (a full relayout refreshes every row: ~7 rows per block at Q_p = 1000)
    constexpr int RG = 8;
    auto row_of = [&](int b) { return b < n1 ? u.lo1 + b : u.lo2 + (b - n1); };
    for (int b0 = unit0; b0 < nb_rows; b0 += RG * ustride) {
        int na[RG];
#pragma unroll
        for (int i = 0; i < RG; ++i) {
            const int b = b0 + i * ustride;
            na[i] = b < nb_rows ? A.node[row_of(b)] : -1;
        }
        for (int c = 4 * threadIdx.x; c < pitch; c += 4 * blockDim.x) {
            const int4 nd = __ldg(reinterpret_cast<const int4 *>(A.node + c));
            DT v[RG][4];
#pragma unroll
            for (int i = 0; i < RG; ++i) {
                if (na[i] < 0) continue;
                const DT *crow = C + static_cast<size_t>(na[i]) * n;
                v[i][0] = __ldg(crow + nd.x); v[i][1] = __ldg(crow + nd.y);
                v[i][2] = __ldg(crow + nd.z); v[i][3] = __ldg(crow + nd.w);
            }
#pragma unroll
            for (int i = 0; i < RG; ++i) {
                if (na[i] < 0) continue;
                DT *drow = Dp + static_cast<size_t>(row_of(b0 + i * ustride)) * pitch;
                *reinterpret_cast<int4 *>(drow + c) = make_int4(bits(v[i][0]), bits(v[i][1]), bits(v[i][2]), bits(v[i][3]));
            }
        }
    }
    // re-scans: one unit per 8 routes, after the row units
    for (int b = unit0; b < total; b += ustride) {
        if (b < nb_rows) continue;
        const int j = (b - nb_rows) * 8 + static_cast<int>(threadIdx.x >> 5);
        if (j < n_routes) scan_route<DT, TW>(A, u.full ? j : (j == 0 && u.r1 >= 0 ? u.r1 : u.r2), threadIdx.x & 31);
    }
}

// Phase 2 (after phase 1 completed): the columns of the changed ranges, from the
// refreshed rows by symmetry, Dp[a][c] = Dp[c][a] (c is symmetric; host-checked),
// as a tiled transpose through shared memory: a unit is 32 rows a x 128 changed
// columns c; the changed rows are read along a (128-byte coalesced reads of the
// just-written rows, L2-resident) and written along c.  Scattered 4-byte gathers
// from C cost 105 MB of DRAM reads per update at n = 10^4; a warp per row a with
// lanes along c read one sector per lane.  Requires blockDim.x to be a multiple of 32.
template <class DT>
__device__ __forceinline__ void update_cols(DT *__restrict__ Dp, int pitch, int Qp, const UpdateSpec u, int unit0,
                                            int ustride) {
    if (u.full) return;  // every row was refreshed
    constexpr int TC = 128;   // changed columns per unit (many loads in flight per thread)
    __shared__ DT tile[TC][33];
    const int n1 = u.hi1 - u.lo1, n2 = u.hi2 - u.lo2, nc = n1 + n2;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int ncb = (nc + TC - 1) / TC, nab = (Qp + 31) / 32;
    auto col = [&](int j) { return j < n1 ? u.lo1 + j : u.lo2 + (j - n1); };
    for (int t = unit0; t < nab * ncb; t += ustride) {
        const int a0 = (t / ncb) * 32, c0 = (t % ncb) * TC;
        const int a = a0 + lane;
        if (nw == 8) {   // every load of the unit in flight before the first store (latency-bound otherwise)
            DT v[TC / 8];
#pragma unroll
            for (int q = 0; q < TC / 8; ++q) {
                const int j = c0 + warp + 8 * q;
                v[q] = (j < nc && a < Qp) ? Dp[static_cast<size_t>(col(j)) * pitch + a] : DT(0);
            }
#pragma unroll
            for (int q = 0; q < TC / 8; ++q) tile[warp + 8 * q][lane] = v[q];
        } else {
            for (int cl = warp; cl < TC; cl += nw) {   // changed row c = col(c0 + cl), lanes along a
                const int j = c0 + cl;
                if (j < nc && a < Qp) tile[cl][lane] = Dp[static_cast<size_t>(col(j)) * pitch + a];
            }
        }
        __syncthreads();
        for (int al = warp; al < 32; al += nw) {   // row a0 + al, lanes along the changed columns
            const int ar = a0 + al;
            if (ar >= Qp) continue;
            DT *drow = Dp + static_cast<size_t>(ar) * pitch;
#pragma unroll
            for (int q = 0; q < TC / 32; ++q) {
                const int j = c0 + q * 32 + lane;
                if (j < nc) drow[col(j)] = tile[q * 32 + lane][al];
            }
        }
        __syncthreads();
    }
}

template <class DT, bool TW>
__global__ void __launch_bounds__(256) k_update(ScanArgs<DT> A, DT *__restrict__ Dp, int pitch, int Qp, int R,
                                                UpdateSpec u) {
    update_rows<DT, TW>(A, Dp, pitch, R, u, blockIdx.x, gridDim.x);
}
template <class DT>
__global__ void __launch_bounds__(256) k_update_cols(DT *__restrict__ Dp, int pitch, int Qp, UpdateSpec u) {
    update_cols<DT>(Dp, pitch, Qp, u, blockIdx.x, gridDim.x);
}

// Device-resident apply + update in ONE launch (blockIdx.y = solution): block 0
// picks the best key and splices the changed routes (tga_pick.cuh), a grid
// barrier over the gridDim.x blocks of the solution (all co-resident: the grid
// is at most one block per SM), then every block refreshes Dp rows / columns
// and re-scans routes of the changed span read from the descriptor.
// Generation (sense-reversing) grid barrier over the nblocks blocks of one
// solution: counter[0] counts arrivals and is reset by the last arriver before it
// advances the generation word counter[2]; waiters spin on the generation.  No
// counter grows across launches, so any number of steps and any mix of grid
// sizes (single solution / population batch) share the descriptor safely.
__device__ __forceinline__ void solution_barrier(int32_t *counter, int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile int32_t *gen = counter + 2;
        const int32_t g = *gen;            // cannot advance before this block arrives
        __threadfence();
        if (atomicAdd(counter, 1) == nblocks - 1) {
            *reinterpret_cast<volatile int32_t *>(counter) = 0;
            __threadfence();
            atomicAdd(counter + 2, 1);
        } else {
            while (*gen == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// Multi-block device step (the Update step of §5.3.5,
// P:437) with no grid barrier between the pick and the update: every block
// decodes the best move itself (decode_best, a warp of key compares and one
// binary search), snapshots the OLD node ids of the 1-2 changed routes into its
// shared memory, and signals arrival; only then may block 0 rewrite the slot
// arrays (it waits for every arrival, which happen early).  New node ids come
// from the snapshot through the pieces, so the Dp rows, the changed columns and
// the re-scans of the changed routes all run at once.  Columns are gathered
// straight from C while Qp is small; above that they are copied from the
// refreshed rows by symmetry behind one barrier (C rows would miss L2).
// A route that outgrew its slots takes the full relayout path of pick_apply_body.
constexpr int kDirectColsQp = 2560;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Arrivals of one launch: every block adds 1 to counter once; block 0 alone waits
// for all nblocks and then resets the counter for the next launch (launches of one
// stream never overlap, and every block has arrived once the count is reached).
__device__ __forceinline__ void wait_arrivals(int32_t *counter, int nblocks) {
    // the arrivals follow the snapshot loads in each block (program order); no fence needed
    while (*reinterpret_cast<volatile int32_t *>(counter) < nblocks) __nanosleep(32);
    *reinterpret_cast<volatile int32_t *>(counter) = 0;
}

template <class DT, bool TW>
__device__ __forceinline__ void pick_update_multi(const DevState &S, const ScanArgs<DT> &A, uint32_t mask,
                                                  uint32_t cmask, int integer, int32_t *smr, int snap_cap,
                                                  unsigned long long *pr) {
    const int tid = threadIdx.x, R = S.R, G = gridDim.x, b = blockIdx.x;
    int32_t *sb = smr, *sl = smr + (R + 1);
    int32_t *snap = smr + 2 * (R + 1);  // old node ids of the changed ranges
    int32_t *nn = snap + snap_cap;      // new node ids of the changed ranges
    const bool direct = S.Qp <= kDirectColsQp;
    __shared__ uint64_t skeys[kNV];
    __shared__ Decoded dm;
    // ---- 1. stage the old route bases / lengths and the keys; decode (every block)
    for (int r = tid; r <= R; r += blockDim.x) {
        sb[r] = S.rbase[r];
        sl[r] = r < R ? S.rlenR[r] : 0;
    }
    if (tid < kNV) skeys[tid] = S.keys[tid];
    __syncthreads();
    if (tid == 0) probe(pr, 1);
    if (pr) S.acc[43] = gtimer();   // diagnostics: block 0 start of decode (globaltimer)
    // the old node ids of the changed routes' first pwin slots ride with the decode
    const int pwin = min(128, snap_cap / 2);
    if (tid < 32) decode_best(skeys, mask, integer, sb, sl, R, S.Qc, dm, snap, S.node, pwin, S.pitch);
    __syncthreads();
    if (tid == 0) probe(pr, 2);
    const int n1 = dm.applied && !dm.full ? dm.hi[0] - dm.lo[0] : 0;
    const int n2 = dm.applied && !dm.full ? dm.hi[1] - dm.lo[1] : 0;
    const int lo0 = dm.lo[0], lo1 = dm.lo[1];
    // ---- 2. new node ids of the changed ranges straight from the old slots through the
    // pieces (start / end depot and spare slots: 0), then arrive -- every read of an old
    // node id of this block is done before block 0 may overwrite them
    for (int j = tid; j < n1 + n2; j += blockDim.x) {
        const int q = j < n1 ? 0 : 1;
        const NewRoute &nr = dm.nr[q];
        const int p = j - (q ? n1 : 0);  // position in the route (base == lo[q])
        int32_t nd = 0;
        if (p >= 1 && p <= nr.L) {
            int off = p - 1, k = 0;
            while (off >= nr.p[k].len) { off -= nr.p[k].len; ++k; }
            const Piece &pc = nr.p[k];
            const int os = sb[pc.src] + (pc.rev ? pc.start + pc.len - 1 - off : pc.start + off);
            const int r0 = os - dm.plo[0], r1 = os - dm.plo[1];
            nd = (r0 >= 0 && r0 < pwin) ? snap[r0] : ((r1 >= 0 && r1 < pwin) ? snap[pwin + r1] : S.node[os]);
        }
        nn[j] = nd;
    }
    __syncthreads();
    if (tid == 0) atomicAdd(S.desc + 9, 1);
    pdl_trigger();  // this block is resident and arrived: a dependent grid cannot starve the wait below
    // ---- 3. roles of the update work.  Direct columns (small Qp): every block does ONE kind of
    // unit, so its chain is two rounds of loads: the re-scans on the last blocks, the changed Dp
    // rows on the first ones, the closed-form counts on the block before the re-scans, the
    // columns of every other row on the blocks between.
    // Symmetric columns (large Qp): rows and re-scans on every block, then a barrier.
    const int nrows = n1 + n2;
    // block 0 keeps only the final slot-array writes (it is the one that waits for
    // every arrival): rows on blocks 1 .. nrows, columns after them, counts, re-scans last
    const bool split_roles = dm.applied && !dm.full && direct && G >= nrows + dm.nrt + 4;
    const int scan0 = split_roles ? G - dm.nrt : 1;                  // first scanning block
    const int row0 = split_roles ? 1 : 0, row_blocks = split_roles ? nrows : G;
    const int col0 = split_roles ? nrows + 1 : 0, col_blocks = split_roles ? G - dm.nrt - nrows - 2 : G;
    // the closed-form counts of the evaluated (old) lengths, on a block of their own when
    // the roles are split (else on a block that does not rebuild a route)
    if (b == (split_roles ? scan0 - 1 : G / 2)) neighbourhood_counts(S, cmask, sl);
    if (!dm.applied) {
        if (b == 0 && tid == 0) {
            S.desc[0] = 0;
            wait_arrivals(S.desc + 9, G);  // every block has read the keys
            for (int v = 0; v < kNV; ++v) S.keys[v] = ~0ull;  // consumed: the next eval needs no memset
        }
        return;
    }
    if (dm.full) {  // relayout: block 0 alone rewrites every slot after all blocks staged
        __syncthreads();
        if (b == 0) {
            if (tid == 0) wait_arrivals(S.desc + 9, G);
            __syncthreads();
            pick_apply_body(S, mask, cmask, integer, smr, pr, false);  // resets the keys too
        }
        solution_barrier(S.desc + 8, G);
        const volatile int32_t *desc = S.desc;
        const UpdateSpec u{desc[1], desc[2], desc[3], desc[4], desc[5], desc[6], desc[7]};
        update_rows<DT, TW>(A, static_cast<DT *>(S.Dp), S.pitch, R, u, b, G);
        return;
    }
    if (tid == 0) probe(pr, 3);
    __syncthreads();
    if (tid == 0) probe(pr, 4);
    auto in_chg = [&](int c) -> int { return (c >= lo0 && c < lo0 + n1) ? c - lo0 : ((c >= lo1 && c < lo1 + n2) ? n1 + c - lo1 : -1); };
    const DT *__restrict__ C = A.C;
    const int n = A.n_nodes, pitch = S.pitch, Qp = S.Qp;
    DT *__restrict__ Dp = static_cast<DT *>(S.Dp);
    // 4a. re-scan of the changed routes (one block each; the longest chains)
    for (int q = 0; q < dm.nrt; ++q) {
        if (b == (scan0 + q) % G) {   // block-uniform: the whole block rebuilds the route
            const int r = dm.nr[q].r, base = dm.lo[q], off = q ? n1 : 0;
            scan_route_block<DT, TW>(A, r, base, dm.nr[q].L, dm.hi[q] - base,
                                     [&](int x) { return nn[off + x - base]; }, [&](int x) { return x; },
                                     (q == 0 && S.acc[31]) ? S.acc + 40 : nullptr);
            if (tid == 0 && S.acc[31]) S.acc[44 + q] = gtimer();   // diagnostics: scan end (globaltimer)
        }
    }
    // 4b. Dp rows of the changed slots: Dp[a][c] = c(new node(a), node(c)), c < pitch
    if (b >= row0 && b < row0 + row_blocks) {
        constexpr int B = 4;   // column chunks per thread with all their loads in flight
        const int step = 4 * static_cast<int>(blockDim.x);
        for (int j = b - row0; j < nrows; j += row_blocks) {
            const int a = j < n1 ? lo0 + j : lo1 + (j - n1);
            const DT *crow = C + static_cast<size_t>(nn[j]) * n;
            DT *drow = Dp + static_cast<size_t>(a) * pitch;
            for (int cb = 4 * tid; cb < pitch; cb += B * step) {
                int4 nd[B];
#pragma unroll
                for (int k = 0; k < B; ++k) {
                    const int c = cb + k * step;
                    nd[k] = c < pitch ? *reinterpret_cast<const int4 *>(S.node + c) : make_int4(0, 0, 0, 0);
                }
                DT v[B][4];
#pragma unroll
                for (int k = 0; k < B; ++k) {
                    const int c = cb + k * step;
                    int t;
                    if ((t = in_chg(c)) >= 0) nd[k].x = nn[t];
                    if ((t = in_chg(c + 1)) >= 0) nd[k].y = nn[t];
                    if ((t = in_chg(c + 2)) >= 0) nd[k].z = nn[t];
                    if ((t = in_chg(c + 3)) >= 0) nd[k].w = nn[t];
                    v[k][0] = __ldg(crow + nd[k].x); v[k][1] = __ldg(crow + nd[k].y);
                    v[k][2] = __ldg(crow + nd[k].z); v[k][3] = __ldg(crow + nd[k].w);
                }
#pragma unroll
                for (int k = 0; k < B; ++k) {
                    const int c = cb + k * step;
                    if (c < pitch)
                        *reinterpret_cast<int4 *>(drow + c) = make_int4(bits(v[k][0]), bits(v[k][1]), bits(v[k][2]), bits(v[k][3]));
                }
            }
        }
    }
    // 4c. columns of the changed slots in every other row (a warp per row; the row's
    // node ids of both of a warp's rows are loaded before any gather)
    if (direct && b >= col0 && b < col0 + col_blocks) {
        const int warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
        const int stride = col_blocks * nw;
        for (int a0 = (b - col0) * nw + warp; a0 < Qp; a0 += 2 * stride) {
            const int a1 = a0 + stride;
            const int32_t na0 = S.node[a0], na1 = a1 < Qp ? S.node[a1] : 0;
            const bool w0 = in_chg(a0) < 0, w1 = a1 < Qp && in_chg(a1) < 0;  // changed rows: written whole above
            const DT *c0 = C + static_cast<size_t>(na0) * n, *c1 = C + static_cast<size_t>(na1) * n;
            DT *d0 = Dp + static_cast<size_t>(a0) * pitch, *d1 = Dp + static_cast<size_t>(a1) * pitch;
            for (int j = lane; j < nrows; j += 32) {
                const int c = j < n1 ? lo0 + j : lo1 + (j - n1);
                const DT v0 = w0 ? __ldg(c0 + nn[j]) : DT(0), v1 = w1 ? __ldg(c1 + nn[j]) : DT(0);
                if (w0) d0[c] = v0;
                if (w1) d1[c] = v1;
            }
        }
    }
    if (tid == 0) probe(pr, 5);
    // ---- 5. block 0: the slot arrays of the changed routes, once every block has its snapshot
    if (b == 0) {
        if (tid == 0) wait_arrivals(S.desc + 9, G);
        __syncthreads();
        for (int j = tid; j < n1 + n2; j += blockDim.x) {
            const int q = j < n1 ? 0 : 1;
            const int x = j < n1 ? lo0 + j : lo1 + (j - n1);
            const int p = j - (q ? n1 : 0), L = dm.nr[q].L, r = dm.nr[q].r;
            const bool live = p <= L + 1;
            S.node[x] = nn[j];
            if (S.slot_of && p >= 1 && p <= L) S.slot_of[nn[j]] = x;
            S.route[x] = live ? r : -1;
            S.pos[x] = live ? p : 0;
            S.rlen[x] = live ? L : -1;
            S.canon[x] = p <= L ? x : -1;  // validity only (keys index physical slots)
        }
        if (tid < dm.nrt) S.rlenR[dm.nr[tid].r] = dm.nr[tid].L;
        if (tid < kNV) S.keys[tid] = ~0ull;  // consumed: the next eval needs no memset
        if (tid == 0) {
            const int rlo = dm.nr[0].r, rhi = dm.nrt == 2 ? dm.nr[1].r : -1;
            S.desc[1] = lo0; S.desc[2] = lo0 + n1; S.desc[3] = dm.nrt == 2 ? lo1 : 0; S.desc[4] = dm.nrt == 2 ? lo1 + n2 : 0;
            S.desc[5] = rlo; S.desc[6] = rhi; S.desc[7] = 0;
            S.desc[0] = 1;
            atomicAdd(S.acc + kAccApplied, 1ull);
        }
    }
    if (!direct) {
        solution_barrier(S.desc + 8, G);  // every changed row is written before the columns copy it
        if (tid == 0) probe(pr, 6);
        const UpdateSpec u{lo0, lo0 + n1, dm.nrt == 2 ? lo1 : 0, dm.nrt == 2 ? lo1 + n2 : 0, dm.nr[0].r,
                           dm.nrt == 2 ? dm.nr[1].r : -1, 0};
        update_cols<DT>(Dp, pitch, Qp, u, b, G);
    }
    __syncthreads();
    if (tid == 0) probe(pr, 7);
    if (pr) S.acc[46] = gtimer();
}

template <class DT, bool TW, bool MULTI>
__device__ __forceinline__ void pick_update_entry(const DevState &S, const ScanArgs<DT> &A, uint32_t mask,
                                                  uint32_t cmask, int integer, int snap_cap, int32_t *smr) {
    unsigned long long *pr = (blockIdx.x == 0 && threadIdx.x == 0 && S.acc[31]) ? S.acc + 32 : nullptr;
    probe(pr, 0);
    if (gridDim.x == 1) pdl_trigger();
    if (MULTI && snap_cap > 0 && gridDim.x > 1) {
        pick_update_multi<DT, TW>(S, A, mask, cmask, integer, smr, snap_cap, pr);
        return;
    }
    // one block per solution (population batches), or the shared memory cannot
    // hold the snapshot: block 0 picks and splices, grid barrier, update
    if (blockIdx.x == 0) pick_apply_body(S, mask, cmask, integer, smr, pr);
    if (gridDim.x > 1) solution_barrier(S.desc + 8, gridDim.x);
    else __syncthreads();
    if (gridDim.x > 1) pdl_trigger();  // every block of this grid is resident (it passed the barrier)
    probe(pr, 4);
    const volatile int32_t *desc = S.desc;
    if (desc[0] == 0) return;
    const UpdateSpec u{desc[1], desc[2], desc[3], desc[4], desc[5], desc[6], desc[7]};
    update_rows<DT, TW>(A, static_cast<DT *>(S.Dp), S.pitch, S.R, u, blockIdx.x, gridDim.x);
    probe(pr, 5);
    if (u.full) return;
    if (gridDim.x > 1) solution_barrier(S.desc + 8, gridDim.x);  // rows before the columns read them
    else __syncthreads();
    probe(pr, 6);
    update_cols<DT>(static_cast<DT *>(S.Dp), S.pitch, S.Qp, u, blockIdx.x, gridDim.x);
    __syncthreads();
    probe(pr, 7);
}

// population batches: blockIdx.y = solution, per-solution state read from device arrays.
// k_pick_update_b (one block per solution) compiles out the multi-block path, whose code
// and registers (112 vs 64 with time windows) would otherwise bound the residency of the
// 1024-block population launch; k_pick_update keeps it (small batches, several blocks each)
template <class DT, bool TW>
__global__ void __launch_bounds__(256) k_pick_update(const DevState *__restrict__ states,
                                                     const ScanArgs<DT> *__restrict__ scans, uint32_t mask,
                                                     uint32_t cmask, int integer, int snap_cap) {
    extern __shared__ int32_t smr[];
    pdl_wait();  // the keys (and, two launches back, the slot arrays) come from stream predecessors
    pick_update_entry<DT, TW, true>(states[blockIdx.y], scans[blockIdx.y], mask, cmask, integer, snap_cap, smr);
}
template <class DT, bool TW>
__global__ void __launch_bounds__(256, 4) k_pick_update_b(const DevState *__restrict__ states,
                                                          const ScanArgs<DT> *__restrict__ scans, uint32_t mask,
                                                          uint32_t cmask, int integer, int snap_cap) {
    extern __shared__ int32_t smr[];
    pdl_wait();
    pick_update_entry<DT, TW, false>(states[blockIdx.y], scans[blockIdx.y], mask, cmask, integer, snap_cap, smr);
}
// one solution: its state passed by value in the parameter space, so every pointer and
// size of the chain (route bases, keys, node ids, C, the record arrays) is a constant-bank
// read instead of a dependent global load in front of the first data load
template <class DT, bool TW>
__global__ void __launch_bounds__(256) k_pick_update1(const __grid_constant__ DevState S,
                                                      const __grid_constant__ ScanArgs<DT> A, uint32_t mask,
                                                      uint32_t cmask, int integer, int snap_cap) {
    extern __shared__ int32_t smr[];
    pdl_wait();
    const bool tl = S.acc[31] != 0 && blockIdx.x < kTimelineBlocks;   // diagnostics: per-block timeline
    if (tl && threadIdx.x == 0) S.acc[kTimeline + 2 * blockIdx.x] = gtimer();
    pick_update_entry<DT, TW, true>(S, A, mask, cmask, integer, snap_cap, smr);
    if (tl) {
        __syncthreads();
        if (threadIdx.x == 0) S.acc[kTimeline + 2 * blockIdx.x + 1] = gtimer();
    }
}

constexpr int kPickSmemMax = 180 * 1024;   // + the static shared memory (<= 227 KB per block)
cudaError_t launch_pick_update(const DevState *states, const void *scans, int n_sol, bool tw, bool is_int,
                               uint32_t mask, uint32_t cmask, int max_routes, int max_cap, int blocks_per_sol,
                               cudaStream_t st, const DevState *h_state, const void *h_scan) {
    // old path: sb, sl, nb (3 x (R+1) ints) + the shared snapshot of the two changed routes;
    // multi-block path: sb, sl + old and new node ids of the two changed routes
    const int smem_old = 3 * (max_routes + 1) * 4 + 2 * max_cap * 4;
    const int smem_multi = 2 * (max_routes + 1) * 4 + 4 * max_cap * 4;
    const bool multi = blocks_per_sol > 1 && smem_multi <= kPickSmemMax;
    const int smem = multi ? std::max(smem_old, smem_multi) : smem_old;
    const int snap_cap = multi ? 2 * max_cap : 0;
    dim3 g(blocks_per_sol, n_sol);
    if (smem > kPickSmemMax) return cudaErrorInvalidValue;
    {  // dynamic + static shared memory above the 48 KB default needs the opt-in (static: ~20 KB);
       // set once per device to the largest size any launch uses
        static PerDevice pd;
        once_per_device(pd, [](int) {
            cudaFuncSetAttribute(k_pick_update<int32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update<int32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update_b<int32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update_b<int32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update_b<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update_b<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update1<int32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update1<int32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update1<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
            cudaFuncSetAttribute(k_pick_update1<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPickSmemMax);
        });
    }
    cudaError_t e;
    const int coop = blocks_per_sol > 1 ? 1 : 0;   // its blocks wait for each other
    if (n_sol == 1 && h_state && h_scan) {   // by value: no dependent loads of the state itself
        const DevState &S = *h_state;
        if (is_int) {
            const auto &A = *static_cast<const ScanArgs<int32_t> *>(h_scan);
            e = tw ? launch_pdl(2, k_pick_update1<int32_t, true>, g, dim3(256), smem, st, coop, S, A, mask, cmask, 1, snap_cap)
                   : launch_pdl(2, k_pick_update1<int32_t, false>, g, dim3(256), smem, st, coop, S, A, mask, cmask, 1, snap_cap);
        } else {
            const auto &A = *static_cast<const ScanArgs<float> *>(h_scan);
            e = tw ? launch_pdl(2, k_pick_update1<float, true>, g, dim3(256), smem, st, coop, S, A, mask, cmask, 0, snap_cap)
                   : launch_pdl(2, k_pick_update1<float, false>, g, dim3(256), smem, st, coop, S, A, mask, cmask, 0, snap_cap);
        }
    } else {
        const auto *si = static_cast<const ScanArgs<int32_t> *>(scans);
        const auto *sf = static_cast<const ScanArgs<float> *>(scans);
        if (multi) {
            if (is_int) e = tw ? launch_pdl(2, k_pick_update<int32_t, true>, g, dim3(256), smem, st, coop, states, si, mask, cmask, 1, snap_cap)
                               : launch_pdl(2, k_pick_update<int32_t, false>, g, dim3(256), smem, st, coop, states, si, mask, cmask, 1, snap_cap);
            else e = tw ? launch_pdl(2, k_pick_update<float, true>, g, dim3(256), smem, st, coop, states, sf, mask, cmask, 0, snap_cap)
                        : launch_pdl(2, k_pick_update<float, false>, g, dim3(256), smem, st, coop, states, sf, mask, cmask, 0, snap_cap);
        } else {
            if (is_int) e = tw ? launch_pdl(2, k_pick_update_b<int32_t, true>, g, dim3(256), smem, st, coop, states, si, mask, cmask, 1, snap_cap)
                               : launch_pdl(2, k_pick_update_b<int32_t, false>, g, dim3(256), smem, st, coop, states, si, mask, cmask, 1, snap_cap);
            else e = tw ? launch_pdl(2, k_pick_update_b<float, true>, g, dim3(256), smem, st, coop, states, sf, mask, cmask, 0, snap_cap)
                        : launch_pdl(2, k_pick_update_b<float, false>, g, dim3(256), smem, st, coop, states, sf, mask, cmask, 0, snap_cap);
        }
    }
    note_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ============================================================== TMA / mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}
// 2-D TMA tile load: box at (x = column, y = row) of the tensor map into smem.
__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// ============================================================== inter-route evaluation
// Tile: TU u-rows x TV v-columns of the (physical) slot pair space; the Dp box
// with a halo (rows u0-1 .. u0+TU+2, cols v0-4 .. v0+TV+3) is TMA-loaded into
// shared memory (double-buffered across the persistent tile loop).
// Thread mapping: lane -> v = v0 + lane + 32*j (j < VPT); warp -> UPW rows.
// One tile of the inter-route candidate space (rows u0.., columns v0..), Dp box
// already in shared memory; running (score, index) keys per variant in `best`.
template <class DT, bool TW, uint32_t MASK, bool DUMP = false>
__device__ __forceinline__ void inter_tile(const SolView<DT> &S, const DT *__restrict__ tile, const int u0,
                                           const int v0, const ScoreParams &sp, uint64_t (&best)[kNV],
                                           unsigned long long *dump = nullptr) {
    constexpr int TU = kTileU, TV = kTileV, VPT = TV / 32, UPW = TU / (kInterThreads / 32);
    constexpr int BW = kBoxW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // Dp(x, y) from the staged box
    auto Dt = [&](int x, int y) -> DT { return tile[(x - u0 + 1) * BW + (y - v0 + kBoxX0)]; };
    // fold one candidate key into the variant's running best (+ the test-only dump; only
    // cells of the candidate space write it -- a cell with route(u) >= route(v) evaluates
    // its streams masked, and its (v, u) mirror holds the real candidates)
    auto take = [&](int var, uint64_t k, uint32_t idx, bool in_space) {
        best[var] = umin64(best[var], k);
        if constexpr (DUMP) {
            if (in_space) dump_put(dump, S.Qc * S.Qc, var, idx, k);
        }
    };
    // VRPSPDTW (S.fwdP != null; a warp-uniform branch): the load a new route is checked
    // with is its largest load L_M, concatenated from the prefix / segment / suffix
    // records (Eq. 3a-d) instead of the delivery sums
    const bool pd = S.fwdP != nullptr;
    auto segP = [&](int x, int N) -> LoadRec {   // slots x..x+N-1
        LoadRec r = ld_single(S.dem[S.node[x]], S.pick[S.node[x]]);
        for (int k = 1; k < N; ++k) r = ld_cat(r, ld_single(S.dem[S.node[x + k]], S.pick[S.node[x + k]]));
        return r;
    };
#pragma unroll 1
    for (int j = 0; j < VPT; ++j) {
        const int v = v0 + lane + 32 * j;
        const int cv = S.canon[v];
        const int rv = S.route[v];
        const int pv = S.pos[v];
        const int Lb = S.rlen[v];
        const int Wb = (rv >= 0) ? S.rW[rv] : 0;
        const float TVb = (TW && rv >= 0) ? S.rTV[rv] : 0.f;
#pragma unroll 1
        for (int i = 0; i < UPW; ++i) {
            const int u = u0 + warp * UPW + i;
            const int cu = S.canon[u];
            const int ru = S.route[u];
            if (cu < 0) continue;  // warp-uniform: end depot / padding row
            const bool pair = (cv >= 0) && (ru < rv);
            const int pu = S.pos[u];
            const int La = S.rlen[u];
            const int Wa = S.rW[ru];
            const float TVa = TW ? S.rTV[ru] : 0.f;
            // flat index over PHYSICAL slots (u * pitch + v): order-isomorphic to the canonical
            // index (both orders are (route, position) lexicographic); the host maps it back
            const uint32_t idx_uv = static_cast<uint32_t>(u) * S.Qc + static_cast<uint32_t>(v);
            const uint32_t idx_vu = static_cast<uint32_t>(v) * S.Qc + static_cast<uint32_t>(u);

            // ---- 2-opt* (3-Seq(0,0) P:346; Eq. 14)
            if (MASK & (1u << 1)) {
                const DT dD = Dt(u, v + 1) + Dt(u + 1, v) - S.enext[u] - S.enext[v];
                int la = S.fwdL[u] + S.bwdL[v + 1];
                int lb = S.fwdL[v] + S.bwdL[u + 1];
                if (pd && pair) {
                    la = ld_cat(S.fwdP[u], S.bwdP[v + 1]).z;
                    lb = ld_cat(S.fwdP[v], S.bwdP[u + 1]).z;
                }
                float ta = 0.f, tb = 0.f;
                if (TW) {
                    ta = tw_cat(S.fwdT[u], S.bwdT[v + 1], static_cast<float>(Dt(u, v + 1))).w;
                    tb = tw_cat(S.fwdT[v], S.bwdT[u + 1], static_cast<float>(Dt(u + 1, v))).w;
                }
                take(1, score_key<DT, TW>(sp, pair, dD, la, lb, Wa, Wb, ta, tb, TVa, TVb, idx_uv), idx_uv, pair);
            }
            // ---- relocate (N=1) / or-opt (N=2,3): both directions (Eq. 13)
#pragma unroll
            for (int N = 1; N <= 3; ++N) {
                if (!(MASK & (1u << (1 + N)))) continue;
                const DT *bridge = N == 1 ? S.bridge1 : (N == 2 ? S.bridge2 : S.bridge3);
                const TwRec *segT = N == 1 ? nullptr : (N == 2 ? S.seg2T : S.seg3T);
                {   // segment u..u+N-1 (route a) inserted after v (route b)
                    const bool ok = pair && pu >= 1 && pu + N - 1 <= La;
                    const DT dD = bridge[u] - S.enext[u - 1] - S.enext[u + N - 1] + Dt(u, v) +
                                  Dt(u + N - 1, v + 1) - S.enext[v];
                    const int s = S.fwdL[u + N - 1] - S.fwdL[u - 1];
                    int la = Wa - s, lb = Wb + s;
                    if (pd && ok) {
                        la = ld_cat(S.fwdP[u - 1], S.bwdP[u + N]).z;
                        lb = ld_cat(ld_cat(S.fwdP[v], segP(u, N)), S.bwdP[v + 1]).z;
                    }
                    float ta = 0.f, tb = 0.f;
                    if (TW) {
                        const TwRec sg = N == 1 ? S.node_tw[S.node[u]] : segT[u];
                        ta = tw_cat(S.fwdT[u - 1], S.bwdT[u + N], static_cast<float>(bridge[u])).w;
                        const TwRec X = tw_cat(S.fwdT[v], sg, static_cast<float>(Dt(u, v)));
                        tb = tw_cat(X, S.bwdT[v + 1], static_cast<float>(Dt(u + N - 1, v + 1))).w;
                    }
                    take(1 + N, score_key<DT, TW>(sp, ok, dD, la, lb, Wa, Wb, ta, tb, TVa, TVb, idx_uv), idx_uv, pair);
                }
                {   // segment v..v+N-1 (route b) inserted after u (route a)
                    const bool ok = pair && pv >= 1 && pv + N - 1 <= Lb;
                    const DT dD = bridge[v] - S.enext[v - 1] - S.enext[v + N - 1] + Dt(u, v) +
                                  Dt(u + 1, v + N - 1) - S.enext[u];
                    const int s = S.fwdL[v + N - 1] - S.fwdL[v - 1];
                    int la = Wa + s, lb = Wb - s;
                    if (pd && ok) {
                        lb = ld_cat(S.fwdP[v - 1], S.bwdP[v + N]).z;
                        la = ld_cat(ld_cat(S.fwdP[u], segP(v, N)), S.bwdP[u + 1]).z;
                    }
                    float ta = 0.f, tb = 0.f;
                    if (TW) {
                        const TwRec sg = N == 1 ? S.node_tw[S.node[v]] : segT[v];
                        tb = tw_cat(S.fwdT[v - 1], S.bwdT[v + N], static_cast<float>(bridge[v])).w;
                        const TwRec X = tw_cat(S.fwdT[u], sg, static_cast<float>(Dt(u, v)));
                        ta = tw_cat(X, S.bwdT[u + 1], static_cast<float>(Dt(u + 1, v + N - 1))).w;
                    }
                    take(1 + N, score_key<DT, TW>(sp, ok, dD, la, lb, Wa, Wb, ta, tb, TVa, TVb, idx_vu), idx_vu, pair);
                }
            }
            // ---- swap (1,1) / cross-exchange (N1,N2) (3-Seq(N1,N2) P:346)
#pragma unroll
            for (int sv = 0; sv < 6; ++sv) {
                const int vid = 5 + sv;
                if (!(MASK & (1u << vid))) continue;
                const int N1 = sv == 0 ? 1 : (sv <= 2 ? 1 : (sv <= 4 ? 2 : 3));
                const int N2 = sv == 0 ? 1 : (sv == 1 ? 2 : (sv == 2 ? 3 : (sv == 3 ? 2 : 3)));
                auto seg = [&](int x, int N) -> TwRec {
                    return N == 1 ? S.node_tw[S.node[x]] : (N == 2 ? S.seg2T[x] : S.seg3T[x]);
                };
                {   // N1-segment at u (route a), N2-segment at v (route b)
                    const bool ok = pair && pu >= 1 && pu + N1 - 1 <= La && pv >= 1 && pv + N2 - 1 <= Lb;
                    const DT dD = Dt(u - 1, v) + Dt(u + N1, v + N2 - 1) + Dt(u, v - 1) + Dt(u + N1 - 1, v + N2) -
                                  S.enext[u - 1] - S.enext[u + N1 - 1] - S.enext[v - 1] - S.enext[v + N2 - 1];
                    const int sa = S.fwdL[u + N1 - 1] - S.fwdL[u - 1];
                    const int sb = S.fwdL[v + N2 - 1] - S.fwdL[v - 1];
                    int la = Wa - sa + sb, lb = Wb - sb + sa;
                    if (pd && ok) {   // A' = F(u-1) + seg(v,N2) + B(u+N1), B' = F(v-1) + seg(u,N1) + B(v+N2)
                        la = ld_cat(ld_cat(S.fwdP[u - 1], segP(v, N2)), S.bwdP[u + N1]).z;
                        lb = ld_cat(ld_cat(S.fwdP[v - 1], segP(u, N1)), S.bwdP[v + N2]).z;
                    }
                    float ta = 0.f, tb = 0.f;
                    if (TW) {
                        const TwRec A1 = tw_cat(S.fwdT[u - 1], seg(v, N2), static_cast<float>(Dt(u - 1, v)));
                        ta = tw_cat(A1, S.bwdT[u + N1], static_cast<float>(Dt(u + N1, v + N2 - 1))).w;
                        const TwRec B1 = tw_cat(S.fwdT[v - 1], seg(u, N1), static_cast<float>(Dt(u, v - 1)));
                        tb = tw_cat(B1, S.bwdT[v + N2], static_cast<float>(Dt(u + N1 - 1, v + N2))).w;
                    }
                    take(vid, score_key<DT, TW>(sp, ok, dD, la, lb, Wa, Wb, ta, tb, TVa, TVb, idx_uv),
                         idx_uv, pair);
                }
                if (N1 != N2) {   // N1-segment at v (route b), N2-segment at u (route a)
                    const bool ok = pair && pv >= 1 && pv + N1 - 1 <= Lb && pu >= 1 && pu + N2 - 1 <= La;
                    const DT dD = Dt(u, v - 1) + Dt(u + N2 - 1, v + N1) + Dt(u - 1, v) + Dt(u + N2, v + N1 - 1) -
                                  S.enext[v - 1] - S.enext[v + N1 - 1] - S.enext[u - 1] - S.enext[u + N2 - 1];
                    const int sb = S.fwdL[v + N1 - 1] - S.fwdL[v - 1];
                    const int sa = S.fwdL[u + N2 - 1] - S.fwdL[u - 1];
                    int la = Wa - sa + sb, lb = Wb - sb + sa;
                    if (pd && ok) {   // B' = F(v-1) + seg(u,N2) + B(v+N1), A' = F(u-1) + seg(v,N1) + B(u+N2)
                        lb = ld_cat(ld_cat(S.fwdP[v - 1], segP(u, N2)), S.bwdP[v + N1]).z;
                        la = ld_cat(ld_cat(S.fwdP[u - 1], segP(v, N1)), S.bwdP[u + N2]).z;
                    }
                    float ta = 0.f, tb = 0.f;
                    if (TW) {
                        const TwRec B1 = tw_cat(S.fwdT[v - 1], seg(u, N2), static_cast<float>(Dt(u, v - 1)));
                        tb = tw_cat(B1, S.bwdT[v + N1], static_cast<float>(Dt(u + N2 - 1, v + N1))).w;
                        const TwRec A1 = tw_cat(S.fwdT[u - 1], seg(v, N1), static_cast<float>(Dt(u - 1, v)));
                        ta = tw_cat(A1, S.bwdT[u + N2], static_cast<float>(Dt(u + N2, v + N1 - 1))).w;
                    }
                    take(vid, score_key<DT, TW>(sp, ok, dD, la, lb, Wa, Wb, ta, tb, TVa, TVb, idx_vu),
                         idx_vu, pair);
                }
            }
            // ---- reversed segments ("Relocate and Swap can incorporate reversed
            // subsequences by exchanging the first and last node index tensors, as in 2-opt"):
            // the segment's records come from its nodes in reverse order; c is symmetric
            // (host-checked), so the reversed segment's own distance is unchanged
            auto segR_T = [&](int x, int N) -> TwRec {   // slots x+N-1, ..., x
                TwRec r = S.node_tw[S.node[x + N - 1]];
                for (int k = N - 2; k >= 0; --k) r = tw_cat(r, S.node_tw[S.node[x + k]], static_cast<float>(S.enext[x + k]));
                return r;
            };
            auto segR_P = [&](int x, int N) -> LoadRec {
                LoadRec r = ld_single(S.dem[S.node[x + N - 1]], S.pick[S.node[x + N - 1]]);
                for (int k = N - 2; k >= 0; --k) r = ld_cat(r, ld_single(S.dem[S.node[x + k]], S.pick[S.node[x + k]]));
                return r;
            };
#pragma unroll
            for (int N = 2; N <= 3; ++N) {   // or-opt N reversed: variants 23, 24
                const int vid = 21 + N;
                if (!(MASK & (1u << vid))) continue;
                const DT *bridge = N == 2 ? S.bridge2 : S.bridge3;
                {   // segment u..u+N-1 (route a) inserted reversed after v (route b): B' = F(v) + rev + B(v+1)
                    const bool ok = pair && pu >= 1 && pu + N - 1 <= La;
                    const DT dD = bridge[u] - S.enext[u - 1] - S.enext[u + N - 1] + Dt(u + N - 1, v) + Dt(u, v + 1) -
                                  S.enext[v];
                    const int s = S.fwdL[u + N - 1] - S.fwdL[u - 1];
                    int la = Wa - s, lb = Wb + s;
                    if (pd && ok) {
                        la = ld_cat(S.fwdP[u - 1], S.bwdP[u + N]).z;
                        lb = ld_cat(ld_cat(S.fwdP[v], segR_P(u, N)), S.bwdP[v + 1]).z;
                    }
                    float ta = 0.f, tb = 0.f;
                    if (TW) {
                        ta = tw_cat(S.fwdT[u - 1], S.bwdT[u + N], static_cast<float>(bridge[u])).w;
                        const TwRec X = tw_cat(S.fwdT[v], segR_T(u, N), static_cast<float>(Dt(u + N - 1, v)));
                        tb = tw_cat(X, S.bwdT[v + 1], static_cast<float>(Dt(u, v + 1))).w;
                    }
                    take(vid, score_key<DT, TW>(sp, ok, dD, la, lb, Wa, Wb, ta, tb, TVa, TVb, idx_uv), idx_uv, pair);
                }
                {   // segment v..v+N-1 (route b) inserted reversed after u (route a): A' = F(u) + rev + B(u+1)
                    const bool ok = pair && pv >= 1 && pv + N - 1 <= Lb;
                    const DT dD = bridge[v] - S.enext[v - 1] - S.enext[v + N - 1] + Dt(u, v + N - 1) + Dt(u + 1, v) -
                                  S.enext[u];
                    const int s = S.fwdL[v + N - 1] - S.fwdL[v - 1];
                    int la = Wa + s, lb = Wb - s;
                    if (pd && ok) {
                        lb = ld_cat(S.fwdP[v - 1], S.bwdP[v + N]).z;
                        la = ld_cat(ld_cat(S.fwdP[u], segR_P(v, N)), S.bwdP[u + 1]).z;
                    }
                    float ta = 0.f, tb = 0.f;
                    if (TW) {
                        tb = tw_cat(S.fwdT[v - 1], S.bwdT[v + N], static_cast<float>(bridge[v])).w;
                        const TwRec X = tw_cat(S.fwdT[u], segR_T(v, N), static_cast<float>(Dt(u, v + N - 1)));
                        ta = tw_cat(X, S.bwdT[u + 1], static_cast<float>(Dt(u + 1, v))).w;
                    }
                    take(vid, score_key<DT, TW>(sp, ok, dD, la, lb, Wa, Wb, ta, tb, TVa, TVb, idx_vu), idx_vu, pair);
                }
            }
#pragma unroll
            for (int N = 2; N <= 3; ++N) {   // cross (N, N), both segments reversed: variants 25, 26
                const int vid = 23 + N;
                if (!(MASK & (1u << vid))) continue;
                // A' = F(u-1) + rev(v..v+N-1) + B(u+N),  B' = F(v-1) + rev(u..u+N-1) + B(v+N)
                const bool ok = pair && pu >= 1 && pu + N - 1 <= La && pv >= 1 && pv + N - 1 <= Lb;
                const DT dD = Dt(u - 1, v + N - 1) + Dt(u + N, v) + Dt(u + N - 1, v - 1) + Dt(u, v + N) -
                              S.enext[u - 1] - S.enext[u + N - 1] - S.enext[v - 1] - S.enext[v + N - 1];
                const int sa = S.fwdL[u + N - 1] - S.fwdL[u - 1];
                const int sb = S.fwdL[v + N - 1] - S.fwdL[v - 1];
                int la = Wa - sa + sb, lb = Wb - sb + sa;
                if (pd && ok) {
                    la = ld_cat(ld_cat(S.fwdP[u - 1], segR_P(v, N)), S.bwdP[u + N]).z;
                    lb = ld_cat(ld_cat(S.fwdP[v - 1], segR_P(u, N)), S.bwdP[v + N]).z;
                }
                float ta = 0.f, tb = 0.f;
                if (TW) {
                    const TwRec A1 = tw_cat(S.fwdT[u - 1], segR_T(v, N), static_cast<float>(Dt(u - 1, v + N - 1)));
                    ta = tw_cat(A1, S.bwdT[u + N], static_cast<float>(Dt(u + N, v))).w;
                    const TwRec B1 = tw_cat(S.fwdT[v - 1], segR_T(u, N), static_cast<float>(Dt(u + N - 1, v - 1)));
                    tb = tw_cat(B1, S.bwdT[v + N], static_cast<float>(Dt(u, v + N))).w;
                }
                take(vid, score_key<DT, TW>(sp, ok, dD, la, lb, Wa, Wb, ta, tb, TVa, TVb, idx_uv), idx_uv, pair);
            }
        }
    }
}

// two resident CTAs per SM (<= 128 registers): the all-variant time-window instantiations
// would take ~157 and run one 256-thread CTA per SM on a latency-bound, gather-heavy body
#ifndef TGA_INTER_MINB
#define TGA_INTER_MINB 2
#endif
template <class DT, bool TW, uint32_t MASK, bool DUMP = false>
__global__ void __launch_bounds__(kInterThreads, TGA_INTER_MINB) k_inter(const __grid_constant__ SolView<DT> S, const __grid_constant__ CUtensorMap tmap,
                                                         const uint32_t *__restrict__ tiles, int t_lo, int t_hi,
                                                         ScoreParams sp, uint64_t *__restrict__ keys,
                                                         unsigned long long *dump) {
    constexpr int TU = kTileU, TV = kTileV, VPT = TV / 32, UPW = TU / (kInterThreads / 32);
    constexpr int BW = kBoxW, BH = kBoxH;
    constexpr int NV = kNV;  // inter variant ids 1..10 and the reversed-segment ones 23..26
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // TMA destinations must be 128-byte aligned in the shared window: align at run time
    unsigned char *smem_al = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    DT *buf0 = reinterpret_cast<DT *>(smem_al);
    DT *buf1 = reinterpret_cast<DT *>(smem_al + kBoxBytesPadded);
    __shared__ uint64_t bar[2];
    __shared__ unsigned long long red[NV];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    if (tid < NV) red[tid] = kNoKey;
    __syncthreads();

    uint64_t best[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) best[i] = kNoKey;

    auto issue = [&](int t, int b) {
        const uint32_t ij = tiles[t];
        const int I = ij >> 16, J = ij & 0xFFFF;
        mbar_expect_tx(&bar[b], kBoxBytes);
        tma_load_2d(b ? buf1 : buf0, &tmap, J * TV - kBoxX0, I * TU - 1, &bar[b]);
    };

    int t = t_lo + blockIdx.x;
    if (tid == 0 && t < t_hi) issue(t, 0);
    uint32_t phase0 = 0, phase1 = 0;
    for (int it = 0; t < t_hi; t += gridDim.x, ++it) {
        const int b = it & 1;
        const int tn = t + gridDim.x;
        if (tid == 0 && tn < t_hi) issue(tn, b ^ 1);
        if (b == 0) { mbar_wait(&bar[0], phase0); phase0 ^= 1; }
        else        { mbar_wait(&bar[1], phase1); phase1 ^= 1; }
        const DT *tile = b ? buf1 : buf0;
        const uint32_t ij = tiles[t];
        const int u0 = (ij >> 16) * TU, v0 = (ij & 0xFFFF) * TV;

        inter_tile<DT, TW, MASK, DUMP>(S, tile, u0, v0, sp, best, dump);
        __syncthreads();  // every thread is done with this buffer before it is refilled
    }

    // ---- fused argmin: warp shuffle -> shared -> one 64-bit atomicMin per variant per CTA
#pragma unroll
    for (int i = 1; i < NV; ++i) {
        if (!(MASK & (1u << i))) continue;
        const uint64_t k = warp_min64(best[i]);
        if (lane == 0 && k != kNoKey) atomicMin(&red[i], static_cast<unsigned long long>(k));
    }
    __syncthreads();
    if (tid < NV && (MASK & (1u << tid)) && red[tid] != kNoKey)
        atomicMin(reinterpret_cast<unsigned long long *>(keys) + tid, red[tid]);
}

// population mode: a work item = (solution, tile) of a batch of solutions of one
// instance; every solution has its own Dp (own TMA descriptor, in global
// memory) and its own 23 keys.  Keys are reduced per work item.
template <class DT, bool TW, uint32_t MASK>
__global__ void __launch_bounds__(kInterThreads, TGA_INTER_MINB) k_inter_batch(const SolView<DT> *__restrict__ views,
                                                               const CUtensorMap *__restrict__ maps,
                                                               const uint32_t *__restrict__ work, int n_work,
                                                               ScoreParams sp, uint64_t *__restrict__ keys) {
    constexpr int TU = kTileU, TV = kTileV;
    constexpr int NV = kNV;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem_al = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    DT *buf0 = reinterpret_cast<DT *>(smem_al);
    DT *buf1 = reinterpret_cast<DT *>(smem_al + kBoxBytesPadded);
    __shared__ uint64_t bar[2];
    __shared__ unsigned long long red[NV];
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    if (tid < NV) red[tid] = kNoKey;
    __syncthreads();
    auto issue = [&](int i, int b) {
        const uint32_t w = work[i];
        const int sol = static_cast<int>(w >> 20);
        const uint32_t ij = views[sol].tiles[w & 0xFFFFFu];
        mbar_expect_tx(&bar[b], kBoxBytes);
        tma_load_2d(b ? buf1 : buf0, maps + sol, (ij & 0xFFFF) * TV - kBoxX0, (ij >> 16) * TU - 1, &bar[b]);
    };
    int i = blockIdx.x;
    if (tid == 0 && i < n_work) issue(i, 0);
    uint32_t phase0 = 0, phase1 = 0;
    for (int it = 0; i < n_work; i += gridDim.x, ++it) {
        const int b = it & 1;
        if (tid == 0 && i + static_cast<int>(gridDim.x) < n_work) issue(i + gridDim.x, b ^ 1);
        if (b == 0) { mbar_wait(&bar[0], phase0); phase0 ^= 1; }
        else        { mbar_wait(&bar[1], phase1); phase1 ^= 1; }
        const uint32_t w = work[i];
        const int sol = static_cast<int>(w >> 20);
        const SolView<DT> &S = views[sol];
        const uint32_t ij = S.tiles[w & 0xFFFFFu];
        uint64_t best[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) best[k] = kNoKey;
        inter_tile<DT, TW, MASK>(S, b ? buf1 : buf0, (ij >> 16) * TU, (ij & 0xFFFF) * TV, sp, best);
#pragma unroll
        for (int k = 1; k < NV; ++k) {
            if (!(MASK & (1u << k))) continue;
            const uint64_t m = warp_min64(best[k]);
            if (lane == 0 && m != kNoKey) atomicMin(&red[k], static_cast<unsigned long long>(m));
        }
        __syncthreads();
        if (tid < NV && (MASK & (1u << tid)) && red[tid] != kNoKey) {
            atomicMin(reinterpret_cast<unsigned long long *>(keys) + static_cast<size_t>(sol) * kNV + tid, red[tid]);
            red[tid] = kNoKey;
        }
        __syncthreads();  // buffer b and red[] are reused
    }
}

// ============================================================== intra-route evaluation
// One thread per (slot u, intra variant); the thread walks v along the route so
// the middle segment of Intra-Relocate / Intra-Swap is composed incrementally
// (one Eq. 4 concatenation per step).
__constant__ int kIntraVariants[13] = {0, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22};

template <class DT, bool TW, bool DUMP = false>
__device__ __forceinline__ void intra_body(const SolView<DT> &S, const ScoreParams &sp, uint32_t vmask, int x_lo,
                                           int x_hi, uint64_t *__restrict__ keys, unsigned long long *dump = nullptr) {
    __shared__ unsigned long long red[23];
    if (threadIdx.x < 23) red[threadIdx.x] = kNoKey;
    __syncthreads();
    // a warp takes one variant for 32 consecutive slots (one code path per warp): groups of
    // nv warps (nv = enabled intra variants, vmask holds only intra bits) cover 32 slots,
    // warp k of a group the k-th enabled variant in kIntraVariants order
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int nv = __popc(vmask);
    const int x = x_lo + (t / (32 * nv)) * 32 + (t & 31);
    uint32_t vm = vmask;
    for (int k = (t >> 5) % nv; k > 0; --k) vm &= vm - 1;
    const int var = __ffs(static_cast<int>(vm)) - 1;
    uint64_t best = kNoKey;
    if (x < x_hi && (vmask & (1u << var)) && S.canon[x] >= 0 && S.pos[x] >= 1) {
        const int p = S.pos[x], L = S.rlen[x], r = S.route[x];
        const int base = x - p;
        const int W = S.rW[r];
        const float TV0 = TW ? S.rTV[r] : 0.f;
        const uint32_t cu = static_cast<uint32_t>(S.canon[x]);
        const uint32_t cbase = cu - static_cast<uint32_t>(p);
        auto D = [&](int a, int b) -> DT { return S.Dp[static_cast<size_t>(a) * S.pitch + b]; };
        auto E = [&](int a) -> DT { return S.enext[a]; };
        auto seg = [&](int a, int N) -> TwRec {
            return N == 1 ? S.node_tw[S.node[a]] : (N == 2 ? S.seg2T[a] : S.seg3T[a]);
        };
        // la: the new route's load -- unchanged by an intra-route move without pickups
        // (the delivery sum), its largest load L_M with them (VRPSPDTW, Eq. 3a-d)
        auto key = [&](DT dD, float tv, int q, int la) -> uint64_t {
            const uint32_t idx = static_cast<uint32_t>(x) * S.Qc + static_cast<uint32_t>(base + q);
            const uint64_t k = score_key<DT, TW>(sp, true, dD, la, 0, W, 0, tv, 0.f, TV0, 0.f, idx);
            if constexpr (DUMP) dump_put(dump, S.Qc * S.Qc, var, idx, k);
            return k;
        };
        const bool pd = S.fwdP != nullptr;   // warp-uniform
        auto ldn = [&](int slot) -> LoadRec { return ld_single(S.dem[S.node[slot]], S.pick[S.node[slot]]); };
        auto segP = [&](int a, int N) -> LoadRec {
            LoadRec r = ldn(a);
            for (int k = 1; k < N; ++k) r = ld_cat(r, ldn(a + k));
            return r;
        };
        if (var == 0) {
            // 2-opt: reverse u..v (Eq. 7); loads unchanged; CVRP only (host-checked)
            for (int q = p + 1; q <= L; ++q) {
                const int v = base + q;
                const DT dD = D(x - 1, v) + D(x, v + 1) - E(x - 1) - E(v);
                best = umin64(best, key(dD, 0.f, q, W));
            }
        } else if (var <= 13) {
            // intra relocate / or-opt of x..x+N-1 after the node originally at q
            const int N = var - 10;
            if (p + N - 1 <= L) {
                const DT rem = (N == 1 ? S.bridge1[x] : (N == 2 ? S.bridge2[x] : S.bridge3[x])) -
                               E(x - 1) - E(x + N - 1);
                // forward: route' = [0..u-1] + [u+N..q] + seg + [q+1..]
                TwRec P = make_float4(0.f, 0.f, 0.f, 0.f);
                TwRec sg = make_float4(0.f, 0.f, 0.f, 0.f);
                if (TW) {
                    sg = seg(x, N);
                    const float br = static_cast<float>(N == 1 ? S.bridge1[x] : (N == 2 ? S.bridge2[x] : S.bridge3[x]));
                    if (p + N <= L) P = tw_cat(S.fwdT[x - 1], S.node_tw[S.node[x + N]], br);
                }
                LoadRec PP = make_int4(0, 0, 0, 0), sgP = PP;   // VRPSPDTW: F(u-1) + [u+N..q], the segment
                if (pd) {
                    sgP = segP(x, N);
                    if (p + N <= L) PP = ld_cat(S.fwdP[x - 1], ldn(x + N));
                }
                for (int q = p + N; q <= L; ++q) {
                    const int v = base + q;
                    if (TW && q > p + N) P = tw_cat(P, S.node_tw[S.node[v]], static_cast<float>(E(v - 1)));
                    if (pd && q > p + N) PP = ld_cat(PP, ldn(v));
                    const DT dD = rem + D(v, x) + D(x + N - 1, v + 1) - E(v);
                    float tv = 0.f;
                    if (TW) {
                        const TwRec A2 = tw_cat(P, sg, static_cast<float>(D(v, x)));
                        tv = tw_cat(A2, S.bwdT[v + 1], static_cast<float>(D(x + N - 1, v + 1))).w;
                    }
                    best = umin64(best, key(dD, tv, q, pd ? ld_cat(ld_cat(PP, sgP), S.bwdP[v + 1]).z : W));
                }
                // backward: route' = [0..q] + seg + [q+1..u-1] + [u+N..]
                TwRec T = make_float4(0.f, 0.f, 0.f, 0.f);
                if (TW && p >= 2) {
                    const float br = static_cast<float>(N == 1 ? S.bridge1[x] : (N == 2 ? S.bridge2[x] : S.bridge3[x]));
                    T = tw_cat(S.node_tw[S.node[x - 1]], S.bwdT[x + N], br);
                }
                LoadRec TP = make_int4(0, 0, 0, 0);   // VRPSPDTW: [q+1..u-1] + B(u+N)
                if (pd && p >= 2) TP = ld_cat(ldn(x - 1), S.bwdP[x + N]);
                for (int q = p - 2; q >= 0; --q) {
                    const int v = base + q;
                    if (TW && q < p - 2) T = tw_cat(S.node_tw[S.node[v + 1]], T, static_cast<float>(E(v + 1)));
                    if (pd && q < p - 2) TP = ld_cat(ldn(v + 1), TP);
                    const DT dD = rem + D(v, x) + D(x + N - 1, v + 1) - E(v);
                    float tv = 0.f;
                    if (TW) {
                        const TwRec A2 = tw_cat(S.fwdT[v], sg, static_cast<float>(D(v, x)));
                        tv = tw_cat(A2, T, static_cast<float>(D(x + N - 1, v + 1))).w;
                    }
                    best = umin64(best, key(dD, tv, q, pd ? ld_cat(ld_cat(S.fwdP[v], sgP), TP).z : W));
                }
            }
        } else {
            // intra swap (N1 at u, N2 at v), u+N1 <= v
            const int N1 = (var - 14) / 3 + 1, N2 = (var - 14) % 3 + 1;
            if (p + N1 - 1 <= L) {
                TwRec M = make_float4(0.f, 0.f, 0.f, 0.f);
                const TwRec s1 = TW ? seg(x, N1) : M;
                LoadRec MP = make_int4(0, 0, 0, 0);               // VRPSPDTW: middle [u+N1..v-1]
                const LoadRec s1P = pd ? segP(x, N1) : MP;
                for (int q = p + N1; q + N2 - 1 <= L; ++q) {
                    const int v = base + q;
                    DT dD;
                    float tv = 0.f;
                    int la = W;
                    if (q == p + N1) {  // adjacent: [0..u-1] + seg_v + seg_u + [v+N2..]
                        dD = D(x - 1, v) + D(v + N2 - 1, x) + D(x + N1 - 1, v + N2) - E(x - 1) - E(v - 1) -
                             E(v + N2 - 1);
                        if (TW) {
                            const TwRec R1 = tw_cat(S.fwdT[x - 1], seg(v, N2), static_cast<float>(D(x - 1, v)));
                            const TwRec R3 = tw_cat(R1, s1, static_cast<float>(D(v + N2 - 1, x)));
                            tv = tw_cat(R3, S.bwdT[v + N2], static_cast<float>(D(x + N1 - 1, v + N2))).w;
                        }
                        if (pd) la = ld_cat(ld_cat(ld_cat(S.fwdP[x - 1], segP(v, N2)), s1P), S.bwdP[v + N2]).z;
                    } else {            // [0..u-1] + seg_v + [u+N1..v-1] + seg_u + [v+N2..]
                        if (pd) MP = (q == p + N1 + 1) ? ldn(v - 1) : ld_cat(MP, ldn(v - 1));
                        if (TW) {
                            const TwRec nv1 = S.node_tw[S.node[v - 1]];
                            M = (q == p + N1 + 1) ? nv1 : tw_cat(M, nv1, static_cast<float>(E(v - 2)));
                        }
                        dD = D(x - 1, v) + D(v + N2 - 1, x + N1) + D(v - 1, x) + D(x + N1 - 1, v + N2) - E(x - 1) -
                             E(x + N1 - 1) - E(v - 1) - E(v + N2 - 1);
                        if (TW) {
                            const TwRec R1 = tw_cat(S.fwdT[x - 1], seg(v, N2), static_cast<float>(D(x - 1, v)));
                            const TwRec R2 = tw_cat(R1, M, static_cast<float>(D(v + N2 - 1, x + N1)));
                            const TwRec R3 = tw_cat(R2, s1, static_cast<float>(D(v - 1, x)));
                            tv = tw_cat(R3, S.bwdT[v + N2], static_cast<float>(D(x + N1 - 1, v + N2))).w;
                        }
                        if (pd) la = ld_cat(ld_cat(ld_cat(ld_cat(S.fwdP[x - 1], segP(v, N2)), MP), s1P), S.bwdP[v + N2]).z;
                    }
                    best = umin64(best, key(dD, tv, q, la));
                }
            }
        }
    }
    if (best != kNoKey) atomicMin(&red[var], static_cast<unsigned long long>(best));
    __syncthreads();
    if (threadIdx.x < 23 && red[threadIdx.x] != kNoKey)
        atomicMin(reinterpret_cast<unsigned long long *>(keys) + threadIdx.x, red[threadIdx.x]);
}

template <class DT, bool TW, bool DUMP = false>
__global__ void __launch_bounds__(256) k_intra(const __grid_constant__ SolView<DT> S, ScoreParams sp, uint32_t vmask,
                                               int x_lo, int x_hi, uint64_t *__restrict__ keys, unsigned long long *dump) {
    intra_body<DT, TW, DUMP>(S, sp, vmask, x_lo, x_hi, keys, dump);
}

// population mode: blockIdx.y = solution (BASELINE config 5)
template <class DT, bool TW>
__global__ void __launch_bounds__(256) k_intra_batch(const SolView<DT> *__restrict__ views, ScoreParams sp,
                                                     uint32_t vmask, uint64_t *__restrict__ keys) {
    const SolView<DT> &S = views[blockIdx.y];
    intra_body<DT, TW>(S, sp, vmask, 0, S.Qp, keys + static_cast<size_t>(blockIdx.y) * kNV);
}

// ============================================================== intra-route evaluation, VRPTW (warp-parallel)
// One warp per u slot x, lane <-> insertion / second-segment position q (chunks of
// 32 with carries).  The middle segments of Intra-Relocate / Intra-Swap are
// warp-wide scans of Eq. 4 records (Hillis-Steele with the in-/out-link of each
// element), so every candidate of a route is evaluated in parallel:
//   relocate fwd  (q >= p+N):  [F(x-1) + x+N .. q] + S(x,N) + B(q+1)
//   relocate bwd  (q <= p-2):  F(q) + S(x,N) + [q+1 .. x-1] + B(x+N)
//   swap (N1,N2)  (q >= p+N1): F(x-1) + S(q,N2) + [x+N1 .. q-1] + S(x,N1) + B(q+N2)
__device__ __forceinline__ TwRec shfl_up_rec(TwRec r, int d) {
    return make_float4(__shfl_up_sync(0xffffffffu, r.x, d), __shfl_up_sync(0xffffffffu, r.y, d),
                       __shfl_up_sync(0xffffffffu, r.z, d), __shfl_up_sync(0xffffffffu, r.w, d));
}
__device__ __forceinline__ TwRec shfl_down_rec(TwRec r, int d) {
    return make_float4(__shfl_down_sync(0xffffffffu, r.x, d), __shfl_down_sync(0xffffffffu, r.y, d),
                       __shfl_down_sync(0xffffffffu, r.z, d), __shfl_down_sync(0xffffffffu, r.w, d));
}
__device__ __forceinline__ TwRec shfl_rec(TwRec r, int src) {
    return make_float4(__shfl_sync(0xffffffffu, r.x, src), __shfl_sync(0xffffffffu, r.y, src),
                       __shfl_sync(0xffffffffu, r.z, src), __shfl_sync(0xffffffffu, r.w, src));
}
// inclusive left-to-right scan of lanes >= s (elements with their in-links);
// lanes < s keep their own element.  Returns the in-link of each lane's run.
__device__ __forceinline__ TwRec scan_fwd(TwRec rec, float &inl, int lane, int s) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const TwRec o = shfl_up_rec(rec, d);
        const float oin = __shfl_up_sync(0xffffffffu, inl, d);
        if (lane - d >= s) { rec = tw_cat(o, rec, inl); inl = oin; }
    }
    return rec;
}
// inclusive right-to-left scan of lanes <= e (elements with their out-links)
__device__ __forceinline__ TwRec scan_bwd(TwRec rec, float &outl, int lane, int e) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const TwRec o = shfl_down_rec(rec, d);
        const float oout = __shfl_down_sync(0xffffffffu, outl, d);
        if (lane + d <= e) { rec = tw_cat(rec, o, outl); outl = oout; }
    }
    return rec;
}

// One warp per (u slot x, length A of the segment starting at x): the forward pass
// evaluates relocate N = A after the segment and the swaps (A, b), the backward pass
// relocate N = A before it.  The three lengths are independent scans (no shared
// carries), so splitting them across warps triples the warps in flight without
// adding work (blockIdx.y = A - 1).
template <class DT, int A, bool DUMP = false>
__device__ __forceinline__ void intra_tw_warp(const SolView<DT> &S, const ScoreParams &sp, uint32_t vmask, int x,
                                              unsigned long long *red, unsigned long long *dump = nullptr) {
    const int lane = threadIdx.x & 31;
    constexpr int kRl = 10 + A, kSw0 = 14 + 3 * (A - 1);   // relocate N = A; swaps (A, 1..3)
    auto D = [&](int a, int b) -> DT { return S.Dp[static_cast<size_t>(a) * S.pitch + b]; };
    auto E = [&](int y) -> DT { return S.enext[y]; };
    // ---- slot x: everything indexed by x alone, one round of loads
    const int cx = S.canon[x], p = S.pos[x], L = S.rlen[x], r = S.route[x];
    const TwRec F = S.fwdT[x - 1];
    const TwRec segxA = A == 1 ? S.node_tw[S.node[x]] : (A == 2 ? S.seg2T[x] : S.seg3T[x]);
    const DT Exm1 = E(x - 1), ExA = E(x + A - 1);
    const DT brA = A == 1 ? S.bridge1[x] : (A == 2 ? S.bridge2[x] : S.bridge3[x]);
    if (!(cx >= 0 && p >= 1) || p + A - 1 > L) return;  // warp-uniform
    const int base = x - p;
    const int W = S.rW[r];
    const float TV0 = S.rTV[r];
    auto keyof = [&](bool ok, DT dD, float tv, int q, int var) -> uint64_t {
        const uint32_t idx = static_cast<uint32_t>(x) * S.Qc + static_cast<uint32_t>(base + q);
        const uint64_t k = score_key<DT, true>(sp, ok, dD, W, 0, W, 0, tv, 0.f, TV0, 0.f, idx);
        if constexpr (DUMP) {
            if (ok) dump_put(dump, S.Qc * S.Qc, var, idx, k);
        }
        return k;
    };
    uint64_t bRl = kNoKey, bRlB = kNoKey, bSw[3] = {kNoKey, kNoKey, kNoKey};
    const bool need_rl = (vmask >> kRl) & 1u;
    const bool any_sw = (vmask >> kSw0) & 7u;

    // ------------------------------------------------ forward pass (chunks left to right)
    // G(q) = [x+A .. q] (plain scan from q = p+A); relocate-forward prefixes are
    // F(x-1) + G(q) by associativity of Eq. 4 (exact on integer-valued times)
    if (need_rl || any_sw) {
        TwRec cG = make_float4(0.f, 0.f, 0.f, 0.f);
        bool hG = false;
        const int st = p + A;
        for (int qb = 0; qb <= L; qb += 32) {
            const int q = qb + lane;
            const bool in = q <= L;
            const int v = base + min(q, L);
            // lane data, loaded up front (masked lanes read slots of this or the next route)
            const int nv = S.node[v];
            const DT Evm1 = E(max(v - 1, base)), Ev0 = E(v), Ev1 = E(v + 1), Ev2 = E(v + 2);
            const TwRec bw[3] = {S.bwdT[v + 1], S.bwdT[v + 2], S.bwdT[v + 3]};
            const TwRec sg2 = S.seg2T[v], sg3 = S.seg3T[v];
            const DT dm1 = D(x - 1, v), dxm = D(x, max(v - 1, base));
            DT d0[3], dAm1[4], dA[3];   // Dp(x, v + j), Dp(x + A - 1, v + j), Dp(x + A, v + j)
#pragma unroll
            for (int j = 0; j < 3; ++j) d0[j] = D(x, v + j);
#pragma unroll
            for (int j = 0; j < 4; ++j) dAm1[j] = (A == 1 && j < 3) ? DT(0) : D(x + A - 1, v + j);
            if (A == 1) {
#pragma unroll
                for (int j = 0; j < 3; ++j) dAm1[j] = d0[j];
            }
#pragma unroll
            for (int j = 0; j < 3; ++j) dA[j] = D(x + A, v + j);
            const TwRec sv = S.node_tw[nv];
            const TwRec segv[3] = {sv, sg2, sg3};
            const DT Evb[3] = {Ev0, Ev1, Ev2};  // E(v + b - 1)
            float inl = q >= 1 ? static_cast<float>(Evm1) : 0.f;  // link (q-1 -> q)
            const int s_rel = max(st - qb, 0);
            TwRec Gk = scan_fwd(sv, inl, lane, s_rel);
            if (hG && lane >= s_rel) Gk = tw_cat(cG, Gk, inl);
            TwRec Gm = shfl_up_rec(Gk, 1);  // G(q-1)
            if (lane == 0) Gm = cG;
            if (st <= qb + 31) {  // carry: the run covers the whole chunk from here on
                cG = shfl_rec(Gk, 31);
                hG = true;
            }
            if (need_rl) {  // relocate N = A after q >= p+N:  [F(x-1) + x+N .. q] + S(x,N) + B(q+1)
                const bool ok = in && q >= st;
                const DT rem = brA - Exm1 - ExA;
                const DT dD = rem + d0[0] + dAm1[1] - Ev0;
                const TwRec P = tw_cat(F, Gk, static_cast<float>(brA));
                const TwRec A2 = tw_cat(P, segxA, static_cast<float>(d0[0]));
                const float tv = tw_cat(A2, bw[0], static_cast<float>(dAm1[1])).w;
                bRl = umin64(bRl, keyof(ok, dD, tv, q, kRl));
            }
#pragma unroll
            for (int b = 1; b <= 3; ++b) {
                const int var = kSw0 + (b - 1);
                if (!(vmask & (1u << var))) continue;
                const bool ok = in && q >= p + A && q + b - 1 <= L;
                if (!__any_sync(0xffffffffu, ok)) continue;
                const TwRec R1 = tw_cat(F, segv[b - 1], static_cast<float>(dm1));
                DT dD;
                float tv;
                if (q == p + A) {  // adjacent
                    dD = dm1 + d0[b - 1] + dAm1[b] - Exm1 - Evm1 - Evb[b - 1];
                    const TwRec R3 = tw_cat(R1, segxA, static_cast<float>(d0[b - 1]));
                    tv = tw_cat(R3, bw[b - 1], static_cast<float>(dAm1[b])).w;
                } else {
                    dD = dm1 + dA[b - 1] + dxm + dAm1[b] - Exm1 - ExA - Evm1 - Evb[b - 1];
                    const TwRec R2 = tw_cat(R1, Gm, static_cast<float>(dA[b - 1]));
                    const TwRec R3 = tw_cat(R2, segxA, static_cast<float>(dxm));
                    tv = tw_cat(R3, bw[b - 1], static_cast<float>(dAm1[b])).w;
                }
                bSw[b - 1] = umin64(bSw[b - 1], keyof(ok, dD, tv, q, var));
            }
        }
    }
    // ------------------------------------------------ backward pass: relocate before the segment
    if (need_rl && p >= 2) {
        const int nch = (p - 1) / 32 + 1;  // element positions up to p-1 (lane q reads Suf(q+1))
        const TwRec bwxA = S.bwdT[x + A];
        TwRec cS = make_float4(0.f, 0.f, 0.f, 0.f);
        bool hS = false;
        for (int ci = nch - 1; ci >= 0; --ci) {
            const int qb = ci * 32;
            const int k = qb + lane;                 // element position k in [1, p-1]; lane q uses Suf(q+1)
            const int vk = base + min(max(k, 1), p - 1);
            const int q = qb + lane;
            const int vq = base + min(q, p - 2);
            // lane data, loaded up front
            const int nk = S.node[vk];
            const float outl = static_cast<float>(E(vk));  // link (k -> k+1)
            const DT Evq = E(vq);
            const TwRec Fq = S.fwdT[vq];
            const DT dq0 = D(x, vq), dq1 = D(x + A - 1, vq + 1);
            const TwRec sk = S.node_tw[nk];
            // Suf(k) = [k .. x-1] + B(x+N); the element at k = p-1 carries B(x+N) (link = bridge_N)
            TwRec el = sk;
            float ol = outl;
            if (k == p - 1) { el = tw_cat(sk, bwxA, static_cast<float>(brA)); ol = 0.f; }
            const int e_rel = min(p - 1 - qb, 31);
            TwRec Sf = scan_bwd(el, ol, lane, e_rel);
            if (hS && lane <= e_rel) Sf = tw_cat(Sf, cS, ol);
            const TwRec carry_in = cS;
            const bool had = hS;
            cS = shfl_rec(Sf, 0);
            hS = true;
            // lane q = qb + lane inserts after position q: needs Suf(q+1)
            TwRec Sn = shfl_down_rec(Sf, 1);
            if (lane == 31) Sn = had ? carry_in : Sf;
            const bool ok = q <= p - 2;
            if (!__any_sync(0xffffffffu, ok)) continue;
            const DT rem = brA - Exm1 - ExA;
            const DT dD = rem + dq0 + dq1 - Evq;
            const TwRec A2 = tw_cat(Fq, segxA, static_cast<float>(dq0));
            const float tv = tw_cat(A2, Sn, static_cast<float>(dq1)).w;
            bRlB = umin64(bRlB, keyof(ok, dD, tv, q, kRl));
        }
    }
    auto put = [&](int var, uint64_t b) {
        const uint64_t m = warp_min64(b);
        if (lane == 0 && m != kNoKey && m < red[var]) red[var] = m;  // the warp's private row
    };
    if (need_rl) put(kRl, umin64(bRl, bRlB));
#pragma unroll
    for (int b = 0; b < 3; ++b)
        if (vmask & (1u << (kSw0 + b))) put(kSw0 + b, bSw[b]);
}

template <class DT, bool DUMP>
__device__ __forceinline__ void intra_tw_dispatch(const SolView<DT> &S, const ScoreParams &sp, uint32_t vmask, int x,
                                                  unsigned long long *red, unsigned long long *dump = nullptr) {
    if (blockIdx.y == 0) intra_tw_warp<DT, 1, DUMP>(S, sp, vmask, x, red, dump);
    else if (blockIdx.y == 1) intra_tw_warp<DT, 2, DUMP>(S, sp, vmask, x, red, dump);
    else intra_tw_warp<DT, 3, DUMP>(S, sp, vmask, x, red, dump);
}

template <class DT, bool DUMP = false>
__global__ void __launch_bounds__(256, 3) k_intra_tw(const __grid_constant__ SolView<DT> S, ScoreParams sp,
                                                  uint32_t vmask, int x_lo, int x_hi, uint64_t *__restrict__ keys,
                                                  unsigned long long *dump) {
    __shared__ unsigned long long red[8][23];   // one private row per warp
    for (int i = threadIdx.x; i < 8 * 23; i += blockDim.x) red[i / 23][i % 23] = kNoKey;
    __syncthreads();
    const int x = x_lo + static_cast<int>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (x < x_hi) intra_tw_dispatch<DT, DUMP>(S, sp, vmask, x, red[threadIdx.x >> 5], dump);
    __syncthreads();
    if (threadIdx.x < 23) {
        unsigned long long m = red[0][threadIdx.x];
        for (int w = 1; w < 8; ++w) m = m < red[w][threadIdx.x] ? m : red[w][threadIdx.x];
        if (m != kNoKey) atomicMin(reinterpret_cast<unsigned long long *>(keys) + threadIdx.x, m);
    }
}

// population mode: blockIdx.z = solution
template <class DT>
__global__ void __launch_bounds__(256, 3) k_intra_tw_batch(const SolView<DT> *__restrict__ views, ScoreParams sp,
                                                        uint32_t vmask, uint64_t *__restrict__ keys) {
    __shared__ unsigned long long red[8][23];   // one private row per warp
    for (int i = threadIdx.x; i < 8 * 23; i += blockDim.x) red[i / 23][i % 23] = kNoKey;
    __syncthreads();
    const SolView<DT> &S = views[blockIdx.z];
    const int x = static_cast<int>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (x < S.Qp) intra_tw_dispatch<DT, false>(S, sp, vmask, x, red[threadIdx.x >> 5]);
    __syncthreads();
    if (threadIdx.x < 23) {
        unsigned long long m = red[0][threadIdx.x];
        for (int w = 1; w < 8; ++w) m = m < red[w][threadIdx.x] ? m : red[w][threadIdx.x];
        if (m != kNoKey)
            atomicMin(reinterpret_cast<unsigned long long *>(keys) + static_cast<size_t>(blockIdx.z) * kNV + threadIdx.x, m);
    }
}

// ============================================================== intra-route evaluation, CVRP
// No time windows => no sequential middle segment: every (u, v) pair of a route
// is independent.  A warp owns one u slot, lane <-> v position (strided by 32);
// per variant the warp argmin is one 32-bit REDUX.MIN of (score << 5 | lane):
// lanes hold consecutive canonical v, so the lowest lane is the lowest index.
// Loads are unchanged by intra moves (Eq. 3f), so feasibility is the route's.
template <bool DUMP = false>
__global__ void __launch_bounds__(256) k_intra_cvrp(const SolView<int32_t> S, ScoreParams sp, uint32_t vmask,
                                                    int x_lo, int x_hi, uint64_t *__restrict__ keys,
                                                    unsigned long long *dump) {
    __shared__ unsigned long long red[8][23];   // one private row per warp
    for (int i = threadIdx.x; i < 8 * 23; i += blockDim.x) red[i / 23][i % 23] = kNoKey;
    __syncthreads();
    const int x = x_lo + static_cast<int>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (x < x_hi) intra_cvrp_warp<DUMP>(S, sp, vmask, x, red[threadIdx.x >> 5], nullptr, dump);
    __syncthreads();
    if (threadIdx.x < 23) {
        unsigned long long m = red[0][threadIdx.x];
        for (int w = 1; w < 8; ++w) m = m < red[w][threadIdx.x] ? m : red[w][threadIdx.x];
        if (m != kNoKey) atomicMin(reinterpret_cast<unsigned long long *>(keys) + threadIdx.x, m);
    }
}

// ============================================================== launchers
static unsigned long long g_launches = 0;
unsigned long long launch_count() { return g_launches; }
// Off by default: measured on B200 (bench.py, replicas graph) every combination
// was slower -- cfg2 23.3 us/step without, 24.5-25.4 with; n=2000 38.8 vs 41.6-44.1.
// TGA_PDL_MODE bits: 1 eval launch, 2 pick launch, 4 eval triggers after its tiles.
bool pdl_enabled(int which) {
    static const int mode = std::getenv("TGA_PDL_MODE") ? std::atoi(std::getenv("TGA_PDL_MODE")) : 0;
    return (mode & which) != 0;
}
void note_launch() { ++g_launches; }

// The per-eval key reset.  Launched as a programmatic dependent (pdl) it waits for its
// stream predecessor before writing the keys; it releases its own dependent (the north-star
// sweep) after that wait, or -- early, when the predecessor is an evaluation of the same,
// unchanged solution, so the dependent's pre-wait reads of Dp / records are safe -- at once,
// so consecutive sweeps of an evaluation loop overlap.
__global__ void k_fill_u64(uint64_t *__restrict__ p, size_t n, uint64_t v, int early) {
    if (early) pdl_trigger();
    pdl_wait();
    if (!early) pdl_trigger();
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}
cudaError_t launch_fill_u64(uint64_t *p, size_t n, uint64_t v, cudaStream_t st, bool pdl, bool early) {
    if (n == 0) return cudaSuccess;
    const int block = n <= 32 ? 32 : 256;
    const int grid = static_cast<int>(std::min<size_t>((n + block - 1) / block, 1184));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_fill_u64, p, n, v, early ? 1 : 0);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaGetLastError();
}

template <class DT>
cudaError_t launch_dp(DT *Dp, int pitch, const int32_t *node, const DT *C, int n, int Qp, int lo, int hi,
                      bool full, cudaStream_t st) {
    if (hi <= lo) return cudaSuccess;
    {
        dim3 grid(std::max(1, std::min(8, (pitch / 4 + 255) / 256)), hi - lo);
        k_dp_rows<DT><<<grid, 256, 0, st>>>(Dp, pitch, node, C, n, lo, hi);
        ++g_launches;
    }
    if (!full) {
        dim3 grid((hi - lo + 31) / 32, (Qp + 7) / 8);
        k_dp_cols<DT><<<grid, dim3(32, 8), 0, st>>>(Dp, pitch, node, C, n, Qp, lo, hi);
        ++g_launches;
    }
    return cudaGetLastError();
}

template <class DT>
cudaError_t launch_scan(const ScanArgs<DT> &A, bool tw, int r_lo, int r_hi, cudaStream_t st) {
    if (r_hi <= r_lo) return cudaSuccess;
    const int warps = r_hi - r_lo;
    const int blocks = (warps * 32 + 255) / 256;
    if (tw) k_scan<DT, true><<<blocks, 256, 0, st>>>(A, r_lo, r_hi);
    else    k_scan<DT, false><<<blocks, 256, 0, st>>>(A, r_lo, r_hi);
    ++g_launches;
    return cudaGetLastError();
}

template <class DT>
cudaError_t launch_update(const ScanArgs<DT> &A, bool tw, DT *Dp, int pitch, int Qp, int R, const UpdateSpec &u,
                          cudaStream_t st) {
    const int n_routes = u.full ? R : (u.r1 >= 0) + (u.r2 >= 0);
    const int grid = (u.hi1 - u.lo1) + (u.hi2 - u.lo2) + (n_routes + 7) / 8;
    if (grid <= 0) return cudaSuccess;
    if (tw) k_update<DT, true><<<grid, 256, 0, st>>>(A, Dp, pitch, Qp, R, u);
    else    k_update<DT, false><<<grid, 256, 0, st>>>(A, Dp, pitch, Qp, R, u);
    ++g_launches;
    if (!u.full) {
        k_update_cols<DT><<<(Qp + 7) / 8, 256, 0, st>>>(Dp, pitch, Qp, u);
        ++g_launches;
    }
    return cudaGetLastError();
}
template cudaError_t launch_update<int32_t>(const ScanArgs<int32_t> &, bool, int32_t *, int, int, int,
                                            const UpdateSpec &, cudaStream_t);
template cudaError_t launch_update<float>(const ScanArgs<float> &, bool, float *, int, int, int, const UpdateSpec &,
                                          cudaStream_t);

template <class DT, bool TW, uint32_t MASK>
static cudaError_t launch_inter_t(const SolView<DT> &S, const CUtensorMap &map, const uint32_t *tiles, int t_lo,
                                  int t_hi, const ScoreParams &sp, uint64_t *keys, int grid, cudaStream_t st) {
    auto kern = k_inter<DT, TW, MASK>;
    const int smem = 2 * kBoxBytesPadded + 128;
    static PerDevice pd;
    once_per_device(pd, [&](int) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
    kern<<<grid, kInterThreads, smem, st>>>(S, map, tiles, t_lo, t_hi, sp, keys, nullptr);
    ++g_launches;
    return cudaGetLastError();
}

// compiled MASK groups; a request is decomposed into these
template <class DT, bool TW>
static cudaError_t launch_inter_tw(uint32_t mask, const SolView<DT> &S, const CUtensorMap &map, const uint32_t *tiles,
                                   int t_lo, int t_hi, const ScoreParams &sp, uint64_t *keys, int grid,
                                   cudaStream_t st) {
    cudaError_t err = cudaSuccess;
    auto run = [&](auto kmask) {
        if (err == cudaSuccess)
            err = launch_inter_t<DT, TW, decltype(kmask)::value>(S, map, tiles, t_lo, t_hi, sp, keys, grid, st);
    };
    constexpr uint32_t ALL = 0x7FEu, NS = (1u << 1) | (1u << 2) | (1u << 5);
    if ((mask & ALL) == ALL) { run(std::integral_constant<uint32_t, ALL>{}); return err; }
    if ((mask & NS) == NS) { run(std::integral_constant<uint32_t, NS>{}); mask &= ~NS; }
    if (mask & (1u << 1)) run(std::integral_constant<uint32_t, (1u << 1)>{});
    if (mask & (1u << 2)) run(std::integral_constant<uint32_t, (1u << 2)>{});
    if (mask & (3u << 3)) run(std::integral_constant<uint32_t, (3u << 3)>{});
    if (mask & (1u << 5)) run(std::integral_constant<uint32_t, (1u << 5)>{});
    if (mask & (0x1Fu << 6)) run(std::integral_constant<uint32_t, (0x1Fu << 6)>{});
    if (mask & kRevMask) run(std::integral_constant<uint32_t, kRevMask>{});   // reversed segments
    return err;
}

template <class DT>
cudaError_t launch_inter(uint32_t mask, bool tw, const SolView<DT> &S, const CUtensorMap &map, const uint32_t *tiles,
                         int t_lo, int t_hi, const ScoreParams &sp, uint64_t *keys, int grid, cudaStream_t st) {
    if (t_hi <= t_lo || !(mask & (0x7FEu | kRevMask))) return cudaSuccess;
    return tw ? launch_inter_tw<DT, true>(mask, S, map, tiles, t_lo, t_hi, sp, keys, grid, st)
              : launch_inter_tw<DT, false>(mask, S, map, tiles, t_lo, t_hi, sp, keys, grid, st);
}

template <class DT>
cudaError_t launch_intra(uint32_t mask, bool tw, const SolView<DT> &S, const ScoreParams &sp, int x_lo, int x_hi,
                         uint64_t *keys, cudaStream_t st, bool small_dist, bool warp_tw) {
    const uint32_t intra = mask & ((1u << 0) | (0x7u << 11) | (0x1FFu << 14));
    if (x_hi <= x_lo || !intra) return cudaSuccess;
    if constexpr (std::is_same<DT, int32_t>::value) {
        if (!tw && small_dist) {
            const int blocks = (x_hi - x_lo + 7) / 8;
            k_intra_cvrp<false><<<blocks, 256, 0, st>>>(S, sp, intra, x_lo, x_hi, keys, nullptr);
            ++g_launches;
            return cudaGetLastError();
        }
    }
    if (tw && !(intra & 1u) && warp_tw) {  // warp-parallel VRPTW kernel (long routes)
        const dim3 blocks((x_hi - x_lo + 7) / 8, 3);   // y: the segment length A at u
        k_intra_tw<DT, false><<<blocks, 256, 0, st>>>(S, sp, intra, x_lo, x_hi, keys, nullptr);
        ++g_launches;
        return cudaGetLastError();
    }
    const int threads = (x_hi - x_lo + 31) / 32 * 32 * __builtin_popcount(intra);
    const int blocks = (threads + 255) / 256;
    if (tw) k_intra<DT, true, false><<<blocks, 256, 0, st>>>(S, sp, intra, x_lo, x_hi, keys, nullptr);
    else    k_intra<DT, false, false><<<blocks, 256, 0, st>>>(S, sp, intra, x_lo, x_hi, keys, nullptr);
    ++g_launches;
    return cudaGetLastError();
}

// ---- test-only DUMP instantiations (tga_debug_eval_dump): the same kernels and launch
// geometry as launch_inter / launch_intra, every evaluated candidate's key stored in dump
template <class DT>
cudaError_t launch_eval_dump(uint32_t mask, bool tw, const SolView<DT> &S, const CUtensorMap &map,
                             const uint32_t *tiles, int t_lo, int t_hi, const ScoreParams &sp, uint64_t *keys,
                             int grid, int x_lo, int x_hi, bool inter, bool small_dist, bool warp_tw,
                             cudaStream_t st, unsigned long long *dump) {
    constexpr uint32_t ALL = 0x7FEu;
    if (inter && t_hi > t_lo && (mask & ALL)) {
        const int smem = 2 * kBoxBytesPadded + 128;
        auto kern = tw ? k_inter<DT, true, ALL, true> : k_inter<DT, false, ALL, true>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<grid, kInterThreads, smem, st>>>(S, map, tiles, t_lo, t_hi, sp, keys, dump);
        ++g_launches;
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (t_hi > t_lo && (mask & kRevMask)) {   // reversed segments: always the generic kernel
        const int smem = 2 * kBoxBytesPadded + 128;
        auto kern = tw ? k_inter<DT, true, kRevMask, true> : k_inter<DT, false, kRevMask, true>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        kern<<<grid, kInterThreads, smem, st>>>(S, map, tiles, t_lo, t_hi, sp, keys, dump);
        ++g_launches;
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const uint32_t intra = mask & ((1u << 0) | (0x7u << 11) | (0x1FFu << 14));
    if (x_hi <= x_lo || !intra) return cudaSuccess;
    if constexpr (std::is_same<DT, int32_t>::value) {
        if (!tw && small_dist) {
            k_intra_cvrp<true><<<(x_hi - x_lo + 7) / 8, 256, 0, st>>>(S, sp, intra, x_lo, x_hi, keys, dump);
            ++g_launches;
            return cudaGetLastError();
        }
    }
    if (tw && !(intra & 1u) && warp_tw) {
        k_intra_tw<DT, true><<<dim3((x_hi - x_lo + 7) / 8, 3), 256, 0, st>>>(S, sp, intra, x_lo, x_hi, keys, dump);
        ++g_launches;
        return cudaGetLastError();
    }
    const int threads = (x_hi - x_lo + 31) / 32 * 32 * __builtin_popcount(intra);
    if (tw) k_intra<DT, true, true><<<(threads + 255) / 256, 256, 0, st>>>(S, sp, intra, x_lo, x_hi, keys, dump);
    else    k_intra<DT, false, true><<<(threads + 255) / 256, 256, 0, st>>>(S, sp, intra, x_lo, x_hi, keys, dump);
    ++g_launches;
    return cudaGetLastError();
}
template cudaError_t launch_eval_dump<int32_t>(uint32_t, bool, const SolView<int32_t> &, const CUtensorMap &,
                                               const uint32_t *, int, int, const ScoreParams &, uint64_t *, int, int,
                                               int, bool, bool, bool, cudaStream_t, unsigned long long *);
template cudaError_t launch_eval_dump<float>(uint32_t, bool, const SolView<float> &, const CUtensorMap &,
                                             const uint32_t *, int, int, const ScoreParams &, uint64_t *, int, int, int,
                                             bool, bool, bool, cudaStream_t, unsigned long long *);

template <class DT, bool TW>
static cudaError_t launch_inter_batch_tw(uint32_t mask, const SolView<DT> *views, const CUtensorMap *maps,
                                         const uint32_t *work, int n_work, const ScoreParams &sp, uint64_t *keys,
                                         int grid, cudaStream_t st) {
    cudaError_t err = cudaSuccess;
    const int smem = 2 * kBoxBytesPadded + 128;
    auto run = [&](auto kmask) {
        if (err != cudaSuccess) return;
        auto kern = k_inter_batch<DT, TW, decltype(kmask)::value>;
        static PerDevice pd;
        once_per_device(pd, [&](int) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
        kern<<<grid, kInterThreads, smem, st>>>(views, maps, work, n_work, sp, keys);
        ++g_launches;
        err = cudaGetLastError();
    };
    constexpr uint32_t ALL = 0x7FEu, NS = (1u << 1) | (1u << 2) | (1u << 5);
    if ((mask & ALL) == ALL) { run(std::integral_constant<uint32_t, ALL>{}); return err; }
    if ((mask & NS) == NS) { run(std::integral_constant<uint32_t, NS>{}); mask &= ~NS; }
    if (mask & (1u << 1)) run(std::integral_constant<uint32_t, (1u << 1)>{});
    if (mask & (1u << 2)) run(std::integral_constant<uint32_t, (1u << 2)>{});
    if (mask & (3u << 3)) run(std::integral_constant<uint32_t, (3u << 3)>{});
    if (mask & (1u << 5)) run(std::integral_constant<uint32_t, (1u << 5)>{});
    if (mask & (0x1Fu << 6)) run(std::integral_constant<uint32_t, (0x1Fu << 6)>{});
    if (mask & kRevMask) run(std::integral_constant<uint32_t, kRevMask>{});
    return err;
}

template <class DT>
cudaError_t launch_batch(uint32_t mask, bool tw, const SolView<DT> *views, const CUtensorMap *maps,
                         const uint32_t *work, int n_work, int n_sol, int max_qp, const ScoreParams &sp,
                         uint64_t *keys, int grid, cudaStream_t st, bool warp_tw) {
    cudaError_t e = cudaSuccess;
    if (n_work > 0 && (mask & (0x7FEu | kRevMask)))
        e = tw ? launch_inter_batch_tw<DT, true>(mask, views, maps, work, n_work, sp, keys, grid, st)
               : launch_inter_batch_tw<DT, false>(mask, views, maps, work, n_work, sp, keys, grid, st);
    const uint32_t intra = mask & ((1u << 0) | (0x7u << 11) | (0x1FFu << 14));
    if (e == cudaSuccess && intra && n_sol > 0) {
        dim3 g(((max_qp + 31) / 32 * 32 * __builtin_popcount(intra) + 255) / 256, n_sol);
        if (tw && !(intra & 1u) && warp_tw)
            k_intra_tw_batch<DT><<<dim3((max_qp + 7) / 8, 3, n_sol), 256, 0, st>>>(views, sp, intra, keys);
        else if (tw) k_intra_batch<DT, true><<<g, 256, 0, st>>>(views, sp, intra, keys);
        else    k_intra_batch<DT, false><<<g, 256, 0, st>>>(views, sp, intra, keys);
        ++g_launches;
        e = cudaGetLastError();
    }
    return e;
}
template cudaError_t launch_batch<int32_t>(uint32_t, bool, const SolView<int32_t> *, const CUtensorMap *,
                                           const uint32_t *, int, int, int, const ScoreParams &, uint64_t *, int,
                                           cudaStream_t, bool);
template cudaError_t launch_batch<float>(uint32_t, bool, const SolView<float> *, const CUtensorMap *,
                                         const uint32_t *, int, int, int, const ScoreParams &, uint64_t *, int,
                                         cudaStream_t, bool);

// explicit instantiations
template cudaError_t launch_dp<int32_t>(int32_t *, int, const int32_t *, const int32_t *, int, int, int, int, bool,
                                        cudaStream_t);
template cudaError_t launch_dp<float>(float *, int, const int32_t *, const float *, int, int, int, int, bool,
                                      cudaStream_t);
template cudaError_t launch_scan<int32_t>(const ScanArgs<int32_t> &, bool, int, int, cudaStream_t);
template cudaError_t launch_scan<float>(const ScanArgs<float> &, bool, int, int, cudaStream_t);
template cudaError_t launch_inter<int32_t>(uint32_t, bool, const SolView<int32_t> &, const CUtensorMap &,
                                           const uint32_t *, int, int, const ScoreParams &, uint64_t *, int,
                                           cudaStream_t);
template cudaError_t launch_inter<float>(uint32_t, bool, const SolView<float> &, const CUtensorMap &, const uint32_t *,
                                         int, int, const ScoreParams &, uint64_t *, int, cudaStream_t);
template cudaError_t launch_intra<int32_t>(uint32_t, bool, const SolView<int32_t> &, const ScoreParams &, int, int,
                                           uint64_t *, cudaStream_t, bool, bool);
template cudaError_t launch_intra<float>(uint32_t, bool, const SolView<float> &, const ScoreParams &, int, int,
                                         uint64_t *, cudaStream_t, bool, bool);

}  // namespace tga
