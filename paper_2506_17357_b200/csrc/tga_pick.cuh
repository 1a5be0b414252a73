// tga_device_step.cu -- device-resident best-improvement step (
// Alg. A2 lines 5-8; the "Update" step of §5.3.5, without a
// GPU-CPU round trip -- the paper's observed bottleneck).
//
//   pick_apply_body  one CTA per solution: candidate counts of the evaluated
//                  neighbourhood (closed forms over route lengths), best key
//                  over the operator mask (lowest (score, variant, index)),
//                  decode, and -- if improving -- the splice of the 1-2 changed
//                  routes directly in the slot arrays (snapshot of the changed
//                  span, piece-wise remap), new route bases / lengths / canonical
//                  offsets, and a descriptor of the changed span.
//   (k_pick_update in tga_kernels.cu) Dp row/column refresh of the span + re-scan of its routes,
//                  bounds read from the descriptor (grid-stride; no host sync).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "tga_device.cuh"
#include "tga_launch.h"

namespace tga {

namespace pick {
// a piece of a new route: customers [start, start+len) of old route `src`
// (1-based positions), possibly reversed (2-opt)
struct Piece {
    int src, start, len, rev;
};
struct NewRoute {
    int r, L, np;
    Piece p[5];
};

__device__ __forceinline__ void add_piece(NewRoute &nr, int src, int a, int b, int rev = 0) {  // [a, b] inclusive
    if (b >= a) nr.p[nr.np++] = Piece{src, a, b - a + 1, rev};
}

__device__ __forceinline__ int find_route(const int32_t *cbase, int R, int c) {
    int lo = 0, hi = R - 1;  // largest r with cbase[r] <= c
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cbase[mid] <= c) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ int64_t pz(int64_t x) { return x > 0 ? x : 0; }
}  // namespace pick
using namespace pick;

// phase probe (diagnostics): clock64 of block 0 at phase k into acc[32 + k] when acc[31] != 0
__device__ __forceinline__ void probe(unsigned long long *pr, int k) {
    if (pr) pr[k] = static_cast<unsigned long long>(clock64());
}

// Exact candidate counts of the evaluated neighbourhood (closed forms over the
// route lengths sl[0..R-1] staged in shared memory), added to acc[0..22].
// Block-wide (every thread must call it).
__device__ __forceinline__ void neighbourhood_counts(const DevState &S, uint32_t mask, const int32_t *sl) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R = S.R;
    constexpr int NS = 27;
    __shared__ long long wsum[8][NS];
    __syncthreads();
    {
        long long loc[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) loc[k] = 0;
        for (int r = tid; r < R; r += blockDim.x) {
            const int64_t L = sl[r], X = L + 1;
            const int64_t x1 = pz(L), x2 = pz(L - 1), x3 = pz(L - 2);
            loc[0] += X;
            loc[1] += X * X;
            loc[2] += x1; loc[3] += x2; loc[4] += x3;
            loc[5] += x1 * X; loc[6] += x2 * X; loc[7] += x3 * X;
            loc[8] += x1 * x1; loc[9] += x1 * x2; loc[10] += x1 * x3;
            loc[11] += x2 * x2; loc[12] += x2 * x3; loc[13] += x3 * x3;
            loc[14] += L * (L - 1) / 2;
            loc[15] += x1 * pz(L - 1); loc[16] += x2 * pz(L - 2); loc[17] += x3 * pz(L - 3);
#pragma unroll
            for (int a = 1; a <= 3; ++a)
#pragma unroll
                for (int b = 1; b <= 3; ++b) {
                    const int64_t M = L - a - b + 1;
                    loc[18 + 3 * (a - 1) + (b - 1)] += M >= 1 ? M * (M + 1) / 2 : 0;
                }
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            long long v = loc[k];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0) wsum[warp][k] = v;
        }
    }
    __syncthreads();
    __shared__ long long sums[NS];
    if (tid < NS) {
        long long v = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) v += wsum[w][tid];
        sums[tid] = v;
    }
    __syncthreads();   // sums[] complete before any thread reads it (racecheck)
    if (tid < kNV && (mask & (1u << tid))) {  // one variant per thread
        const long long S1 = sums[0], S2 = sums[1];
        const int v0 = tid;
        // reversed-segment variants: the candidate spaces of or-opt N and cross (N, N)
        const int v = v0 == 23 ? 3 : (v0 == 24 ? 4 : (v0 == 25 ? 8 : (v0 == 26 ? 10 : v0)));
        long long c;
        if (v == 0) c = sums[14];
        else if (v == 1) c = (S1 * S1 - S2) / 2;
        else if (v <= 4) c = sums[v] * S1 - sums[v + 3];
        else if (v <= 10) {
            const int n1s[6] = {1, 1, 1, 2, 2, 3}, n2s[6] = {1, 2, 3, 2, 3, 3}, pidx[6] = {8, 9, 10, 11, 12, 13};
            const int k = v - 5;
            const long long ordered = sums[1 + n1s[k]] * sums[1 + n2s[k]] - sums[pidx[k]];
            c = (n1s[k] == n2s[k]) ? ordered / 2 : ordered;
        } else if (v <= 13) c = sums[v + 4];
        else c = sums[v + 4];
        atomicAdd(S.acc + v0, static_cast<unsigned long long>(c));  // fire-and-forget (RED)
    }
}


// ------------------------------------------------------------------ redundant decode
// The best move decoded by one warp of EVERY block of the multi-block step (no
// barrier before the update work): lowest (score, variant) over the evaluated
// keys (Eq. 16c, reading 5), improving iff score < 0, the 1-2 new routes as
// pieces of old routes.  sb / sl = old route bases / lengths in shared memory.
struct Decoded {
    int applied, full, nrt;  // move applied?  changed route outgrew its slots?  #routes changed
    NewRoute nr[2];          // nr[0] = lower route index
    int lo[2], hi[2];        // old (== new) slot ranges of the changed routes
    int plo[2];              // first slots of the prefetched windows (routes of u and of v)
};

// lane 0 of the decode: the 1-2 new routes of variant v at (ra, pa), (rb, pb) as pieces
// of old routes, their slot ranges and whether they still fit
__device__ __forceinline__ void decode_pieces(const int32_t *sb, const int32_t *sl, int ra, int rb, int pa, int pb,
                                              int v, Decoded &dm) {
    const int La = sl[ra], Lb = sl[rb];
    const bool one = v == 0 || (v >= 11 && v < 23);
    // pieces with static indices (empty pieces have len 0 and are skipped by the walk)
    Piece A0{}, A1{}, A2{}, A3{}, A4{}, B0{}, B1{}, B2{};
    int na = 0, nb = 0;
    auto pc = [](int src, int a, int b, int rev = 0) { return Piece{src, a, b >= a ? b - a + 1 : 0, rev}; };
    if (v == 1) {  // 2-opt*
        A0 = pc(ra, 1, pa); A1 = pc(rb, pb + 1, Lb); na = 2;
        B0 = pc(rb, 1, pb); B1 = pc(ra, pa + 1, La); nb = 2;
    } else if (v >= 2 && v <= 4) {  // relocate / or-opt
        const int N = v - 1;
        A0 = pc(ra, 1, pa - 1); A1 = pc(ra, pa + N, La); na = 2;
        B0 = pc(rb, 1, pb); B1 = pc(ra, pa, pa + N - 1); B2 = pc(rb, pb + 1, Lb); nb = 3;
    } else if (v >= 5 && v <= 10) {  // swap / cross: (N1, N2) = (1,1) (1,2) (1,3) (2,2) (2,3) (3,3)
        const int q = v - 5;
        const int N1 = q < 3 ? 1 : (q < 5 ? 2 : 3), N2 = q < 3 ? q + 1 : (q < 5 ? q - 1 : 3);
        A0 = pc(ra, 1, pa - 1); A1 = pc(rb, pb, pb + N2 - 1); A2 = pc(ra, pa + N1, La); na = 3;
        B0 = pc(rb, 1, pb - 1); B1 = pc(ra, pa, pa + N1 - 1); B2 = pc(rb, pb + N2, Lb); nb = 3;
    } else if (v == 0) {  // 2-opt
        A0 = pc(ra, 1, pa - 1); A1 = pc(ra, pa, pb, 1); A2 = pc(ra, pb + 1, La); na = 3;
    } else if (v == 23 || v == 24) {  // or-opt, the segment inserted reversed
        const int N = v - 21;
        A0 = pc(ra, 1, pa - 1); A1 = pc(ra, pa + N, La); na = 2;
        B0 = pc(rb, 1, pb); B1 = pc(ra, pa, pa + N - 1, 1); B2 = pc(rb, pb + 1, Lb); nb = 3;
    } else if (v == 25 || v == 26) {  // cross (N, N), both segments reversed
        const int N = v - 23;
        A0 = pc(ra, 1, pa - 1); A1 = pc(rb, pb, pb + N - 1, 1); A2 = pc(ra, pa + N, La); na = 3;
        B0 = pc(rb, 1, pb - 1); B1 = pc(ra, pa, pa + N - 1, 1); B2 = pc(rb, pb + N, Lb); nb = 3;
    } else if (v >= 11 && v <= 13) {  // intra relocate
        const int N = v - 10;
        if (pb > pa) {
            A0 = pc(ra, 1, pa - 1); A1 = pc(ra, pa + N, pb); A2 = pc(ra, pa, pa + N - 1); A3 = pc(ra, pb + 1, La);
        } else {
            A0 = pc(ra, 1, pb); A1 = pc(ra, pa, pa + N - 1); A2 = pc(ra, pb + 1, pa - 1); A3 = pc(ra, pa + N, La);
        }
        na = 4;
    } else {  // intra swap
        const int N1 = (v - 14) / 3 + 1, N2 = (v - 14) % 3 + 1;
        A0 = pc(ra, 1, pa - 1); A1 = pc(ra, pb, pb + N2 - 1); A2 = pc(ra, pa + N1, pb - 1);
        A3 = pc(ra, pa, pa + N1 - 1); A4 = pc(ra, pb + N2, La); na = 5;
    }
    const int LA = A0.len + A1.len + A2.len + A3.len + A4.len, LB = B0.len + B1.len + B2.len;
    const int ia = (one || ra < rb) ? 0 : 1;  // nr[0] = lower route of the span
    NewRoute &A = dm.nr[ia];
    A.r = ra; A.L = LA; A.np = na;
    A.p[0] = A0; A.p[1] = A1; A.p[2] = A2; A.p[3] = A3; A.p[4] = A4;
    bool fits = LA + 2 <= sb[ra + 1] - sb[ra];
    dm.lo[ia] = sb[ra];
    dm.hi[ia] = sb[ra + 1];
    if (!one) {
        NewRoute &B = dm.nr[ia ^ 1];
        B.r = rb; B.L = LB; B.np = nb;
        B.p[0] = B0; B.p[1] = B1; B.p[2] = B2;
        fits = fits && LB + 2 <= sb[rb + 1] - sb[rb];
        dm.lo[ia ^ 1] = sb[rb];
        dm.hi[ia ^ 1] = sb[rb + 1];
    } else {
        dm.lo[1] = dm.hi[1] = 0;
    }
    dm.nrt = one ? 1 : 2;
    dm.full = fits ? 0 : 1;
    dm.applied = 1;
}

// snap / node / pwin (optional): the old node ids of the first pwin slots of the (up to) two
// changed routes are loaded by the whole warp as soon as the routes are known -- in flight
// while lane 0 builds the pieces -- and left in snap[0 .. pwin) / snap[pwin .. 2 pwin)
// (slots below nlim, the length of node).
__device__ __forceinline__ void decode_best(const uint64_t *__restrict__ keys, uint32_t mask, int integer,
                                            const int32_t *sb, const int32_t *sl, int R, int Qc, Decoded &dm,
                                            int32_t *snap = nullptr, const int32_t *node = nullptr, int pwin = 0,
                                            int nlim = 0) {
    const int lane = threadIdx.x & 31;
    const uint64_t k = (lane < kNV && ((mask >> lane) & 1u)) ? keys[lane] : ~0ull;
    const bool valid = k != ~0ull;
    const uint32_t hi = valid ? static_cast<uint32_t>(k >> 32) : 0xFFFFFFFFu;
    const uint32_t mhi = __reduce_min_sync(0xFFFFFFFFu, hi);
    const uint32_t win = __ballot_sync(0xFFFFFFFFu, valid && hi == mhi);
    bool improving = false;
    if (win) {
        if (integer) {
            improving = mhi < 0x80000000u;  // int32 score < 0
        } else {
            const uint32_t u = (mhi & 0x80000000u) ? (mhi ^ 0x80000000u) : ~mhi;
            improving = __uint_as_float(u) < 0.0f;
        }
    }
    if (!improving) {
        if (lane == 0) dm.applied = 0;
        return;
    }
    const int v = __ffs(win) - 1;  // lowest variant among the lowest scores (reading 5)
    const uint32_t idx = static_cast<uint32_t>(__shfl_sync(0xFFFFFFFFu, k, v) & 0xFFFFFFFFu);
    // lanes 0 / 1 locate the u / v slot (physical) in parallel: largest r with sb[r] <= x
    const int x = lane == 0 ? static_cast<int>(idx / static_cast<uint32_t>(Qc)) : static_cast<int>(idx % static_cast<uint32_t>(Qc));
    int ra_ = 0;
    if (lane < 2) {
        int a = 0, b = R - 1;
        while (a < b) {
            const int m = (a + b + 1) >> 1;
            if (sb[m] <= x) a = m;
            else b = m - 1;
        }
        ra_ = a;
    }
    const int ra = __shfl_sync(0xFFFFFFFFu, ra_, 0), rb = __shfl_sync(0xFFFFFFFFu, ra_, 1);
    const int pa = __shfl_sync(0xFFFFFFFFu, x, 0) - sb[ra], pb = __shfl_sync(0xFFFFFFFFu, x, 1) - sb[rb];
    constexpr int kPre = 4;   // slots per lane and route: windows of up to 128 slots
    int32_t pre[2][kPre];
    if (snap) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            // the whole window, across route ends: every old slot in it is then served
            // from the snapshot, whichever route (of the two) it belongs to
            const int lo = sb[q ? rb : ra];
#pragma unroll
            for (int k = 0; k < kPre; ++k) {
                const int o = k * 32 + lane;
                pre[q][k] = (o < pwin && lo + o < nlim) ? node[lo + o] : 0;
            }
        }
    }
    if (lane == 0) {
        dm.plo[0] = sb[ra];
        dm.plo[1] = sb[rb];
        decode_pieces(sb, sl, ra, rb, pa, pb, v, dm);
    }
    if (snap) {   // the loads were in flight during the piece building above
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int k = 0; k < kPre; ++k) {
                const int o = k * 32 + lane;
                if (o < pwin) snap[q * pwin + o] = pre[q][k];
            }
    }
}

// ------------------------------------------------------------------ pick + apply
// Route arrays (base, length, canonical base) are staged in shared memory so the
// serial parts (decode, binary searches over routes) never wait on global loads.

__device__ __forceinline__ void pick_apply_body(const DevState &S, uint32_t mask, uint32_t cmask, int integer,
                                                int32_t *smr, unsigned long long *pr, bool do_counts = true) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R = S.R;
    int32_t *sb = smr, *sl = smr + (R + 1), *nb = smr + 2 * (R + 1);  // old bases, old lengths, new bases
    for (int r = tid; r <= R; r += blockDim.x) {
        sb[r] = S.rbase[r];
        sl[r] = r < R ? S.rlenR[r] : 0;
    }
    __shared__ uint64_t skeys[kNV];
    if (tid < kNV) skeys[tid] = S.keys[tid];
    if (do_counts) neighbourhood_counts(S, cmask, sl);
    __syncthreads();
    if (tid < kNV) S.keys[tid] = ~0ull;  // consumed (block 0 is the only reader): the next eval needs no memset
    if (tid == 0) probe(pr, 1);
    // ---- 2. best key over the mask, decode, pieces of the new routes
    __shared__ NewRoute nr[2];
    __shared__ int sh_n, sh_rlo, sh_rhi, sh_lo, sh_hi, sh_d, sh_applied;
    if (tid == 0) {
        int bv = -1;
        uint64_t bk = ~0ull;
        for (int v = 0; v < kNV; ++v) {
            if (!(mask & (1u << v))) continue;
            const uint64_t k = skeys[v];
            if (k == ~0ull) continue;
            if (bv < 0 || (k >> 32) < (bk >> 32)) { bv = v; bk = k; }
        }
        bool improving = false;
        if (bv >= 0) {
            const uint32_t ord = static_cast<uint32_t>(bk >> 32);
            if (integer) {
                improving = ord < 0x80000000u;  // int32 score < 0
            } else {
                const uint32_t u = (ord & 0x80000000u) ? (ord ^ 0x80000000u) : ~ord;
                improving = __uint_as_float(u) < 0.0f;
            }
        }
        sh_applied = 0;
        if (improving) {
            const uint32_t idx = static_cast<uint32_t>(bk & 0xFFFFFFFFu);
            const int xu = static_cast<int>(idx / static_cast<uint32_t>(S.Qc));  // physical slots
            const int xv = static_cast<int>(idx % static_cast<uint32_t>(S.Qc));
            // physical slot -> (route, position) from the staged bases (no global round trip)
            auto rp = [&](int x, int &r, int &p) {
                int a = 0, b = R - 1;
                while (a < b) {
                    const int m = (a + b + 1) >> 1;
                    if (sb[m] <= x) a = m;
                    else b = m - 1;
                }
                r = a;
                p = x - sb[a];
            };
            int ra, pa, rb, pb;
            rp(xu, ra, pa);
            rp(xv, rb, pb);
            const int La = sl[ra], Lb = sl[rb];
            const int v = bv;
            NewRoute A{ra, 0, 0, {}}, B{rb, 0, 0, {}};
            int nroutes = 2;
            if (v == 1) {  // 2-opt*
                add_piece(A, ra, 1, pa); add_piece(A, rb, pb + 1, Lb);
                add_piece(B, rb, 1, pb); add_piece(B, ra, pa + 1, La);
            } else if (v >= 2 && v <= 4) {  // relocate / or-opt
                const int N = v - 1;
                add_piece(A, ra, 1, pa - 1); add_piece(A, ra, pa + N, La);
                add_piece(B, rb, 1, pb); add_piece(B, ra, pa, pa + N - 1); add_piece(B, rb, pb + 1, Lb);
            } else if (v >= 5 && v <= 10) {  // swap / cross
                const int n1s[6] = {1, 1, 1, 2, 2, 3}, n2s[6] = {1, 2, 3, 2, 3, 3};
                const int N1 = n1s[v - 5], N2 = n2s[v - 5];
                add_piece(A, ra, 1, pa - 1); add_piece(A, rb, pb, pb + N2 - 1); add_piece(A, ra, pa + N1, La);
                add_piece(B, rb, 1, pb - 1); add_piece(B, ra, pa, pa + N1 - 1); add_piece(B, rb, pb + N2, Lb);
            } else if (v == 0) {  // 2-opt
                nroutes = 1;
                add_piece(A, ra, 1, pa - 1); add_piece(A, ra, pa, pb, 1); add_piece(A, ra, pb + 1, La);
            } else if (v == 23 || v == 24) {  // or-opt, the segment inserted reversed
                const int N = v - 21;
                add_piece(A, ra, 1, pa - 1); add_piece(A, ra, pa + N, La);
                add_piece(B, rb, 1, pb); add_piece(B, ra, pa, pa + N - 1, 1); add_piece(B, rb, pb + 1, Lb);
            } else if (v == 25 || v == 26) {  // cross (N, N), both segments reversed
                const int N = v - 23;
                add_piece(A, ra, 1, pa - 1); add_piece(A, rb, pb, pb + N - 1, 1); add_piece(A, ra, pa + N, La);
                add_piece(B, rb, 1, pb - 1); add_piece(B, ra, pa, pa + N - 1, 1); add_piece(B, rb, pb + N, Lb);
            } else if (v >= 11 && v <= 13) {  // intra relocate
                nroutes = 1;
                const int N = v - 10;
                if (pb > pa) {
                    add_piece(A, ra, 1, pa - 1); add_piece(A, ra, pa + N, pb);
                    add_piece(A, ra, pa, pa + N - 1); add_piece(A, ra, pb + 1, La);
                } else {
                    add_piece(A, ra, 1, pb); add_piece(A, ra, pa, pa + N - 1);
                    add_piece(A, ra, pb + 1, pa - 1); add_piece(A, ra, pa + N, La);
                }
            } else {  // intra swap
                nroutes = 1;
                const int N1 = (v - 14) / 3 + 1, N2 = (v - 14) % 3 + 1;
                add_piece(A, ra, 1, pa - 1); add_piece(A, ra, pb, pb + N2 - 1); add_piece(A, ra, pa + N1, pb - 1);
                add_piece(A, ra, pa, pa + N1 - 1); add_piece(A, ra, pb + N2, La);
            }
            for (int k = 0; k < A.np; ++k) A.L += A.p[k].len;
            for (int k = 0; k < B.np; ++k) B.L += B.p[k].len;
            if (nroutes == 1 || ra < rb) { nr[0] = A; nr[1] = B; }  // nr[0] = lower route of the span
            else { nr[0] = B; nr[1] = A; }
            sh_n = nroutes;
            sh_rlo = nr[0].r;
            sh_rhi = nroutes == 2 ? nr[1].r : nr[0].r;
            // do the changed routes still fit in their slot capacity?
            bool fits = nr[0].L + 2 <= sb[nr[0].r + 1] - sb[nr[0].r];
            if (nroutes == 2) fits = fits && (nr[1].L + 2 <= sb[nr[1].r + 1] - sb[nr[1].r]);
            sh_d = fits ? 0 : 1;  // 1 = full relayout
            sh_applied = 1;
        }
    }
    __syncthreads();
    if (tid == 0) probe(pr, 2);
    if (!sh_applied) {
        if (tid == 0) S.desc[0] = 0;
        return;  // uniform across the block
    }
    const int rlo = sh_rlo, rhi = sh_rhi, full = sh_d, nrt = sh_n;
    auto nlen = [&](int r) { return r == nr[0].r ? nr[0].L : (nrt == 2 && r == nr[1].r ? nr[1].L : sl[r]); };
    auto changed = [&](int r) -> const NewRoute * {
        return r == nr[0].r ? &nr[0] : ((nrt == 2 && r == nr[1].r) ? &nr[1] : nullptr);
    };
    // node id of new slot p (1..L) of route r: through its pieces, or unchanged
    auto old_slot = [&](int r, int p) {
        const NewRoute *chg = changed(r);
        if (!chg) return sb[r] + p;
        int off = p - 1, k = 0;
        while (off >= chg->p[k].len) { off -= chg->p[k].len; ++k; }
        const Piece &pc = chg->p[k];
        return sb[pc.src] + (pc.rev ? pc.start + pc.len - 1 - off : pc.start + off);
    };
    // old node id of an old slot: from the shared snapshot of the changed routes
    // (fits case) or the global snapshot of the whole layout (relayout)
    __shared__ int snap_off[2], snap_base[2], snap_n;
    extern __shared__ int32_t smr_all[];
    int32_t *snap = smr_all + 3 * (R + 1);  // after sb, sl, nb
    auto old_node = [&](int os) -> int32_t {
        if (full) return S.scratch[os];
        for (int k = 0; k < snap_n; ++k) {
            const int rel = os - snap_base[k];
            if (rel >= 0 && rel < (k + 1 < snap_n ? snap_off[k + 1] : 1 << 30) - snap_off[k]) return snap[snap_off[k] + rel];
        }
        return 0;
    };
    auto write_slot = [&](int x, int r, int p, int L, int span_lo) {
        (void)span_lo;
        if (p <= L + 1) {
            S.node[x] = (p >= 1 && p <= L) ? old_node(old_slot(r, p)) : 0;
            if (S.slot_of && p >= 1 && p <= L) S.slot_of[S.node[x]] = x;
            S.route[x] = r;
            S.pos[x] = p;
            S.rlen[x] = L;
            S.canon[x] = p <= L ? x : -1;  // validity only (keys index physical slots)
        } else {  // spare slot
            S.node[x] = 0;
            S.route[x] = -1;
            S.pos[x] = 0;
            S.rlen[x] = -1;
            S.canon[x] = -1;
        }
    };
    if (!full) {
        // ---- 3. snapshot the changed routes' old node ids in shared memory, rewrite just them
        if (tid == 0) {
            snap_n = nrt;
            snap_off[0] = 0;
            snap_base[0] = sb[nr[0].r];
            if (nrt == 2) { snap_off[1] = sb[nr[0].r + 1] - sb[nr[0].r]; snap_base[1] = sb[nr[1].r]; }
        }
        __syncthreads();
        for (int k = 0; k < nrt; ++k) {
            const int r = nr[k].r;
            for (int x = sb[r] + tid; x < sb[r + 1]; x += blockDim.x) snap[snap_off[k] + x - sb[r]] = S.node[x];
        }
        __syncthreads();
        const int span_lo = 0;
        for (int k = 0; k < nrt; ++k) {
            const int r = nr[k].r, L = nr[k].L;
            for (int x = sb[r] + tid; x < sb[r + 1]; x += blockDim.x) write_slot(x, r, x - sb[r], L, span_lo);
        }
        if (tid < nrt) S.rlenR[nr[tid].r] = nr[tid].L;
        if (tid == 0) {
            S.desc[1] = sb[rlo]; S.desc[2] = sb[rlo + 1];
            S.desc[3] = nrt == 2 ? sb[rhi] : 0; S.desc[4] = nrt == 2 ? sb[rhi + 1] : 0;
            S.desc[5] = rlo; S.desc[6] = nrt == 2 ? rhi : -1; S.desc[7] = 0;
        }
    } else {
        // ---- a changed route outgrew its slots: full relayout with fresh spare slots
        if (tid == 0) {
            int b = 0;
            for (int r = 0; r < R; ++r) { nb[r] = b; b += nlen(r) + 2 + S.slack; }
            nb[R] = b;  // == Qp
        }
        for (int x = tid; x < S.Qp; x += blockDim.x) S.scratch[x] = S.node[x];
        __syncthreads();
        for (int x = tid; x < S.Qp; x += blockDim.x) {
            int a = 0, b = R - 1;  // largest r with nb[r] <= x
            while (a < b) {
                const int m = (a + b + 1) >> 1;
                if (nb[m] <= x) a = m;
                else b = m - 1;
            }
            write_slot(x, a, x - nb[a], nlen(a), 0);
        }
        __syncthreads();
        for (int r = tid; r <= R; r += blockDim.x) {
            if (r < R) S.rlenR[r] = nlen(r);
            S.rbase[r] = nb[r];
        }
        if (tid == 0) {
            S.desc[1] = 0; S.desc[2] = S.Qp; S.desc[3] = 0; S.desc[4] = 0;
            S.desc[5] = -1; S.desc[6] = -1; S.desc[7] = 1;
        }
    }
    if (tid == 0) {
        S.desc[0] = 1;
        atomicAdd(S.acc + kAccApplied, 1ull);
        probe(pr, 3);
    }
}

}  // namespace tga
