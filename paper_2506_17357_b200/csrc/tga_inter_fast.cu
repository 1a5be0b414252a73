// tga_inter_fast.cu -- fused inter-route sweep, CVRP feasible-only fast path (sm_100a).
//
// Same candidate space, scores and keys as k_inter (Fig. `operators`
// P:107-149; Eq. 2 / 3f; Eq. 16), organised for instruction economy:
//   * tile = U rows (u) x 128 columns (v); a CTA of 4 warps, lane <-> column;
//     the warp walks its U rows in canonical order, so a plain strict '<' on a
//     32-bit score keeps the lowest canonical index per (variant, direction)
//     stream (reading 5) -- no 64-bit key per candidate;
//   * the Dp box (rows u0-1..u0+U+2, cols v0-4..v0+131) is one TMA tile load,
//     the U+4 row records one bulk copy, both double-buffered across the
//     persistent tile loop on mbarriers;
//   * every row-only or column-only term (removal gains, segment loads, route
//     loads, validity) is precomputed in the 80-byte SlotRec; validity is a
//     poisoned load, so each candidate is: a few adds, one capacity compare,
//     one select and one compare-and-keep.
#include <cuda.h>
#include <cuda_runtime.h>
#include <climits>
#include <cstdlib>
#include <cstdint>

#include "tga_device.cuh"
#include "tga_launch.h"
#include "tga_tma.cuh"

namespace tga {

// diagnostics (TGA_INTER_PROBE=1): per-CTA %globaltimer stamps, 8 per CTA:
// 0 start, 1 intra done, 2 first tile data arrived, 3 tiles done, 4 end
__device__ unsigned long long g_inter_probe[8 * 4096];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

namespace {
// running best of one (variant, direction) stream inside a tile, packed in 32
// bits: (score + 2^25) << 5 | row-in-tile.  The score of the integer fast path
// is bounded by 8 * max c < 2^25 (host-checked: fast_ok), rows are < 32, so an
// unsigned min keeps the lowest score and, among equal scores, the lowest row --
// the lowest canonical index, since the column is fixed per lane (reading 5).
// An infeasible candidate maps to 0xFFFFFFFF and never wins.
// mul32 is 32 held in an opaque register: the pack is then one IMAD (fma pipe) instead
// of a LEA on the alu pipe, which the integer-heavy tile body saturates first (both
// pipes issue every 2 cycles per SMSP, B300_MICROARCH "Pipe rates").
__device__ __forceinline__ void keep(uint32_t &b, bool feas, int32_t dD, int row, uint32_t mul32) {
    const uint32_t k = static_cast<uint32_t>(dD) * mul32 + static_cast<uint32_t>((1 << 30) + row);
    b = min(b, feas ? k : 0xFFFFFFFFu);
}
__device__ __forceinline__ void fold(uint64_t &acc, uint32_t b, bool direct, int u0, uint32_t v, uint32_t Qc) {
    if (b != 0xFFFFFFFFu) {
        const int32_t s = static_cast<int32_t>(b >> 5) - (1 << 25);
        const uint32_t u = static_cast<uint32_t>(u0) + (b & 31u);
        const uint32_t idx = direct ? u * Qc + v : v * Qc + u;
        acc = umin64(acc, pack_key(ord_score(s), idx));
    }
}
}  // namespace

// The candidate streams of one (row u, column v) cell with route(u) < route(v)
// (stream slots above): D(di, dj) = Dp(u + di, v + dj); put(slot, ok, score)
// receives every candidate.  Feasible-only (PEN = false): ok = feasibility
// (capacity, and time windows in the T_V = 0 form of SlotTW), score = the
// distance delta dD (Eq. 2, 13, 14).  Penalised (PEN, CVRP; records with the old
// excess folded in, see SlotRec): ok = the candidate is structurally valid (no
// poisoned load), score = dD + w_Q (max(L_a' - Q, 0) + max(L_b' - Q, 0)) - w_Q
// (ex_a + ex_b) = dD + w_Q dL_V (Eq. 16a, reading 4).
template <bool TW, bool PEN, uint32_t MASK, class DF, class PF>
__device__ __forceinline__ void cell_streams(const SlotRec &A, const SlotRec &V, const SlotTW &AT, const SlotTW &VT,
                                             int32_t cap, int32_t wQ, DF D, PF put) {
    static_assert(!(TW && PEN), "penalised fast path: CVRP only");
    constexpr int32_t kValid = kPoison / 2;   // any poisoned load exceeds it
    // penalty of the two new route loads
    auto pen = [&](int32_t la, int32_t lb) -> int32_t { return wQ * (max(la - cap, 0) + max(lb - cap, 0)); };
    // time-window check of  F + seg + B  (Eq. 4 in the T_V = 0 form of SlotTW):
    // start after ef + t1 <= seg latest start, completion + t2 <= suffix latest start
    auto tw3 = [&](float ef, int32_t t1, float sTE, float sTL, float sTD, int32_t t2, float lb) -> bool {
        const float x = ef + static_cast<float>(t1);
        return (x <= sTL) & (fmaxf(x, sTE) + sTD + static_cast<float>(t2) <= lb);
    };
    // ---- 2-opt*: A' = F(u) + B(v+1), B' = F(v) + B(u+1)    (Eq. 14)
    if (MASK & (1u << 1)) {
        const int32_t d01 = D(0, 1), d10 = D(1, 0);
        const int32_t dD = d01 + d10 + A.ne + V.ne;
        const int32_t la = A.fL + V.bL1, lb = V.fL + A.bL1;
        if (PEN) {
            put(0, max(la, lb) < kValid, dD + pen(la, lb));
        } else {
            bool ok = max(la, lb) <= cap;
            if (TW) ok = ok & (AT.EF + static_cast<float>(d01) <= VT.LBN[0]) &
                         (VT.EF + static_cast<float>(d10) <= AT.LBN[0]);
            put(0, ok, dD);
        }
    }
    // ---- relocate / or-opt, both directions                   (Eq. 13)
#pragma unroll
    for (int N = 1; N <= 3; ++N) {
        if (!(MASK & (1u << (1 + N)))) continue;
        const int32_t d00 = D(0, 0), dN1 = D(N - 1, 1), d1N = D(1, N - 1);
        const int32_t d1 = A.rem[N - 1] + d00 + dN1 + V.ne;  // seg(u) after v
        const int32_t d2 = V.rem[N - 1] + d00 + d1N + A.ne;  // seg(v) after u
        if (PEN) {
            const int32_t lb1 = V.W + A.so[N - 1], lb2 = A.W + V.so[N - 1];
            put(2 * N - 1, lb1 < kValid, d1 + pen(A.W - A.so[N - 1], lb1));
            put(2 * N, lb2 < kValid, d2 + pen(lb2, V.W - V.so[N - 1]));
        } else {
            bool ok1 = V.W + A.so[N - 1] <= cap;
            if (TW) ok1 = ok1 & tw3(VT.EF, d00, AT.sTE[N - 1], AT.sTL[N - 1], AT.sTD[N - 1], dN1, VT.LBN[0]);
            put(2 * N - 1, ok1, d1);
            bool ok2 = A.W + V.so[N - 1] <= cap;
            if (TW) ok2 = ok2 & tw3(AT.EF, d00, VT.sTE[N - 1], VT.sTL[N - 1], VT.sTD[N - 1], d1N, AT.LBN[0]);
            put(2 * N, ok2, d2);
        }
    }
    // ---- swap (1,1) / cross-exchange (N1,N2), N1 <= N2
#pragma unroll
    for (int sv = 0; sv < 6; ++sv) {
        constexpr int n1s[6] = {1, 1, 1, 2, 2, 3}, n2s[6] = {1, 2, 3, 2, 3, 3};
        constexpr int slot[6] = {7, 8, 10, 12, 13, 15};
        const int N1 = n1s[sv], N2 = n2s[sv];
        if (!(MASK & (1u << (5 + sv)))) continue;
        {   // N1-segment at u, N2-segment at v
            const int32_t a = D(-1, 0), bq = D(N1, N2 - 1), c = D(0, -1), dq = D(N1 - 1, N2);
            const int32_t dD = a + bq + c + dq + A.sE[N1 - 1] + V.sE[N2 - 1];
            const int32_t la = A.sA[N1 - 1] + V.sS[N2 - 1], lb = V.sA[N2 - 1] + A.sS[N1 - 1];
            if (PEN) {
                put(slot[sv], max(la, lb) < kValid, dD + pen(la, lb));
            } else {
                bool ok = max(la, lb) <= cap;
                if (TW)  // A' = F(u-1) + S(v,N2) + B(u+N1),  B' = F(v-1) + S(u,N1) + B(v+N2)
                    ok = ok & tw3(AT.EFm, a, VT.sTE[N2 - 1], VT.sTL[N2 - 1], VT.sTD[N2 - 1], bq, AT.LBN[N1 - 1]) &
                         tw3(VT.EFm, c, AT.sTE[N1 - 1], AT.sTL[N1 - 1], AT.sTD[N1 - 1], dq, VT.LBN[N2 - 1]);
                put(slot[sv], ok, dD);
            }
        }
        if (N1 != N2) {   // N1-segment at v, N2-segment at u
            const int32_t c = D(0, -1), bq = D(N2 - 1, N1), a = D(-1, 0), dq = D(N2, N1 - 1);
            const int32_t dD = c + bq + a + dq + V.sE[N1 - 1] + A.sE[N2 - 1];
            const int32_t lb = V.sA[N1 - 1] + A.sS[N2 - 1], la = A.sA[N2 - 1] + V.sS[N1 - 1];
            if (PEN) {
                put(slot[sv] + 1, max(la, lb) < kValid, dD + pen(la, lb));
            } else {
                bool ok = max(la, lb) <= cap;
                if (TW)  // B' = F(v-1) + S(u,N2) + B(v+N1),  A' = F(u-1) + S(v,N1) + B(u+N2)
                    ok = ok & tw3(VT.EFm, c, AT.sTE[N2 - 1], AT.sTL[N2 - 1], AT.sTD[N2 - 1], bq, VT.LBN[N1 - 1]) &
                         tw3(AT.EFm, a, VT.sTE[N1 - 1], VT.sTL[N1 - 1], VT.sTD[N1 - 1], dq, AT.LBN[N2 - 1]);
                put(slot[sv] + 1, ok, dD);
            }
        }
    }
}

#ifndef TGA_FAST_CTA_SYNC
#define TGA_FAST_CTA_SYNC 0   // 1: the former __syncthreads per tile before a stage is refilled
#endif

// The fast-path tile plan of one solution, decoded arithmetically (no plan table to
// load before the first TMA can be issued): tiles of U rows x kFastTV columns of the
// upper triangle, R = kFastTV / U row bands per column band.  Tiles t < nI are the
// diagonal tiles (row band I = t, column band I / R; the lightest, so one-tile-per-CTA
// launches put the intra-route units beside them), then the full tiles (I < R J)
// column by column: before column J lie R J (J - 1) / 2 of them.  fast_plan (host)
// lists the same order; tile (I, J) exists iff I U < Qp, J kFastTV < Qp and
// I U < J kFastTV + kFastTV - 1.
__host__ __device__ __forceinline__ void fast_tile_of(int t, int nI, int R, int &I, int &J) {
    if (t < nI) { I = t; J = t / R; return; }
    const int q = t - nI;
    int j = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(q) / static_cast<float>(R))) * 0.5f);
    while (j > 1 && R * j * (j - 1) / 2 > q) --j;
    while (R * (j + 1) * j / 2 <= q) ++j;
    J = j;
    I = q - R * j * (j - 1) / 2;
}

// one work item of the fused sweep: tile (I, J) of one solution
struct FastItem {
    const SlotRec *rec;
    const SlotTW *rectw;
    const CUtensorMap *map;
    uint64_t *keys;
    uint32_t Qc;
    int sol, I, J;
};

// Work items of one launch: w = w0, w0 + stride, ... < w1; item(w) describes it.
// One solution: the tiles of its plan, strided over the CTAs; a population batch:
// a contiguous run of (solution, tile) items per CTA, so the running minima are
// flushed into a solution's keys only when the run moves on to the next solution.
// stream slots: 0 2opt* | 1,2 reloc1 d/r | 3,4 oropt2 | 5,6 oropt3 | 7 swap11 |
// 8,9 cross12 | 10,11 cross13 | 12 cross22 | 13,14 cross23 | 15 cross33
// stream slot k -> (variant, direct): direct = the key index is u * Qc + v (the
// N1-segment / moved segment / cut is at the row slot u), else v * Qc + u
__device__ __forceinline__ int stream_variant(int k) {
    return k == 0 ? 1 : (k <= 6 ? 1 + (k + 1) / 2 : (k == 7 ? 5 : (k <= 9 ? 6 : (k <= 11 ? 7 : (k == 12 ? 8 : (k <= 14 ? 9 : 10))))));
}
__device__ __forceinline__ bool stream_direct(int k) {
    return (k == 0 || k == 7 || k == 12 || k == 15) ? true : (k <= 6 ? (k & 1) == 1 : (k == 8 || k == 10 || k == 13));
}

// SC (population batches): one column region shared by both stages (rows and box stay
// double-buffered) -- a lane reads its column record once per tile into registers, so the
// region is refilled, on its own mbarrier bar[2], only when the run moves to another
// (solution, column band), after every warp has read the last tile of the old one; the
// CTA's buffers shrink from 63 to 45 KB (time windows): 4 CTAs per SM instead of 3.
template <int U, bool TW, uint32_t MASK, bool DUMP, bool PEN, class ItemF, bool SC = false>
__device__ __forceinline__ void fast_body(ItemF item, int w0, int w1, int wstride, uint64_t *bar,
                                          unsigned long long (*red)[23], unsigned char *sm, int32_t cap,
                                          const SolView<int32_t> &SV, const ScoreParams &sp, uint32_t imask,
                                          int x_lo, int x_hi, int icta, int incta, int flags,
                                          uint64_t *keys0 = nullptr, unsigned long long *dump = nullptr) {
    using G = FastGeom<U, TW>;
    constexpr int BW = G::BoxW;
    constexpr int NV = 11;
    // stage b at sm + b * Stage: box | row records | column records | TW rows | TW columns
    // (SC: stage b at sm + b * StageSC: box | row records | TW rows; the columns after both)
    constexpr int StageSC = G::BoxPad + G::RowBytes + G::RowTW;
    constexpr int SB = SC ? StageSC : G::Stage;
    int32_t *const dp0 = reinterpret_cast<int32_t *>(sm);
    int32_t *const dp1 = reinterpret_cast<int32_t *>(sm + SB);
    SlotRec *const rows0 = reinterpret_cast<SlotRec *>(sm + G::BoxPad);
    SlotRec *const rows1 = reinterpret_cast<SlotRec *>(sm + SB + G::BoxPad);
    SlotRec *const cols0 = reinterpret_cast<SlotRec *>(SC ? sm + 2 * StageSC : sm + G::BoxPad + G::RowBytes);
    SlotRec *const cols1 = reinterpret_cast<SlotRec *>(SC ? sm + 2 * StageSC : sm + G::Stage + G::BoxPad + G::RowBytes);
    SlotTW *const trows0 = reinterpret_cast<SlotTW *>(sm + G::BoxPad + G::RowBytes + (SC ? 0 : G::ColBytes));
    SlotTW *const trows1 = reinterpret_cast<SlotTW *>(sm + SB + G::BoxPad + G::RowBytes + (SC ? 0 : G::ColBytes));
    SlotTW *const tcols0 = reinterpret_cast<SlotTW *>(SC ? sm + 2 * StageSC + G::ColBytes
                                                         : sm + G::BoxPad + G::RowBytes + G::ColBytes + G::RowTW);
    SlotTW *const tcols1 = reinterpret_cast<SlotTW *>(SC ? sm + 2 * StageSC + G::ColBytes
                                                         : sm + G::Stage + G::BoxPad + G::RowBytes + G::ColBytes + G::RowTW);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool prb = (flags & 2) && tid == 0 && blockIdx.x < 4096;

    uint64_t acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = kNoKey;

    // A stage keeps the column records of its last tile: when its next tile has the same
    // (solution, column band) -- consecutive items of a population run are ordered by column
    // band -- only the Dp box and the row records are copied (the column records are the
    // largest part of a tile's traffic).  s_colkey[b] is written by the one thread that
    // refills stage b, after every warp has released it.
    __shared__ int s_colkey[2];
    __shared__ int s_cout;   // SC: warps done with the column region's current content
    if (tid == 0) { s_colkey[0] = s_colkey[1] = -1; s_cout = 0; }
    __syncthreads();
    auto colkey = [](const FastItem &f) { return f.sol * 1024 + f.J; };
    auto issue_cols = [&](const FastItem &f) {   // SC: the shared column region, on bar[2]
        f_expect(&bar[2], G::ColBytes + G::ColTW);
        f_bulk(cols0, f.rec + f.J * kFastTV, G::ColBytes, &bar[2]);
        if (TW) f_bulk(tcols0, f.rectw + f.J * kFastTV, G::ColTW, &bar[2]);
    };
    auto issue = [&](const FastItem &f, int b) {
        uint64_t *br = b ? &bar[1] : &bar[0];
        const int key = f.sol * 1024 + f.J;
        const bool cols = !SC && s_colkey[b] != key;
        s_colkey[b] = key;   // before the arrive below publishes it to the stage's next refiller
        f_expect(br, G::BoxBytes + G::RowBytes + G::RowTW + (cols ? G::ColBytes + G::ColTW : 0));
        f_tma2d(b ? dp1 : dp0, f.map, f.J * kFastTV - 4, f.I * U - 1, br);
        f_bulk(b ? rows1 : rows0, f.rec + f.I * U, G::RowBytes, br);
        if (cols) f_bulk(b ? cols1 : cols0, f.rec + f.J * kFastTV, G::ColBytes, br);
        if (TW) {
            f_bulk(b ? trows1 : trows0, f.rectw + f.I * U, G::RowTW, br);
            if (cols) f_bulk(b ? tcols1 : tcols0, f.rectw + f.J * kFastTV, G::ColTW, br);
        }
    };
    // ---- fused argmin of the running minima: warp REDUX -> the warp's private shared
    // row -> one 64-bit atomicMin per variant per CTA into the solution's keys
    auto flush = [&](uint64_t *keys) {
#pragma unroll
        for (int i = 1; i < NV; ++i) {
            if (!(MASK & (1u << i))) continue;
            const uint64_t k = warp_min64(acc[i]);
            if (lane == 0 && k < red[warp][i]) red[warp][i] = k;
            acc[i] = kNoKey;
        }
        __syncthreads();
        if (tid < 23) {
            unsigned long long m = red[0][tid];
#pragma unroll
            for (int w = 1; w < kFastThreads / 32; ++w) m = m < red[w][tid] ? m : red[w][tid];
            if (m != kNoKey) atomicMin(reinterpret_cast<unsigned long long *>(keys) + tid, m);
        }
        __syncthreads();
        for (int i = tid; i < (kFastThreads / 32) * 23; i += kFastThreads) red[i / 23][i % 23] = kNoKey;
    };

    int w = w0;
    FastItem cur{};
    if (w < w1) cur = item(w);
#if TGA_FAST_CTA_SYNC
    if (tid == 0 && w < w1) issue(cur, 0);
#else
    // buffer release without a CTA barrier: each warp counts itself out of a stage when it has
    // read it; the last one out refills it with the tile two iterations ahead. Warps whose
    // columns skip more rows (route order, end depots) run up to one tile ahead instead of
    // waiting at a __syncthreads per tile.
    __shared__ int s_out[2];
    if (tid == 0) {
        s_out[0] = 0;
        s_out[1] = 0;
        if (SC && w < w1) issue_cols(cur);
        if (w < w1) issue(cur, 0);                              // arrive (release) publishes s_out
        if (w + wstride < w1) issue(item(w + wstride), 1);
    }
#endif
    // intra-route CVRP work of this launch (one u slot per warp) while the first
    // tile's TMA is in flight: the whole neighbourhood is one kernel
    if (imask) {
        const int n_units = (x_hi - x_lo + 3) / 4;
        for (int j = icta; j < n_units; j += incta) {
            const int x = x_lo + 4 * j + warp;
            if (x < x_hi)
                intra_cvrp_warp<DUMP>(SV, sp, imask, x, red[warp],
                                      ((flags & 2) && warp == 0 && j == icta && blockIdx.x < 4096) ? g_inter_probe + 8 * blockIdx.x + 4 : nullptr,
                                      dump);
        }
    }
    if (prb) g_inter_probe[8 * blockIdx.x + 1] = gtime();
    uint64_t *keys = w < w1 ? cur.keys : keys0;   // keys0: intra-only CTAs of one solution
    int sol = cur.sol;
    const uint32_t mul32 = static_cast<uint32_t>(flags >> 8);   // 32, a kernel parameter: keep() packs with IMAD
    uint32_t ph0 = 0u, ph1 = 0u, phc = 0u;
    int held = -1;   // SC: the (solution, column band) key the column region holds for this warp
    for (int it = 0; w < w1; w += wstride, ++it) {
        const int b = it & 1;
        const FastItem f = cur;
        if (w + wstride < w1) {
            cur = item(w + wstride);
#if TGA_FAST_CTA_SYNC
            if (tid == 0) issue(cur, b ^ 1);
#endif
        }
        if (f.sol != sol) {   // a batch run moved on to the next solution (CTA-uniform)
            flush(keys);
            keys = f.keys;
            sol = f.sol;
        }
        const uint32_t Qc = f.Qc;
        const int u0 = f.I * U, v0 = f.J * kFastTV;
        const int col = warp * 32 + lane;   // column inside the tile
        const int v = v0 + col;
        if (b) { f_wait(&bar[1], ph1); ph1 ^= 1u; } else { f_wait(&bar[0], ph0); ph0 ^= 1u; }
        if (prb && it == 0) g_inter_probe[8 * blockIdx.x + 2] = gtime();
        if (SC && colkey(f) != held) {   // warp-uniform: a new column epoch
            f_wait(&bar[2], phc);
            phc ^= 1u;
            held = colkey(f);
        }
        // ---- this lane's column record, bulk-copied with the tile (five 16-byte LDS)
        const SlotRec V = (b ? cols1 : cols0)[col];
        SlotTW VT{};
        if (TW) VT = (b ? tcols1 : tcols0)[col];
        if (SC && w + wstride < w1 && colkey(cur) != colkey(f)) {
            // the last tile of this column epoch: once every warp has its records in registers,
            // the last one out refills the region with the next epoch's columns
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&s_cout, 1) == kFastThreads / 32 - 1) {
                    s_cout = 0;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the copy
                    issue_cols(cur);
                }
            }
            __syncwarp();
        }
        const SlotTW *TR = b ? trows1 : trows0;
        (void)TR;
        const int32_t *T = b ? dp1 : dp0;
        const SlotRec *RW = b ? rows1 : rows0;
        // Dp(u0 + i + di, v + dj), i = row index in the tile
        auto D = [&](int i, int di, int dj) -> int32_t { return T[(i + 1 + di) * BW + (col + 4 + dj)]; };

        uint32_t run[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) run[k] = 0xFFFFFFFFu;

        // the body is large: fully unrolled over the 16 rows it overflows the instruction
        // cache (ncu: 38 % no_inst stalls in the TW batch kernel, 8 % at cfg4), so it is
        // unrolled by 4 rows with time windows, by 8 without (measured best: cfg4 inter
        // 365 -> 351 us at 8, 424 us at 4)
        constexpr int kRowUnroll = TW ? 4 : 8;
#pragma unroll kRowUnroll
        for (int i = 0; i < U; ++i) {
            const SlotRec &A = RW[i];       // row u = u0 + i (broadcast reads)
            const int32_t ru = A.r;
            const int u = u0 + i;            // physical row slot (key index = u * pitch + v)
            if (ru < 0) continue;            // warp-uniform: end depot / spare / padding row
            if (!(ru < V.r)) continue;       // pair must span two routes, route(u) < route(v)
            const SlotTW &AT = TR[TW ? i : 0];
            cell_streams<TW, PEN, MASK>(A, V, AT, VT, cap, sp.wQ, [&](int di, int dj) { return D(i, di, dj); },
                                   [&](int k, bool ok, int32_t dD) {
                                       keep(run[k], ok, dD, i, mul32);
                                       if constexpr (DUMP) {   // test-only: every candidate's key
                                           const uint32_t uu = static_cast<uint32_t>(u), vv = static_cast<uint32_t>(v);
                                           const uint32_t idx = stream_direct(k) ? uu * Qc + vv : vv * Qc + uu;
                                           dump_put(dump, Qc * Qc, stream_variant(k), idx,
                                                    ok ? pack_key(ord_score(dD), idx) : kNoKey);
                                       }
                                   });
        }
#if !TGA_FAST_CTA_SYNC
        // this warp is done with stage b (every shared read above has returned its value)
        __syncwarp();
        int last = 0;
        if (lane == 0) {
            __threadfence_block();
            last = atomicAdd(&s_out[b], 1) == kFastThreads / 32 - 1;
            if (last) {
                s_out[b] = 0;
                if (w + 2 * wstride < w1) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA writes
                    issue(item(w + 2 * wstride), b);
                }
            }
        }
        (void)last;
#endif
        // ---- fold this tile's streams into the per-variant 64-bit keys
        if (V.r >= 0) {
            const uint32_t cv = static_cast<uint32_t>(v);  // physical column slot
            if (MASK & (1u << 1)) fold(acc[1], run[0], true, u0, cv, Qc);
#pragma unroll
            for (int N = 1; N <= 3; ++N) {
                if (!(MASK & (1u << (1 + N)))) continue;
                fold(acc[1 + N], run[2 * N - 1], true, u0, cv, Qc);
                fold(acc[1 + N], run[2 * N], false, u0, cv, Qc);
            }
            if (MASK & (1u << 5)) fold(acc[5], run[7], true, u0, cv, Qc);
            if (MASK & (1u << 6)) { fold(acc[6], run[8], true, u0, cv, Qc); fold(acc[6], run[9], false, u0, cv, Qc); }
            if (MASK & (1u << 7)) { fold(acc[7], run[10], true, u0, cv, Qc); fold(acc[7], run[11], false, u0, cv, Qc); }
            if (MASK & (1u << 8)) fold(acc[8], run[12], true, u0, cv, Qc);
            if (MASK & (1u << 9)) { fold(acc[9], run[13], true, u0, cv, Qc); fold(acc[9], run[14], false, u0, cv, Qc); }
            if (MASK & (1u << 10)) fold(acc[10], run[15], true, u0, cv, Qc);
        }
#if TGA_FAST_CTA_SYNC
        __syncthreads();  // buffer b is refilled two iterations later
#endif
    }

    if (flags & 1) pdl_trigger();
    if (keys) flush(keys);
}


// The launch: CTAs [0, split) evaluate the variants of MASK over every tile,
// CTAs [split, grid) those of MASK2 (0 = none) -- the all-variant sweep is split
// in two halves of similar work so that small neighbourhoods get twice the CTAs
// (and each CTA half the registers' worth of running minima); the intra-route
// work rides with the second half.
template <int U, bool TW, uint32_t MASK, uint32_t MASK2, bool DUMP = false, bool PEN = false>
__global__ void __launch_bounds__(kFastThreads) k_inter_fast(const SlotRec *__restrict__ rec,
                                                             const SlotTW *__restrict__ rectw,
                                                             const __grid_constant__ CUtensorMap tmap,
                                                             const uint32_t *__restrict__ tiles, int t_lo, int t_hi,
                                                             uint32_t Qc, int32_t cap, uint64_t *__restrict__ keys,
                                                             const __grid_constant__ SolView<int32_t> SV,
                                                             ScoreParams sp, uint32_t imask, int x_lo, int x_hi,
                                                             int flags, int split, unsigned long long *dump) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (s_u32(smem_raw) & 127u)) & 127u);
    __shared__ uint64_t bar[2];
    __shared__ unsigned long long red[kFastThreads / 32][23];   // per-warp minima (no shared 64-bit atomics)
    const int tid = threadIdx.x;
    if ((flags & 2) && tid == 0 && blockIdx.x < 4096) g_inter_probe[8 * blockIdx.x] = gtime();
    if (tid == 0) {
        f_mbar_init(&bar[0]);
        f_mbar_init(&bar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < (kFastThreads / 32) * 23; i += kFastThreads) red[i / 23][i % 23] = kNoKey;
    if (!(flags & 1)) pdl_trigger();  // no inter-CTA waits here: a dependent grid may launch now
    __syncthreads();
    pdl_wait();                       // Dp / records / keys are written by the stream predecessors
    const int cta = static_cast<int>(blockIdx.x);
    const int nI = (SV.Qp + U - 1) / U;
    // a CTA's first tile is decoded arithmetically (no plan-table load before its first TMA);
    // later tiles of a persistent CTA come from the plan table (one load, issued a tile ahead:
    // the arithmetic decode costs every thread ~2 x 50 instructions per tile)
    const int first_wave = t_lo + static_cast<int>(gridDim.x);
    auto item = [&](int t) -> FastItem {
        int I, J;
        if (t < first_wave) {
            fast_tile_of(t, nI, kFastTV / U, I, J);
        } else {
            const uint32_t ij = __ldg(tiles + t);
            I = static_cast<int>(ij >> 16);
            J = static_cast<int>(ij & 0xFFFFu);
        }
        return FastItem{rec, rectw, &tmap, keys, Qc, 0, I, J};
    };
    if (MASK2 == 0 || cta < split) {
        const int n = MASK2 ? split : static_cast<int>(gridDim.x);
        fast_body<U, TW, MASK, DUMP, PEN>(item, t_lo + cta, t_hi, n, bar, red, sm, cap, SV, sp, MASK2 ? 0u : imask, x_lo,
                                     x_hi, cta, n, flags, keys, dump);
    } else {
        const int n = static_cast<int>(gridDim.x) - split;
        fast_body<U, TW, MASK2, DUMP, PEN>(item, t_lo + cta - split, t_hi, n, bar, red, sm, cap, SV, sp, imask, x_lo, x_hi,
                                      cta - split, n, flags, keys, dump);
    }
    if ((flags & 2) && tid == 0 && blockIdx.x < 4096) g_inter_probe[8 * blockIdx.x + 3] = gtime();
}

static bool inter_probe_on() {
    static const bool on = std::getenv("TGA_INTER_PROBE") != nullptr;
    return on;
}

// resident CTAs (whole GPU) of one instantiation with one / two pipeline stages
template <int U, bool TW, uint32_t MASK, uint32_t MASK2, bool PEN>
static void fast_capacity(int &res1, int &res2) {
    static PerDevice pd;
    static int r1[kMaxDevices], r2[kMaxDevices];
    const int d = once_per_device(pd, [](int dev) {
        auto kern = k_inter_fast<U, TW, MASK, MASK2, false, PEN>;
        using G = FastGeom<U, TW>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::Smem);
        int sms = 0, b1 = 0, b2 = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, kern, kFastThreads, G::Smem1);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, kern, kFastThreads, G::Smem);
        r1[dev] = std::max(1, b1) * std::max(1, sms);
        r2[dev] = std::max(1, b2) * std::max(1, sms);
    });
    res1 = r1[d];
    res2 = r2[d];
}

template <int U, bool TW, uint32_t MASK, uint32_t MASK2, bool PEN>
static cudaError_t launch_fast_t(const SlotRec *rec, const SlotTW *rectw, const CUtensorMap &map, const uint32_t *tiles,
                                 int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys, int units_max,
                                 cudaStream_t st, const SolView<int32_t> &SV, const ScoreParams &sp, uint32_t imask,
                                 int x_lo, int x_hi) {
    auto kern = k_inter_fast<U, TW, MASK, MASK2, false, PEN>;
    using G = FastGeom<U, TW>;
    // resident CTAs with one / two pipeline stages (a persistent grid never exceeds them)
    int res1 = 0, res2 = 0;
    fast_capacity<U, TW, MASK, MASK2, PEN>(res1, res2);
    const int groups = MASK2 ? 2 : 1;
    const int tiles_n = t_hi - t_lo;
    const int units = imask ? (x_hi - x_lo + 3) / 4 : 0;
    int per_group = std::max(tiles_n, MASK2 ? 0 : units);
    int smem = G::Smem1, grid;
    if (per_group * groups <= res1) {
        grid = std::max(1, per_group) * groups;   // one tile per CTA: a single stage
    } else {
        smem = G::Smem;
        grid = std::max(groups, std::min(per_group * groups, std::min(res2, units_max)));
    }
    const int split = MASK2 ? grid / 2 : grid;
    // bits 0-1: PDL trigger placement, probe; bits 8+: the constant 32 for keep() (opaque to ptxas)
    const int flags = (pdl_enabled(4) ? 1 : 0) | (inter_probe_on() ? 2 : 0) | (32 << 8);
    const cudaError_t e = launch_pdl(1, kern, dim3(grid), dim3(kFastThreads), smem, st, 0, rec, rectw, map, tiles, t_lo,
                                     t_hi, Qc, cap, keys, SV, sp, imask, x_lo, x_hi, flags, split,
                                     static_cast<unsigned long long *>(nullptr));
    note_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <int U, bool TW, bool PEN = false>
static cudaError_t launch_fast_u(uint32_t mask, const SlotRec *rec, const SlotTW *rectw, const CUtensorMap &map,
                                 const uint32_t *tiles,
                                 int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys, int max_grid,
                                 cudaStream_t st, const SolView<int32_t> &SV, const ScoreParams &sp, uint32_t imask,
                                 int x_lo, int x_hi) {
    if (!(mask & 0x7FEu)) return cudaSuccess;
    cudaError_t err = cudaSuccess;
    // the intra-route work rides along with the first launch
    auto run = [&](auto kmask, auto kmask2) {
        if (err != cudaSuccess) return;
        err = launch_fast_t<U, TW, decltype(kmask)::value, decltype(kmask2)::value, PEN>(
            rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, max_grid, st, SV, sp, imask, x_lo, x_hi);
        imask = 0;
    };
    using Z = std::integral_constant<uint32_t, 0u>;
    // all inter variants: {2-opt*, relocate, or-opt, swap(1,1), cross(2,2)} | {cross (1,2) (1,3) (2,3) (3,3)}
    constexpr uint32_t ALL = 0x7FEu, HA = 0x13Eu, HB = 0x6C0u, NS = (1u << 1) | (1u << 2) | (1u << 5);
    static_assert((HA | HB) == ALL && (HA & HB) == 0, "halves");
    if ((mask & ALL) == ALL) {
        // split in halves only while both halves still get one tile per resident CTA
        // (small neighbourhoods: twice the CTAs); above that the halves would pay the
        // per-tile loads and folds twice
        int r1 = 0, r2 = 0;
        fast_capacity<U, TW, HA, HB, PEN>(r1, r2);
        if (2 * (t_hi - t_lo) <= r1)
            run(std::integral_constant<uint32_t, HA>{}, std::integral_constant<uint32_t, HB>{});
        else
            run(std::integral_constant<uint32_t, ALL>{}, Z{});
        return err;
    }
    if ((mask & NS) == NS) { run(std::integral_constant<uint32_t, NS>{}, Z{}); mask &= ~NS; }
    if (mask & (1u << 1)) run(std::integral_constant<uint32_t, (1u << 1)>{}, Z{});
    if (mask & (1u << 2)) run(std::integral_constant<uint32_t, (1u << 2)>{}, Z{});
    if (mask & (3u << 3)) run(std::integral_constant<uint32_t, (3u << 3)>{}, Z{});
    if (mask & (1u << 5)) run(std::integral_constant<uint32_t, (1u << 5)>{}, Z{});
    if (mask & (0x1Fu << 6)) run(std::integral_constant<uint32_t, (0x1Fu << 6)>{}, Z{});
    return err;
}

#ifndef TGA_BATCH_SHARED_COLS
#define TGA_BATCH_SHARED_COLS 1
#endif
constexpr bool kBatchSharedCols = TGA_BATCH_SHARED_COLS != 0;
// Population batch (BASELINE config 5) on the fast path: a contiguous run of
// (solution, tile) items per CTA; the running minima are flushed into a
// solution's keys when the run moves on to the next solution.
template <int U, bool TW, uint32_t MASK>
__global__ void __launch_bounds__(kFastThreads) k_inter_fast_batch(const FastSol *__restrict__ sols,
                                                                   const CUtensorMap *__restrict__ maps,
                                                                   const uint32_t *__restrict__ work, int n_work,
                                                                   int32_t cap, ScoreParams sp, int flags) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (s_u32(smem_raw) & 127u)) & 127u);
    __shared__ uint64_t bar[3];
    __shared__ unsigned long long red[kFastThreads / 32][23];
    const int tid = threadIdx.x;
    if (tid == 0) {
        f_mbar_init(&bar[0]);
        f_mbar_init(&bar[1]);
        f_mbar_init(&bar[2]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < (kFastThreads / 32) * 23; i += kFastThreads) red[i / 23][i % 23] = kNoKey;
    __syncthreads();
    const int cta = static_cast<int>(blockIdx.x), G = static_cast<int>(gridDim.x);
    const int w0 = static_cast<int>(static_cast<long long>(n_work) * cta / G);
    const int w1 = static_cast<int>(static_cast<long long>(n_work) * (cta + 1) / G);
    auto item = [&](int w) -> FastItem {
        const uint32_t c = work[w];
        const int k = static_cast<int>(c >> 20);
        const FastSol f = sols[k];
        return FastItem{f.rec, f.rectw, maps + k, f.keys, f.Qc, k, static_cast<int>((c >> 10) & 0x3FFu),
                        static_cast<int>(c & 0x3FFu)};
    };
    const SolView<int32_t> none{};
    fast_body<U, TW, MASK, false, false, decltype(item), kBatchSharedCols>(item, w0, w1, 1, bar, red, sm, cap, none, sp,
                                                                         0u, 0, 0, 0, 1, flags);
}

// the batch kernel's dynamic shared memory: two box + row stages and one column region (SC)
template <int U, bool TW>
constexpr int batch_smem() {
    using G = FastGeom<U, TW>;
    return kBatchSharedCols ? 2 * (G::BoxPad + G::RowBytes + G::RowTW) + G::ColBytes + G::ColTW + 128 : G::Smem;
}
template <int U, bool TW, uint32_t MASK>
static cudaError_t launch_fast_batch_t(const FastSol *sols, const CUtensorMap *maps, const uint32_t *work, int n_work,
                                       int32_t cap, const ScoreParams &sp, int max_grid, cudaStream_t st) {
    auto kern = k_inter_fast_batch<U, TW, MASK>;
    using G = FastGeom<U, TW>;
    static PerDevice pd;
    static int res_cap[kMaxDevices];
    const int d = once_per_device(pd, [](int dev) {
        auto k = k_inter_fast_batch<U, TW, MASK>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, batch_smem<U, TW>());
        int sms = 0, b = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kFastThreads, batch_smem<U, TW>());
        res_cap[dev] = std::max(1, b) * std::max(1, sms);
    });
    const int res = res_cap[d];
    const int grid = std::max(1, std::min(n_work, std::min(res, max_grid)));
    kern<<<grid, kFastThreads, batch_smem<U, TW>(), st>>>(sols, maps, work, n_work, cap, sp, 32 << 8);
    note_launch();
    return cudaGetLastError();
}

template <int U, bool TW>
static cudaError_t launch_fast_batch_u(uint32_t mask, const FastSol *sols, const CUtensorMap *maps,
                                       const uint32_t *work, int n_work, int32_t cap, const ScoreParams &sp,
                                       int max_grid, cudaStream_t st) {
    if (!(mask & 0x7FEu) || n_work <= 0) return cudaSuccess;
    cudaError_t err = cudaSuccess;
    auto run = [&](auto kmask) {
        if (err == cudaSuccess)
            err = launch_fast_batch_t<U, TW, decltype(kmask)::value>(sols, maps, work, n_work, cap, sp, max_grid, st);
    };
    constexpr uint32_t ALL = 0x7FEu, NS = (1u << 1) | (1u << 2) | (1u << 5);
    if ((mask & ALL) == ALL) { run(std::integral_constant<uint32_t, ALL>{}); return err; }
    if ((mask & NS) == NS) { run(std::integral_constant<uint32_t, NS>{}); mask &= ~NS; }
    if (mask & (1u << 1)) run(std::integral_constant<uint32_t, (1u << 1)>{});
    if (mask & (1u << 2)) run(std::integral_constant<uint32_t, (1u << 2)>{});
    if (mask & (3u << 3)) run(std::integral_constant<uint32_t, (3u << 3)>{});
    if (mask & (1u << 5)) run(std::integral_constant<uint32_t, (1u << 5)>{});
    if (mask & (0x1Fu << 6)) run(std::integral_constant<uint32_t, (0x1Fu << 6)>{});
    return err;
}

cudaError_t launch_inter_fast_batch(int U, bool tw, uint32_t mask, const FastSol *sols, const CUtensorMap *maps,
                                    const uint32_t *work, int n_work, int32_t cap, const ScoreParams &sp,
                                    int max_grid, cudaStream_t st) {
    if (U != 16) return cudaErrorInvalidValue;
    return tw ? launch_fast_batch_u<16, true>(mask, sols, maps, work, n_work, cap, sp, max_grid, st)
              : launch_fast_batch_u<16, false>(mask, sols, maps, work, n_work, cap, sp, max_grid, st);
}

// ============================================================== edge-based evaluation (ETGA)
// Edge-based extraction for inter-route operators: only the cells
// (u, v) whose node pair the edge mask M keeps are evaluated -- the customer
// pairs of the granular neighbourhood (host-built, reading 21), every
// (customer, start depot of another route) cell and every pair of start depots.
// Each thread evaluates one cell with the same stream formulas as the tile
// kernel (cell_streams), reading its 5x5 Dp neighbourhood and the two records
// from L2; slot_of[node] (k_slot_of) maps the static node pairs to the current
// slots.  Intra-route variants stay full.
__global__ void __launch_bounds__(256) k_slot_of(const int32_t *__restrict__ node, const int32_t *__restrict__ pos,
                                                 const int32_t *__restrict__ rlen, int Qp, int32_t *__restrict__ slot_of) {
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < Qp; x += gridDim.x * blockDim.x) {
        const int p = pos[x];
        if (p >= 1 && p <= rlen[x]) slot_of[node[x]] = x;
    }
}

template <bool TW, uint32_t MASK>
__global__ void __launch_bounds__(256, 2) k_etga(const SlotRec *__restrict__ rec, const SlotTW *__restrict__ rectw,
                                              const int32_t *__restrict__ Dp, int pitch, uint32_t Qc,
                                              const int32_t *__restrict__ slot_of, const int32_t *__restrict__ rbase,
                                              const int32_t *__restrict__ pos, const int32_t *__restrict__ rlen,
                                              const int2 *__restrict__ pairs, int n_pairs, int n_cust, int R,
                                              int32_t cap, uint64_t *__restrict__ keys,
                                              unsigned long long *__restrict__ counts, int w_lo, int w_hi) {
    constexpr int NV = 11;
    __shared__ unsigned long long red[8][23];
    __shared__ unsigned long long csum[8][NV];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t acc[NV];
    uint32_t nc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) { acc[i] = kNoKey; nc[i] = 0u; }
    const int n_dep = n_cust * R;
    const int stride = gridDim.x * blockDim.x;
    // one cell (u, v) evaluated with the streams of mask CM
    auto eval_cell = [&](auto kmask, int u, int v) {
        constexpr uint32_t CM = decltype(kmask)::value;
        SlotRec A = rec[u], V = rec[v];
        if (A.r < 0 || V.r < 0 || A.r == V.r) return;
        if (A.r > V.r) {
            const int t = u; u = v; v = t;
            const SlotRec T = A; A = V; V = T;
        }
        SlotTW AT{}, VT{};
        if (TW) { AT = rectw[u]; VT = rectw[v]; }
        // rows / columns clamped into the matrix: u - 1 of the first start depot (slot 0)
        // or u + 3 past the last slot only feed candidates that are invalid anyway
        auto D = [&](int di, int dj) -> int32_t {
            const int r = min(max(u + di, 0), pitch - 1), c = min(max(v + dj, 0), pitch - 1);
            return __ldg(Dp + static_cast<size_t>(r) * pitch + c);
        };
        const uint32_t idx_d = static_cast<uint32_t>(u) * Qc + static_cast<uint32_t>(v);
        const uint32_t idx_r = static_cast<uint32_t>(v) * Qc + static_cast<uint32_t>(u);
        // slot -> (variant, direction) of the stream layout
        cell_streams<TW, false, CM>(A, V, AT, VT, cap, 0, D, [&](int k, bool ok, int32_t dD) {
            const int var = stream_variant(k);
            const bool direct = stream_direct(k);
            if (ok) acc[var] = umin64(acc[var], pack_key(ord_score(dD), direct ? idx_d : idx_r));
        });
        // structurally valid candidates of the cell (the oracle's masked count)
        const int pu = pos[u], pv = pos[v], Lu = rlen[u], Lv = rlen[v];
        auto segok = [](int p, int n, int L) -> uint32_t { return (p >= 1 && p + n - 1 <= L) ? 1u : 0u; };
        if (CM & (1u << 1)) nc[1] += 1u;
    #pragma unroll
        for (int N = 1; N <= 3; ++N)
            if (CM & (1u << (1 + N))) nc[1 + N] += segok(pu, N, Lu) + segok(pv, N, Lv);
    #pragma unroll
        for (int sv = 0; sv < 6; ++sv) {
            constexpr int n1s[6] = {1, 1, 1, 2, 2, 3}, n2s[6] = {1, 2, 3, 2, 3, 3};
            const int N1 = n1s[sv], N2 = n2s[sv];
            if (!(CM & (1u << (5 + sv)))) continue;
            nc[5 + sv] += segok(pu, N1, Lu) * segok(pv, N2, Lv);
            if (N1 != N2) nc[5 + sv] += segok(pv, N1, Lv) * segok(pu, N2, Lu);
        }
    };
    // cells with a start depot only have 2-opt* and relocate candidates (a segment never
    // starts at a depot): their swap / cross streams are not evaluated
    constexpr uint32_t DEPOT_MASK = MASK & 0x1Eu;
    for (int w = w_lo + blockIdx.x * blockDim.x + tid; w < w_hi; w += stride) {
        if (w < n_pairs) {
            const int2 pr = pairs[w];
            eval_cell(std::integral_constant<uint32_t, MASK>{}, slot_of[pr.x], slot_of[pr.y]);
        } else if (w < n_pairs + n_dep) {   // (customer j, start depot of route a)
            const int k = w - n_pairs;
            eval_cell(std::integral_constant<uint32_t, DEPOT_MASK>{}, rbase[k % R], slot_of[k / R + 1]);
        } else {                            // (start depot of a, start depot of b), a < b
            const int k = w - n_pairs - n_dep;
            const int a = k / R, b = k % R;
            if (a < b) eval_cell(std::integral_constant<uint32_t, DEPOT_MASK>{}, rbase[a], rbase[b]);
        }
    }
    // fused argmin + counts: warp -> the warp's shared row -> one atomic per variant per CTA
#pragma unroll
    for (int i = 1; i < NV; ++i) {
        const uint64_t k = warp_min64(acc[i]);
        const uint32_t c = __reduce_add_sync(0xffffffffu, nc[i]);
        if (lane == 0) { red[warp][i] = k; csum[warp][i] = c; }
    }
    __syncthreads();
    if (tid >= 1 && tid < NV) {
        unsigned long long m = kNoKey, c = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            m = m < red[w][tid] ? m : red[w][tid];
            c += csum[w][tid];
        }
        if (m != kNoKey) atomicMin(reinterpret_cast<unsigned long long *>(keys) + tid, m);
        if (counts && c) atomicAdd(counts + tid, c);
    }
}

template <bool TW>
static cudaError_t launch_etga_t(uint32_t mask, const EtgaArgs &a, cudaStream_t st) {
    cudaError_t err = cudaSuccess;
    const int cells = a.w_hi - a.w_lo;
    if (cells <= 0 || !(mask & 0x7FEu)) return cudaSuccess;
    const int grid = std::max(1, std::min((cells + 255) / 256, a.sm_count * 8));
    auto run = [&](auto kmask) {
        if (err != cudaSuccess) return;
        k_etga<TW, decltype(kmask)::value><<<grid, 256, 0, st>>>(a.rec, a.rectw, a.Dp, a.pitch, a.Qc, a.slot_of, a.rbase,
                                                                 a.pos, a.rlen, a.pairs, a.n_pairs, a.n_cust, a.R,
                                                                 a.cap, a.keys, a.counts, a.w_lo, a.w_hi);
        note_launch();
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
    return err;
}

cudaError_t launch_etga(uint32_t mask, bool tw, const EtgaArgs &a, cudaStream_t st, bool build_slot_of) {
    cudaError_t e = cudaSuccess;
    if (build_slot_of) {   // device steps keep the map current; host layout uploads invalidate it
        const int grid = std::max(1, std::min((a.Qp + 255) / 256, a.sm_count * 4));
        k_slot_of<<<grid, 256, 0, st>>>(a.node, a.pos, a.rlen, a.Qp, a.slot_of);
        note_launch();
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return tw ? launch_etga_t<true>(mask, a, st) : launch_etga_t<false>(mask, a, st);
}

// test-only: the DUMP instantiation of the all-variant fused sweep (U = 16), every
// candidate's key stored in dump (tga_debug_eval_dump); same tile plan and body
template <bool TW, bool PEN>
static cudaError_t launch_fast_dump_t(const SlotRec *rec, const SlotTW *rectw, const CUtensorMap &map,
                                      const uint32_t *tiles, int t_lo, int t_hi, uint32_t Qc, int32_t cap,
                                      uint64_t *keys, cudaStream_t st, const SolView<int32_t> &SV,
                                      const ScoreParams &sp, uint32_t imask, int x_lo, int x_hi,
                                      unsigned long long *dump) {
    constexpr uint32_t ALL = 0x7FEu;
    auto kern = k_inter_fast<16, TW, ALL, 0u, true, PEN>;
    using G = FastGeom<16, TW>;
    static PerDevice pd;
    once_per_device(pd, [&](int) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::Smem); });
    const int units = imask ? (x_hi - x_lo + 3) / 4 : 0;
    const int grid = std::max(1, std::max(t_hi - t_lo, units));
    kern<<<grid, kFastThreads, G::Smem1, st>>>(rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, SV, sp, imask, x_lo,
                                               x_hi, 32 << 8, grid, dump);
    note_launch();
    return cudaGetLastError();
}
cudaError_t launch_inter_fast_dump(bool tw, const SlotRec *rec, const SlotTW *rectw, const CUtensorMap &map,
                                   const uint32_t *tiles, int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys,
                                   cudaStream_t st, const SolView<int32_t> &SV, const ScoreParams &sp, uint32_t imask,
                                   int x_lo, int x_hi, unsigned long long *dump) {
    if (sp.mode == 1)
        return tw ? cudaErrorInvalidValue
                  : launch_fast_dump_t<false, true>(rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, st, SV, sp, imask,
                                                    x_lo, x_hi, dump);
    return tw ? launch_fast_dump_t<true, false>(rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, st, SV, sp, imask, x_lo,
                                                x_hi, dump)
              : launch_fast_dump_t<false, false>(rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, st, SV, sp, imask,
                                                 x_lo, x_hi, dump);
}

cudaError_t launch_inter_fast(int U, uint32_t mask, const SlotRec *rec, const SlotTW *rectw, const CUtensorMap &map,
                              const uint32_t *tiles, int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys,
                              int max_grid, cudaStream_t st, const SolView<int32_t> &SV, const ScoreParams &sp,
                              uint32_t imask, int x_lo, int x_hi) {
    if (sp.mode == 1) {   // penalised records (CVRP): U = 16 tiles
        if (rectw) return cudaErrorInvalidValue;
        return launch_fast_u<16, false, true>(mask, rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, max_grid, st, SV,
                                              sp, imask, x_lo, x_hi);
    }
    if (rectw)
        return U == 8 ? launch_fast_u<8, true>(mask, rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, max_grid, st, SV,
                                               sp, imask, x_lo, x_hi)
                      : launch_fast_u<16, true>(mask, rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, max_grid, st,
                                                SV, sp, imask, x_lo, x_hi);
    return U == 8 ? launch_fast_u<8, false>(mask, rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, max_grid, st, SV,
                                            sp, imask, x_lo, x_hi)
                  : launch_fast_u<16, false>(mask, rec, rectw, map, tiles, t_lo, t_hi, Qc, cap, keys, max_grid, st, SV,
                                             sp, imask, x_lo, x_hi);
}

}  // namespace tga

// host-side decode of the fast-path tile order (tests: a bijection onto the plan set)
extern "C" int32_t tga_debug_fast_tile(int32_t t, int32_t nI, int32_t R, int32_t *I, int32_t *J) {
    if (!I || !J || R < 1 || nI < 0 || t < 0) return -1;
    int i, j;
    tga::fast_tile_of(t, nI, R, i, j);
    *I = i;
    *J = j;
    return 0;
}

extern "C" int32_t tga_debug_inter_probe(uint64_t *out, int32_t n) {
    return cudaMemcpyFromSymbol(out, tga::g_inter_probe, sizeof(uint64_t) * static_cast<size_t>(n)) == cudaSuccess ? 0 : -5;
}
