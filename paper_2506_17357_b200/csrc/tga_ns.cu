// tga_ns.cu -- the north-star sweep: fused 2-opt* + relocate (N = 1) + swap (1,1)
// inter-route evaluation, CVRP, feasible-only score (sm_100a).
//
// Same candidates, scores, feasibility and keys as the all-variant tile kernel
// (Fig. `operators` P:107-149; Eq. 2, Eq. 3f, Eq. 13-14
// P:372-388; score and argmin Eq. 16), restricted to the three
// operators of the north-star sweep and organised for instruction count:
//   * tile = 32 rows x 128 columns; 4 warps stacked in rows (8 rows each), a lane
//     owns 4 CONSECUTIVE columns, so one 16-byte shared load brings the Dp values
//     of 4 cells, a row's record (a warp-uniform broadcast) serves 4 cells, and
//     the 8 rows are unrolled with the Dp rows u-1, u, u+1 kept in registers;
//   * every term that depends on the row alone or the column alone is folded
//     before the row loop: per column  cap - load  bounds and the -e(v) terms,
//     per row the  -e(u) * 32 + row  key addends (compact NsRow records), so a
//     candidate costs one or two IADD3, one IMAD (its 32-bit key
//     score * 32 + 2^28 + row), one or two ISETP and one predicated IMNMX;
//   * one running minimum per (stream, column): with the column fixed, the row
//     order is the canonical order of both key directions (u * Q + v and
//     v * Q + u, reading 5), so the key needs no column bits until the tile end,
//     where the 4 columns are merged in 32 bits and converted to 64-bit
//     (score, canonical index) keys once per stream;
//   * one tile per CTA when the grid covers the plan (the usual case), one Dp box
//     (34 x 136 int32) + row and column records per tile on one mbarrier; the
//     per-variant minima leave the CTA as one 64-bit atomicMin each.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

#include "tga_device.cuh"
#include "tga_launch.h"
#include "tga_tma.cuh"

namespace tga {

// diagnostics (TGA_NS_PROBE=1): per-CTA %globaltimer stamps, 4 per CTA:
// 0 start, 1 first tile's data arrived, 2 tiles done, 3 end
__device__ unsigned long long g_ns_probe[4 * 4096];
__device__ __forceinline__ unsigned long long ns_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

namespace {
constexpr int kNsW = 4;                         // warps per CTA (stacked in rows)
constexpr int kNsTV = 128;                      // 32 lanes x 4 columns
constexpr int kNsBoxW = kNsTV + 8;              // cols v0-4 .. v0+131 (16-byte aligned TMA x)
constexpr int kNsColF = 10;                     // per-column terms, SoA in shared memory
constexpr uint32_t kNsNone = 0xFFFFFF00u;       // "no feasible candidate": survives *4 + c and + RW c
constexpr int32_t kNsOff = 1 << 28;             // key offset B: score * S + B + row >= 0 for |score| < B / S

// geometry of the RW-rows-per-warp instantiation: tile = 4 RW rows x 128 columns;
// shared memory: the column-term planes | per warp: its Dp box (RW + 2 rows) | per
// warp: its row records -- every warp waits only for its own box and rows
template <int RW>
struct NsGeom {
    static constexpr int TU = kNsW * RW;                        // rows per tile
    static constexpr int RB = kNsTV / TU;                       // row bands per column band
    static constexpr int BoxH = RW + 2;                         // a warp's rows u-1 .. u+RW
    static constexpr int BoxBytes = kNsBoxW * BoxH * 4;
    static constexpr int BoxPad = (BoxBytes + 127) / 128 * 128;
    static constexpr int ColBytes = kNsColF * kNsTV * 4;        // column-term planes of the tile
    static constexpr int RowBytes = RW * 80;                    // a warp's row records
    static constexpr int RowPad = (RowBytes + 127) / 128 * 128;
    static constexpr int OffBox = ColBytes;
    static constexpr int OffRows = OffBox + kNsW * BoxPad;
    static constexpr int Smem = OffRows + kNsW * RowPad + 128;
    static constexpr int S = 4 * RW;                            // key = score * S + B + row (row < RW)
    static constexpr int LS = RW == 4 ? 4 : (RW == 8 ? 5 : 6);  // log2 S
    static_assert(RW == 4 || RW == 8 || RW == 16, "rows per warp");
};

// per-row terms of one tile row (built from the SlotRec once per tile)
struct __align__(16) NsRow {
    int32_t r, fL, bL1, so0;     // route (-1: not a canonical slot), 2-opt* loads, relocate-out load
    int32_t cW, sA0, cS, a2;     // cap - W, swap load, cap - sS0, ne * S + B + row
    int32_t aR, aS, pad0, pad1;  // rem0 * S + B + row, sE0 * S + B + row
};
}  // namespace

// tile t of the plan (RB row bands of TU rows per 128-column band): the diagonal tiles
// (row band I, column band I / RB) that do not close their column band, then the full
// tiles column by column (RB J (J - 1) / 2 of them precede column band J), then the
// lightest diagonal tiles (I % RB == RB - 1: only the band's last TU columns can lie
// above their rows) -- a grid one wave short of the plan gives its extra tiles, these,
// to CTAs that started with a diagonal tile
__host__ __device__ __forceinline__ void ns_tile_of(int t, int nI, int nJ, int RB, int &I, int &J) {
    const int n3 = nI / RB, n0 = nI - n3, F = RB * nJ * (nJ - 1) / 2;
    if (t < n0) { I = (t / (RB - 1)) * RB + t % (RB - 1); J = I / RB; return; }
    if (t >= n0 + F) { I = RB * (t - n0 - F) + RB - 1; J = I / RB; return; }
    const int q = t - n0;
    int j = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(q) / static_cast<float>(RB))) * 0.5f);
    while (j > 1 && RB * j * (j - 1) / 2 > q) --j;
    while (RB * (j + 1) * j / 2 <= q) ++j;
    J = j;
    I = q - RB * j * (j - 1) / 2;
}

template <int RW, bool DUMP>
__global__ void __launch_bounds__(kNsW * 32, DUMP ? 1 : (RW == 16 ? 4 : 5))
    k_ns_sweep(const SlotRec *__restrict__ rec, const int32_t *__restrict__ nsc, int pitch,
               const __grid_constant__ CUtensorMap tmap, int Qp, int t_lo, int t_hi, uint32_t Qc, int32_t cap,
               uint64_t *__restrict__ keys, uint32_t mulS, uint32_t one, int flags, unsigned long long *dump) {
    using G = NsGeom<RW>;
    constexpr int TU = G::TU;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (s_u32(smem_raw) & 127u)) & 127u);
    const int32_t(*colS)[kNsTV] = reinterpret_cast<const int32_t(*)[kNsTV]>(sm);   // [term][column]
    __shared__ uint64_t bar[kNsW + 1];                          // per warp (box + rows), [kNsW] columns
    __shared__ int s_tile[2][2];                                // (u0, v0) of the tile of iteration parity
    __shared__ NsRow nrow[TU];
    __shared__ unsigned long long red[kNsW][3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool prb = (flags & 1) && tid == 0 && blockIdx.x < 4096;
    if (prb) g_ns_probe[4 * blockIdx.x] = ns_gtime();
    const int nI = (Qp + TU - 1) / TU, nJ = (Qp + kNsTV - 1) / kNsTV;
    const int G_ = static_cast<int>(gridDim.x);
    int t = t_lo + static_cast<int>(blockIdx.x);
    // thread 0 issues a tile: the column-term planes first (every warp needs them), then
    // each warp's Dp box and row records on the warp's own barrier
    auto issue = [&](int u0, int v0) {
        f_expect(&bar[kNsW], G::ColBytes);
#pragma unroll
        for (int f = 0; f < kNsColF; ++f)
            f_bulk(sm + f * kNsTV * 4, nsc + static_cast<size_t>(f) * pitch + v0, kNsTV * 4, &bar[kNsW]);
#pragma unroll
        for (int w = 0; w < kNsW; ++w) {
            f_expect(&bar[w], G::BoxBytes + G::RowBytes);
            f_tma2d(sm + G::OffBox + w * G::BoxPad, &tmap, v0 - 4, u0 + w * RW - 1, &bar[w]);
            f_bulk(sm + G::OffRows + w * G::RowPad, rec + u0 + w * RW, G::RowBytes, &bar[w]);
        }
    };
    if (tid == 0) {
#pragma unroll
        for (int w = 0; w <= kNsW; ++w) f_mbar_init(&bar[w]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (t < t_hi) {   // the first tile's loads are in flight before anything else runs
            int I, J;
            ns_tile_of(t, nI, nJ, G::RB, I, J);
            s_tile[0][0] = I * TU;
            s_tile[0][1] = J * kNsTV;
            issue(I * TU, J * kNsTV);
        }
    }
    // a programmatic dependent (the next evaluation's key reset, which waits for this grid
    // before it writes) may launch now
    pdl_trigger();
    uint64_t acc[3] = {kNoKey, kNoKey, kNoKey};   // 2-opt*, relocate, swap (1,1)
    __syncthreads();
    uint32_t phase = 0u;
    for (int it = 0; t < t_hi; t += G_, ++it) {
        const int u0 = s_tile[it & 1][0], v0 = s_tile[it & 1][1];
        const int32_t *const box = reinterpret_cast<const int32_t *>(sm + G::OffBox + warp * G::BoxPad);
        const SlotRec *const rows = reinterpret_cast<const SlotRec *>(sm + G::OffRows + warp * G::RowPad);
        f_wait(&bar[warp], phase);
        if (prb && phase == 0u) g_ns_probe[4 * blockIdx.x + 1] = ns_gtime();
        // ---- this warp's RW rows as NsRow (lanes 0..RW-1)
        const int uw = u0 + warp * RW;   // first row of the warp
        if (lane < RW) {
            const SlotRec &A = rows[lane];
            NsRow n;
            n.r = A.r; n.fL = A.fL; n.bL1 = A.bL1; n.so0 = A.so[0];
            n.cW = cap - A.W; n.sA0 = A.sA[0]; n.cS = cap - A.sS[0];
            n.a2 = A.ne * G::S + kNsOff + lane;
            n.aR = A.rem[0] * G::S + kNsOff + lane;
            n.aS = A.sE[0] * G::S + kNsOff + lane;
            n.pad0 = n.pad1 = 0;
            nrow[warp * RW + lane] = n;
        }
        __syncwarp();
        f_wait(&bar[kNsW], phase);   // the column-term planes
        phase ^= 1u;
        int32_t Vr[4], Vne[4], Vrem[4], VsE[4], cbL1[4], cfL[4], cW[4], cS[4], Vso[4], VsA[4];
        auto col4 = [&](int f, int32_t (&x)[4]) {
            const int4 q = *reinterpret_cast<const int4 *>(&colS[f][4 * lane]);
            x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
        };
        col4(0, Vr); col4(1, Vne); col4(2, Vrem); col4(3, VsE); col4(4, cbL1);
        col4(5, cfL); col4(6, cW); col4(7, cS); col4(8, Vso); col4(9, VsA);
        int rmaxV = max(max(Vr[0], Vr[1]), max(Vr[2], Vr[3]));
        rmaxV = __reduce_max_sync(0xffffffffu, rmaxV);   // rows of a route >= every column's are skipped
        uint32_t run0[4], run1[4], run2[4], run3[4];   // 2-opt*, relocate u->v, relocate v->u, swap
#pragma unroll
        for (int c = 0; c < 4; ++c) run0[c] = run1[c] = run2[c] = run3[c] = kNsNone;
        // Dp(u, v0 + 4 lane + c) for the warp's rows: box row (u - uw + 1), box col 4 + 4 lane + c
        const int32_t *bcol = box + 4 + 4 * lane;
        auto ld4 = [&](int brow) { return *reinterpret_cast<const int4 *>(bcol + brow * kNsBoxW); };
        constexpr int br0 = 1;           // box row of the warp's first row
        int4 dm = ld4(br0 - 1), d0 = ld4(br0);
#pragma unroll
        for (int i = 0; i < RW; ++i) {
            const int4 d1 = ld4(br0 + i + 1);
            const int32_t dl = bcol[(br0 + i) * kNsBoxW - 1], dr = bcol[(br0 + i) * kNsBoxW + 4];
            const NsRow A = nrow[warp * RW + i];
            if (A.r >= 0 && A.r < rmaxV) {   // warp-uniform
                const int32_t D0[4] = {d0.x, d0.y, d0.z, d0.w};
                const int32_t Dm[4] = {dm.x, dm.y, dm.z, dm.w};
                const int32_t D1[4] = {d1.x, d1.y, d1.z, d1.w};
                const int32_t Dr[4] = {d0.y, d0.z, d0.w, dr};    // Dp(u, v + 1)
                const int32_t Dl[4] = {dl, d0.x, d0.y, d0.z};    // Dp(u, v - 1)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    // Keys  score * S + (B + row),  the sums built mostly with IMAD (x * S + y) on the
                    // fma pipe: the compares and minima already fill the alu pipe (both issue every
                    // 2 cycles per SMSP), so 12 alu + 10 fma instructions per cell beat 16 + 4.
                    // (inline PTX: the compiler would otherwise re-associate x S + y S into (x + y) S)
                    auto mad = [&](int32_t x, uint32_t y) {
                        uint32_t r;
                        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(mulS), "r"(y));
                        return r;
                    };
                    uint32_t t;
                    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(Dr[c]), "r"(one), "r"(Vne[c]));
                    const uint32_t u = mad(D1[c], static_cast<uint32_t>(A.a2));
                    // 2-opt*: A' = F(u) + B(v+1), B' = F(v) + B(u+1): dD = Dp(u,v+1) + Dp(u+1,v) - e(u) - e(v)  (Eq. 14)
                    const uint32_t k0 = mad(static_cast<int32_t>(t), u);
                    // relocate u after v: rem(u) + Dp(u,v) + Dp(u,v+1) - e(v);  v after u: rem(v) + Dp(u,v) + Dp(u+1,v) - e(u)  (Eq. 13)
                    const uint32_t k1 = mad(static_cast<int32_t>(t), mad(D0[c], static_cast<uint32_t>(A.aR)));
                    const uint32_t k2 = mad(D0[c], mad(Vrem[c], u));
                    // swap (1,1): A' = F(u-1) + v + B(u+1), B' = F(v-1) + u + B(v+1)
                    const uint32_t k3 = mad(Dr[c], mad(D1[c], mad(Dm[c] + Dl[c] + VsE[c], static_cast<uint32_t>(A.aS))));
                    // feasibility (Eq. 16b) and the keep, branch-free on predicates: the pair must
                    // span two routes, route(u) < route(v); every new route load <= cap (the loads
                    // of an invalid role are poisoned, so it fails the same compares)
                    asm("{\n\t.reg .pred v, p;\n\t"
                        "setp.lt.s32 v, %4, %5;\n\t"
                        "setp.le.and.s32 p, %6, %7, v;\n\t"
                        "setp.le.and.s32 p, %8, %9, p;\n\t"
                        "@p min.u32 %0, %0, %18;\n\t"
                        "setp.le.and.s32 p, %10, %11, v;\n\t"
                        "@p min.u32 %1, %1, %19;\n\t"
                        "setp.le.and.s32 p, %12, %13, v;\n\t"
                        "@p min.u32 %2, %2, %20;\n\t"
                        "setp.le.and.s32 p, %14, %15, v;\n\t"
                        "setp.le.and.s32 p, %16, %17, p;\n\t"
                        "@p min.u32 %3, %3, %21;\n\t}"
                        : "+r"(run0[c]), "+r"(run1[c]), "+r"(run2[c]), "+r"(run3[c])
                        : "r"(A.r), "r"(Vr[c]), "r"(A.fL), "r"(cbL1[c]), "r"(A.bL1), "r"(cfL[c]), "r"(A.so0), "r"(cW[c]),
                          "r"(Vso[c]), "r"(A.cW), "r"(A.sA0), "r"(cS[c]), "r"(VsA[c]), "r"(A.cS), "r"(k0), "r"(k1),
                          "r"(k2), "r"(k3));
                    if constexpr (DUMP) {   // test-only: every candidate of a valid cell (kNoKey if infeasible)
                        const bool valid = A.r < Vr[c];
                        const bool ok0 = valid & (A.fL <= cbL1[c]) & (A.bL1 <= cfL[c]);
                        const bool ok1 = valid & (A.so0 <= cW[c]);
                        const bool ok2 = valid & (Vso[c] <= A.cW);
                        const bool ok3 = valid & (A.sA0 <= cS[c]) & (VsA[c] <= A.cS);
                        if (valid) {
                            const uint32_t u = static_cast<uint32_t>(uw + i), v = static_cast<uint32_t>(v0 + 4 * lane + c);
                            const uint32_t st = Qc * Qc;
                            auto key = [&](bool ok, uint32_t k, uint32_t idx) -> unsigned long long {
                                return ok ? pack_key(ord_score(static_cast<int32_t>(k >> G::LS) - (kNsOff >> G::LS)), idx)
                                          : kNoKey;
                            };
                            dump_put(dump, st, 1, u * Qc + v, key(ok0, k0, u * Qc + v));
                            dump_put(dump, st, 2, u * Qc + v, key(ok1, k1, u * Qc + v));
                            dump_put(dump, st, 2, v * Qc + u, key(ok2, k2, v * Qc + u));
                            dump_put(dump, st, 5, u * Qc + v, key(ok3, k3, u * Qc + v));
                        }
                    }
                }
            }
            dm = d0;
            d0 = d1;
        }
        // the next tile's origin, decoded before the barrier that lets thread 0 refill the stage
        if (tid == 0 && t + G_ < t_hi) {
            int I, J;
            ns_tile_of(t + G_, nI, nJ, G::RB, I, J);
            s_tile[(it + 1) & 1][0] = I * TU;
            s_tile[(it + 1) & 1][1] = J * kNsTV;
        }
        // ---- merge the 4 columns in 32 bits, then one 64-bit key per stream
        //  direct (u * Q + v):  order (score, row, c)  ->  run * 4 + c
        //  reversed (v * Q + u): order (score, c, row)  ->  run + RW c
        uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu, m3 = 0xFFFFFFFFu;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            m0 = min(m0, run0[c] * 4u + static_cast<uint32_t>(c));
            m1 = min(m1, run1[c] * 4u + static_cast<uint32_t>(c));
            m2 = min(m2, run2[c] + static_cast<uint32_t>(RW * c));
            m3 = min(m3, run3[c] * 4u + static_cast<uint32_t>(c));
        }
        const uint32_t vb = static_cast<uint32_t>(v0 + 4 * lane);
        constexpr uint32_t kOrd = 0x80000000u - static_cast<uint32_t>(kNsOff >> G::LS);   // ord_score(score) - (score + B/S)
        auto direct = [&](uint64_t &a, uint32_t m) {
            if (m < 0xF0000000u) {
                const uint32_t u = static_cast<uint32_t>(uw) + ((m >> 2) & (RW - 1)), v = vb + (m & 3u);
                a = umin64(a, pack_key((m >> (G::LS + 2)) + kOrd, u * Qc + v));
            }
        };
        direct(acc[0], m0);
        direct(acc[1], m1);
        direct(acc[2], m3);
        if (m2 < 0xF0000000u) {
            const uint32_t u = static_cast<uint32_t>(uw) + (m2 & (RW - 1)), v = vb + ((m2 / RW) & 3u);
            acc[1] = umin64(acc[1], pack_key((m2 >> G::LS) + kOrd, v * Qc + u));
        }
        if (t + G_ < t_hi) {   // another tile: every warp is done with the stage
            __syncthreads();
            if (tid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(s_tile[(it + 1) & 1][0], s_tile[(it + 1) & 1][1]);
            }
        }
    }
    if (prb) g_ns_probe[4 * blockIdx.x + 2] = ns_gtime();
    // ---- fused argmin: warp minimum -> shared row -> one atomicMin per variant per CTA
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const uint64_t m = warp_min64(acc[k]);
        if (lane == 0) red[warp][k] = m;
    }
    __syncthreads();
    // the keys were reset by the stream predecessor (a programmatic dependent launch may
    // have started this grid while it ran): wait for it before the first key update
    pdl_wait();
    if (tid < 3) {
        unsigned long long m = red[0][tid];
#pragma unroll
        for (int w = 1; w < kNsW; ++w) m = m < red[w][tid] ? m : red[w][tid];
        const int var = tid == 0 ? 1 : (tid == 1 ? 2 : 5);
        if (m != kNoKey) atomicMin(reinterpret_cast<unsigned long long *>(keys) + var, m);
    }
    if (prb) g_ns_probe[4 * blockIdx.x + 3] = ns_gtime();
}

int ns_rows_per_warp(int Qp, int sm_count) {
    // the largest RW whose plan still gives every SM ~2.5 tiles (parallelism for the
    // latency-bound small sweeps, fewer per-tile overheads for the large ones)
    if (const char *e = std::getenv("TGA_NS_RW")) {
        const int v = std::atoi(e);
        if (v == 4 || v == 8 || v == 16) return v;
    }
    for (int rw : {16, 8})
        if (ns_tile_count(Qp, rw) >= (5 * sm_count) / 2) return rw;
    return 4;
}

int ns_tile_count(int Qp, int rw) {
    const int TU = kNsW * rw, RB = kNsTV / TU;
    const int nI = (Qp + TU - 1) / TU, nJ = (Qp + kNsTV - 1) / kNsTV;
    return nI + RB * nJ * (nJ - 1) / 2;
}

int ns_box_rows(int rw) { return rw + 2; }
int ns_box_cols() { return kNsBoxW; }

template <int RW, bool DUMP>
static int ns_capacity() {
    static PerDevice pd;
    static int res[kMaxDevices];
    const int d = once_per_device(pd, [](int dev) {
        cudaFuncSetAttribute(k_ns_sweep<RW, DUMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, NsGeom<RW>::Smem);
        int sms = 0, b = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_ns_sweep<RW, DUMP>, kNsW * 32, NsGeom<RW>::Smem);
        res[dev] = std::max(1, b) * std::max(1, sms);
    });
    return res[d];
}

template <int RW>
static cudaError_t launch_ns_t(const SlotRec *rec, const int32_t *nsc, int pitch, const CUtensorMap &map, int Qp,
                               int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys, bool after_reset,
                               cudaStream_t st, unsigned long long *dump) {
    const int tiles = t_hi - t_lo;
    static const int probe = std::getenv("TGA_NS_PROBE") != nullptr;
    static const bool no_pdl = std::getenv("TGA_NS_NO_PDL") != nullptr;   // A/B override
    constexpr int Smem = NsGeom<RW>::Smem;
    const uint32_t mulS = static_cast<uint32_t>(NsGeom<RW>::S);   // a kernel parameter: one IMAD per key
    if (dump) {
        const int grid = std::min(tiles, ns_capacity<RW, true>());
        k_ns_sweep<RW, true><<<grid, kNsW * 32, Smem, st>>>(rec, nsc, pitch, map, Qp, t_lo, t_hi, Qc, cap, keys, mulS, 1u,
                                                            0, dump);
        note_launch();
        return cudaGetLastError();
    }
    // after the key-reset kernel: a programmatic dependent launch, so the sweep's launch,
    // TMA loads and evaluation overlap the reset (k_ns_sweep waits only before its key
    // updates; the reset itself starts after every earlier write of the stream completed)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(std::min(tiles, ns_capacity<RW, false>()));
    cfg.blockDim = dim3(kNsW * 32);
    cfg.dynamicSmemBytes = Smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (after_reset && !no_pdl) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_ns_sweep<RW, false>, rec, nsc, pitch, map, Qp, t_lo, t_hi, Qc, cap,
                                             keys, mulS, 1u, probe ? 1 : 0, static_cast<unsigned long long *>(nullptr));
    note_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_ns_sweep(int rw, const SlotRec *rec, const int32_t *nsc, int pitch, const CUtensorMap &map, int Qp,
                            int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys, bool after_reset,
                            cudaStream_t st, unsigned long long *dump) {
    if (t_hi <= t_lo) return cudaSuccess;
    switch (rw) {
        case 4: return launch_ns_t<4>(rec, nsc, pitch, map, Qp, t_lo, t_hi, Qc, cap, keys, after_reset, st, dump);
        case 8: return launch_ns_t<8>(rec, nsc, pitch, map, Qp, t_lo, t_hi, Qc, cap, keys, after_reset, st, dump);
        case 16: return launch_ns_t<16>(rec, nsc, pitch, map, Qp, t_lo, t_hi, Qc, cap, keys, after_reset, st, dump);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace tga

// host-side decode of the NS tile order (tests: a bijection onto the plan)
extern "C" int32_t tga_debug_ns_tile(int32_t t, int32_t nI, int32_t nJ, int32_t RB, int32_t *I, int32_t *J) {
    if (!I || !J || nI < 0 || nJ < 0 || t < 0 || RB < 2) return -1;
    int i, j;
    tga::ns_tile_of(t, nI, nJ, RB, i, j);
    *I = i;
    *J = j;
    return 0;
}

extern "C" int32_t tga_debug_ns_probe(uint64_t *out, int32_t n) {
    return cudaMemcpyFromSymbol(out, tga::g_ns_probe, sizeof(uint64_t) * static_cast<size_t>(n)) == cudaSuccess ? 0 : -5;
}
