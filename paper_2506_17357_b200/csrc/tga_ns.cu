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
constexpr int kNsRW = 8;                        // rows per warp
constexpr int kNsW = 4;                         // warps per CTA (stacked in rows)
constexpr int kNsTU = kNsRW * kNsW;             // 32 rows per tile
constexpr int kNsTV = 128;                      // 32 lanes x 4 columns
constexpr int kNsBoxW = kNsTV + 8;              // cols v0-4 .. v0+131 (16-byte aligned TMA x)
constexpr int kNsBoxH = kNsTU + 2;              // rows u0-1 .. u0+32
constexpr int kNsBoxBytes = kNsBoxW * kNsBoxH * 4;
constexpr int kNsBoxPad = (kNsBoxBytes + 127) / 128 * 128;
constexpr int kNsRowBytes = kNsTU * 80;
constexpr int kNsSmem = kNsBoxPad + kNsRowBytes + 128;
constexpr int kNsColF = 10;                     // per-column terms, SoA in shared memory
constexpr uint32_t kNsNone = 0xFFFFFF00u;       // "no feasible candidate": survives *4 + c and + 8 c
constexpr uint32_t kNsOff = 1u << 28;           // key offset: score * 32 + 2^28 + row >= 0 for |score| < 2^23

// per-row terms of one tile row (built from the SlotRec once per tile)
struct __align__(16) NsRow {
    int32_t r, fL, bL1, so0;     // route (-1: not a canonical slot), 2-opt* loads, relocate-out load
    int32_t cW, sA0, cS, a2;     // cap - W, swap load, cap - sS0, ne * 32 + 2^28 + row8
    int32_t aR, aS, pad0, pad1;  // rem0 * 32 + 2^28 + row8, sE0 * 32 + 2^28 + row8
};
}  // namespace

// tile t of the plan: the diagonal tiles (row band I, column band I / 4) whose rows
// start the column band's first three quarters, then the full tiles column by column
// (2 J (J - 1) of them precede column band J), then the lightest diagonal tiles
// (I % 4 == 3: only the band's last 32 columns can lie above their rows) -- so a grid
// one wave short of the plan gives its extra tiles, these, to CTAs that started with
// a diagonal tile
__host__ __device__ __forceinline__ void ns_tile_of(int t, int nI, int nJ, int &I, int &J) {
    const int n3 = nI / 4, n0 = nI - n3, F = 2 * nJ * (nJ - 1);
    if (t < n0) { I = (t / 3) * 4 + t % 3; J = I >> 2; return; }
    if (t >= n0 + F) { I = 4 * (t - n0 - F) + 3; J = I >> 2; return; }
    const int q = t - n0;
    int j = static_cast<int>((1.0f + sqrtf(1.0f + 2.0f * static_cast<float>(q))) * 0.5f);
    while (j > 1 && 2 * j * (j - 1) > q) --j;
    while (2 * (j + 1) * j <= q) ++j;
    J = j;
    I = q - 2 * j * (j - 1);
}

template <bool DUMP>
__global__ void __launch_bounds__(kNsW * 32, 5)
    k_ns_sweep(const SlotRec *__restrict__ rec, const __grid_constant__ CUtensorMap tmap, int Qp, int t_lo, int t_hi,
               uint32_t Qc, int32_t cap, uint64_t *__restrict__ keys, uint32_t mul32, int flags,
               unsigned long long *dump) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *sm = smem_raw + ((128u - (s_u32(smem_raw) & 127u)) & 127u);
    int32_t *const box = reinterpret_cast<int32_t *>(sm);
    const SlotRec *const rows = reinterpret_cast<const SlotRec *>(sm + kNsBoxPad);
    __shared__ uint64_t bar;
    __shared__ NsRow nrow[kNsTU];
    __shared__ __align__(16) int32_t colS[kNsColF][kNsTV];   // column terms: [field][column]
    __shared__ unsigned long long red[kNsW][3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool prb = (flags & 1) && tid == 0 && blockIdx.x < 4096;
    if (prb) g_ns_probe[4 * blockIdx.x] = ns_gtime();
    const int nI = (Qp + kNsTU - 1) / kNsTU, nJ = (Qp + kNsTV - 1) / kNsTV;
    int t = t_lo + static_cast<int>(blockIdx.x);
    auto issue = [&](int tt) {
        int I, J;
        ns_tile_of(tt, nI, nJ, I, J);
        f_expect(&bar, kNsBoxBytes + kNsRowBytes);
        f_tma2d(box, &tmap, J * kNsTV - 4, I * kNsTU - 1, &bar);
        f_bulk(sm + kNsBoxPad, rec + I * kNsTU, kNsRowBytes, &bar);
    };
    if (tid == 0) {
        f_mbar_init(&bar);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (t < t_hi) issue(t);   // the first Dp box is in flight before anything else runs
    }
    uint64_t acc[3] = {kNoKey, kNoKey, kNoKey};   // 2-opt*, relocate, swap (1,1)
    __syncthreads();
    uint32_t phase = 0u;
    for (; t < t_hi; t += static_cast<int>(gridDim.x)) {
        int I, J;
        ns_tile_of(t, nI, nJ, I, J);
        const int u0 = I * kNsTU, v0 = J * kNsTV;
        {   // column terms of the tile: thread t reads record v0 + t from L2 (in flight with
            // the box) and stores its per-column terms as SoA, so that a lane later reads its 4
            // consecutive columns' terms with one conflict-free 16-byte load per term
            const SlotRec V = rec[v0 + tid];
            colS[0][tid] = V.r; colS[1][tid] = V.ne; colS[2][tid] = V.rem[0]; colS[3][tid] = V.sE[0];
            colS[4][tid] = cap - V.bL1; colS[5][tid] = cap - V.fL; colS[6][tid] = cap - V.W;
            colS[7][tid] = cap - V.sS[0]; colS[8][tid] = V.so[0]; colS[9][tid] = V.sA[0];
        }
        f_wait(&bar, phase);
        if (prb && phase == 0u) g_ns_probe[4 * blockIdx.x + 1] = ns_gtime();
        phase ^= 1u;
        // ---- this warp's 8 rows as NsRow (lanes 0..7)
        const int uw = u0 + warp * kNsRW;   // first row of the warp
        if (lane < kNsRW) {
            const SlotRec &A = rows[warp * kNsRW + lane];
            NsRow n;
            n.r = A.r; n.fL = A.fL; n.bL1 = A.bL1; n.so0 = A.so[0];
            n.cW = cap - A.W; n.sA0 = A.sA[0]; n.cS = cap - A.sS[0];
            n.a2 = A.ne * 32 + static_cast<int32_t>(kNsOff) + lane;
            n.aR = A.rem[0] * 32 + static_cast<int32_t>(kNsOff) + lane;
            n.aS = A.sE[0] * 32 + static_cast<int32_t>(kNsOff) + lane;
            n.pad0 = n.pad1 = 0;
            nrow[warp * kNsRW + lane] = n;
        }
        __syncthreads();
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
        // Dp(u, v0 + 4 lane + c) for the warp's rows: box row (u - u0 + 1), box col 4 + 4 lane + c
        const int32_t *bcol = box + 4 + 4 * lane;
        auto ld4 = [&](int brow) { return *reinterpret_cast<const int4 *>(bcol + brow * kNsBoxW); };
        const int br0 = warp * kNsRW + 1;   // box row of the warp's first row
        int4 dm = ld4(br0 - 1), d0 = ld4(br0);
#pragma unroll
        for (int i = 0; i < kNsRW; ++i) {
            const int4 d1 = ld4(br0 + i + 1);
            const int32_t dl = bcol[(br0 + i) * kNsBoxW - 1], dr = bcol[(br0 + i) * kNsBoxW + 4];
            const NsRow A = nrow[warp * kNsRW + i];
            if (A.r >= 0 && A.r < rmaxV) {   // warp-uniform
                const int32_t D0[4] = {d0.x, d0.y, d0.z, d0.w};
                const int32_t Dm[4] = {dm.x, dm.y, dm.z, dm.w};
                const int32_t D1[4] = {d1.x, d1.y, d1.z, d1.w};
                const int32_t Dr[4] = {d0.y, d0.z, d0.w, dr};    // Dp(u, v + 1)
                const int32_t Dl[4] = {dl, d0.x, d0.y, d0.z};    // Dp(u, v - 1)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    // 2-opt*: A' = F(u) + B(v+1), B' = F(v) + B(u+1)      (Eq. 14)
                    const uint32_t k0 = static_cast<uint32_t>(Dr[c] + D1[c] + Vne[c]) * mul32 + static_cast<uint32_t>(A.a2);
                    // relocate u after v / v after u                    (Eq. 13)
                    const uint32_t k1 = static_cast<uint32_t>(D0[c] + Dr[c] + Vne[c]) * mul32 + static_cast<uint32_t>(A.aR);
                    const uint32_t k2 = static_cast<uint32_t>(D0[c] + D1[c] + Vrem[c]) * mul32 + static_cast<uint32_t>(A.a2);
                    // swap (1,1): A' = F(u-1) + v + B(u+1), B' = F(v-1) + u + B(v+1)
                    const uint32_t k3 = static_cast<uint32_t>(Dm[c] + D1[c] + Dl[c] + Dr[c] + VsE[c]) * mul32 +
                                        static_cast<uint32_t>(A.aS);
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
                                return ok ? pack_key(ord_score(static_cast<int32_t>(k >> 5) - (1 << 23)), idx) : kNoKey;
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
        // ---- merge the 4 columns in 32 bits, then one 64-bit key per stream
        //  direct (u * Q + v):  order (score, row, c)  ->  run * 4 + c
        //  reversed (v * Q + u): order (score, c, row)  ->  run + 8 c
        uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu, m3 = 0xFFFFFFFFu;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            m0 = min(m0, run0[c] * 4u + static_cast<uint32_t>(c));
            m1 = min(m1, run1[c] * 4u + static_cast<uint32_t>(c));
            m2 = min(m2, run2[c] + 8u * static_cast<uint32_t>(c));
            m3 = min(m3, run3[c] * 4u + static_cast<uint32_t>(c));
        }
        const uint32_t vb = static_cast<uint32_t>(v0 + 4 * lane);
        auto direct = [&](uint64_t &a, uint32_t m) {
            if (m < 0xF0000000u) {
                const uint32_t ord = (m >> 7) + (0x80000000u - (1u << 23));   // ord_score(score)
                const uint32_t u = static_cast<uint32_t>(uw) + ((m >> 2) & 7u), v = vb + (m & 3u);
                a = umin64(a, pack_key(ord, u * Qc + v));
            }
        };
        direct(acc[0], m0);
        direct(acc[1], m1);
        direct(acc[2], m3);
        if (m2 < 0xF0000000u) {
            const uint32_t ord = (m2 >> 5) + (0x80000000u - (1u << 23));
            const uint32_t u = static_cast<uint32_t>(uw) + (m2 & 7u), v = vb + ((m2 >> 3) & 3u);
            acc[1] = umin64(acc[1], pack_key(ord, v * Qc + u));
        }
        if (t + static_cast<int>(gridDim.x) < t_hi) {   // another tile: every warp is done with the stage
            __syncthreads();
            if (tid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(t + static_cast<int>(gridDim.x));
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

int ns_tile_count(int Qp) {
    const int nI = (Qp + kNsTU - 1) / kNsTU, nJ = (Qp + kNsTV - 1) / kNsTV;
    return nI + 2 * nJ * (nJ - 1);
}

int ns_box_rows() { return kNsBoxH; }
int ns_box_cols() { return kNsBoxW; }

template <bool DUMP>
static int ns_capacity() {
    static PerDevice pd;
    static int res[kMaxDevices];
    const int d = once_per_device(pd, [](int dev) {
        cudaFuncSetAttribute(k_ns_sweep<DUMP>, cudaFuncAttributeMaxDynamicSharedMemorySize, kNsSmem);
        int sms = 0, b = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_ns_sweep<DUMP>, kNsW * 32, kNsSmem);
        res[dev] = std::max(1, b) * std::max(1, sms);
    });
    return res[d];
}

cudaError_t launch_ns_sweep(const SlotRec *rec, const CUtensorMap &map, int Qp, int t_lo, int t_hi, uint32_t Qc,
                            int32_t cap, uint64_t *keys, bool after_reset, cudaStream_t st, unsigned long long *dump) {
    if (t_hi <= t_lo) return cudaSuccess;
    const int tiles = t_hi - t_lo;
    static const int probe = std::getenv("TGA_NS_PROBE") != nullptr;
    static const bool no_pdl = std::getenv("TGA_NS_NO_PDL") != nullptr;   // A/B override
    if (dump) {
        const int grid = std::min(tiles, ns_capacity<true>());
        k_ns_sweep<true><<<grid, kNsW * 32, kNsSmem, st>>>(rec, map, Qp, t_lo, t_hi, Qc, cap, keys, 32u, 0, dump);
        note_launch();
        return cudaGetLastError();
    }
    // after the key-reset kernel: a programmatic dependent launch, so the sweep's launch,
    // TMA loads and evaluation overlap the reset (k_ns_sweep waits only before its key
    // updates; the reset itself starts after every earlier write of the stream completed)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(std::min(tiles, ns_capacity<false>()));
    cfg.blockDim = dim3(kNsW * 32);
    cfg.dynamicSmemBytes = kNsSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (after_reset && !no_pdl) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_ns_sweep<false>, rec, map, Qp, t_lo, t_hi, Qc, cap, keys, 32u,
                                             probe ? 1 : 0, static_cast<unsigned long long *>(nullptr));
    note_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tga

// host-side decode of the NS tile order (tests: a bijection onto the plan)
extern "C" int32_t tga_debug_ns_tile(int32_t t, int32_t nI, int32_t nJ, int32_t *I, int32_t *J) {
    if (!I || !J || nI < 0 || nJ < 0 || t < 0) return -1;
    int i, j;
    tga::ns_tile_of(t, nI, nJ, i, j);
    *I = i;
    *J = j;
    return 0;
}

extern "C" int32_t tga_debug_ns_probe(uint64_t *out, int32_t n) {
    return cudaMemcpyFromSymbol(out, tga::g_ns_probe, sizeof(uint64_t) * static_cast<size_t>(n)) == cudaSuccess ? 0 : -5;
}
