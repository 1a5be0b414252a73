// tga_launch.h -- host-side launch interface of the TGA kernels (internal).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>
#include <algorithm>
#include <utility>
#include <mutex>

#include "tga_device.cuh"

namespace tga {

// inter-route tile geometry (see k_inter)
constexpr int kInterThreads = 256;
constexpr int kTileU = 32;                      // u rows per tile
constexpr int kTileV = 64;                      // v columns per tile
// Dp box columns v0-4 .. v0+TV+3: the innermost TMA coordinate must be a
// multiple of 16 bytes (measured on B200: an unaligned x traps as an illegal
// instruction), so the left halo is 4 columns wide instead of 1.
constexpr int kBoxW = kTileV + 8;
constexpr int kBoxX0 = 4;                       // columns left of v0 in the box
constexpr int kBoxH = kTileU + 4;               // Dp box rows:    u0-1 .. u0+TU+2
constexpr int kBoxBytes = kBoxW * kBoxH * 4;
constexpr int kBoxBytesPadded = (kBoxBytes + 127) / 128 * 128;
constexpr int kPitchAlign = 128;                // Dp pitch: multiple of every tile width

// CVRP fast path (k_inter_fast<U>): 4 warps, tile = U rows x 128 columns,
// U = 8 for small neighbourhoods (more tiles than resident CTAs), 16 otherwise
constexpr int kFastThreads = 128;
constexpr int kFastTV = 128;
template <int U, bool TW = false>
struct FastGeom {
    static constexpr int BoxW = kFastTV + 8;                    // cols v0-4 .. v0+131 (16-byte aligned TMA x)
    static constexpr int BoxH = U + 4;                          // rows u0-1 .. u0+U+2
    static constexpr int BoxBytes = BoxW * BoxH * 4;
    static constexpr int BoxPad = (BoxBytes + 127) / 128 * 128;
    static constexpr int RowBytes = U * 80;                     // row records (bulk copy)
    static constexpr int ColBytes = kFastTV * 80;               // column records (bulk copy)
    static constexpr int RowTW = TW ? U * 64 : 0;               // time-window parts
    static constexpr int ColTW = TW ? kFastTV * 64 : 0;
    // one pipeline stage = box + row/column records; two stages when a CTA
    // walks several tiles (double buffering), one when it has a single tile
    static constexpr int Stage = BoxPad + RowBytes + ColBytes + RowTW + ColTW;
    static constexpr int Smem = 2 * Stage + 128;
    static constexpr int Smem1 = Stage + 128;
    static_assert(RowBytes % 128 == 0 && ColBytes % 128 == 0 && Stage % 128 == 0, "bulk copy alignment");
};
constexpr int kGuard = 8;                       // guard slots before/after every slot array

template <class DT>
struct ScanArgs {
    int n_nodes;
    const DT *C;
    const int32_t *demand;
    const TwRec *node_tw;
    const int32_t *node;
    const int32_t *rbase, *rlenR;
    int32_t *fwdL, *bwdL;
    DT *enext, *fwdD, *bwdD;
    DT *bridge1, *bridge2, *bridge3;
    TwRec *fwdT, *bwdT, *seg2T, *seg3T;
    int32_t *rW;
    float *rTV;
    DT *rD;
    const int32_t *canon;
    int32_t capacity;
    int32_t pen_wQ;    // penalised fast-path records: w_load (0 = feasible-only records)
    SlotRec *rec;      // CVRP fast-path records (int DT only); may be null
    SlotTW *rectw;     // VRPTW (TW-I) fast-path records; may be null
    int32_t *nsc;      // north-star sweep column terms, SoA [kNscF][nsc_pitch] (ns_col_terms); may be null
    int32_t nsc_pitch;
    // VRPSPDTW (pickups): per node p_i, and per slot the Eq. 3a-d load records
    // (L_I, L_O, L_M, 0) of the prefix [0..x] / suffix [x..L+1]; all null without pickups
    const int32_t *pickup;
    int4 *fwdP, *bwdP;
};
// the north-star sweep's per-slot column terms (tga_ns.cu), one plane each:
// r, ne, rem0, sE0, cap - bL1, cap - fL, cap - W, cap - sS0, so0, sA0  (SlotRec fields)
constexpr int kNscF = 10;

// what an update refreshes: up to two slot ranges (the changed routes' whole
// slot capacity) with their routes, or everything (full relayout)
struct UpdateSpec {
    int lo1, hi1, lo2, hi2, r1, r2, full;
};

// per-solution device state of the device-resident step (k_pick_apply / k_update_dev)
// diagnostics: DevState::acc[kTimeline + 2b], [.. + 1] = globaltimer at the start / end of block b
// of the single-solution pick/update launch (armed by tga_solution_debug_probe)
constexpr int kTimeline = 64, kTimelineBlocks = 512, kAccWords = kTimeline + 2 * kTimelineBlocks;
struct DevState {
    int32_t *node, *route, *pos, *rlen, *canon;   // slot arrays (guarded)
    int32_t *rbase, *rlenR, *cbase;              // per route
    int32_t *scratch;                            // snapshot of a changed span (cap ints)
    uint64_t *keys;                              // 23 packed keys of the last evaluation (reset to ~0 once consumed)
    int32_t *desc;                               // [0] applied, [1..7] UpdateSpec, [8] grid-barrier count, [9] arrivals, [10] barrier generation
    unsigned long long *acc;                     // [23] candidate counts + [23] applied moves
    int32_t *slot_of;                            // ETGA node -> slot map kept current by the step (or null)
    void *Dp;
    int32_t R, Qc, Qp, pitch, slack;
};
// mask: the evaluated variants (pick); cmask: the variants whose closed-form counts are added
cudaError_t launch_pick_update(const DevState *states, const void *scans, int n_sol, bool tw, bool is_int,
                               uint32_t mask, uint32_t cmask, int max_routes, int max_cap, int blocks_per_sol,
                               cudaStream_t st, const DevState *h_state = nullptr, const void *h_scan = nullptr);

template <class DT>
cudaError_t launch_dp(DT *Dp, int pitch, const int32_t *node, const DT *C, int n, int Qp, int lo, int hi,
                      bool full, cudaStream_t st);
template <class DT>
cudaError_t launch_update(const ScanArgs<DT> &A, bool tw, DT *Dp, int pitch, int Qp, int R, const UpdateSpec &u,
                          cudaStream_t st);
template <class DT>
cudaError_t launch_scan(const ScanArgs<DT> &A, bool tw, int r_lo, int r_hi, cudaStream_t st);
template <class DT>
cudaError_t launch_inter(uint32_t mask, bool tw, const SolView<DT> &S, const CUtensorMap &map, const uint32_t *tiles,
                         int t_lo, int t_hi, const ScoreParams &sp, uint64_t *keys, int grid, cudaStream_t st);
template <class DT>
cudaError_t launch_intra(uint32_t mask, bool tw, const SolView<DT> &S, const ScoreParams &sp, int x_lo, int x_hi,
                         uint64_t *keys, cudaStream_t st, bool small_dist = false, bool warp_tw = false);
template <class DT>
cudaError_t launch_batch(uint32_t mask, bool tw, const SolView<DT> *views, const CUtensorMap *maps,
                         const uint32_t *work, int n_work, int n_sol, int max_qp, const ScoreParams &sp,
                         uint64_t *keys, int grid, cudaStream_t st, bool warp_tw = false);
// test-only DUMP instantiations (tga_debug_eval_dump): every evaluated candidate's key
// at dump[variant * pitch^2 + physical flat index]
template <class DT>
cudaError_t launch_eval_dump(uint32_t mask, bool tw, const SolView<DT> &S, const CUtensorMap &map,
                             const uint32_t *tiles, int t_lo, int t_hi, const ScoreParams &sp, uint64_t *keys,
                             int grid, int x_lo, int x_hi, bool inter, bool small_dist, bool warp_tw,
                             cudaStream_t st, unsigned long long *dump);
cudaError_t launch_inter_fast_dump(bool tw, const SlotRec *rec, const SlotTW *rectw, const CUtensorMap &map,
                                   const uint32_t *tiles, int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys,
                                   cudaStream_t st, const SolView<int32_t> &SV, const ScoreParams &sp, uint32_t imask,
                                   int x_lo, int x_hi, unsigned long long *dump);
unsigned long long launch_count();
void note_launch();
// p[0..n) = v on stream st: the per-eval key reset as a kernel node (a memset node
// between two kernels costs ~3 us more inside a graph on B200, tools/graph_floor.cu)
// pdl: launched as a programmatic dependent of its stream predecessor (it waits for it before
// writing); early: release its own dependent before that wait (see k_fill_u64)
cudaError_t launch_fill_u64(uint64_t *p, size_t n, uint64_t v, cudaStream_t st, bool pdl = false, bool early = false);

// Programmatic dependent launch (PDL): the kernel may be scheduled while its
// stream predecessor is still running; it calls pdl_wait() before its first
// global read of data any predecessor writes (griddepcontrol.wait returns once
// the predecessor grid has completed and its writes are visible), and
// pdl_trigger() once its own CTAs are all resident (so a dependent grid can
// never take the SM slots a grid barrier of this kernel waits for).
// Enabled per launch site with TGA_PDL_MODE (see pdl_enabled; off by default).
bool pdl_enabled(int which = 1);
// One-time per-device setup (kernel attributes, occupancy-derived capacities):
// f(dev) runs once per CUDA device ordinal, thread-safely; callers index their
// cached values by the returned ordinal (a process may drive several devices).
constexpr int kMaxDevices = 64;
struct PerDevice {
    std::once_flag flag[kMaxDevices];
};
template <class F>
int once_per_device(PerDevice &pd, F f) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = kMaxDevices - 1;
    std::call_once(pd.flag[dev], f, dev);
    return dev;
}
// cooperative != 0: the launch guarantees that every block of the grid is resident
// at once (or fails with cudaErrorCooperativeLaunchTooLarge instead of deadlocking)
// -- required by kernels whose blocks wait for each other (grid barriers).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(int which, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       int cooperative, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled(which) ? 1 : 0;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = cooperative;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// population batch on the fast path: per-solution pointers, work = (k << 20 | I << 10 | J)
struct FastSol {
    const SlotRec *rec;
    const SlotTW *rectw;
    uint64_t *keys;
    uint32_t Qc;
    int32_t pad;
};
cudaError_t launch_inter_fast_batch(int U, bool tw, uint32_t mask, const FastSol *sols, const CUtensorMap *maps,
                                    const uint32_t *work, int n_work, int32_t cap, const ScoreParams &sp,
                                    int max_grid, cudaStream_t st);
// edge-based inter-route evaluation (ETGA): cells [w_lo, w_hi) of
// {customer pairs of the edge mask} + {customer, start depot} + {start depot pairs}
struct EtgaArgs {
    const SlotRec *rec;
    const SlotTW *rectw;
    const int32_t *Dp;
    int pitch;
    uint32_t Qc;
    const int32_t *node, *pos, *rlen, *rbase;
    int32_t *slot_of;
    const int2 *pairs;
    int n_pairs, n_cust, R, Qp;
    int32_t cap;
    uint64_t *keys;
    unsigned long long *counts;   // per-variant evaluated candidates (may be null)
    int w_lo, w_hi, sm_count;
};
cudaError_t launch_etga(uint32_t mask, bool tw, const EtgaArgs &a, cudaStream_t st, bool build_slot_of);
// north-star sweep (tga_ns.cu): 2-opt* + relocate + swap (1,1), CVRP feasible-only;
// rw rows per warp (4, 8, 16: tiles of 4 rw x 128), tiles [t_lo, t_hi) of its plan
// (ns_tile_count); nsc: the column-term planes (ScanArgs::nsc); map: Dp with box
// {ns_box_cols(), ns_box_rows(rw)} (one warp's rows + halo); after_reset: the
// stream predecessor is the key reset (launch_fill_u64), so the sweep is launched as its
// programmatic dependent
int ns_rows_per_warp(int Qp, int sm_count);
int ns_tile_count(int Qp, int rw);
int ns_box_rows(int rw);
int ns_box_cols();
cudaError_t launch_ns_sweep(int rw, const SlotRec *rec, const int32_t *nsc, int pitch, const CUtensorMap &map, int Qp,
                            int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys, bool after_reset,
                            cudaStream_t st, unsigned long long *dump);
cudaError_t launch_inter_fast(int U, uint32_t mask, const SlotRec *rec, const SlotTW *rectw, const CUtensorMap &map,
                              const uint32_t *tiles, int t_lo, int t_hi, uint32_t Qc, int32_t cap, uint64_t *keys,
                              int max_grid, cudaStream_t st, const SolView<int32_t> &SV, const ScoreParams &sp,
                              uint32_t imask, int x_lo, int x_hi);

}  // namespace tga
