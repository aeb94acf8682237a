// sdmm_gather.cu -- K4: the RBGP4 product on tcgen05 WITHOUT densification.
//
// Replaces kronsparse.sdmm._tile_worker (reference sdmm.py:148-205) for compute="bf16" when
// the dense element blocks g_b are at least 16 x 16 (the tensor-core factorisations,
// SURVEY §7 hard part 1).  Transposed formulation, per output tile (tile-row tbm of W,
// 128 batch columns n0..n0+127):
//
//     D^T (128 batch cols x tm rows) += I^T (128 x tk) * W_tile^T (tk x tm)
//
// and the MMA shapes follow the graph product instead of a dense tile:
//   M = 128 batch columns (the I slab's columns; MN-major A, 128B swizzle, as TMA lands it)
//   N = bm output rows (one g_b row block ui of the tile-row)
//   K = 16 input rows inside one g_b column block, i.e. the slab rows
//       (adj_i[ui][ink] * bk + 16 kk) -- the gather is the descriptor's start address
//   B = the compressed values of row block ui, slots (ink * bk + 16 kk): exactly the
//       (rows x d_t) tile of RcubsMatrix.values (sorted-column order, rcubs.py:79-98),
//       TMA-staged K-major with the 32/64/128-byte swizzle that matches its row length.
// A step (one g_o neighbour of the tile-row, sdmm.py:167-176) is u_i * d_i * bk/16 MMAs;
// no zero is ever multiplied, nothing is densified, and the only shared-memory traffic is
// the TMA fill, the MMA operand reads and the epilogue staging.
//
// Warp roles (192 threads): warps 0-3 epilogue (TMEM lanes 32w.. = batch columns), warp 4
// TMA producer (I slab + W tile of a step on ONE mbarrier), warp 5 TMEM allocation + MMA
// issue.  Ring of ns stages, one full / one empty barrier each: the producer of step s waits
// for the MMA commit of step s - ns.  Split-K (small N): the steps of a tile are cut into
// ksplit slices run by the CTAs of one cluster; slices > 0 park their fp32 tile in their own
// shared memory and the leader adds them over DSMEM in fixed slice order (deterministic).
//
// Implicit-im2col convolution (K3 on this kernel): A is the NHWC pixel x channel tile of the
// tap-shifted 4-D TMA box (K-major, 128B swizzle), O is NHWC.
#include "common.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <cstring>
#include <vector>

namespace rbgp4 {
namespace {

constexpr int kGThreads = 192;

// Debug builds only (option debug, RBGP4_DEBUG=1): bit 8 -- CTA (0,0,0) stamps clock64 per
// step: [0] producer issued, [1] MMA saw full, [2] MMA issue done; [3][0..3] setup / epilogue
// marks; bit 512 -- every CTA stamps %globaltimer (ns) at entry and exit.
constexpr int kGTraceSteps = 256;
constexpr int kCtaStamps = 4096;
#if RBGP4_DEBUG
__device__ unsigned long long g_gtrace[4][kGTraceSteps];
__device__ unsigned long long g_cta_stamp[2][kCtaStamps];
#endif
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void gtrace(int debug, int ev, int step) {
#if RBGP4_DEBUG
    if ((debug & 8) && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && step < kGTraceSteps)
        g_gtrace[ev][step] = clock64();
#endif
}
__device__ __forceinline__ void cta_stamp(int debug, int which, int cta_id) {
#if RBGP4_DEBUG
    if ((debug & 512) && threadIdx.x == 0 && cta_id < kCtaStamps) g_cta_stamp[which][cta_id] = gtimer();
#endif
}
constexpr int kBatch = 128;  // MMA M: batch columns (or pixels) per CTA
constexpr int kMaxMma = 256; // MMAs per step (u_i * d_i * bk / 16)
constexpr int kMaxCols = 64; // relayout partials per tile (u_i * d_i)
constexpr int kMaxSched = 256; // steps whose (adjacency slot, slab row) are staged in shared memory

struct GParams {
    int64_t n_cols, ld_out;
    int32_t tm, tk, d_o, d_t, u_i, d_i, bm, bk;
    int32_t ns;                 // ring stages
    int32_t i_bytes, w_bytes;   // per stage
    int32_t w_swz;              // W row bytes = swizzle span (32 / 64 / 128)
    int32_t ksplit, sps;        // split-K slices (cluster z) and steps per slice
    int32_t tmem_cols;
    int32_t debug;
    const int32_t *sched;       // step schedule (rbgp4_prepare) or null
    // relayout mode (rbgp4_prepare): W tiles re-laid out by g_i column block, one MMA of
    // N = d_r * bm per column block into its own TMEM columns; cols[ui][ink] = TMEM column of
    // row block ui's partial for its ink-th neighbour (summed in the epilogue)
    const int32_t *cols;
    int32_t d_r, mma_n, w_rows;  // users per column block, MMA N, W tile rows per step
    // multicast pairs (rbgp4_prepare): the u_o tile-rows of a column block form one cluster;
    // pair[tbm][s] = the tile-row reading the same I slab at step s (or -1).  Paired CTAs each
    // fetch one 64-column atom of the slab and multicast it to both, so L2 streams I once.
    const int32_t *pair;
    int32_t mc;
    int32_t sym, stage_off;  // symmetric split-K epilogue; output staging offset in the ring
    int32_t persistent, u_o; // persistent tile loop (many-wave grids); tile-rows
    // M-split: the 2 CTAs of a cluster (grid z) own the two halves of a tile's rows and run all
    // steps, each fetching one 64-column atom of the shared I slab and multicasting it to both
    int32_t msplit;
    // implicit-im2col convolution
    int32_t conv, c_in, img_h, img_w, kw, pad, relu, stride;  // img_h/img_w: OUTPUT map
};

// MMA_N (= bm, or d_r * bm in relayout mode) is a template constant so the instruction
// descriptor is an immediate: computed at run time, ptxas rematerialised it from the constant
// bank through a uniform->vector->uniform round trip before every UTCHMMA (tools/k4_trace.py)
template <bool OUT_BF16, bool CONV, int MMA_N>
__global__ void __launch_bounds__(kGThreads, 2)
gather_kernel(const __grid_constant__ CUtensorMap imap, const __grid_constant__ CUtensorMap wmap,
              const __grid_constant__ CUtensorMap omap, const GParams p,
              const int32_t *__restrict__ adj_o, const int32_t *__restrict__ adj_i) {
    extern __shared__ unsigned char smem_raw[];
    // MMA table, one uint2 per MMA of a step: x = A offset | B offset << 16 (16-byte units,
    // relative to the stage), y = TMEM column of D | 1 << 31 on the first MMA into it
    __shared__ uint2 mma_tab[kMaxMma];
    // relayout: TMEM column of each (row block, neighbour) partial, read by the epilogue
    __shared__ int32_t s_cols[kMaxCols];
    // the producer's step list, read from global memory by its lanes during setup (the first
    // slab no longer waits behind two dependent global loads)
    __shared__ int32_t s_j[kMaxSched], s_krow[kMaxSched];
    unsigned char *ring = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = p.i_bytes + p.w_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + size_t(p.ns) * stage_bytes);
    uint64_t *empty = full + p.ns;
    uint64_t *tmem_full = empty + p.ns;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 0);
    const int cta_id = int(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
    cta_stamp(DBG(p.debug), 0, cta_id);
    const int64_t n0 = int64_t(blockIdx.x) * kBatch;
    const int tbm = blockIdx.y;
    const int64_t m0 = int64_t(tbm) * p.tm;
    const int half = p.msplit ? int(blockIdx.z) : 0;
    const int kslice = p.msplit ? 0 : int(blockIdx.z);
    const int n_ui = p.msplit ? p.u_i / 2 : p.u_i;  // row blocks of this CTA
    const int ui0 = half * n_ui;
    const int s_begin = kslice * p.sps;
    const int nsteps = min(p.d_o, s_begin + p.sps) - s_begin;
    const int32_t *orow = adj_o + int64_t(tbm) * p.d_o;
    const int32_t *srow = p.sched ? p.sched + int64_t(tbm) * p.d_o + s_begin : nullptr;
    const int32_t *prow = p.mc ? p.pair + int64_t(tbm) * p.d_o : nullptr;

    const bool staged_sched = nsteps <= kMaxSched;
    if (warp == 4 && staged_sched) {
        for (int i = lane; i < nsteps; i += 32) {
            const int j = srow ? srow[i] : s_begin + i;
            s_j[i] = j;
            s_krow[i] = orow[j] * p.tk;
        }
    }
    if (warp == 4 && lane == 0) {
        // empty[st] of step s completes on two arrivals in multicast mode: this CTA's release
        // of the slot and its step-s partner's (or this CTA's commit twice when unpaired)
        for (int i = 0; i < p.ns; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], (p.mc || p.msplit) ? 2 : 1); }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&imap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    }
    const int kk_n = p.bk / 16;
    const int v_blocks = p.cols ? p.u_i * p.d_i / p.d_r : 0;  // g_i column blocks (relayout)
    const int n_mma = (p.cols ? v_blocks : n_ui * p.d_i) * kk_n;
    if (warp == 5) {
        // the in-tile gather pattern g_i (x) g_b is the same for every step and tile-row
        // (sdmm.py:183-186).  Direct mode: MMA (ui, ink, kk) reads slab rows
        // adj_i[ui][ink]*bk + 16kk and compressed slots ink*bk + 16kk of row block ui.
        // Relayout mode: MMA (kb, kk) reads slab rows kb*bk + 16kk once for all d_r row
        // blocks that use column block kb (their rows are contiguous in the re-laid tile).
        for (int i = lane; i < n_mma; i += 32) {
            const int kk = i % kk_n;
            int krow, b_row, slot, dcol;
            if (p.cols) {
                const int kb = i / kk_n;
                krow = kb * p.bk + 16 * kk;
                b_row = kb * p.d_r * p.bm;
                slot = 16 * kk;
                dcol = b_row;
            } else {
                const int ink = (i / kk_n) % p.d_i, ur = i / (kk_n * p.d_i);  // ur: row block in this CTA
                krow = adj_i[(ui0 + ur) * p.d_i + ink] * p.bk + 16 * kk;
                b_row = ur * p.bm;
                slot = ink * p.bk + 16 * kk;
                dcol = ur * p.bm;
            }
            const uint32_t a_off = CONV ? uint32_t((krow / 64) * (kBatch * 128) + (krow % 64) * 2)
                                        : uint32_t(krow * 128);
            const uint32_t b_off = uint32_t(p.i_bytes + b_row * p.w_swz + slot * 2);
            mma_tab[i] = make_uint2((a_off >> 4) | ((b_off >> 4) << 16),
                                    uint32_t(dcol) | ((kk == 0 && (p.cols || slot == 0)) ? 0x80000000u : 0u));
        }
        if (p.cols)
            for (int i = lane; i < p.u_i * p.d_i; i += 32) s_cols[i] = p.cols[i];
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)), "r"(uint32_t(p.tmem_cols)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (p.mc || p.msplit) {
        // peers must see the initialised barriers before any multicast lands or arrives
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 1);
    // programmatic dependent launch: the next kernel in the stream may be scheduled now (its
    // setup overlaps this kernel); it waits in griddepcontrol.wait before reading anything
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 4) {
        // ================= TMA producer: I slab + W tile of each step, one barrier ======
        // The weights are never the previous kernel's output: the W tiles of the first ring's
        // worth of steps are requested before waiting on it.  The I slabs may be its output, so
        // they wait (griddepcontrol.wait is a no-op without a programmatic dependency).
        const int pre = (DBG(p.debug) & 128) ? 0 : min(p.ns, nsteps);
        if (elect_one()) {
            for (int s = 0; s < pre; ++s) {
                const int j = staged_sched ? s_j[s] : srow ? srow[s] : s_begin + s;
                mbar_expect_tx(&full[s], uint32_t(stage_bytes));
                unsigned char *wdst = ring + size_t(s) * stage_bytes + p.i_bytes;
                if (p.cols)
                    tma_load_2d(wdst, &wmap, &full[s], 0, (tbm * p.d_o + j) * p.w_rows);
                else
                    tma_load_2d(wdst, &wmap, &full[s], j * p.d_t, int32_t(m0) + ui0 * p.bm);
            }
        }
        __syncwarp();
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int s = 0; s < nsteps; ++s) {
            const int st = s % p.ns;
            if (DBG(p.debug) & 256) mbar_wait_sleep(&empty[st], ((s / p.ns) & 1) ^ 1, 64);
            else mbar_wait(&empty[st], ((s / p.ns) & 1) ^ 1);
            // g_o adjacency slot of this step and its first slab row
            const int j = staged_sched ? s_j[s] : srow ? srow[s] : s_begin + s;
            const int32_t krow = staged_sched ? s_krow[s] : orow[j] * p.tk;
            const bool leader = elect_one();
            if (leader && (DBG(p.debug) & 128)) {
                mbar_arrive(&full[st]);  // ablation: no loads (MMA / pipeline skeleton only)
                gtrace(DBG(p.debug), 0, s);
            } else if (leader) {
                if (s >= pre) mbar_expect_tx(&full[st], uint32_t(stage_bytes));
                unsigned char *dst = ring + size_t(st) * stage_bytes;
                if constexpr (CONV) {
                    // K rows [krow, krow + tk) = tap (i, j), channels [c0, c0 + tk): per 64-channel
                    // atom one 4-D box of 128 pixels (rows of the map, tap-shifted; OOB = padding)
                    const int tap = krow / p.c_in, c0 = krow - tap * p.c_in;
                    const int ti = tap / p.kw, tj = tap - ti * p.kw;
                    const int hw = p.img_h * p.img_w;
                    const int b0 = int(n0 / hw), h0 = int(n0 % hw) / p.img_w;
                    const int pb = p.mc ? prow[s] : p.msplit ? 1 - half : -1;
                    const int me = p.msplit ? half : tbm;
                    for (int a = 0; a < p.tk / 64; ++a) {
                        if (pb >= 0 && p.msplit) {  // row halves: channel atoms alternate, both receive
                            if ((a & 1) != half) continue;
                            tma_load_4d_mc(dst + a * (kBatch * 128), &imap, &full[st], c0 + 64 * a,
                                           tj - p.pad, h0 * p.stride + ti - p.pad, b0, uint16_t(3u));
                        } else if (pb >= 0) {  // paired: channel atoms alternate between the two CTAs
                            if ((a & 1) != (me < pb ? 0 : 1)) continue;
                            tma_load_4d_mc(dst + a * (kBatch * 128), &imap, &full[st], c0 + 64 * a,
                                           tj - p.pad, h0 * p.stride + ti - p.pad, b0,
                                           uint16_t((1u << tbm) | (1u << pb)));
                        } else {
                            tma_load_4d(dst + a * (kBatch * 128), &imap, &full[st], c0 + 64 * a,
                                        tj - p.pad, h0 * p.stride + ti - p.pad, b0);
                        }
                    }
                } else if (p.msplit) {
                    // the two row halves share every slab: fetch atom `half` for both CTAs
                    tma_load_3d_mc(dst + half * p.tk * 128, &imap, &full[st], 0, krow, int32_t(n0 / 64) + half,
                                   uint16_t(3u));
                } else if (p.mc) {
                    // one-atom boxes (64 cols x tk rows); paired: fetch atom h for both CTAs
                    const int pb = prow[s];
                    if (pb >= 0) {
                        const int h = tbm < pb ? 0 : 1;
                        tma_load_3d_mc(dst + h * p.tk * 128, &imap, &full[st], 0, krow, int32_t(n0 / 64) + h,
                                       uint16_t((1u << tbm) | (1u << pb)));
                    } else {
                        tma_load_3d(dst, &imap, &full[st], 0, krow, int32_t(n0 / 64));
                        tma_load_3d(dst + p.tk * 128, &imap, &full[st], 0, krow, int32_t(n0 / 64) + 1);
                    }
                } else {
                    // (64 cols, tk rows, 2 atoms) box: MN-major, atom-major in shared memory
                    tma_load_3d(dst, &imap, &full[st], 0, krow, int32_t(n0 / 64));
                }
                if (s < pre) {
                    // W tile already requested before griddepcontrol.wait
                } else if (p.cols)  // re-laid tiles: (bk, rows) view, tile (tbm, j) = w_rows rows
                    tma_load_2d(dst + p.i_bytes, &wmap, &full[st], 0, (tbm * p.d_o + j) * p.w_rows);
                else  // this CTA's rows of the compressed tile
                    tma_load_2d(dst + p.i_bytes, &wmap, &full[st], j * p.d_t, int32_t(m0) + ui0 * p.bm);
                gtrace(DBG(p.debug), 0, s);
            }
            __syncwarp();
        }
    } else if (warp == 5) {
        // ================= MMA issuer =================
        const uint32_t tmem_d = *tmem_slot;
        // idesc: D f32, A/B bf16, A MN-major (SDMM: I slab) or K-major (conv: NHWC tile),
        // B K-major (compressed W rows), N = bm, M = 128
        const uint32_t a_mn = CONV ? 0u : 1u;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (0u << 16) |
                               (uint32_t(MMA_N >> 3) << 17) | (uint32_t(kBatch >> 4) << 24);
        const uint32_t ring_a = smem_u32(ring);
        const uint32_t w_code = p.w_swz == 128 ? 2u : p.w_swz == 64 ? 4u : 6u;
        // descriptors of stage 0; a stage / table entry only moves the 14-bit start field
        const uint64_t a_desc0 = CONV ? smem_desc(ring_a, 0, 1024, 2u)
                                      : smem_desc(ring_a, uint32_t(p.tk) * 128, 1024, 2u);
        const uint64_t b_desc0 = smem_desc(ring_a, 0, 8 * p.w_swz, w_code);
        // up to kRegMma table entries live in registers for the whole kernel (plain shared
        // loads the compiler can hoist); larger patterns stream the table from shared memory
        constexpr int kRegMma = 32;
        uint32_t rx[kRegMma], ry[kRegMma];
#pragma unroll
        for (int i = 0; i < kRegMma; ++i) {
            const uint2 e = i < n_mma ? mma_tab[i] : make_uint2(0, 0);
            rx[i] = e.x;
            ry[i] = e.y;
        }
        const bool in_regs = n_mma <= kRegMma;
        const bool no_mma = DBG(p.debug) & 2;
        const bool fast8 = MMA_N == 32 && p.cols && p.bk == 16 && v_blocks == 8 && p.w_swz == 32 &&
                           !(DBG(p.debug) & 16384);
        for (int s = 0; s < nsteps; ++s) {
            const int st = s % p.ns;
            mbar_wait(&full[st], (s / p.ns) & 1);
            tc_fence_after();
            if (elect_one()) {
                gtrace(DBG(p.debug), 1, s);
                const uint32_t st16 = uint32_t(st * stage_bytes) >> 4;
                const uint64_t a_st = a_desc0 + st16, b_st = b_desc0 + st16;
                if (no_mma) {
                } else if (fast8) {
                    // relayout, TC16 factorisation (8 column blocks of 16 rows, N = 32): every
                    // offset is an immediate, so a step is 8 UTCHMMAs and a few uniform adds.
                    // A rows kb*16..+15: SDMM slab rows of 128 B; conv: 32-byte K offset inside
                    // the 64-channel atom (kb % 4) of atom kb / 4
                    const uint32_t acc = s > 0 ? 1u : 0u;
                    const uint64_t bd = b_st + (uint32_t(p.i_bytes) >> 4);
#pragma unroll
                    for (int kb = 0; kb < 8; ++kb) {
                        constexpr uint32_t kAtom16 = uint32_t(kBatch * 128) >> 4;
                        const uint32_t a16 = CONV ? uint32_t(kb / 4) * kAtom16 + uint32_t(kb % 4) * 2
                                                  : uint32_t(kb * 16 * 8);
                        tc_mma<false>(tmem_d + uint32_t(kb * MMA_N), a_st + a16,
                                      bd + uint32_t(kb * ((MMA_N * 32) >> 4)), idesc, acc);
                    }
                } else if (p.cols) {
                    // relayout: every descriptor is uniform arithmetic of (kb, kk) -- no table,
                    // no register-to-uniform moves on the issue path
                    const uint32_t n_blk = uint32_t(p.d_r * p.bm);
                    const uint32_t b_blk16 = (n_blk * uint32_t(p.w_swz)) >> 4;
                    uint64_t bd = b_st + (uint32_t(p.i_bytes) >> 4);
                    uint32_t dcol = tmem_d;
                    for (int kb = 0; kb < v_blocks; ++kb) {
                        for (int kk = 0; kk < kk_n; ++kk) {
                            const uint32_t krow = uint32_t(kb * p.bk + 16 * kk);
                            const uint32_t a16 = CONV ? (((krow >> 6) * (kBatch * 128)) + (krow & 63) * 2) >> 4
                                                      : krow * 8;  // krow * 128 bytes
                            tc_mma<false>(dcol, a_st + a16, bd + uint32_t(2 * kk), idesc,
                                          (s > 0 || kk > 0) ? 1u : 0u);
                        }
                        bd += b_blk16;
                        dcol += n_blk;
                    }
                } else if (in_regs) {
#pragma unroll
                    for (int i = 0; i < kRegMma; ++i)
                        if (i < n_mma)
                            tc_mma<false>(tmem_d + (ry[i] & 0xFFFFu), a_st + (rx[i] & 0xFFFFu), b_st + (rx[i] >> 16),
                                          idesc, (s > 0 || !(ry[i] >> 31)) ? 1u : 0u);
                } else {
                    for (int i = 0; i < n_mma; ++i) {
                        const uint2 e = mma_tab[i];
                        tc_mma<false>(tmem_d + (e.y & 0xFFFFu), a_st + (e.x & 0xFFFFu), b_st + (e.x >> 16), idesc,
                                      (s > 0 || !(e.y >> 31)) ? 1u : 0u);
                    }
                }
                if (p.msplit) {
                    tc_commit_mc(&empty[st], uint16_t(3u));  // both halves fill every slot
                } else if (p.mc) {
                    // release slot st for step s + ns to the CTAs that will fill it: this one and
                    // its step-(s + ns) partner
                    const int sn = s + p.ns;
                    const int pb = sn < nsteps ? prow[sn] : -1;
                    if (pb >= 0) {
                        tc_commit_mc(&empty[st], uint16_t((1u << tbm) | (1u << pb)));
                    } else {
                        tc_commit(&empty[st]);
                        tc_commit(&empty[st]);
                    }
                } else {
                    tc_commit(&empty[st]);
                }
                gtrace(DBG(p.debug), 2, s);
            }
            __syncwarp();
        }
        if (elect_one()) tc_commit(tmem_full);
        __syncwarp();
        if (!(DBG(p.debug) & (4096 | 8192))) {
            // hand the accumulator to the epilogue warps through a named barrier: they sleep
            // in bar.sync for the whole main loop instead of polling tmem_full (polling warps
            // measured to slow this warp's MMA issue)
            mbar_wait(tmem_full, 0);
            tc_fence_before();
            asm volatile("bar.arrive 2, 160;" ::: "memory");
        }
    } else {
        // ================= epilogue (warps 0-3): TMEM lane = batch column =================
        if (DBG(p.debug) & 4096) mbar_wait_sleep(tmem_full, 0, 256);  // A/B: polling with back-off
        else if (DBG(p.debug) & 8192) mbar_wait_parked(tmem_full, 0);
        else asm volatile("bar.sync 2, 160;" ::: "memory");
        tc_fence_after();
        if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 2);
    }

    const uint32_t tmem_d = *tmem_slot;
    const uint32_t ring_a = smem_u32(ring);
    const int t = warp * 32 + lane;  // batch column inside the tile (warps 0-3)
    const uint32_t lane_base = tmem_d + (uint32_t(warp * 32) << 16);
    // output rows c..c+31 of this thread's batch column: direct mode reads the accumulator
    // columns as they are; relayout mode sums each row block's d_i partial accumulators
    auto load_rows = [&](int c, uint32_t (&r)[32]) {
        if (!p.cols) {
            TMEM_LD_32x32b_X32(lane_base + uint32_t(c), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            return;
        }
        if (p.d_i == 2) {
            uint32_t v[2][2][16];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int row = c + 16 * h, ui = row / p.bm, m = row % p.bm;
#pragma unroll
                for (int ink = 0; ink < 2; ++ink)
                    TMEM_LD_32x32b_X16(lane_base + uint32_t(s_cols[ui * 2 + ink] + m), v[h][ink]);
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    r[16 * h + q] = __float_as_uint(__uint_as_float(v[h][0][q]) + __uint_as_float(v[h][1][q]));
            return;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int row = c + 16 * h, ui = row / p.bm, m = row % p.bm;
            float acc[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] = 0.0f;
            for (int ink = 0; ink < p.d_i; ++ink) {
                uint32_t v[16];
                TMEM_LD_32x32b_X16(lane_base + uint32_t(s_cols[ui * p.d_i + ink] + m), v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < 16; ++q) acc[q] += __uint_as_float(v[q]);
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) r[16 * h + q] = __float_as_uint(acc[q]);
        }
    };
    // ---- output rows of this CTA: everything (no split), nothing (legacy split, slices > 0),
    // or its own 1/ksplit of the rows (symmetric split: each slice reduces and stores a part)
    const int rp = p.msplit ? p.tm / 2 : p.sym ? p.tm / p.ksplit : p.tm;
    const int r_lo = p.msplit ? half * rp : p.sym ? kslice * rp : 0;
    const int t_lo = p.msplit ? r_lo : 0;  // TMEM holds only this CTA's rows in M-split mode
    const bool outputs = p.sym || p.msplit || kslice == 0;
    // symmetric split: receive buffer [source slot][rp rows][128 cols] fp32 at the ring start,
    // output staging after it
    const uint32_t recv = ring_a;
    const uint32_t stage_base = ring_a + uint32_t(p.sym ? p.stage_off : 0);
    unsigned char *stage_ptr = ring + (p.sym ? p.stage_off : 0);
    if (p.ksplit > 1 && p.sym) {
        // the receive buffers alias the rings: every slice's main loop must be over (slices run
        // different step counts) before any partial lands in a peer
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 4);
        if (warp < 4) {
            // push the partial rows other slices own: posted DSMEM stores into their receive buffer
            for (int c = 0; c < p.tm; c += 32) {
                const int owner = c / rp;
                if (owner == kslice) continue;
                uint32_t r[32];
                load_rows(c, r);
                const int slot = kslice < owner ? kslice : kslice - 1;
                // generic address of the owner's receive row (mapa on a generic address), then
                // plain stores the compiler can issue back to back (volatile asm serialised them)
                float *mine = reinterpret_cast<float *>(ring) + (int64_t(slot) * rp + (c - owner * rp)) * kBatch + t;
                float *dstp;
                asm volatile("mapa.u64 %0, %1, %2;" : "=l"(dstp) : "l"(mine), "r"(owner));
#pragma unroll
                for (int q = 0; q < 32; ++q) dstp[q * kBatch] = __uint_as_float(r[q]);
            }
        }
        if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 5);
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 6);
    } else if (p.ksplit > 1) {
        // legacy: slices > 0 park the whole fp32 partial tile in their own shared memory
        if (kslice > 0 && warp < 4) {
            for (int c = 0; c < p.tm; c += 32) {
                uint32_t r[32];
                load_rows(c, r);
#pragma unroll
                for (int q = 0; q < 32; ++q) sts32(ring_a + uint32_t(((c + q) * kBatch + t) * 4), r[q]);
            }
        }
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (outputs && warp < 4 && !(DBG(p.debug) & 4)) {
        constexpr int kOutElt = OUT_BF16 ? 2 : 4;
        for (int c = r_lo; c < r_lo + rp; c += 32) {
            uint32_t r[32];
            load_rows(c - t_lo, r);
            if (DBG(p.debug) & 1024) {
                if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 9);
            } else if (p.sym) {
                // plain shared loads (the static __shared__ base keeps them LDS) so ptxas can keep
                // all of them in flight; volatile asm loads measured latency-serialised
                const float *rb = reinterpret_cast<const float *>(smem_raw + (ring - smem_raw));
                for (int k = 0; k < p.ksplit - 1; ++k) {
                    const float *src = rb + (int64_t(k) * rp + (c - r_lo)) * kBatch + t;
#pragma unroll
                    for (int q = 0; q < 32; ++q)
                        r[q] = __float_as_uint(__uint_as_float(r[q]) + src[q * kBatch]);
                }
            } else {
                for (int k = 1; k < p.ksplit; ++k) {
                    // peer slice k's partial, same offsets in its shared memory (DSMEM)
                    uint32_t peer;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(ring_a), "r"(k));
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        float v;
                        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v)
                                     : "r"(peer + uint32_t(((c + q) * kBatch + t) * 4)));
                        r[q] = __float_as_uint(__uint_as_float(r[q]) + v);
                    }
                }
            }
            const int cr = c - r_lo;  // row inside this CTA's output range
            if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 10);
            if (DBG(p.debug) & 2048) continue;
            if constexpr (CONV) {
                // NHWC: pixel t holds channels c..c+31 -> 4 x 16-byte chunks of its 128-byte
                // rows in 64-channel atoms [atom][pixel][128 B], 128B-swizzled (chunk ^ pixel%8)
#pragma unroll
                for (int q = 0; q < 32; ++q)
                    if (p.relu) r[q] = __float_as_uint(fmaxf(__uint_as_float(r[q]), 0.0f));
                if constexpr (OUT_BF16) {
                    const uint32_t atom = stage_base + uint32_t((cr / 64) * (kBatch * 128) + t * 128);
                    const uint32_t ch0 = uint32_t(cr % 64) / 8;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t w[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r[q * 8 + 2 * h]),
                                                                      __uint_as_float(r[q * 8 + 2 * h + 1]));
                            w[h] = *reinterpret_cast<uint32_t *>(&b2);
                        }
                        sts128(atom + (((ch0 + q) ^ uint32_t(t & 7)) << 4), w[0], w[1], w[2], w[3]);
                    }
                } else {
                    const uint32_t atom = stage_base + uint32_t((cr / 32) * (kBatch * 128) + t * 128);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        sts128(atom + ((uint32_t(q) ^ uint32_t(t & 7)) << 4), r[4 * q], r[4 * q + 1],
                               r[4 * q + 2], r[4 * q + 3]);
                }
            } else {
                // row-major O: column t of rows c..c+31 -> [atom of 128/elt cols][row][128 B],
                // 128B-swizzled (chunk ^ row%8); lanes = consecutive columns
                constexpr int kAtomCols = 128 / kOutElt;
                const uint32_t atom = stage_base + uint32_t((t / kAtomCols) * (rp * 128));
                const uint32_t cb = uint32_t(t % kAtomCols) * kOutElt;  // byte inside the row
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const uint32_t row = uint32_t(cr + q);
                    const uint32_t addr = atom + row * 128 + ((((cb >> 4) ^ (row & 7))) << 4) + (cb & 15);
                    if constexpr (OUT_BF16) {
                        const __nv_bfloat16 bv = __float2bfloat16_rn(__uint_as_float(r[q]));
                        sts16(addr, *reinterpret_cast<const uint16_t *>(&bv));
                    } else {
                        sts32(addr, r[q]);
                    }
                }
            }
        }
        if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 7);
        fence_async_smem();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 8);
        if (warp == 0 && elect_one()) {
            if constexpr (CONV) {
                constexpr int kAtomCh = 128 / kOutElt;
                for (int a = 0; a < rp / kAtomCh; ++a)
                    tma_store_2d(&omap, stage_ptr + a * (kBatch * 128), int32_t(m0) + r_lo + a * kAtomCh,
                                 int32_t(n0));
            } else {
                constexpr int kAtomCols = 128 / kOutElt;
                for (int a = 0; a < kBatch / kAtomCols; ++a)
                    tma_store_2d(&omap, stage_ptr + a * (rp * 128), int32_t(n0) + a * kAtomCols,
                                 int32_t(m0) + r_lo);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
    }
    if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 3);
    if ((p.ksplit > 1 && !p.sym) || p.mc || p.msplit) {
        // peers keep their shared memory alive until the leader has read it (legacy split);
        // multicast peers may still arrive on this CTA's barriers
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                     "r"(uint32_t(p.tmem_cols)));
    }
    cta_stamp(DBG(p.debug), 1, cta_id);
}

// ---------------------------------------------------------------- persistent variant
// Many-wave grids (e.g. the VGG layers at batch 32768: 16k+ tiles): one CTA per SM loops over
// tiles (column block-major, so the u_o tile-rows sharing a slab run side by side).  The ring
// and its phases continue across tiles; the accumulator is double-buffered in TMEM, so the
// epilogue warps drain tile i (straight from registers to global memory, coalesced) while the
// MMA warp already accumulates tile i+1 and the producer streams without a pipeline restart.
// Setup, TMEM allocation and the first-load latency are paid once per SM instead of per tile.
template <bool OUT_BF16, bool CONV, int MMA_N>
__global__ void __launch_bounds__(kGThreads, 1)
gather_persistent_kernel(const __grid_constant__ CUtensorMap imap, const __grid_constant__ CUtensorMap wmap,
                         const GParams p, const int32_t *__restrict__ adj_o, const int32_t *__restrict__ adj_i,
                         void *__restrict__ out, int64_t n_tiles) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ uint2 mma_tab[kMaxMma];
    __shared__ int32_t s_cols[kMaxCols];  // relayout: TMEM column of each (row block, neighbour) partial
    unsigned char *ring = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = p.i_bytes + p.w_bytes;
    // relayout (TC16 only here, the immediate-offset loop): 8 MMAs of N = 32 per step into the
    // tile's d_i partial accumulators (tm * d_i columns per buffer)
    const bool rl = p.cols != nullptr;
    const int acc_cols = rl ? p.tm * p.d_i : p.tm;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + size_t(p.ns) * stage_bytes);
    uint64_t *empty = full + p.ns;
    uint64_t *acc_full = empty + p.ns;     // [2]: last MMA of a tile committed
    uint64_t *acc_empty = acc_full + 2;    // [2]: the epilogue has read the accumulator
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int kk_n = p.bk / 16;
    const int n_mma = p.u_i * p.d_i * kk_n;
    const int u_o = p.u_o;
    if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 0);
    cta_stamp(DBG(p.debug), 0, int(blockIdx.x));

    if (warp == 4 && lane == 0) {
        for (int i = 0; i < p.ns; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 4); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&imap)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    }
    if (warp == 5) {
        for (int i = lane; i < n_mma; i += 32) {
            const int kk = i % kk_n, ink = (i / kk_n) % p.d_i, ui = i / (kk_n * p.d_i);
            const int krow = adj_i[ui * p.d_i + ink] * p.bk + 16 * kk;
            const int slot = ink * p.bk + 16 * kk;
            const uint32_t a_off = CONV ? uint32_t((krow / 64) * (kBatch * 128) + (krow % 64) * 2)
                                        : uint32_t(krow * 128);
            const uint32_t b_off = uint32_t(p.i_bytes + ui * p.bm * p.w_swz + slot * 2);
            mma_tab[i] = make_uint2((a_off >> 4) | ((b_off >> 4) << 16),
                                    uint32_t(ui * p.bm) | (slot == 0 ? 0x80000000u : 0u));
        }
        if (rl)
            for (int i = lane; i < p.u_i * p.d_i; i += 32) s_cols[i] = p.cols[i];
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)), "r"(uint32_t(p.tmem_cols)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint32_t tmem_d = *tmem_slot;
    if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 1);

    if (warp == 4) {
        // ================= producer: I slab + W tile of every step of every tile =================
        asm volatile("griddepcontrol.wait;" ::: "memory");
        int64_t g = 0;
        for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            const int tbm = int(tile % u_o);
            const int64_t n0 = (tile / u_o) * kBatch;
            const int32_t *orow = adj_o + int64_t(tbm) * p.d_o;
            const int32_t *srow = p.sched ? p.sched + int64_t(tbm) * p.d_o : nullptr;
            for (int s = 0; s < p.d_o; ++s, ++g) {
                const int st = int(g % p.ns);
                mbar_wait(&empty[st], uint32_t((g / p.ns) & 1) ^ 1u);
                const int j = srow ? srow[s] : s;
                const int32_t krow = orow[j] * p.tk;
                if (elect_one()) {
                    mbar_expect_tx(&full[st], uint32_t(stage_bytes));
                    unsigned char *dst = ring + size_t(st) * stage_bytes;
                    if constexpr (CONV) {
                        const int tap = krow / p.c_in, c0 = krow - tap * p.c_in;
                        const int ti = tap / p.kw, tj = tap - ti * p.kw;
                        const int hw = p.img_h * p.img_w;
                        const int b0 = int(n0 / hw), h0 = int(n0 % hw) / p.img_w;
                        for (int a = 0; a < p.tk / 64; ++a)
                            tma_load_4d(dst + a * (kBatch * 128), &imap, &full[st], c0 + 64 * a, tj - p.pad,
                                        h0 * p.stride + ti - p.pad, b0);
                    } else {
                        tma_load_3d(dst, &imap, &full[st], 0, krow, int32_t(n0 / 64));
                    }
                    if (rl)  // re-laid tiles: (bk, rows) view, tile (tbm, j) = w_rows rows
                        tma_load_2d(dst + p.i_bytes, &wmap, &full[st], 0, (tbm * p.d_o + j) * p.w_rows);
                    else
                        tma_load_2d(dst + p.i_bytes, &wmap, &full[st], j * p.d_t, tbm * p.tm);
                    gtrace(DBG(p.debug), 0, int(g));
                }
                __syncwarp();
            }
        }
    } else if (warp == 5) {
        // ================= MMA issuer: accumulator b = tile parity =================
        const uint32_t a_mn = CONV ? 0u : 1u;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (0u << 16) |
                               (uint32_t(MMA_N >> 3) << 17) | (uint32_t(kBatch >> 4) << 24);
        const uint32_t ring_a = smem_u32(ring);
        const uint32_t w_code = p.w_swz == 128 ? 2u : p.w_swz == 64 ? 4u : 6u;
        const uint64_t a_desc0 = CONV ? smem_desc(ring_a, 0, 1024, 2u) : smem_desc(ring_a, uint32_t(p.tk) * 128, 1024, 2u);
        const uint64_t b_desc0 = smem_desc(ring_a, 0, 8 * p.w_swz, w_code);
        constexpr int kRegMma = 32;
        uint32_t rx[kRegMma], ry[kRegMma];
#pragma unroll
        for (int i = 0; i < kRegMma; ++i) {
            const uint2 e = i < n_mma ? mma_tab[i] : make_uint2(0, 0);
            rx[i] = e.x;
            ry[i] = e.y;
        }
        int64_t g = 0, it = 0;
        for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const int b = int(it & 1);
            mbar_wait(&acc_empty[b], uint32_t((it >> 1) & 1) ^ 1u);  // epilogue done with it
            tc_fence_after();
            const uint32_t d_base = tmem_d + uint32_t(b * acc_cols);
            for (int s = 0; s < p.d_o; ++s, ++g) {
                const int st = int(g % p.ns);
                mbar_wait(&full[st], uint32_t((g / p.ns) & 1));
                tc_fence_after();
                if (elect_one()) {
                    gtrace(DBG(p.debug), 1, int(g));
                    const uint32_t st16 = uint32_t(st * stage_bytes) >> 4;
                    const uint64_t a_st = a_desc0 + st16, b_st = b_desc0 + st16;
                    if constexpr (MMA_N == 32) {
                        if (rl) {  // same immediate-offset step as gather_kernel's fast path
                            const uint32_t acc = s > 0 ? 1u : 0u;
                            const uint64_t bd = b_st + (uint32_t(p.i_bytes) >> 4);
#pragma unroll
                            for (int kb = 0; kb < 8; ++kb) {
                                constexpr uint32_t kAtom16 = uint32_t(kBatch * 128) >> 4;
                                const uint32_t a16 = CONV ? uint32_t(kb / 4) * kAtom16 + uint32_t(kb % 4) * 2
                                                          : uint32_t(kb * 16 * 8);
                                tc_mma<false>(d_base + uint32_t(kb * MMA_N), a_st + a16,
                                              bd + uint32_t(kb * ((MMA_N * 32) >> 4)), idesc, acc);
                            }
                        }
                    }
                    if (rl) {
                    } else if (n_mma <= kRegMma) {
#pragma unroll
                        for (int i = 0; i < kRegMma; ++i)
                            if (i < n_mma)
                                tc_mma<false>(d_base + (ry[i] & 0xFFFFu), a_st + (rx[i] & 0xFFFFu), b_st + (rx[i] >> 16),
                                              idesc, (s > 0 || !(ry[i] >> 31)) ? 1u : 0u);
                    } else {
                        for (int i = 0; i < n_mma; ++i) {
                            const uint2 e = mma_tab[i];
                            tc_mma<false>(d_base + (e.y & 0xFFFFu), a_st + (e.x & 0xFFFFu), b_st + (e.x >> 16), idesc,
                                          (s > 0 || !(e.y >> 31)) ? 1u : 0u);
                        }
                    }
                    tc_commit(&empty[st]);
                    if (s == p.d_o - 1) tc_commit(&acc_full[b]);
                    gtrace(DBG(p.debug), 2, int(g));
                }
                __syncwarp();
            }
        }
    } else {
        // ================= epilogue (warps 0-3): TMEM lane = batch column / pixel =================
        const int t = warp * 32 + lane;
        int64_t it = 0;
        for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
            const int b = int(it & 1);
            const int tbm = int(tile % u_o);
            const int64_t n0 = (tile / u_o) * kBatch;
            const int64_t m0 = int64_t(tbm) * p.tm;
            if (DBG(p.debug) & 4096) mbar_wait_sleep(&acc_full[b], uint32_t((it >> 1) & 1), 64);
            else mbar_wait_parked(&acc_full[b], uint32_t((it >> 1) & 1));
            tc_fence_after();
            if (threadIdx.x == 0 && it < 4) gtrace(DBG(p.debug), 3, int(2 + 2 * it));
            const uint32_t lane_base = tmem_d + (uint32_t(warp * 32) << 16) + uint32_t(b * acc_cols);
            const int64_t col = n0 + t;
            const bool ok = col < p.n_cols;
            for (int c = 0; c < p.tm; c += 32) {
                uint32_t r[32];
                if (rl) {  // rows c..c+31: two 16-row halves, each the sum of its row block's 2 partials
                    uint32_t v[2][2][16];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        // row -> (row block ui, row m inside it); bm is 16 or 32 on this path
                        const int row = c + 16 * h, ui = row / p.bm, m = row - ui * p.bm;
#pragma unroll
                        for (int ink = 0; ink < 2; ++ink)
                            TMEM_LD_32x32b_X16(lane_base + uint32_t(s_cols[ui * 2 + ink] + m), v[h][ink]);
                    }
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int q = 0; q < 16; ++q)
                            r[16 * h + q] = __float_as_uint(__uint_as_float(v[h][0][q]) + __uint_as_float(v[h][1][q]));
                } else {
                    TMEM_LD_32x32b_X32(lane_base + uint32_t(c), r);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                }
                if (!ok) continue;
                if constexpr (CONV) {
                    // NHWC: this pixel's channels m0+c .. +31 are contiguous
#pragma unroll
                    for (int q = 0; q < 32; ++q)
                        if (p.relu) r[q] = __float_as_uint(fmaxf(__uint_as_float(r[q]), 0.0f));
                    if constexpr (OUT_BF16) {
                        uint4 *dst = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(out) + col * p.ld_out + m0 + c);
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            uint32_t w[4];
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(r[q * 8 + 2 * h]),
                                                                          __uint_as_float(r[q * 8 + 2 * h + 1]));
                                w[h] = *reinterpret_cast<uint32_t *>(&b2);
                            }
                            dst[q] = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    } else {
                        uint4 *dst = reinterpret_cast<uint4 *>(static_cast<float *>(out) + col * p.ld_out + m0 + c);
#pragma unroll
                        for (int q = 0; q < 8; ++q) dst[q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                    }
                } else {
                    // row-major O: lanes = consecutive columns of one row (coalesced)
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        if constexpr (OUT_BF16)
                            static_cast<__nv_bfloat16 *>(out)[(m0 + c + q) * p.ld_out + col] =
                                __float2bfloat16_rn(__uint_as_float(r[q]));
                        else
                            static_cast<float *>(out)[(m0 + c + q) * p.ld_out + col] = __uint_as_float(r[q]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (threadIdx.x == 0 && it < 4) gtrace(DBG(p.debug), 3, int(3 + 2 * it));
            if (lane == 0) mbar_arrive(&acc_empty[b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(uint32_t(p.tmem_cols)));
    }
    if (threadIdx.x == 0) gtrace(DBG(p.debug), 3, 11);
    cta_stamp(DBG(p.debug), 1, int(blockIdx.x));
}

constexpr size_t kGSmemCap = 227 * 1024;

struct GPlan {
    GParams p;
    size_t smem;
    dim3 grid;
    int64_t n_tiles;
};

CUtensorMapSwizzle swizzle_of(int span) {
    return span == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
         : span == 64  ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
}

}  // namespace

// Shapes K4 takes: bf16, g_r = (1,1), g_b blocks of >= 16 x 16 (multiples of 16), a tile-row
// of <= 256 rows (a multiple of 32), I slabs of <= 256 rows.  Direct mode needs one compressed
// W row to be a swizzle span (32/64/128 bytes); relayout mode (prepared values) needs g_i
// biregular, tm * d_i <= 256 (W tile rows per step = TMEM columns) and bk * 2 a span.
int gather_relayout_ok(const ChainDims &c) {
    if (c.rm != 1 || c.rk != 1 || c.bm % 16 || c.bk % 16 || c.tm % 32 || c.tm > 256) return 0;
    if ((c.u_i * c.d_i) % c.v_i) return 0;
    const int d_r = c.u_i * c.d_i / c.v_i;
    const int span = c.bk * 2;
    if (span != 32 && span != 64 && span != 128) return 0;
    if (c.tm * c.d_i > 256 || d_r * c.bm > 256) return 0;
    if (opts().relayout == 0) return 0;
    if (opts().relayout == 1) return 1;
    // default where the immediate-offset MMA loop applies (TC16: 8 column blocks of 16 rows,
    // N = 32, d_i = 2): half the MMAs of the direct mode and no per-MMA descriptor arithmetic.
    // Elsewhere the generic relayout loop loses to the direct mode (measured), so it is opt-in.
    return (c.bk == 16 && c.v_i == 8 && d_r * c.bm == 32 && c.d_i == 2) ? 1 : 0;
}

int gather_plan(const ChainDims &c, int compute, bool conv, bool relayout, GPlan *out, bool pairs = false) {
    if (compute != RBGP4_COMPUTE_BF16) return 0;
    if (opts().dense) return 0;  // A/B switch: force the densify kernel (K2)
    if (c.rm != 1 || c.rk != 1 || c.bm % 16 || c.bk % 16 || c.tm % 32 || c.tm > 256 || c.tk > 256) return 0;
    if (relayout && !gather_relayout_ok(c)) return 0;
    const int w_row = relayout ? c.bk * 2 : c.d_t * 2;
    if (w_row != 32 && w_row != 64 && w_row != 128) return 0;
    if (conv && c.tk % 64) return 0;
    GParams p{};
    p.n_cols = c.n_cols; p.ld_out = c.ld_out;
    p.tm = c.tm; p.tk = c.tk; p.d_o = c.d_o; p.d_t = c.d_t; p.u_i = c.u_i; p.d_i = c.d_i;
    p.bm = c.bm; p.bk = c.bk;
    p.d_r = relayout ? c.u_i * c.d_i / c.v_i : 1;
    p.mma_n = relayout ? p.d_r * c.bm : c.bm;
    p.w_rows = relayout ? c.tm * c.d_i : c.tm;
    if (p.mma_n != 16 && p.mma_n != 32 && p.mma_n != 48 && p.mma_n != 64 && p.mma_n != 128) return 0;
    const int n_mma = (relayout ? c.v_i : c.u_i * c.d_i) * (c.bk / 16);
    if (n_mma > kMaxMma) return 0;
    p.i_bytes = c.tk * kBatch * 2;
    const int64_t col_blocks = (c.n_cols + kBatch - 1) / kBatch;
    const int64_t tiles = col_blocks * c.u_o;
    // many waves: one persistent CTA per SM loops over the tiles (no split, no pairs)
    p.u_o = c.u_o;
    // (relayout: only the TC16 shape, whose immediate-offset step the persistent kernel has; there
    // the persistent loop also wins below a wave -- conv10 N = 4096: 20.8 vs 24.6 us with split-K
    // clusters, N = 8192: 30.4 vs 42.8 us, N = 1024: 19.1 vs 19.3 us -- so the SDMM always takes
    // it from half a wave up (at 32 tiles the two are even); the implicit-im2col conv measured
    // slower that way (conv_fused 78.3 -> 74.6 TF/s) and keeps the split-K clusters)
    const bool rl_fast = c.bk == 16 && c.v_i == 8 && c.d_i == 2 && c.u_i * c.d_i / c.v_i * c.bm == 32;
    p.persistent = ((tiles >= 2 * kNumSMs || (relayout && rl_fast && !conv && tiles >= kNumSMs / 2) ||
                     opts().persistent == 1) &&
                    (!relayout || rl_fast) && opts().persistent != 0) ? 1 : 0;
    // M-split (opt-in, option msplit=1): the two row halves of each tile on two CTAs (2 per
    // SM) that share every I slab by multicast and need no reduction.  Correct, but on conv10
    // it measured 30.1 us against 26.0 us for the split-K default (half the MMAs per CTA do
    // not make up for running all steps), so it is not chosen by itself.
    p.msplit = (!p.persistent && !relayout && c.u_i % 2 == 0 && (c.tm / 2) % 32 == 0 &&
                (!conv || (c.tk / 64) % 2 == 0) && opts().msplit) ? 1 : 0;
    p.w_rows = p.msplit ? c.tm / 2 : p.w_rows;
    p.w_bytes = p.w_rows * w_row;  // = tm * d_t * 2 (half of it in M-split)
    p.w_swz = w_row;
    const size_t stage = size_t(p.i_bytes) + p.w_bytes;
    // dynamic: alignment slack + barriers + ring; the static tables count against the same
    // 227 KB per-CTA limit
    const size_t fixed = 1024 + 8 * (2 * 16 + 1) + 16 + 64;
    const size_t statics = size_t(kMaxMma) * 8 + size_t(kMaxCols) * 4 + size_t(kMaxSched) * 8 + 256;
    // Occupancy: a CTA's steps are a serial latency chain (load -> MMA issue -> commit), so
    // when one tile per SM would leave SMs idle, the steps of a tile are split over a cluster
    // (DSMEM reduction) and two CTAs share an SM with 2-stage rings (measured on the VGG
    // shapes: 2 CTAs/SM x 2 stages beats 1 CTA/SM x 5 stages).  Large grids keep 1 CTA/SM
    // with the deepest ring that fits.
    int ks = 1;
    bool dual = p.msplit;
    if (tiles < kNumSMs && !p.msplit) {
        // (more than 4 slices measured slower: the DSMEM reduction grows with the slices)
        while (ks < 4 && tiles * ks * 2 <= 2 * kNumSMs && c.d_o >= ks * 2 * 2) ks *= 2;
        dual = tiles * ks > kNumSMs;
    }
    if (opts().ksplit > 0) ks = std::min(8, int(opts().ksplit));
    if (p.persistent || p.msplit) ks = 1;
    if (p.persistent) dual = false;
    int ns = dual ? 2 : int(std::min<size_t>(16, (kGSmemCap - fixed - statics) / stage));
    if (opts().stages > 0) ns = std::max(2, std::min(16, int(opts().stages)));
    if (fixed + statics + size_t(ns) * stage > kGSmemCap) return 0;
    p.ns = ns;
    p.tmem_cols = 32;
    while (p.tmem_cols < (relayout ? c.tm * c.d_i : c.tm / (p.msplit ? 2 : 1)) * (p.persistent ? 2 : 1))
        p.tmem_cols *= 2;
    if (p.tmem_cols > 512) p.persistent = 0, p.tmem_cols = 256;
    p.sps = (c.d_o + ks - 1) / ks;
    p.ksplit = (c.d_o + p.sps - 1) / p.sps;
    p.debug = DBG(opts().debug);
    // multicast pairs: the u_o tile-rows of a column block as one cluster (<= 8 portable)
    // (SDMM slabs are two 64-column atoms; conv slabs must have an even number of channel atoms)
    // (relayout: measured slower with pairs -- 26.6 vs 25.2 us on conv10 -- so never paired)
    p.mc = (pairs && p.ksplit == 1 && !p.persistent && !p.msplit && !relayout && c.u_o >= 2 && c.u_o <= 8 &&
            (!conv || (c.tk / 64) % 2 == 0) && opts().multicast != 0) ? 1 : 0;
    out->p = p;
    out->smem = fixed + size_t(ns) * stage;
    out->grid = p.persistent ? dim3(unsigned(std::min<int64_t>(tiles, kNumSMs)), 1, 1)
                             : dim3(unsigned(col_blocks), unsigned(c.u_o), unsigned(p.msplit ? 2 : p.ksplit));
    out->n_tiles = tiles;
    return 1;
}

// symmetric split-K epilogue: each of the ksplit slices reduces and stores tm / ksplit rows
// (32-row chunks; conv: whole 128-byte channel atoms), receiving the other slices' partials by
// posted DSMEM stores; the receive buffer and the output staging share the idle ring
void set_symmetric(GPlan *pl, int oelt, bool conv) {
    GParams &p = pl->p;
    p.sym = 0;
    p.stage_off = 0;
    if (p.ksplit <= 1 || p.tm % p.ksplit || !opts().sym) return;
    const int rp = p.tm / p.ksplit;
    if (rp % 32 || (conv && rp % (128 / oelt))) return;
    const size_t recv = size_t(p.ksplit - 1) * rp * kBatch * 4;
    const size_t off = (recv + 1023) & ~size_t(1023);
    if (off + size_t(rp) * oelt * 128 > size_t(p.ns) * (p.i_bytes + p.w_bytes)) return;
    p.sym = 1;
    p.stage_off = int32_t(off);
}

// ---------------------------------------------------------------- prepared relayout
// prepared K4 section: [cols i32 u_i x d_i][users i32 v_i x d_r x 2][values bf16 u_o x d_o x tm x d_t]
// Tile (tbm, j) of the re-laid values lists, for each g_i column block kb, its d_r user row
// blocks (ascending) x bm rows x bk slots: value(kb, u, m, k) = W[tbm*tm + ui*bm + m]
// [j*d_t + ink*bk + k] with (ui, ink) = users[kb][u].  A permutation of RcubsMatrix.values
// (same bytes, still the succinct format), so one MMA covers a column block.
namespace {
size_t a16(size_t x) { return (x + 15) & ~size_t(15); }
__global__ void relayout_kernel(const __nv_bfloat16 *__restrict__ values, int64_t row_nnz, int tm, int d_t,
                                int d_o, int bm, int bk, int d_r, const int32_t *__restrict__ users,
                                int64_t total, __nv_bfloat16 *__restrict__ out) {
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tile = idx / (int64_t(tm) * d_t);
        const int r = int(idx - tile * tm * d_t);
        const int k = r % bk, m = (r / bk) % bm, u = (r / (bk * bm)) % d_r, kb = r / (bk * bm * d_r);
        const int tbm = int(tile / d_o), j = int(tile % d_o);
        const int ui = users[(kb * d_r + u) * 2], ink = users[(kb * d_r + u) * 2 + 1];
        out[idx] = values[(int64_t(tbm) * tm + ui * bm + m) * row_nnz + int64_t(j) * d_t + ink * bk + k];
    }
}
}  // namespace

// values-only refresh of the relayout (training: new values, same pattern): the users table
// written by gather_prepare stays in the prepared buffer; stream-ordered, no host work
int gather_prepare_values(const ChainDims &c, const void *values, void *k4, cudaStream_t stream) {
    const int d_r = c.u_i * c.d_i / c.v_i;
    const int32_t *cols_d;
    const void *vals_d;
    gather_prep_views(c, k4, &cols_d, &vals_d);
    const int32_t *users_d = reinterpret_cast<const int32_t *>(static_cast<char *>(k4) + a16(size_t(c.u_i) * c.d_i * 4));
    const int64_t total = c.rows * c.row_nnz;
    relayout_kernel<<<int(std::min<int64_t>((total + 255) / 256, 4 * kNumSMs)), 256, 0, stream>>>(
        static_cast<const __nv_bfloat16 *>(values), c.row_nnz, c.tm, c.d_t, c.d_o, c.bm, c.bk, d_r, users_d, total,
        static_cast<__nv_bfloat16 *>(const_cast<void *>(vals_d)));
    RBGP4_CHECK_LAUNCH("relayout_kernel launch");
    return RBGP4_OK;
}

size_t gather_prep_bytes(const ChainDims &c) {
    if (!gather_relayout_ok(c)) return 0;
    const int d_r = c.u_i * c.d_i / c.v_i;
    return a16(size_t(c.u_i) * c.d_i * 4) + a16(size_t(c.v_i) * d_r * 8) + size_t(c.rows) * c.row_nnz * 2;
}

void gather_prep_views(const ChainDims &c, const void *k4, const int32_t **cols, const void **vals) {
    const int d_r = c.u_i * c.d_i / c.v_i;
    *cols = static_cast<const int32_t *>(k4);
    *vals = static_cast<const char *>(k4) + a16(size_t(c.u_i) * c.d_i * 4) + a16(size_t(c.v_i) * d_r * 8);
}

int gather_prepare(const ChainDims &c, const void *values, const int32_t *adj_i_host, void *k4,
                   cudaStream_t stream) {
    const int d_r = c.u_i * c.d_i / c.v_i;
    std::vector<int32_t> cols(size_t(c.u_i) * c.d_i), users(size_t(c.v_i) * d_r * 2, -1);
    std::vector<int> fill(c.v_i, 0);
    for (int ui = 0; ui < c.u_i; ++ui)
        for (int ink = 0; ink < c.d_i; ++ink) {
            const int kb = adj_i_host[ui * c.d_i + ink];
            if (kb < 0 || kb >= c.v_i || fill[kb] >= d_r) {
                set_error("gather relayout: g_i is not biregular (column %d)", kb);
                return RBGP4_EINVAL;
            }
            const int u = fill[kb]++;
            users[(size_t(kb) * d_r + u) * 2] = ui;
            users[(size_t(kb) * d_r + u) * 2 + 1] = ink;
            cols[size_t(ui) * c.d_i + ink] = (kb * d_r + u) * c.bm;  // TMEM column of the partial
        }
    const int32_t *cols_d;
    const void *vals_d;
    gather_prep_views(c, k4, &cols_d, &vals_d);
    int32_t *users_d = reinterpret_cast<int32_t *>(static_cast<char *>(k4) + a16(size_t(c.u_i) * c.d_i * 4));
    cudaError_t e = cudaMemcpyAsync(const_cast<int32_t *>(cols_d), cols.data(), cols.size() * 4,
                                    cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(users_d, users.data(), users.size() * 4, cudaMemcpyHostToDevice, stream);
    const int64_t total = c.rows * c.row_nnz;
    if (e == cudaSuccess) {
        relayout_kernel<<<int(std::min<int64_t>((total + 255) / 256, 4 * kNumSMs)), 256, 0, stream>>>(
            static_cast<const __nv_bfloat16 *>(values), c.row_nnz, c.tm, c.d_t, c.d_o, c.bm, c.bk, d_r,
            users_d, total, static_cast<__nv_bfloat16 *>(const_cast<void *>(vals_d)));
        e = cudaGetLastError();
        if (e == cudaSuccess) note_launch();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // host tables are temporaries
    if (e != cudaSuccess) {
        set_error("gather relayout: %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    return RBGP4_OK;
}

namespace {
template <bool OUT_BF16, bool CONV>
int gather_launch_typed(const GPlan &pl, const CUtensorMap &imap, const CUtensorMap &wmap,
                        const CUtensorMap &omap, const int32_t *adj_o, const int32_t *adj_i,
                        void *out, cudaStream_t stream) {
    if (pl.p.persistent) {
        void (*pk)(CUtensorMap, CUtensorMap, GParams, const int32_t *, const int32_t *, void *, int64_t) = nullptr;
        switch (pl.p.mma_n) {
            case 16: pk = gather_persistent_kernel<OUT_BF16, CONV, 16>; break;
            case 32: pk = gather_persistent_kernel<OUT_BF16, CONV, 32>; break;
            case 48: pk = gather_persistent_kernel<OUT_BF16, CONV, 48>; break;
            case 64: pk = gather_persistent_kernel<OUT_BF16, CONV, 64>; break;
            case 128: pk = gather_persistent_kernel<OUT_BF16, CONV, 128>; break;
            default:
                set_error("gather kernel: no instantiation for MMA N = %d", pl.p.mma_n);
                return RBGP4_EUNSUPPORTED;
        }
        cudaError_t e = cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
        if (e != cudaSuccess) {
            set_error("cudaFuncSetAttribute(gather persistent): %s", cudaGetErrorString(e));
            (void)cudaGetLastError();  // not sticky: do not leave it for the next launch check
            return RBGP4_ECUDA;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = pl.grid;
        cfg.blockDim = dim3(kGThreads);
        cfg.dynamicSmemBytes = pl.smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = opts().pdl ? 1 : 0;
        note_kernel(pl.p.conv ? "K4 conv" : "K4 gather");
        e = cudaLaunchKernelEx(&cfg, pk, imap, wmap, pl.p, adj_o, adj_i, out, pl.n_tiles);
        if (e != cudaSuccess) {
            set_error("gather_persistent_kernel launch (%u CTAs, smem %zu): %s", pl.grid.x, pl.smem,
                      cudaGetErrorString(e));
            return RBGP4_ECUDA;
        }
        RBGP4_CHECK_LAUNCH("gather_persistent_kernel launch");
        return RBGP4_OK;
    }
    void (*kern)(CUtensorMap, CUtensorMap, CUtensorMap, GParams, const int32_t *, const int32_t *) = nullptr;
    switch (pl.p.mma_n) {
        case 16: kern = gather_kernel<OUT_BF16, CONV, 16>; break;
        case 32: kern = gather_kernel<OUT_BF16, CONV, 32>; break;
        case 48: kern = gather_kernel<OUT_BF16, CONV, 48>; break;
        case 64: kern = gather_kernel<OUT_BF16, CONV, 64>; break;
        case 128: kern = gather_kernel<OUT_BF16, CONV, 128>; break;
        default:
            set_error("gather kernel: no instantiation for MMA N = %d", pl.p.mma_n);
            return RBGP4_EUNSUPPORTED;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(gather): %s", cudaGetErrorString(e));
        (void)cudaGetLastError();  // not sticky: do not leave it for the next launch check
        return RBGP4_ECUDA;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = pl.grid;
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = pl.p.mc ? pl.grid.y : 1;
    attr[0].val.clusterDim.z = unsigned(pl.p.msplit ? 2 : pl.p.ksplit);
    int na = (pl.p.ksplit > 1 || pl.p.mc || pl.p.msplit) ? 1 : 0;
    cudaLaunchAttribute attrs[2];
    if (na) attrs[0] = attr[0];
    if (opts().pdl) {
        attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = unsigned(na);
    note_kernel(pl.p.conv ? "K4 conv" : "K4 gather");
    e = cudaLaunchKernelEx(&cfg, kern, imap, wmap, omap, pl.p, adj_o, adj_i);
    if (e != cudaSuccess) {
        set_error("gather_kernel launch (grid %u x %u x %u, smem %zu): %s", pl.grid.x, pl.grid.y,
                  pl.grid.z, pl.smem, cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    RBGP4_CHECK_LAUNCH("gather_kernel launch");
    return RBGP4_OK;
}

int encode_w_map(CUtensorMap *wmap, const ChainDims &c, const GParams &p, const void *values) {
    auto enc = encode_fn();
    cuuint64_t wdims[2], wstrides[1];
    cuuint32_t wbox[2];
    if (p.cols) {  // re-laid tiles: (bk, u_o * d_o * w_rows)
        wdims[0] = cuuint64_t(c.bk); wdims[1] = cuuint64_t(c.u_o) * c.d_o * p.w_rows;
        wstrides[0] = cuuint64_t(c.bk) * 2;
        wbox[0] = cuuint32_t(c.bk); wbox[1] = cuuint32_t(p.w_rows);
    } else {       // RcubsMatrix.values as stored: (row_nnz, rows)
        wdims[0] = cuuint64_t(c.row_nnz); wdims[1] = cuuint64_t(c.rows);
        wstrides[0] = cuuint64_t(c.row_nnz) * 2;
        wbox[0] = cuuint32_t(c.d_t); wbox[1] = cuuint32_t(p.msplit ? c.tm / 2 : c.tm);
    }
    cuuint32_t estr[2] = {1, 1};
    if (reinterpret_cast<uintptr_t>(values) % 16 != 0 || wstrides[0] % 16 != 0) {
        set_error("gather path needs 16-byte aligned values rows");
        return RBGP4_EUNSUPPORTED;
    }
    CUresult r = enc(wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(values), wdims, wstrides,
                     wbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(p.w_swz),
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled(values) failed (%d)", int(r));
        return RBGP4_ECUDA;
    }
    return RBGP4_OK;
}
}  // namespace

int launch_gather(const ChainDims &c, int out_dtype, const void *values, const int32_t *adj_o,
                  const int32_t *adj_i, const int32_t *sched, const int32_t *pair, const void *k4,
                  const void *inp, void *out, cudaStream_t stream) {
    const int oelt = out_dtype == RBGP4_BF16 ? 2 : 4;
    GPlan pl;
    if (!gather_plan(c, RBGP4_COMPUTE_BF16, false, k4 != nullptr, &pl, pair != nullptr)) return RBGP4_EUNSUPPORTED;
    pl.p.sched = sched;
    pl.p.pair = pair;
    if (k4) gather_prep_views(c, k4, &pl.p.cols, &values);
    set_symmetric(&pl, oelt, false);
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(inp) % 16 == 0 && (c.ld_in * 2) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(out) % 16 == 0 && (c.ld_out * oelt) % 16 == 0,
                  "gather path needs 16-byte aligned I / O rows");
    CUtensorMap imap, wmap, omap;
    cuuint32_t estr[3] = {1, 1, 1};
    {
        // I as (64 cols, K rows, N/64 atoms): one box = a whole 128-column slab, atom-major
        cuuint64_t dims[3] = {64, cuuint64_t(c.cols), cuuint64_t((c.n_cols + 63) / 64)};
        cuuint64_t strides[2] = {cuuint64_t(c.ld_in) * 2, 128};
        cuuint32_t box[3] = {64, cuuint32_t(c.tk), (pl.p.mc || pl.p.msplit) ? 1u : 2u};
        if (c.n_cols % 64) {
            // ragged last atom: a 2-atom view would read past the row; fall back to the
            // column-exact 2-D view with one box per atom (OOB columns zero-filled)
            set_error("gather path: n_cols %% 64 != 0");
            return RBGP4_EUNSUPPORTED;
        }
        CUresult r = enc(&imap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(inp), dims, strides,
                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(I) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    if (int rc = encode_w_map(&wmap, c, pl.p, values)) return rc;
    {
        cuuint64_t odims[2] = {cuuint64_t(c.n_cols), cuuint64_t(c.rows)};
        cuuint64_t ostrides[1] = {cuuint64_t(c.ld_out) * oelt};
        cuuint32_t obox[2] = {cuuint32_t(128 / oelt),
                              cuuint32_t(pl.p.msplit ? c.tm / 2 : pl.p.sym ? c.tm / pl.p.ksplit : c.tm)};
        CUresult r = enc(&omap, oelt == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         2, out, odims, ostrides, obox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(O) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    return oelt == 2 ? gather_launch_typed<true, false>(pl, imap, wmap, omap, adj_o, adj_i, out, stream)
                     : gather_launch_typed<false, false>(pl, imap, wmap, omap, adj_o, adj_i, out, stream);
}

int gather_supported(const ChainDims &c, int compute, int out_dtype, bool relayout) {
    GPlan pl;
    (void)out_dtype;
    return c.n_cols % 64 == 0 && gather_plan(c, compute, false, relayout, &pl);
}

int gather_conv_supported(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, bool relayout) {
    GPlan pl;
    if (!gather_plan(c, RBGP4_COMPUTE_BF16, true, relayout, &pl)) return 0;
    const int oh = (cv->height + 2 * cv->pad - cv->kh) / cv->stride + 1;
    const int ow = (cv->width + 2 * cv->pad - cv->kw) / cv->stride + 1;
    const int hw = oh * ow;
    // a 128-pixel tile = whole output rows of one image, or whole images
    const bool tiles = (kBatch <= hw) ? (hw % kBatch == 0 && kBatch % ow == 0) : (kBatch % hw == 0);
    return tiles && cv->c_in % 64 == 0 && cv->c_in % c.tk == 0 && (cv->stride == 1 || cv->stride == 2) &&
           ow * cv->stride <= 256 && (c.rows * (out_dtype == RBGP4_BF16 ? 2 : 4)) % 16 == 0;
}

int launch_gather_conv(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, const void *values,
                       const int32_t *adj_o, const int32_t *adj_i, const int32_t *sched, const int32_t *pair,
                       const void *k4, const void *x, void *out, cudaStream_t stream) {
    const int oelt = out_dtype == RBGP4_BF16 ? 2 : 4;
    GPlan pl;
    if (!gather_plan(c, RBGP4_COMPUTE_BF16, true, k4 != nullptr, &pl, pair != nullptr)) return RBGP4_EUNSUPPORTED;
    pl.p.sched = sched;
    pl.p.pair = pair;
    if (k4) gather_prep_views(c, k4, &pl.p.cols, &values);
    set_symmetric(&pl, oelt, true);
    pl.p.conv = 1;
    pl.p.ld_out = int64_t(c.rows);  // NHWC: a pixel row holds c_out channels
    pl.p.c_in = cv->c_in;
    const int oh = (cv->height + 2 * cv->pad - cv->kh) / cv->stride + 1;
    const int ow = (cv->width + 2 * cv->pad - cv->kw) / cv->stride + 1;
    pl.p.img_h = oh;
    pl.p.img_w = ow;
    pl.p.stride = cv->stride;
    pl.p.kw = cv->kw;
    pl.p.pad = cv->pad;
    pl.p.relu = cv->relu;
    auto enc = encode_fn();
    RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0,
                  "conv input / output must be 16-byte aligned");
    const int hw = oh * ow;
    const int th = kBatch <= hw ? kBatch / ow : oh;
    const int tb = kBatch <= hw ? 1 : kBatch / hw;
    CUtensorMap imap, wmap, omap;
    const cuuint32_t sd = cuuint32_t(cv->stride);
    cuuint32_t estr[4] = {1, sd, sd, 1};        // strided conv: every stride-th input pixel
    const cuuint32_t ones4[4] = {1, 1, 1, 1};   // W and O maps
    {
        const int64_t ihw = int64_t(cv->height) * cv->width;
        cuuint64_t dims[4] = {cuuint64_t(cv->c_in), cuuint64_t(cv->width), cuuint64_t(cv->height),
                              cuuint64_t(cv->batch)};
        cuuint64_t strides[3] = {cuuint64_t(cv->c_in) * 2, cuuint64_t(cv->width) * cv->c_in * 2,
                                 cuuint64_t(ihw) * cv->c_in * 2};
        cuuint32_t box[4] = {64, cuuint32_t(ow) * sd, cuuint32_t(th) * sd, cuuint32_t(tb)};
        CUresult r = enc(&imap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(x), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(conv input) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    if (int rc = encode_w_map(&wmap, c, pl.p, values)) return rc;
    {
        // NHWC output as (c_out, pixels): box = one 128-byte channel atom x 128 pixels
        cuuint64_t odims[2] = {cuuint64_t(c.rows), cuuint64_t(c.n_cols)};
        cuuint64_t ostrides[1] = {cuuint64_t(c.rows) * oelt};
        cuuint32_t obox[2] = {cuuint32_t(128 / oelt), cuuint32_t(kBatch)};
        CUresult r = enc(&omap, oelt == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         2, out, odims, ostrides, obox, ones4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(conv output) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    return oelt == 2 ? gather_launch_typed<true, true>(pl, imap, wmap, omap, adj_o, adj_i, out, stream)
                     : gather_launch_typed<false, true>(pl, imap, wmap, omap, adj_o, adj_i, out, stream);
}

}  // namespace rbgp4

#if RBGP4_DEBUG
// debug builds only (not part of include/rbgp4.h): copy the K4 CTA-0 trace to the host
extern "C" int rbgp4_debug_trace_gather(unsigned long long *host, int n) {
    if (n > 4 * rbgp4::kGTraceSteps) n = 4 * rbgp4::kGTraceSteps;
    return cudaMemcpyFromSymbol(host, rbgp4::g_gtrace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -3;
}

// debug-only: per-CTA entry / exit %globaltimer stamps (RBGP4_TC_DEBUG bit 512)
extern "C" int rbgp4_debug_cta_stamps(unsigned long long *host, int n) {
    if (n > 2 * rbgp4::kCtaStamps) n = 2 * rbgp4::kCtaStamps;
    return cudaMemcpyFromSymbol(host, rbgp4::g_cta_stamp, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -3;
}
#endif  // RBGP4_DEBUG
