// sdmm_tc.cu -- K2: RBGP4 product on the 5th-generation tensor cores (tcgen05).
//
// Replaces kronsparse.sdmm._tile_worker (reference sdmm.py:148-205) for the
// bf16 / tf32 compute modes.  Formulation ("densified tile"):
// a CTA owns 128 rows of one W tile-row (M = 128 MMA rows) and TN <= 256
// output columns.  It walks g_o's adjacency row only (structurally zero
// tiles are skipped, as in the reference), and per step s
//
//   B (I slab)  I[adj_o[tbm][s]*tk : +tk, n0 : n0+TN]  -- TMA, 128B swizzle
//               (32 B atoms for tf32), MN-major UMMA operand (I is row-major,
//               N contiguous, so no transpose is ever materialised)
//   A (W tile)  the 128 x tk dense tile, K-major 32/64/128B swizzle, built in
//               shared memory from the COMPRESSED values (128 x d_t): the
//               in-tile pattern g_r (x) g_i (x) g_b is the same for every
//               step and every tile-row, so the zero positions are written
//               once at kernel start and each step only scatters the d_t
//               nonzeros of each row to their (fixed) positions.
//   D          += A * B   with tk*E/32 tcgen05.mma (M=128, N=TN, K=32 bytes),
//               fp32 accumulation in TMEM (TN columns).
//
// Warp roles (224 threads):  warps 0-3 densify A and run the epilogue
// (tcgen05.ld 32x32b -> registers -> 16-byte global stores; warp w owns TMEM
// lanes 32w..32w+31 = output rows);  warp 4 lane 0 issues the I-slab TMA
// loads; warp 6 lane 0 the compressed-W TMA loads (separate rings so the I
// stream never waits on densify progress); warp 5 allocates TMEM and lane 0
// issues the MMAs.  An NS-stage mbarrier
// ring links them:  full (TMA tx bytes + 4 densify-warp arrivals), empty (one commit),
// empty (tcgen05.commit), tmem_full (last commit).
//
// Roofline: bound by HBM for the VGG/WRN layer shapes (compressed W + I +
// O once); the MMA does 1/(1-sp_i) times the useful work, which stays under
// the HBM time while (1-sp_i) * P_tc >= AI * BW (SURVEY §7 hard part 1).
#include "common.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

namespace rbgp4 {
namespace {

constexpr int kThreads = 224;

// Debug trace (RBGP4_TC_DEBUG bit 8): CTA 0 stamps clock64 at every role hand-off.
// Layout: [event][step], event = 0 B issued, 1 W issued, 2 densify start, 3 densify end,
// 4 MMA start, 5 MMA end; [6][0] setup done, [6][1] epilogue start, [6][2] epilogue end;
// 7 MMA saw full_b, 8 densify saw full_w (per W stage).
// (debug builds only: option debug, RBGP4_DEBUG=1)
constexpr int kTraceSteps = 512;
#if RBGP4_DEBUG
__device__ unsigned long long g_trace[10][kTraceSteps];
#endif
__device__ __forceinline__ void trace(const int debug, int ev, int step) {
#if RBGP4_DEBUG
    if ((debug & 8) && blockIdx.x == 0 && blockIdx.y == 0 && step < kTraceSteps)
        g_trace[ev][step] = clock64();
#endif
}
constexpr int kBlockM = 128;

struct TcParams {
    int64_t n_cols, ld_out, row_nnz;
    int64_t ws_ld;           // split-K workspace row pitch: n_cols rounded up to 4 floats (16 B)
    int32_t tm, tk, d_o, d_t, u_i, v_i, d_i, rk, bm, bk;
    int32_t tn;              // MMA N (columns per CTA), multiple of 16, <= 256
    int32_t rows_valid;      // 128, or 64 when tm == 64 (upper half of A is zero)
    int32_t na, nb, nw;      // ring depths: dense A tiles, I slabs, compressed W tiles
    int32_t w_tma;           // compressed W tiles staged by TMA (else read by the densify warps)
    int32_t ws;              // steps per W stage (one TMA box carries ws consecutive W tiles)
    int32_t i3d;             // one 3-D TMA per I slab (all column atoms) instead of one per atom
    int32_t a_swz;           // K-major swizzle span of A in bytes: 32 / 64 / 128
    int32_t a_stage_bytes, b_stage_bytes, w_stage_bytes;
    int32_t debug;           // ablation bits (RBGP4_TC_DEBUG): 1 no densify, 2 no MMA, 4 no epilogue
    int32_t ksplit, sps;     // split-K: CTAs per output tile (one cluster) and steps per slice
    int32_t adj_smem;        // g_i adjacency staged in shared memory for the table build
    const uint16_t *prep;    // precomputed scatter table [phase][j][row] (rbgp4_prepare) or null
    const int32_t *sched;    // step schedule [tile-row][s] -> g_o adjacency slot (rbgp4_prepare) or null
    int32_t table_in_regs;   // densify keeps each row's offsets in registers (else smem table)
    int32_t tmem_cols;       // TMEM allocation (power of two)
    // implicit-im2col convolution (K3): I is never materialised; x is NHWC bf16 and the
    // slab of step s is the tap (i, j) / channel block of its K rows, fetched by a 4-D TMA
    // box at the tap-shifted coordinates (out-of-bounds = zero padding); O is NHWC.
    // (img_h, img_w = OUTPUT map; the input map is stride x larger, read by strided TMA boxes)
    int32_t conv, c_in, img_h, img_w, kw, pad, relu, th, tb, stride;
    int32_t ostore;          // epilogue stages the output tile in shared memory and TMA-stores it
    // persistent tile loop (many-wave conv / SDMM grids, tm <= 128, no split-K): CTAs stride over
    // n_tiles tiles (column block-major); rings and barrier phases continue across tiles
    int32_t persistent, blocks_m;
    int64_t n_tiles;
    int32_t pstage_bytes;    // persistent: dedicated output staging (the rings are streaming)
    int32_t w_swz;           // swizzle span (bytes) of the compressed-W stage rows: 0 / 32 / 64 / 128
};

// Byte offset, inside one densified A stage, of nonzero j of CTA row r (the scatter map).
// Row r walks j = ((rk*d_i + ink)*bk + k) with counters (reference sdmm.py:183-186).
template <int kElt>
__device__ __forceinline__ void row_offsets(const TcParams &p, const int32_t *adj, int row_in_tile0,
                                            int r, uint16_t *dst, int dst_stride) {
    const int ui = ((row_in_tile0 + r) / p.bm) % p.u_i;
    const int32_t *arow = adj + ui * p.d_i;
    const int sh = p.a_swz == 128 ? 7 : p.a_swz == 64 ? 6 : 5;  // log2(swizzle span)
    const uint32_t rbase = uint32_t(r) << sh;
    int k = 0, ink = 0, rk = 0;
    int kbase = arow[0] * p.bk;  // (rk*v_i + adj_i[ui][ink])*bk
    for (int j = 0; j < p.d_t; ++j) {
        const uint32_t kb = uint32_t(kbase + k) * kElt;  // byte offset along K
        dst[j * dst_stride] =
            uint16_t(((kb >> sh) << (sh + 7)) + swz(rbase + (kb & (p.a_swz - 1)), p.a_swz));
        if (++k == p.bk) {
            k = 0;
            if (++ink == p.d_i) { ink = 0; ++rk; }
            if (rk < p.rk) kbase = (rk * p.v_i + arow[ink]) * p.bk;
        }
    }
}

// rbgp4_prepare: the scatter map depends only on the chain and the tiling, so it is built
// once per matrix into [phase][j][row] (phase = which 128-row block of a tile-row).
template <int kElt>
__global__ void prep_kernel(const TcParams p, const int32_t *__restrict__ adj_i, uint16_t *out) {
    const int phase = blockIdx.x;
    const int r = threadIdx.x;
    if (r < kBlockM)
        row_offsets<kElt>(p, adj_i, phase * p.rows_valid, r,
                          out + size_t(phase) * p.d_t * kBlockM + r, kBlockM);
}

// ---------------------------------------------------------------- the kernel
template <typename E, bool OUT_BF16, bool CONV>
__global__ void __launch_bounds__(kThreads, 1)
tc_kernel(const __grid_constant__ CUtensorMap imap, const __grid_constant__ CUtensorMap wmap,
          const __grid_constant__ CUtensorMap omap, const TcParams p, const E *__restrict__ values, const int32_t *__restrict__ adj_o,
          const int32_t *__restrict__ adj_i, void *__restrict__ out, float *__restrict__ wsp) {
    constexpr bool kTF32 = sizeof(E) == 4;
    constexpr int kElt = sizeof(E);
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned carve-up:
    //   [A ring: na x 128 x tk dense]  [B ring: nb x tk x tn]  [W ring: nw x rows x d_t]
    //   [aoff table 128 x d_t u16]  [barriers]  [tmem ptr]
    unsigned char *base = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *a_buf = base;
    unsigned char *b_buf = a_buf + p.na * p.a_stage_bytes;
    unsigned char *w_buf = b_buf + p.nb * p.b_stage_bytes;
    unsigned char *pstage = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(w_buf + p.nw * p.w_stage_bytes) + 1023) & ~uintptr_t(1023));
    // aoff[j * 128 + r]: byte offset (inside an A stage) of nonzero j of CTA row r
    uint16_t *aoff = reinterpret_cast<uint16_t *>(p.pstage_bytes ? pstage + p.pstage_bytes
                                                                  : w_buf + p.nw * p.w_stage_bytes);
    int32_t *adj_s = reinterpret_cast<int32_t *>(
        (reinterpret_cast<uintptr_t>(aoff + kBlockM * p.d_t) + 15) & ~uintptr_t(15));
    uint64_t *bars = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(adj_s + (p.adj_smem ? p.u_i * p.d_i : 0)) + 7) & ~uintptr_t(7));
    // one barrier ring of nb stages indexed by step (s % nb): the I slab of step s lives in
    // B stage s % nb, its dense A tile in A stage s % na (na <= nb: the A ring only needs to
    // cover densify-ahead, the I ring covers the load latency).  full[s % nb] completes on
    // the TMA transaction bytes + 4 densify-warp arrivals, empty[s % nb] on the MMA commit of
    // step s (one wait and one commit per step for the MMA warp); the A stage of step s is
    // free once empty[(s - na) % nb] has completed for step s - na.
    uint64_t *full_b = bars, *empty_b = full_b + p.nb;
    uint64_t *full_w = empty_b + p.nb, *empty_w = full_w + p.nw;
    uint64_t *tmem_full = empty_w + p.nw;
    uint64_t *tmem_empty = tmem_full + 1;  // persistent: the epilogue has read the accumulator
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) trace(DBG(p.debug), 6, 3);
    // first tile of this CTA (the only one unless persistent)
    const int64_t m0_first = int64_t(p.persistent ? blockIdx.x % p.blocks_m : blockIdx.y) * p.rows_valid;
    const int row_in_tile0 = int(m0_first % p.tm);  // same for every tile (persistent: tm <= 128)
    // split-K: this CTA runs steps [s_begin, s_begin + nsteps) of the tile-row
    const int kslice = blockIdx.z;
    const int s_begin = kslice * p.sps;
    const int nsteps = min(p.d_o, s_begin + p.sps) - s_begin;

    // ---- barriers first, so the TMA producers start streaming before the rest of the
    // setup (TMEM allocation, A-ring zeroing, scatter table) -- that setup only gates
    // the densify warps and the MMA warp, and overlaps the first I-slab loads.
    if (warp == 4 && lane == 0) {
        for (int i = 0; i < p.nb; ++i) { mbar_init(&full_b[i], 1 + 4); mbar_init(&empty_b[i], 1); }
        for (int i = 0; i < p.nw; ++i) { mbar_init(&full_w[i], 1); mbar_init(&empty_w[i], 4); }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&imap)) : "memory");
        if (p.w_tma)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    }
    __syncthreads();
    // programmatic dependent launch: let the next kernel schedule now; every thread waits for
    // the previous kernel (which may have produced I or W) before its first global read
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // g_o adjacency row of this tile-row and the order its slots are walked in: the
    // schedule lets tile-rows that share a K-block read its I slab at the same step
    if (threadIdx.x == 0) trace(DBG(p.debug), 6, 0);

    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(uint32_t(p.tmem_cols)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        tc_fence_before();
        __syncwarp();
        tc_fence_after();
        if (lane == 0) trace(DBG(p.debug), 6, 5);
    }
    if (warp < 4) {
        // ---- densify-warp setup: zero the A ring and load the scatter-offset table.
        // The in-tile pattern is the same for every step, so the (row, j) -> A position
        // map is computed once here and the per-step densify is a pure table-driven
        // scatter (reference index map: sdmm.py:183-186).  Zeros written now are never
        // overwritten: every step fills the same positions.
        const int t = threadIdx.x;
        uint4 z = make_uint4(0, 0, 0, 0);
        uint4 *a4 = reinterpret_cast<uint4 *>(a_buf);
        for (int i = t; i < p.na * p.a_stage_bytes / 16; i += kBlockM) a4[i] = z;
        const int32_t *adj = adj_i;
        if (p.prep != nullptr) {
            // prepared map: one coalesced 16-byte copy into the shared table
            const uint4 *src = reinterpret_cast<const uint4 *>(
                p.prep + size_t(row_in_tile0 / p.rows_valid) * p.d_t * kBlockM);
            uint4 *dst = reinterpret_cast<uint4 *>(aoff);
            for (int i = t; i < p.d_t * kBlockM / 8; i += kBlockM) dst[i] = __ldg(src + i);
        } else {
            if (p.adj_smem) {
                // one coalesced copy instead of d_t dependent global loads per row
                for (int i = t; i < p.u_i * p.d_i; i += kBlockM) adj_s[i] = adj_i[i];
                asm volatile("bar.sync 1, 128;" ::: "memory");
                adj = adj_s;
            }
            row_offsets<kElt>(p, adj, row_in_tile0, t, aoff + t, kBlockM);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // table + zeros complete (warps 0-3)
        if (t == 0) trace(DBG(p.debug), 6, 4);
        if (DBG(p.debug) & 32) asm volatile("bar.sync 2, 160;" ::: "memory");
    }

    // Role loops run warp-uniformly (all 32 lanes wait on the barriers); one lane,
    // picked by elect.sync, issues the TMA / tcgen05 instructions.  Issuing from
    // lane-0-only divergent code made the compiler wrap every UTCHMMA/UTMALDG in an
    // elect loop with R2UR conversions (~500 cycles per step, tools/tc_trace.py).
    if ((DBG(p.debug) & 32) && warp == 4) asm volatile("bar.sync 2, 160;" ::: "memory");  // late start
    const int64_t n_tiles = p.persistent ? p.n_tiles : 1;
    const int64_t tile_stride = p.persistent ? gridDim.x : 1;
    int64_t it = 0;
    for (int64_t tile = p.persistent ? blockIdx.x : 0; tile < n_tiles; tile += tile_stride, ++it) {
    const int64_t n0 = int64_t(p.persistent ? tile / p.blocks_m : blockIdx.x) * p.tn;
    const int64_t m0 = int64_t(p.persistent ? tile % p.blocks_m : blockIdx.y) * p.rows_valid;
    const int64_t tbm = m0 / p.tm;
    const int32_t *orow = adj_o + tbm * p.d_o;
    const int32_t *srow = p.sched ? p.sched + tbm * p.d_o + s_begin : nullptr;
    const int g0 = int(it) * nsteps;  // ring position of this tile's first step
    if (warp == 4) {
        // ================= TMA producer: I slabs (runs ahead by the B ring depth) ==========
        const int atoms = p.tn * kElt / 128;           // 128-byte MN atoms per slab
        const int atom_cols = 128 / kElt;
        const uint32_t atom_bytes = uint32_t(p.tk) * 128;
        for (int s = 0; s < nsteps; ++s) {
            const int st = (g0 + s) % p.nb;
            const uint32_t ph = ((g0 + s) / p.nb) & 1;
            mbar_wait(&empty_b[st], ph ^ 1);
            const int32_t krow = orow[srow ? srow[s] : s_begin + s] * p.tk;
            if (elect_one()) {
                mbar_expect_tx(&full_b[st], uint32_t(p.b_stage_bytes));
                unsigned char *dst = b_buf + st * p.b_stage_bytes;
                if constexpr (CONV) {
                    // K rows [krow, krow + tk) = tap (i, j), channels [c0, c0 + tk); the pixel
                    // tile is tb images x th rows x the full width, shifted by the tap
                    const int tap = krow / p.c_in, c0 = krow - tap * p.c_in;
                    const int ti = tap / p.kw, tj = tap - ti * p.kw;
                    const int hw = p.img_h * p.img_w;
                    const int b0 = int(n0 / hw), h0 = int(n0 % hw) / p.img_w;
                    const uint32_t k_atom_bytes = uint32_t(p.tn) * 128;
                    for (int a = 0; a < p.tk / 64; ++a)
                        tma_load_4d(dst + a * k_atom_bytes, &imap, &full_b[st], c0 + 64 * a,
                                    tj - p.pad, h0 * p.stride + ti - p.pad, b0);
                } else if (p.i3d) {
                    // one instruction for the whole slab: (atom cols, K rows, atoms) box
                    tma_load_3d(dst, &imap, &full_b[st], 0, krow, int32_t(n0) / atom_cols);
                } else {
                    for (int a = 0; a < atoms; ++a)
                        tma_load_2d(dst + a * atom_bytes, &imap, &full_b[st],
                                    int32_t(n0) + a * atom_cols, krow);
                }
                trace(DBG(p.debug), 0, s);
            }
            __syncwarp();
        }
    } else if (warp == 6) {
        // ================= TMA producer: compressed W tiles (own ring, own pace) ============
        if (p.w_tma) {
            const int wstages = (nsteps + p.ws - 1) / p.ws;
            for (int g = 0; g < wstages; ++g) {
                const int st = (g0 + g) % p.nw;
                const uint32_t ph = ((g0 + g) / p.nw) & 1;
                mbar_wait(&empty_w[st], ph ^ 1);
                if (elect_one()) {
                    mbar_expect_tx(&full_w[st], uint32_t(p.w_stage_bytes));
                    const int j = srow ? srow[g] : s_begin + g;  // ws == 1: stage g = step g
                    tma_load_2d(w_buf + st * p.w_stage_bytes, &wmap, &full_w[st], j * p.d_t,
                                int32_t(m0));
                    trace(DBG(p.debug), 1, g);
                }
                __syncwarp();
            }
        }
    } else if (warp == 5) {
        // ================= MMA issuer =================
        const uint32_t tmem_d = *tmem_slot;
        // instruction descriptor: D f32, A/B bf16|tf32, A K-major, B MN-major, N, M=128
        const uint32_t fmt = kTF32 ? 2u : 1u;
        const uint32_t b_mn = CONV ? 0u : 1u;  // conv: B (im2col of NHWC) is K-major
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (b_mn << 16) |
                               (uint32_t(p.tn >> 3) << 17) | (uint32_t(kBlockM >> 4) << 24);
        const int ksteps = p.tk * kElt / 32;
        // Descriptors are built once; per stage / K-step only the 14-bit start-address
        // field (16-byte units, low word) moves, so the issue loop is pure adds.
        const uint64_t a_desc0 =
            smem_desc(smem_u32(a_buf), 0, 8 * p.a_swz, swizzle_layout_code(p.a_swz));
        // MN-major B: bf16 -> SWIZZLE_128B (8-row K groups, SBO 1024);
        // tf32 -> SWIZZLE_128B_BASE32B (32 B chunks, 4-row K groups, SBO 512)
        const uint64_t b_desc0 = CONV ? smem_desc(smem_u32(b_buf), 0, 1024, 2u)  // K-major SW128
                               : kTF32 ? smem_desc(smem_u32(b_buf), uint32_t(p.tk) * 128, 512, 1u)
                                       : smem_desc(smem_u32(b_buf), uint32_t(p.tk) * 128, 1024, 2u);
        const uint32_t bk_jump16 = uint32_t(p.tn - 1) * 8;  // conv: next 64-channel K atom
        const uint32_t a_stage16 = uint32_t(p.a_stage_bytes) >> 4;
        const uint32_t b_stage16 = uint32_t(p.b_stage_bytes) >> 4;
        const uint32_t a_span16 = uint32_t(p.a_swz) >> 4;                // 16B units per atom row
        const uint32_t a_jump16 = uint32_t(kBlockM - 1) * a_span16;        // next K atom
        const uint32_t b_step16 = uint32_t(32 / kElt) * 128 / 16;           // 32/E K-rows
        if (it > 0) {  // persistent: the epilogue must have drained the accumulator
            mbar_wait(tmem_empty, uint32_t((it - 1) & 1));
            tc_fence_after();
        }
        for (int s = 0; s < nsteps; ++s) {
            const int sb = (g0 + s) % p.nb, sa = (g0 + s) % p.na;
            mbar_wait(&full_b[sb], ((g0 + s) / p.nb) & 1);  // I slab landed and A tile densified
            if (lane == 0) trace(DBG(p.debug), 7, s);
            tc_fence_after();
            if (elect_one()) {
                trace(DBG(p.debug), 4, s);
                uint64_t ad = a_desc0 + uint64_t(sa) * a_stage16;
                uint64_t bd = b_desc0 + uint64_t(sb) * b_stage16;
                uint32_t in_atom = 0;
                for (int kk = 0; kk < ksteps; ++kk) {
                    if (!(DBG(p.debug) & 2)) tc_mma<kTF32>(tmem_d, ad, bd, idesc, (s > 0 || kk > 0) ? 1u : 0u);
                    ad += 2;  // 32 bytes along K inside the swizzle atom
                    in_atom += 2;
                    if (in_atom == a_span16) { ad += a_jump16; in_atom = 0; }
                    if constexpr (CONV) {
                        bd += 2;  // K-major B: 32 bytes along K inside its 128 B atom
                        if ((kk & 3) == 3) bd += bk_jump16;
                    } else {
                        bd += b_step16;
                    }
                }
                tc_commit(&empty_b[sb]);  // frees the I slab (and, na steps later, the A tile)
                trace(DBG(p.debug), 5, s);
            }
            __syncwarp();
        }
        if (elect_one()) tc_commit(tmem_full);
        __syncwarp();
    } else {
        // ================= densify (warps 0-3), then epilogue =================
        const int t = threadIdx.x;  // 0..127: this thread densifies CTA row t
        const bool active = t < p.rows_valid;
        constexpr int V = 16 / kElt;          // elements per 16-byte chunk
        constexpr int kRegNnz = 64;           // d_t handled from registers up to this
        const E *vrow = values + (m0 + t) * p.row_nnz;
        // this row's scatter offsets never change: keep them in registers (2 per reg)
        uint32_t offp[kRegNnz / 2];
        // G_b blocks of >= 16 bytes along K (bk % V == 0): each 16-byte chunk of a compressed
        // row lands on one 16-byte unit of the swizzled A tile -> 16-byte stores
        constexpr int kMaxChunks = 16;      // 16-byte chunks per row held in registers
        const bool chunked = p.w_tma && (p.bk % V == 0) && p.d_t <= kMaxChunks * V;
        const bool reg_path = p.w_tma && p.d_t <= kRegNnz;
#pragma unroll
        for (int i = 0; i < kRegNnz / 2; ++i) {
            // element offsets (reg_path) or, when chunked, the offsets of chunk starts
            const int j = chunked ? 2 * i * V : 2 * i;
            const int j2 = chunked ? j + V : j + 1;
            uint32_t lo = j < p.d_t ? aoff[j * kBlockM + t] : 0u;
            uint32_t hi = j2 < p.d_t ? aoff[j2 * kBlockM + t] : 0u;
            offp[i] = lo | (hi << 16);
        }
        // compressed row t of a W stage: ws*d_t elements; when the stage is swizzled (TMA
        // SWIZZLE_32B/64B/128B, rows of exactly w_swz bytes) 16-byte chunk c sits at c ^ wxor
        const uint32_t wrow_bytes = uint32_t(p.ws * p.d_t * kElt);
        const uint32_t wrow = smem_u32(w_buf) + uint32_t(t) * wrow_bytes;
        const uint32_t wxor = p.w_swz ? ((uint32_t(t) * wrow_bytes) >> 7) & uint32_t(p.w_swz / 16 - 1) : 0u;
        for (int s = 0; s < nsteps; ++s) {
            const int gs = g0 + s;  // ring position (continues across persistent tiles)
            const int sa = gs % p.na;
            const int wg = s / p.ws, wsub = s - wg * p.ws;  // W stage and slot inside it
            const int wr = g0 + wg;                         // W ring position (ws == 1)
            if (p.w_tma && wsub == 0) {
                mbar_wait(&full_w[wr % p.nw], (wr / p.nw) & 1);
                if (t == 0) trace(DBG(p.debug), 8, wg);
            }
            if (gs >= p.na) {  // A stage sa was last read by the MMAs of ring step gs - na
                const int sp = gs - p.na;
                mbar_wait(&empty_b[sp % p.nb], (sp / p.nb) & 1);
            }
            if (t == 0) trace(DBG(p.debug), 2, s);
            const uint32_t a = smem_u32(a_buf + sa * p.a_stage_bytes);
            const uint32_t src = wrow + uint32_t((wr % p.nw) * p.w_stage_bytes);
            const uint32_t c0 = uint32_t(wsub * p.d_t * kElt / 16);  // first chunk of this step
            if (active && !(DBG(p.debug) & 1)) {
                if (chunked) {
                    const int nchunks = p.d_t / V;
                    uint4 q[kMaxChunks];
#pragma unroll
                    for (int c = 0; c < kMaxChunks; ++c)
                        if (c < nchunks) q[c] = lds128(src + (((c0 + c) ^ wxor) << 4));
#pragma unroll
                    for (int c = 0; c < kMaxChunks; ++c) {
                        if (c < nchunks) {
                            const uint32_t o = (offp[c / 2] >> (16 * (c & 1))) & 0xFFFFu;
                            sts128(a + o, q[c].x, q[c].y, q[c].z, q[c].w);
                        }
                    }
                } else if (reg_path) {
                    // compressed row t of this step (TMA-staged): 16-byte shared loads,
                    // all issued before the scatter so their latency overlaps
                    uint4 q[kRegNnz / V];
#pragma unroll
                    for (int c = 0; c < kRegNnz / V; ++c)
                        if (c * V < p.d_t) q[c] = lds128(src + (((c0 + c) ^ wxor) << 4));
#pragma unroll
                    for (int c = 0; c < kRegNnz / V; ++c) {
                        if (c * V < p.d_t) {
                            const E *qe = reinterpret_cast<const E *>(&q[c]);
#pragma unroll
                            for (int v = 0; v < V; ++v) {
                                const int j = c * V + v;
                                const uint32_t o = (offp[j / 2] >> (16 * (j & 1))) & 0xFFFFu;
                                sts_elem<E>(a + o, qe[v]);
                            }
                        }
                    }
                } else if (p.w_tma) {
                    for (int j = 0; j < p.d_t; j += V) {
                        uint4 q = lds128(src + (((c0 + j / V) ^ wxor) << 4));
                        const E *qe = reinterpret_cast<const E *>(&q);
#pragma unroll
                        for (int v = 0; v < V; ++v) sts_elem<E>(a + aoff[(j + v) * kBlockM + t], qe[v]);
                    }
                } else {
                    const E *vs = vrow + int64_t(srow ? srow[s] : s_begin + s) * p.d_t;
                    for (int j = 0; j < p.d_t; ++j) sts_elem<E>(a + aoff[j * kBlockM + t], vs[j]);
                }
            }
            // make the generic-proxy stores visible to the tensor core, then one
            // release-arrive per warp (full counts 4 warps + the TMA)
            if (!(DBG(p.debug) & 256)) fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&full_b[gs % p.nb]);
                if (p.w_tma && (wsub == p.ws - 1 || s == nsteps - 1)) mbar_arrive(&empty_w[wr % p.nw]);
            }
            if (t == 0) trace(DBG(p.debug), 3, s);
        }
        // ---- epilogue phase 1: wait for the accumulator; split-K slices > 0 park
        // their fp32 partial tile in the workspace (L2-resident) for the leader
        mbar_wait(tmem_full, uint32_t(it & 1));
        tc_fence_after();
        if (threadIdx.x == 0) trace(DBG(p.debug), 6, 1);
        if (kslice > 0) {
            const uint32_t tmem_d = *tmem_slot;
            const int row = warp * 32 + lane;
            const uint32_t lane_base = tmem_d + (uint32_t(warp * 32) << 16);
            float *dst = wsp + (int64_t(kslice - 1) * (int64_t(gridDim.y) * p.rows_valid) + m0 + row) *
                                   p.ws_ld;
            for (int c = 0; c < p.tn; c += 32) {
                uint32_t r[32];
                TMEM_LD_32x32b_X32(lane_base + uint32_t(c), r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int64_t col = n0 + c;
                if (row >= p.rows_valid || col >= p.n_cols) continue;
                if (col + 32 <= p.n_cols) {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<uint4 *>(dst + col)[q] =
                            make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                } else {
                    for (int q = 0; q < 32 && col + q < p.n_cols; ++q) dst[col + q] = __uint_as_float(r[q]);
                }
            }
        }
    }
    if (p.ksplit > 1) {
        // every thread of every slice: partials written (release) -> leader reads (acquire)
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (warp < 4 && kslice == 0) {
        // ---- epilogue phase 2 (leader): TMEM + partials (fixed slice order) -> output.
        // With p.ostore the tile is staged in shared memory (the A and I rings are free:
        // every MMA has completed) and written by TMA bulk stores -- full 128-byte lines
        // instead of 32 row-strided 16-byte stores per warp instruction.
        const uint32_t tmem_d = *tmem_slot;
        constexpr int kOutElt = OUT_BF16 ? 2 : 4;
        const int row = warp * 32 + lane;
        const bool row_ok = row < p.rows_valid;
        const uint32_t lane_base = tmem_d + (uint32_t(warp * 32) << 16);
        const int64_t slice_stride = int64_t(gridDim.y) * p.rows_valid * p.ws_ld;
        unsigned char *stage_buf = p.pstage_bytes ? pstage : a_buf;  // idle rings unless persistent
        const uint32_t stage = smem_u32(stage_buf);
        for (int c = 0; c < p.tn; c += 32) {
            uint32_t r[32];
            TMEM_LD_32x32b_X32(lane_base + uint32_t(c), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int64_t col = n0 + c;
            if (!row_ok || (DBG(p.debug) & 4)) continue;
            if (!p.ostore && col >= p.n_cols) continue;
            const bool full = col + 32 <= p.n_cols;
            if (p.ksplit > 1 && col < p.n_cols) {
                const float *part = wsp + (m0 + row) * p.ws_ld + col;
                for (int k = 1; k < p.ksplit; ++k, part += slice_stride) {
                    if (full) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 v = __ldcg(reinterpret_cast<const float4 *>(part) + q);
                            r[4 * q] = __float_as_uint(__uint_as_float(r[4 * q]) + v.x);
                            r[4 * q + 1] = __float_as_uint(__uint_as_float(r[4 * q + 1]) + v.y);
                            r[4 * q + 2] = __float_as_uint(__uint_as_float(r[4 * q + 2]) + v.z);
                            r[4 * q + 3] = __float_as_uint(__uint_as_float(r[4 * q + 3]) + v.w);
                        }
                    } else {
                        for (int q = 0; q < 32 && col + q < p.n_cols; ++q)
                            r[q] = __float_as_uint(__uint_as_float(r[q]) + __ldcg(part + q));
                    }
                }
            }
            if constexpr (CONV) {
                if (p.relu) {
#pragma unroll
                    for (int q = 0; q < 32; ++q) r[q] = __float_as_uint(fmaxf(__uint_as_float(r[q]), 0.0f));
                }
                if (p.ostore) {
                    // staging [pixel][rows_valid channels]: lanes = consecutive channels
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const uint32_t addr = stage + uint32_t(((c + q) * p.rows_valid + row) * kOutElt);
                        if constexpr (OUT_BF16) {
                            const __nv_bfloat16 b = __float2bfloat16_rn(__uint_as_float(r[q]));
                            sts16(addr, *reinterpret_cast<const uint16_t *>(&b));
                        } else {
                            sts32(addr, r[q]);
                        }
                    }
                    continue;
                }
                // NHWC output: pixel (col + q) is a row of c_out = p.ld_out channels
                const int64_t ch = m0 + row;
#pragma unroll 4
                for (int q = 0; q < 32; ++q) {
                    if (col + q >= p.n_cols) break;
                    const float v = __uint_as_float(r[q]);
                    if constexpr (OUT_BF16)
                        static_cast<__nv_bfloat16 *>(out)[(col + q) * p.ld_out + ch] = __float2bfloat16_rn(v);
                    else
                        static_cast<float *>(out)[(col + q) * p.ld_out + ch] = v;
                }
                continue;
            }
            if (p.ostore) {
                // staging: 128-byte column atoms of rows_valid rows, 128B-swizzled (chunk ^ row%8)
                if constexpr (OUT_BF16) {
                    const uint32_t atom = stage + uint32_t((c / 64) * p.rows_valid * 128 + row * 128);
                    const uint32_t ch0 = uint32_t(c % 64) / 8;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t w[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(
                                __uint_as_float(r[q * 8 + 2 * h]), __uint_as_float(r[q * 8 + 2 * h + 1]));
                            w[h] = *reinterpret_cast<uint32_t *>(&b2);
                        }
                        sts128(atom + (((ch0 + q) ^ uint32_t(row & 7)) << 4), w[0], w[1], w[2], w[3]);
                    }
                } else {
                    const uint32_t atom = stage + uint32_t((c / 32) * p.rows_valid * 128 + row * 128);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        sts128(atom + ((uint32_t(q) ^ uint32_t(row & 7)) << 4), r[4 * q], r[4 * q + 1],
                               r[4 * q + 2], r[4 * q + 3]);
                }
                continue;
            }
            if constexpr (OUT_BF16) {
                __nv_bfloat16 *dst = static_cast<__nv_bfloat16 *>(out) + (m0 + row) * p.ld_out + col;
                if (full && (reinterpret_cast<uintptr_t>(dst) % 16 == 0)) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t w[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(
                                __uint_as_float(r[q * 8 + 2 * h]), __uint_as_float(r[q * 8 + 2 * h + 1]));
                            w[h] = *reinterpret_cast<uint32_t *>(&b2);
                        }
                        reinterpret_cast<uint4 *>(dst)[q] = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                } else {
                    for (int q = 0; q < 32 && col + q < p.n_cols; ++q)
                        dst[q] = __float2bfloat16_rn(__uint_as_float(r[q]));
                }
            } else {
                float *dst = static_cast<float *>(out) + (m0 + row) * p.ld_out + col;
                if (full && (reinterpret_cast<uintptr_t>(dst) % 16 == 0)) {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<uint4 *>(dst)[q] =
                            make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                } else {
                    for (int q = 0; q < 32 && col + q < p.n_cols; ++q) dst[q] = __uint_as_float(r[q]);
                }
            }
        }
        if (p.ostore && !(DBG(p.debug) & 4)) {
            fence_async_smem();  // staged tile -> visible to the TMA (async proxy)
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (warp == 0 && elect_one()) {
                if constexpr (CONV) {
                    tma_store_2d(&omap, stage_buf, int32_t(m0), int32_t(n0));
                } else {
                    const int atom_cols = 128 / kOutElt;
                    for (int a = 0; a < p.tn / atom_cols; ++a)
                        tma_store_2d(&omap, stage_buf + a * p.rows_valid * 128, int32_t(n0) + a * atom_cols,
                                     int32_t(m0));
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
        }
        if (p.persistent) {  // accumulator drained: the MMA warp may start the next tile
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tmem_empty);
        }
    }
    }  // tile loop
    if (threadIdx.x == 0) trace(DBG(p.debug), 6, 2);
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot),
                     "r"(uint32_t(p.tmem_cols)));
    }
}

// ---------------------------------------------------------------- host side
CUtensorMapSwizzle w_swizzle(int span) {
    return span == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
         : span == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
         : span == 32  ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
}

struct TcPlan {
    TcParams p;
    size_t smem;
    int blocks_m;
};

constexpr size_t kSmemCap = 227 * 1024;

int plan_tc(const ChainDims &c, int compute, TcPlan *out, int force_tn = 0) {
    const int elt = compute == RBGP4_COMPUTE_TF32 ? 4 : 2;
    if (!(c.tm == 64 || c.tm % kBlockM == 0)) {
        set_error("tensor-core path needs tile rows tm = 64 or a multiple of 128 (tm=%d)", c.tm);
        return 0;
    }
    if ((c.tk * elt) % 32 != 0 || c.tk > 256) {
        set_error("tensor-core path needs tk*%d bytes to be a multiple of 32 and tk <= 256 (tk=%d)",
                  elt, c.tk);
        return 0;
    }
    if (c.d_t > 256 || size_t(kBlockM) * c.tk * elt > 65536) {
        set_error("tensor-core path: d_t=%d / tile %dx%d exceeds the 16-bit scatter table", c.d_t,
                  kBlockM, c.tk);
        return 0;
    }
    TcParams p{};
    p.n_cols = c.n_cols; p.ld_out = c.ld_out; p.row_nnz = c.row_nnz;
    p.ws_ld = (c.n_cols + 3) & ~int64_t(3);
    p.tm = c.tm; p.tk = c.tk; p.d_o = c.d_o; p.d_t = c.d_t; p.u_i = c.u_i; p.v_i = c.v_i;
    p.d_i = c.d_i; p.rk = c.rk; p.bm = c.bm; p.bk = c.bk;
    p.rows_valid = c.tm == 64 ? 64 : kBlockM;
    const int kbytes = c.tk * elt;
    p.a_swz = kbytes % 128 == 0 ? 128 : kbytes % 64 == 0 ? 64 : 32;
    p.a_stage_bytes = kBlockM * kbytes;
    // compressed W tiles come in by TMA when a row of one step is whole 16-byte chunks
    p.w_tma = (c.d_t * elt) % 16 == 0 && c.d_t <= 256 ? 1 : 0;
    // W stage: as many consecutive steps as fit one box (<= 256 elements, <= 8 KB)
    // one W box (one step's compressed tile) per W stage: with a step schedule consecutive
    // steps are not contiguous in `values`
    p.ws = 1;
    p.w_stage_bytes = p.w_tma ? p.rows_valid * p.ws * c.d_t * elt : 0;
    {
        const int V = 16 / elt;
        p.table_in_regs = p.w_tma && ((c.bk % V == 0 && c.d_t <= 16 * V) || c.d_t <= 64);
    }
    const int64_t blocks_m = c.rows / p.rows_valid;
    const int tn_min = 128 / elt;  // one 128-byte swizzle atom of B along N
    // tn = 128, or 64 when 128-wide tiles leave more than half the SMs idle
    // (measured on the VGG shapes with tools/tc_time.py)
    int tn = 128;
    while (tn > tn_min && tn / 2 >= c.n_cols) tn /= 2;
    if (tn > tn_min && ((c.n_cols + tn - 1) / tn) * blocks_m * 2 < kNumSMs) tn /= 2;
    if (opts().tc_tn > 0) tn = std::max(tn_min, std::min(256, int(opts().tc_tn)));
    if (force_tn) tn = force_tn;
    p.adj_smem = size_t(c.u_i) * c.d_i * 4 <= 16384 ? 1 : 0;
    // Shared-memory budget (one CTA per SM).  The main loop is bound by I-slab bytes in
    // flight per SM (TMA latency under load is ~2 us: Little's law, tools/tc_trace.py), so:
    //   1. A ring 2 deep (densify one step ahead of the MMA is enough),
    //   2. W ring 2 x <= 8 KB,
    //   3. everything left -> I stages (2..16).
    for (; tn >= tn_min; tn /= 2) {
        if (force_tn && tn != force_tn) break;
        p.tn = tn;
        p.b_stage_bytes = c.tk * tn * elt;
        p.a_stage_bytes = kBlockM * c.tk * elt;
        p.nw = p.w_tma ? 2 : 1;
        const size_t base = 1024 + size_t(kBlockM) * c.d_t * 2 + 64 +
                            (p.adj_smem ? size_t(c.u_i) * c.d_i * 4 + 16 : 0) + 8 * (2 * 16 + 2 * 16 + 2) + 16;
        size_t w_bytes = size_t(p.nw) * p.w_stage_bytes;
        int na = 2;
        if (opts().tc_na > 0) na = std::min(8, int(opts().tc_na));
        const size_t a_ring = size_t(na) * p.a_stage_bytes;
        if (base + w_bytes + a_ring + 2 * size_t(p.b_stage_bytes) > kSmemCap && p.w_tma) {
            // large compressed tiles: read W straight from global in the densify warps
            p.w_tma = 0;
            p.ws = 1;
            p.nw = 1;
            p.w_stage_bytes = 0;
            p.table_in_regs = 0;
            w_bytes = 0;
        }
        if (base + w_bytes + a_ring + 2 * size_t(p.b_stage_bytes) > kSmemCap) continue;
        // I and W rings share the rest: both chains (I slab of step s waits for the MMA of
        // s - nb, W tile of step s for the densify of s - nw) progress nb resp. nw steps per
        // load latency, so maximise min(nb, nw), then nb
        // many waves of tiles: persistent CTAs (setup, TMEM allocation and the pipeline fill
        // once per SM; loads of tile i+1 stream under the epilogue of tile i) with a dedicated
        // output staging area for the TMA-store epilogue
        const int64_t tiles_here = ((c.n_cols + tn - 1) / tn) * blocks_m;
        // Opt-in (option persistent=1): correct and tested, but measured no faster than one CTA
        // per tile on the VGG layers (the densify warps are also the epilogue warps, so the
        // densify -> MMA -> epilogue chain stays serial per tile); K4 has dedicated epilogue warps.
        (void)tiles_here;
        const bool persist = p.rows_valid == c.tm && opts().persistent == 1;
        p.pstage_bytes = persist ? int32_t(size_t(p.rows_valid) * tn * 4) : 0;  // f32 worst case
        const size_t pst = persist ? size_t(p.pstage_bytes) + 1024 : 0;
        if (base + a_ring + pst + 4 * size_t(p.b_stage_bytes) > kSmemCap) { p.pstage_bytes = 0; }
        const size_t avail = kSmemCap - (base + a_ring + (p.pstage_bytes ? pst : 0));
        int nb = 0, nw = 0;
        for (int cand = 16; cand >= 2; --cand) {
            const size_t ib = size_t(cand) * p.b_stage_bytes;
            if (ib + (p.w_tma ? 2 * size_t(p.w_stage_bytes) : 0) > avail) continue;
            const int cw = p.w_tma ? int(std::min<size_t>(cand, (avail - ib) / p.w_stage_bytes)) : 1;
            if (std::min(cand, cw) > std::min(nb, nw) || nb == 0) { nb = cand; nw = cw; }
        }
        if (opts().tc_nb > 0) {
            const int want = std::max(2, std::min(16, int(opts().tc_nb)));
            if (size_t(want) * p.b_stage_bytes + 2 * size_t(p.w_stage_bytes) <= avail) {
                nb = want;
                nw = p.w_tma ? int(std::min<size_t>(want, (avail - size_t(nb) * p.b_stage_bytes) / p.w_stage_bytes)) : 1;
            }
        }
        if (opts().tc_nw > 0 && p.w_tma)
            nw = std::max(2, std::min({16, int(opts().tc_nw), int((avail - size_t(nb) * p.b_stage_bytes) / p.w_stage_bytes)}));
        if (nb < na || nb < 2) continue;
        p.na = na;
        p.nb = nb;
        p.nw = nw;
        w_bytes = size_t(nw) * p.w_stage_bytes;
        const size_t fixed = base + w_bytes + a_ring;
        // compressed-W stage rows of exactly 32/64/128 bytes are TMA-swizzled, so the 32 rows a
        // densify warp reads land on distinct banks (unswizzled 64-byte rows are 16-way conflicted)
        {
            const int wb = p.ws * c.d_t * elt;
            p.w_swz = (p.w_tma && (wb == 32 || wb == 64 || wb == 128) && opts().wswz) ? wb : 0;
        }
        p.tmem_cols = 32;
        while (p.tmem_cols < tn) p.tmem_cols *= 2;
        const int64_t tiles = ((c.n_cols + tn - 1) / tn) * blocks_m;
        // split-K in two (a 2-CTA cluster per tile) only when that still fits one wave;
        // deeper splits measured slower (tools/tc_time.py)
        int ks = (tiles * 2 <= kNumSMs && c.d_o >= 2) ? 2 : 1;
        if (opts().ksplit > 0) ks = std::min(8, int(opts().ksplit));
        p.sps = (c.d_o + ks - 1) / ks;
        p.ksplit = (c.d_o + p.sps - 1) / p.sps;  // no empty slices
        // many waves of tiles: persistent CTAs (setup, TMEM allocation and the pipeline fill
        // once per SM; loads of tile i+1 stream under the epilogue of tile i)
        p.blocks_m = int(blocks_m);
        p.n_tiles = tiles;
        p.persistent = (p.ksplit == 1 && p.pstage_bytes && p.rows_valid == c.tm) ? 1 : 0;
        if (!p.persistent) p.pstage_bytes = 0;
        out->p = p;
        out->smem = fixed + size_t(nb) * p.b_stage_bytes + (p.pstage_bytes ? size_t(p.pstage_bytes) + 1024 : 0);
        out->blocks_m = int(blocks_m);
        return 1;
    }
    set_error("tensor-core path: tile %dx%d does not fit shared memory", c.tm, c.tk);
    return 0;
}

// The TMA-store epilogue stages the whole output tile in the (then idle) A + I rings.
bool staging_fits(const TcPlan &pl, int out_elt) {
    const size_t rings = pl.p.pstage_bytes ? size_t(pl.p.pstage_bytes)
                                           : size_t(pl.p.na) * pl.p.a_stage_bytes + size_t(pl.p.nb) * pl.p.b_stage_bytes;
    return size_t(pl.p.rows_valid) * pl.p.tn * out_elt <= rings && opts().ostore;
}

template <typename E, bool OUT_BF16, bool CONV = false>
int launch_typed(const TcPlan &pl, const CUtensorMap &map, const CUtensorMap &wmap,
                 const CUtensorMap &omap, const void *values, const int32_t *adj_o, const int32_t *adj_i, void *out,
                 float *wsp, cudaStream_t stream) {
    auto kern = tc_kernel<E, OUT_BF16, CONV>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(tc): %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    dim3 grid = pl.p.persistent
                    ? dim3(unsigned(std::min<int64_t>(pl.p.n_tiles, kNumSMs)), 1, 1)
                    : dim3(unsigned((pl.p.n_cols + pl.p.tn - 1) / pl.p.tn), unsigned(pl.blocks_m),
                           unsigned(pl.p.ksplit));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = unsigned(pl.p.ksplit);  // the K slices of one tile co-reside
    cudaLaunchAttribute attrs[2];
    unsigned na = 0;
    if (pl.p.ksplit > 1) attrs[na++] = attr[0];
    if (opts().pdl) {
        attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = na;
    note_kernel(pl.p.conv ? "K2 conv" : "K2 tc");
    e = cudaLaunchKernelEx(&cfg, kern, map, wmap, omap, pl.p, static_cast<const E *>(values), adj_o, adj_i,
                           out, wsp);
    if (e != cudaSuccess) {
        set_error("tc_kernel launch (grid %u x %u x %u, smem %zu): %s", grid.x, grid.y, grid.z,
                  pl.smem, cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    RBGP4_CHECK_LAUNCH("tc_kernel launch");
    return RBGP4_OK;
}

}  // namespace

// ---------------------------------------------------------------- step schedule
// Every tile-row walks only its g_o neighbours (as the reference does), but in which order
// is free for the tensor-core modes (fp32 accumulation; no bit-exactness claim).  When
// d_r(g_o) >= 2, several tile-rows read the same I slab: if they read it at the SAME step,
// their CTAs (same column block, launched in the same wave) request the same lines at about
// the same time and L2 serves them once, instead of a second full pass over I later.  The
// schedule picks, per step, a set of vertex-disjoint K-blocks covering as many tile-rows as
// possible.  For u_o = 4 and right degree 2 (the VGG/WRN factorisations) the K-blocks are the
// edges of a d_o-regular multigraph on 4 vertices, which always splits into the 3 perfect
// matchings {01,23} {02,13} {03,12} (x01 = x23, x02 = x13, x03 = x12 follows from
// regularity), so every slab is read by both of its tile-rows at the same step.
namespace {
struct Lcg {
    uint64_t x;
    uint32_t next() { x = x * 6364136223846793005ull + 1442695040888963407ull; return uint32_t(x >> 33); }
};

// sched[u * d_o + s] = adjacency slot j of tile-row u read at step s; returns #slab reads
int64_t schedule_cost(int u_o, int d_o, const int32_t *adj, const std::vector<int32_t> &sched) {
    std::vector<std::pair<int, int>> reads;  // (step, K-block)
    for (int u = 0; u < u_o; ++u)
        for (int s = 0; s < d_o; ++s) reads.emplace_back(s, adj[u * d_o + sched[u * d_o + s]]);
    std::sort(reads.begin(), reads.end());
    return std::unique(reads.begin(), reads.end()) - reads.begin();
}

void build_schedule(int u_o, int v_o, int d_o, const int32_t *adj, int32_t *out) {
    std::vector<int32_t> best(size_t(u_o) * d_o);
    for (int u = 0; u < u_o; ++u)
        for (int s = 0; s < d_o; ++s) best[u * d_o + s] = s;  // reference order
    int64_t best_cost = schedule_cost(u_o, d_o, adj, best);
    // slot of K-block kb in tile-row u's adjacency row (-1 if not adjacent)
    std::vector<int> slot(size_t(u_o) * v_o, -1);
    std::vector<std::vector<int>> users(v_o);
    for (int u = 0; u < u_o; ++u)
        for (int j = 0; j < d_o; ++j) {
            slot[size_t(u) * v_o + adj[u * d_o + j]] = j;
            users[adj[u * d_o + j]].push_back(u);
        }
    auto consider = [&](const std::vector<int32_t> &cand) {
        const int64_t cost = schedule_cost(u_o, d_o, adj, cand);
        if (cost < best_cost) { best_cost = cost; best = cand; }
    };
    if (u_o == 4) {
        bool deg2 = true;
        for (int kb = 0; kb < v_o; ++kb) deg2 &= users[kb].empty() || users[kb].size() == 2;
        if (deg2) {
            // edges per vertex pair, then the three perfect matchings in turn
            std::vector<int> pairs[4][4];
            for (int kb = 0; kb < v_o; ++kb)
                if (!users[kb].empty()) pairs[users[kb][0]][users[kb][1]].push_back(kb);
            const int mt[3][2][2] = {{{0, 1}, {2, 3}}, {{0, 2}, {1, 3}}, {{0, 3}, {1, 2}}};
            std::vector<int32_t> cand(size_t(u_o) * d_o, -1);
            std::vector<int> step(u_o, 0);
            bool ok = true;
            for (auto &m : mt) {
                const auto &e0 = pairs[m[0][0]][m[0][1]], &e1 = pairs[m[1][0]][m[1][1]];
                ok &= e0.size() == e1.size();
                for (int i = 0; ok && i < int(e0.size()); ++i)
                    for (int h = 0; h < 2; ++h) {
                        const int kb = h ? e1[i] : e0[i];
                        for (int v : {m[h][0], m[h][1]}) cand[v * d_o + step[v]++] = slot[size_t(v) * v_o + kb];
                    }
            }
            for (int u = 0; u < u_o; ++u) ok &= step[u] == d_o;
            if (ok) consider(cand);
        }
    }
    // general case: seeded randomised greedy; per step take vertex-disjoint shared K-blocks,
    // then let leftover tile-rows read a K-block whose sharing is already lost
    Lcg rng{0x9E3779B97F4A7C15ull};
    for (int trial = 0; trial < 48 && u_o > 1; ++trial) {
        std::vector<int32_t> cand(size_t(u_o) * d_o, -1);
        std::vector<std::vector<char>> rem(u_o, std::vector<char>(v_o, 0));
        std::vector<int> left(v_o, 0);  // users that still have kb pending
        for (int u = 0; u < u_o; ++u)
            for (int j = 0; j < d_o; ++j) { rem[u][adj[u * d_o + j]] = 1; ++left[adj[u * d_o + j]]; }
        std::vector<int> order(v_o);
        for (int i = 0; i < v_o; ++i) order[i] = i;
        for (int s = 0; s < d_o; ++s) {
            for (int i = v_o - 1; i > 0; --i) std::swap(order[i], order[rng.next() % (i + 1)]);
            std::vector<char> busy(u_o, 0);
            for (int kb : order) {
                if (left[kb] < 2 || left[kb] != int(users[kb].size())) continue;
                bool free = true;
                for (int u : users[kb]) free &= !busy[u];
                if (!free) continue;
                for (int u : users[kb]) {
                    busy[u] = 1; rem[u][kb] = 0;
                    cand[u * d_o + s] = slot[size_t(u) * v_o + kb];
                }
                left[kb] = 0;
            }
            for (int u = 0; u < u_o; ++u) {
                if (busy[u]) continue;
                int pick = -1;
                for (int j = 0; j < d_o; ++j) {
                    const int kb = adj[u * d_o + j];
                    if (rem[u][kb] && (pick < 0 || left[kb] < left[pick])) pick = kb;
                }
                rem[u][pick] = 0;
                --left[pick];
                cand[u * d_o + s] = slot[size_t(u) * v_o + pick];
            }
        }
        consider(cand);
    }
    std::copy(best.begin(), best.end(), out);
}

size_t scatter_bytes(const ChainDims &c, const TcPlan &pl) {
    const int phases = c.tm / pl.p.rows_valid;
    return (size_t(phases) * c.d_t * kBlockM * sizeof(uint16_t) + 15) & ~size_t(15);
}
}  // namespace

// prepared buffer: [scatter map u16: phase x d_t x 128, 16-byte padded][schedule i32: u_o x d_o,
// padded][K4 relayout section (bf16 only, sdmm_gather.cu)]
namespace {
// schedule then partner table ([tile-row][s] -> tile-row reading the same slab at step s, or -1)
size_t sched_end(const ChainDims &c, const TcPlan &pl) {
    return (scatter_bytes(c, pl) + 2 * size_t(c.u_o) * c.d_o * sizeof(int32_t) + 15) & ~size_t(15);
}
size_t k4_bytes(const ChainDims &c, int compute) {
    return compute == RBGP4_COMPUTE_BF16 ? gather_prep_bytes(c) : 0;
}
size_t k5_bytes(const ChainDims &c, int compute) {
    return compute == RBGP4_COMPUTE_BF16 ? stream_prep_bytes(c) : 0;
}
}  // namespace

size_t tc_prep_size(const ChainDims &c, int compute) {
    TcPlan pl;
    if (!plan_tc(c, compute, &pl)) return 0;
    return sched_end(c, pl) + ((k4_bytes(c, compute) + 15) & ~size_t(15)) + k5_bytes(c, compute);
}

const int32_t *tc_prep_schedule(const ChainDims &c, const TcPlan &pl, const void *prep) {
    return prep ? reinterpret_cast<const int32_t *>(static_cast<const char *>(prep) + scatter_bytes(c, pl))
                : nullptr;
}

const int32_t *tc_prep_pair(const ChainDims &c, const TcPlan &pl, const void *prep) {
    return prep ? tc_prep_schedule(c, pl, prep) + size_t(c.u_o) * c.d_o : nullptr;
}

const void *tc_prep_k4(const ChainDims &c, const TcPlan &pl, int compute, const void *prep) {
    return prep && k4_bytes(c, compute) ? static_cast<const char *>(prep) + sched_end(c, pl) : nullptr;
}

// K5 tables (sdmm_stream.cu) after the K4 section
const void *tc_prep_k5(const ChainDims &c, const TcPlan &pl, int compute, const void *prep) {
    return prep && k5_bytes(c, compute)
               ? static_cast<const char *>(prep) + sched_end(c, pl) + ((k4_bytes(c, compute) + 15) & ~size_t(15))
               : nullptr;
}

int tc_prepare(const ChainDims &c, int compute, const void *values, const int32_t *adj_o,
               const int32_t *adj_i, void *prep, size_t bytes, cudaStream_t stream) {
    TcPlan pl;
    if (!plan_tc(c, compute, &pl)) return RBGP4_EUNSUPPORTED;
    const size_t need = tc_prep_size(c, compute);
    if (prep == nullptr || bytes < need) {
        set_error("rbgp4_prepare needs %zu bytes", need);
        return RBGP4_EWORKSPACE;
    }
    const int phases = c.tm / pl.p.rows_valid;
    if (compute == RBGP4_COMPUTE_TF32)
        prep_kernel<4><<<phases, kBlockM, 0, stream>>>(pl.p, adj_i, static_cast<uint16_t *>(prep));
    else
        prep_kernel<2><<<phases, kBlockM, 0, stream>>>(pl.p, adj_i, static_cast<uint16_t *>(prep));
    RBGP4_CHECK_LAUNCH("prep_kernel launch");
    // the step schedule is a small host-side search over g_o's adjacency (once per matrix)
    std::vector<int32_t> adj(size_t(c.u_o) * c.d_o), sched(adj.size()), adji(size_t(c.u_i) * c.d_i);
    cudaError_t e = cudaMemcpyAsync(adj.data(), adj_o, adj.size() * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(adji.data(), adj_i, adji.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) {
        set_error("rbgp4_prepare: reading the adjacency: %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    build_schedule(c.u_o, c.v_o, c.d_o, adj.data(), sched.data());
    if (!opts().sched)
        for (int u = 0; u < c.u_o; ++u)
            for (int s2 = 0; s2 < c.d_o; ++s2) sched[size_t(u) * c.d_o + s2] = s2;
    // pairs: per step, tile-rows reading the same K-block are matched two by two (symmetric)
    std::vector<int32_t> both(2 * sched.size(), -1);
    std::copy(sched.begin(), sched.end(), both.begin());
    int32_t *pair = both.data() + sched.size();
    for (int s2 = 0; s2 < c.d_o; ++s2)
        for (int u = 0; u < c.u_o; ++u) {
            if (pair[size_t(u) * c.d_o + s2] >= 0) continue;
            const int kb = adj[size_t(u) * c.d_o + sched[size_t(u) * c.d_o + s2]];
            for (int v = u + 1; v < c.u_o; ++v)
                if (pair[size_t(v) * c.d_o + s2] < 0 && adj[size_t(v) * c.d_o + sched[size_t(v) * c.d_o + s2]] == kb) {
                    pair[size_t(u) * c.d_o + s2] = v;
                    pair[size_t(v) * c.d_o + s2] = u;
                    break;
                }
        }
    sched.swap(both);
    e = cudaMemcpyAsync(const_cast<int32_t *>(tc_prep_schedule(c, pl, prep)), sched.data(),
                        sched.size() * sizeof(int32_t), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // `sched` is a host temporary
    if (e != cudaSuccess) {
        set_error("rbgp4_prepare: writing the schedule: %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    if (const void *k5 = tc_prep_k5(c, pl, compute, prep)) {
        if (values == nullptr) {
            set_error("rbgp4_prepare: values needed for the bf16 relayout");
            return RBGP4_EINVAL;
        }
        if (int rc = stream_prepare(c, values, adj.data(), sched.data(), adji.data(), const_cast<void *>(k5), stream))
            return rc;
    }
    if (const void *k4 = tc_prep_k4(c, pl, compute, prep)) {
        if (values == nullptr) {
            set_error("rbgp4_prepare: values needed for the bf16 relayout");
            return RBGP4_EINVAL;
        }
        return gather_prepare(c, values, adji.data(), const_cast<void *>(k4), stream);
    }
    return RBGP4_OK;
}

int tc_prepare_values(const ChainDims &c, int compute, const void *values, void *prep, size_t bytes,
                      cudaStream_t stream) {
    TcPlan pl;
    if (!plan_tc(c, compute, &pl)) return RBGP4_EUNSUPPORTED;
    if (prep == nullptr || bytes < tc_prep_size(c, compute)) {
        set_error("rbgp4_prepare_values needs the %zu-byte buffer of rbgp4_prepare", tc_prep_size(c, compute));
        return RBGP4_EWORKSPACE;
    }
    RBGP4_REQUIRE(values != nullptr, "rbgp4_prepare_values: null values");
    if (const void *k5 = tc_prep_k5(c, pl, compute, prep))
        if (int rc = stream_prepare_values(c, values, const_cast<void *>(k5), stream)) return rc;
    if (const void *k4 = tc_prep_k4(c, pl, compute, prep))
        return gather_prepare_values(c, values, const_cast<void *>(k4), stream);
    return RBGP4_OK;
}

int tc_supported(const ChainDims &c, int compute, int out_dtype) {
    if (out_dtype != RBGP4_F32 && out_dtype != RBGP4_BF16) {
        set_error("tensor-core modes write f32 or bf16 outputs");
        return 0;
    }
    TcPlan pl;
    return plan_tc(c, compute, &pl);
}

size_t tc_workspace_size(const ChainDims &c, int compute) {
    // K4 splits K over DSMEM (either mode)
    if (gather_supported(c, compute, RBGP4_BF16, false) || gather_supported(c, compute, RBGP4_BF16, true))
        return 0;
    TcPlan pl;
    if (!plan_tc(c, compute, &pl) || pl.p.ksplit <= 1) return 0;
    // (ksplit - 1) fp32 partial copies of the output, row-major (rows, ws_ld)
    return size_t(pl.p.ksplit - 1) * size_t(pl.blocks_m) * pl.p.rows_valid * size_t(pl.p.ws_ld) * 4;
}

int launch_tc(const ChainDims &c, int compute, int out_dtype, const void *values,
              const int32_t *adj_o, const int32_t *adj_i, const void *prep, const void *inp,
              void *out, void *workspace, size_t workspace_bytes, cudaStream_t stream) {
    if (c.n_cols == 0) return RBGP4_OK;
    TcPlan pl;
    if (!plan_tc(c, compute, &pl)) return RBGP4_EUNSUPPORTED;
    pl.p.prep = static_cast<const uint16_t *>(prep);
    pl.p.sched = tc_prep_schedule(c, pl, prep);
    // prepared bf16 with a K5 section (TC16 or slice relayout): the streamed kernel (K5)
    {
        const void *k4 = tc_prep_k4(c, pl, compute, prep), *k5 = tc_prep_k5(c, pl, compute, prep);
        if (compute == RBGP4_COMPUTE_BF16 && k5 && (k4 || !stream_shape_ok(c)) && stream_supported(c, out_dtype))
            return launch_stream(c, out_dtype, k4, k5, inp, out, stream);
    }
    // g_b blocks >= 16 x 16: the gathered-block kernel (K4), no densification
    {
        const void *k4 = tc_prep_k4(c, pl, compute, prep);
        if (gather_supported(c, compute, out_dtype, k4 != nullptr))
            return launch_gather(c, out_dtype, values, adj_o, adj_i, pl.p.sched, tc_prep_pair(c, pl, prep), k4,
                                 inp, out, stream);
    }
    const int elt = compute == RBGP4_COMPUTE_TF32 ? 4 : 2;
    if (reinterpret_cast<uintptr_t>(inp) % 16 != 0 || (c.ld_in * elt) % 16 != 0) {
        set_error("tensor-core path needs a 16-byte aligned I with ld_in*%d %% 16 == 0", elt);
        return RBGP4_EUNSUPPORTED;
    }
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    CUtensorMap map;
    cuuint32_t estr[3] = {1, 1, 1};
    const int atom_cols = 128 / elt;
    CUresult r;
    pl.p.i3d = (c.n_cols % atom_cols == 0) ? 1 : 0;
    if (!opts().i3d) pl.p.i3d = 0;
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (opts().promo >= 0)
        promo = opts().promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
              : opts().promo == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : opts().promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (pl.p.i3d) {
        // (atom cols, K rows, N atoms) view: one box = one whole I slab, atom-major in smem
        cuuint64_t dims[3] = {cuuint64_t(atom_cols), cuuint64_t(c.cols), cuuint64_t(c.n_cols / atom_cols)};
        cuuint64_t strides[2] = {cuuint64_t(c.ld_in) * elt, 128};
        cuuint32_t box[3] = {cuuint32_t(atom_cols), cuuint32_t(c.tk), cuuint32_t(pl.p.tn / atom_cols)};
        r = enc(&map, elt == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                const_cast<void *>(inp), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                elt == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[2] = {cuuint64_t(c.n_cols), cuuint64_t(c.cols)};
        cuuint64_t strides[1] = {cuuint64_t(c.ld_in) * elt};
        cuuint32_t box[2] = {cuuint32_t(atom_cols), cuuint32_t(c.tk)};
        r = enc(&map, elt == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                const_cast<void *>(inp), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                elt == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", int(r));
        return RBGP4_ECUDA;
    }
    if (DBG(opts().debug)) {
        pl.p.debug = DBG(opts().debug);
        if (pl.p.debug & 8192)
            fprintf(stderr, "[rbgp4 tc plan] tn=%d na=%d nb=%d nw=%d ws=%d w_tma=%d w_swz=%d ks=%d smem=%zu tmem=%d\n",
                    pl.p.tn, pl.p.na, pl.p.nb, pl.p.nw, pl.p.ws, pl.p.w_tma, pl.p.w_swz, pl.p.ksplit, pl.smem,
                    pl.p.tmem_cols);
        if (pl.p.debug & 16) { pl.p.w_tma = 0; pl.p.nw = 1; pl.p.ws = 1; pl.p.w_stage_bytes = 0; pl.p.w_swz = 0; }
    }
    // output tile store: (n_cols, rows) view, box = one 128-byte column atom x rows of a CTA
    CUtensorMap omap;
    memset(&omap, 0, sizeof(omap));
    {
        const int oelt = out_dtype == RBGP4_BF16 ? 2 : 4;
        pl.p.ostore = staging_fits(pl, oelt) && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
                      (c.ld_out * oelt) % 16 == 0 && (pl.p.tn * oelt) % 128 == 0;
        if (pl.p.ostore) {
            cuuint64_t odims[2] = {cuuint64_t(c.n_cols), cuuint64_t(c.rows)};
            cuuint64_t ostrides[1] = {cuuint64_t(c.ld_out) * oelt};
            cuuint32_t obox[2] = {cuuint32_t(128 / oelt), cuuint32_t(pl.p.rows_valid)};
            r = enc(&omap, oelt == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    out, odims, ostrides, obox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) pl.p.ostore = 0;
        }
    }
    // compressed W tiles: 2-D (row_nnz, rows) view of the values, box (d_t, rows of a CTA)
    CUtensorMap wmap;
    memset(&wmap, 0, sizeof(wmap));
    if (pl.p.w_tma) {
        cuuint64_t wdims[2] = {cuuint64_t(c.row_nnz), cuuint64_t(c.rows)};
        cuuint64_t wstrides[1] = {cuuint64_t(c.row_nnz) * elt};
        cuuint32_t wbox[2] = {cuuint32_t(pl.p.ws * c.d_t), cuuint32_t(pl.p.rows_valid)};
        if (reinterpret_cast<uintptr_t>(values) % 16 != 0) {
            set_error("tensor-core path needs 16-byte aligned values");
            return RBGP4_EUNSUPPORTED;
        }
        r = enc(&wmap, elt == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                2, const_cast<void *>(values), wdims, wstrides, wbox, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, w_swizzle(pl.p.w_swz),
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(values) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    float *wsp = static_cast<float *>(workspace);
    if (pl.p.ksplit > 1 && (wsp == nullptr || workspace_bytes < tc_workspace_size(c, compute))) {
        set_error("split-K (%d slices) needs %zu workspace bytes", pl.p.ksplit,
                  tc_workspace_size(c, compute));
        return RBGP4_EWORKSPACE;
    }
    const bool obf = out_dtype == RBGP4_BF16;
    if (compute == RBGP4_COMPUTE_TF32)
        return obf ? launch_typed<float, true>(pl, map, wmap, omap, values, adj_o, adj_i, out, wsp, stream)
                   : launch_typed<float, false>(pl, map, wmap, omap, values, adj_o, adj_i, out, wsp, stream);
    return obf ? launch_typed<__nv_bfloat16, true>(pl, map, wmap, omap, values, adj_o, adj_i, out, wsp, stream)
               : launch_typed<__nv_bfloat16, false>(pl, map, wmap, omap, values, adj_o, adj_i, out, wsp, stream);
}

// ---------------------------------------------------------------- K3: implicit im2col
namespace {
// output map of a 'same'-padded (pad = (k-1)/2) convolution with stride 1 or 2
void conv_out(const rbgp4_conv_desc &cv, int *oh, int *ow) {
    *oh = (cv.height + 2 * cv.pad - cv.kh) / cv.stride + 1;
    *ow = (cv.width + 2 * cv.pad - cv.kw) / cv.stride + 1;
}
int conv_tile(const rbgp4_conv_desc &cv, int tn, int *th, int *tb) {
    int oh, ow;
    conv_out(cv, &oh, &ow);
    const int hw = oh * ow;
    if (tn % ow) return 0;
    if (tn <= hw) {
        *th = tn / ow;
        *tb = 1;
        return oh % *th == 0;
    }
    *th = oh;
    *tb = tn / hw;
    return tn % hw == 0 && *tb <= 256;
}
}  // namespace

int conv_plan(const ChainDims &c, const rbgp4_conv_desc *cv, TcPlan *pl) {
    RBGP4_REQUIRE(cv != nullptr, "null conv descriptor");
    RBGP4_REQUIRE((cv->stride == 1 || cv->stride == 2) && cv->pad * 2 == cv->kh - 1 && cv->kh == cv->kw,
                  "implicit-im2col path supports 'same'-padded square convolutions of stride 1 or 2 "
                  "(kh=%d, pad=%d, stride=%d)", cv->kh, cv->pad, cv->stride);
    RBGP4_REQUIRE(c.cols == int64_t(cv->kh) * cv->kw * cv->c_in,
                  "chain columns %lld != kh*kw*c_in = %d (tap-major im2col order)", (long long)c.cols,
                  cv->kh * cv->kw * cv->c_in);
    int oh, ow;
    conv_out(*cv, &oh, &ow);
    RBGP4_REQUIRE(c.n_cols == int64_t(cv->batch) * oh * ow,
                  "n_cols %lld != batch*out_height*out_width", (long long)c.n_cols);
    RBGP4_REQUIRE(c.tk % 64 == 0 && cv->c_in % c.tk == 0,
                  "conv path needs tk %% 64 == 0 and c_in %% tk == 0 (tk=%d, c_in=%d)", c.tk, cv->c_in);
    RBGP4_REQUIRE(cv->width <= 256 && cv->height <= 256, "feature map too large for one TMA box");
    // wide pixel tiles when the grid is many waves deep: the per-CTA setup (TMEM, barriers,
    // scatter table, pipeline fill) is amortised over twice the pixels
    const bool wide = c.n_cols >= int64_t(kNumSMs) * 256 * 4 && opts().conv_wide;
    for (int tn : {256, 128, 64}) {
        if (tn == 256 && !wide) continue;
        int th, tb;
        if (!conv_tile(*cv, tn, &th, &tb)) continue;
        if (!plan_tc(c, RBGP4_COMPUTE_BF16, pl, tn)) continue;
        pl->p.conv = 1;
        pl->p.c_in = cv->c_in;
        pl->p.img_h = oh;
        pl->p.img_w = ow;
        pl->p.stride = cv->stride;
        pl->p.kw = cv->kw;
        pl->p.pad = cv->pad;
        pl->p.relu = cv->relu;
        pl->p.th = th;
        pl->p.tb = tb;
        pl->p.ld_out = c.rows;  // NHWC: a pixel row holds c_out channels
        return 1;
    }
    set_error("no pixel tiling of %dx%d maps into 128 or 64 columns", cv->height, cv->width);
    return 0;
}

size_t conv_workspace_size(const ChainDims &c, const rbgp4_conv_desc *cv) {
    if (cv != nullptr && (gather_conv_supported(c, cv, RBGP4_BF16, false) ||
                          gather_conv_supported(c, cv, RBGP4_BF16, true)))
        return 0;
    TcPlan pl;
    if (!conv_plan(c, cv, &pl) || pl.p.ksplit <= 1) return 0;
    return size_t(pl.p.ksplit - 1) * size_t(pl.blocks_m) * pl.p.rows_valid * size_t(pl.p.ws_ld) * 4;
}

int launch_conv(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, const void *values,
                const int32_t *adj_o, const int32_t *adj_i, const void *prep, const void *x,
                void *out, void *workspace, size_t workspace_bytes, cudaStream_t stream) {
    TcPlan pl;
    if (!conv_plan(c, cv, &pl)) return RBGP4_EUNSUPPORTED;
    if (c.n_cols == 0) return RBGP4_OK;
    pl.p.prep = static_cast<const uint16_t *>(prep);
    pl.p.sched = tc_prep_schedule(c, pl, prep);
    {
        const void *k4 = tc_prep_k4(c, pl, RBGP4_COMPUTE_BF16, prep), *k5 = tc_prep_k5(c, pl, RBGP4_COMPUTE_BF16, prep);
        if (k5 && (k4 || !stream_shape_ok(c)) && stream_conv_supported(c, cv, out_dtype))
            return launch_stream_conv(c, cv, out_dtype, k4, k5, x, out, stream);
    }
    if (cv->relu & RBGP4_CONV_POOL2) {
        set_error("rbgp4_conv2d: the fused 2x2 pool runs on the streamed kernel only (this shape: pool separately)");
        return RBGP4_EUNSUPPORTED;
    }
    if (conv_epilogue().res != nullptr) {
        set_error("rbgp4_conv2d_residual: the residual epilogue runs on the streamed kernel only (this shape: add separately)");
        return RBGP4_EUNSUPPORTED;
    }
    {
        const void *k4 = tc_prep_k4(c, pl, RBGP4_COMPUTE_BF16, prep);
        if (gather_conv_supported(c, cv, out_dtype, k4 != nullptr))
            return launch_gather_conv(c, cv, out_dtype, values, adj_o, adj_i, pl.p.sched, tc_prep_pair(c, pl, prep),
                                      k4, x, out, stream);
    }
    RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(x) % 16 == 0 && (cv->c_in * 2) % 16 == 0,
                  "conv input must be 16-byte aligned NHWC bf16");
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    // x: NHWC bf16 as a 4-D tensor (C, W, H, B); box = 64 channels x full width x th rows x tb
    CUtensorMap map, wmap;
    cuuint64_t dims[4] = {cuuint64_t(cv->c_in), cuuint64_t(cv->width), cuuint64_t(cv->height),
                          cuuint64_t(cv->batch)};
    cuuint64_t strides[3] = {cuuint64_t(cv->c_in) * 2, cuuint64_t(cv->width) * cv->c_in * 2,
                             cuuint64_t(cv->height) * cv->width * cv->c_in * 2};
    // strided convolution: the box spans stride x the output extent and loads every stride-th pixel
    const cuuint32_t sd = cuuint32_t(cv->stride);
    cuuint32_t box[4] = {64, cuuint32_t(pl.p.img_w) * sd, cuuint32_t(pl.p.th) * sd, cuuint32_t(pl.p.tb)};
    cuuint32_t estr[4] = {1, sd, sd, 1};
    const cuuint32_t ones4[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(x), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled(conv input) failed (%d)", int(r));
        return RBGP4_ECUDA;
    }
    // NHWC output store: (c_out, pixels) view, box = the CTA's channels x tn pixels
    CUtensorMap omap;
    memset(&omap, 0, sizeof(omap));
    {
        const int oelt = out_dtype == RBGP4_BF16 ? 2 : 4;
        pl.p.ostore = staging_fits(pl, oelt) && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
                      (c.rows * oelt) % 16 == 0 && pl.p.rows_valid * oelt >= 16;
        if (pl.p.ostore) {
            cuuint64_t odims[2] = {cuuint64_t(c.rows), cuuint64_t(c.n_cols)};
            cuuint64_t ostrides[1] = {cuuint64_t(c.rows) * oelt};
            cuuint32_t obox[2] = {cuuint32_t(pl.p.rows_valid), cuuint32_t(pl.p.tn)};
            r = enc(&omap, oelt == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    out, odims, ostrides, obox, ones4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) pl.p.ostore = 0;
        }
    }
    memset(&wmap, 0, sizeof(wmap));
    if (pl.p.w_tma) {
        cuuint64_t wdims[2] = {cuuint64_t(c.row_nnz), cuuint64_t(c.rows)};
        cuuint64_t wstrides[1] = {cuuint64_t(c.row_nnz) * 2};
        cuuint32_t wbox[2] = {cuuint32_t(pl.p.ws * c.d_t), cuuint32_t(pl.p.rows_valid)};
        r = enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(values), wdims,
                wstrides, wbox, ones4, CU_TENSOR_MAP_INTERLEAVE_NONE, w_swizzle(pl.p.w_swz),
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(values) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    float *wsp = static_cast<float *>(workspace);
    if (pl.p.ksplit > 1 && (wsp == nullptr || workspace_bytes < conv_workspace_size(c, cv))) {
        set_error("split-K conv needs %zu workspace bytes", conv_workspace_size(c, cv));
        return RBGP4_EWORKSPACE;
    }
    return out_dtype == RBGP4_BF16
               ? launch_typed<__nv_bfloat16, true, true>(pl, map, wmap, omap, values, adj_o, adj_i, out, wsp, stream)
               : launch_typed<__nv_bfloat16, false, true>(pl, map, wmap, omap, values, adj_o, adj_i, out, wsp, stream);
}

}  // namespace rbgp4

#if RBGP4_DEBUG
// debug builds only (not part of include/rbgp4.h): copy the CTA-0 trace to the host
extern "C" int rbgp4_debug_trace(unsigned long long *host, int n) {
    if (n > 10 * rbgp4::kTraceSteps) n = 10 * rbgp4::kTraceSteps;
    return cudaMemcpyFromSymbol(host, rbgp4::g_trace, sizeof(unsigned long long) * n) == cudaSuccess
               ? 0 : -3;
}
#endif  // RBGP4_DEBUG
