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

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

namespace rbgp4 {
namespace {

constexpr int kThreads = 224;

// Debug trace (RBGP4_TC_DEBUG bit 8): CTA 0 stamps clock64 at every role hand-off.
// Layout: [event][step], event = 0 B issued, 1 W issued, 2 densify start, 3 densify end,
// 4 MMA start, 5 MMA end; [6][0] setup done, [6][1] epilogue start, [6][2] epilogue end;
// 7 MMA saw full_b, 8 densify saw full_w (per W stage).
constexpr int kTraceSteps = 512;
__device__ unsigned long long g_trace[10][kTraceSteps];
__device__ __forceinline__ void trace(const int debug, int ev, int step) {
    if ((debug & 8) && blockIdx.x == 0 && blockIdx.y == 0 && step < kTraceSteps)
        g_trace[ev][step] = clock64();
}
constexpr int kBlockM = 128;

struct TcParams {
    int64_t n_cols, ld_out, row_nnz;
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
    int32_t table_in_regs;   // densify keeps each row's offsets in registers (else smem table)
    int32_t a_tmem;          // A tiles assembled in TMEM (tcgen05.st) and read by TS-mode MMAs
    int32_t a_tcols;         // TMEM columns per A stage (tk * elt / 4)
    int32_t tmem_cols;       // TMEM allocation (power of two)
    // implicit-im2col convolution (K3): I is never materialised; x is NHWC bf16 and the
    // slab of step s is the tap (i, j) / channel block of its K rows, fetched by a 4-D TMA
    // box at the tap-shifted coordinates (out-of-bounds = zero padding); O is NHWC.
    int32_t conv, c_in, img_h, img_w, kw, pad, relu, th, tb;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef RBGP4_MBAR_POLL
#define RBGP4_MBAR_POLL 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
#if RBGP4_MBAR_POLL
    // pure polling: test_wait never suspends the thread
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr), "r"(parity) : "memory");
#else
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr), "r"(parity) : "memory");
#endif
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int32_t x, int32_t y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void sts16(uint32_t addr, uint16_t v) {
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
template <typename E>
__device__ __forceinline__ void sts_elem(uint32_t addr, E v) {
    if constexpr (sizeof(E) == 2) sts16(addr, *reinterpret_cast<uint16_t *>(&v));
    else sts32(addr, *reinterpret_cast<uint32_t *>(&v));
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int32_t x, int32_t y, int32_t z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int32_t x, int32_t y, int32_t z, int32_t w) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .pred p;\n.reg .b32 r;\n"
        "elect.sync r|p, 0xffffffff;\n"
        "selp.b32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                     "r"(smem_u32(bar)) : "memory");
}
template <bool TF32>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
    if constexpr (TF32) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
    }
}
// A from TMEM (TS): A must be K-major (lane = row), B from shared memory.
template <bool TF32>
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
    if constexpr (TF32) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n}\n" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u));
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n}\n" ::"r"(d_tmem),
            "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0u));
    }
}
#define TMEM_ST_32x32b_X32(taddr, r)                                                        \
    asm volatile(                                                                           \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"  \
        "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" \
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),        \
        "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),      \
        "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]),  \
        "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),  \
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory")
// one of q[0..3] by a runtime index without local memory (SEL chains)
__device__ __forceinline__ uint4 sel4(const uint4 &a, const uint4 &b, const uint4 &c, const uint4 &d,
                                      uint32_t idx) {
    const bool o = idx & 1, t = idx & 2;
    uint4 x, y, r;
    x.x = o ? b.x : a.x; x.y = o ? b.y : a.y; x.z = o ? b.z : a.z; x.w = o ? b.w : a.w;
    y.x = o ? d.x : c.x; y.y = o ? d.y : c.y; y.z = o ? d.z : c.z; y.w = o ? d.w : c.w;
    r.x = t ? y.x : x.x; r.y = t ? y.y : x.y; r.z = t ? y.z : x.z; r.w = t ? y.w : x.w;
    return r;
}

// UMMA shared-memory matrix descriptor (sm_100: version 1 at bit 46).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout & 7) << 61;
    return d;
}
__device__ __forceinline__ uint32_t swizzle_layout_code(int span) {
    return span == 128 ? 2u : span == 64 ? 4u : 6u;  // SWIZZLE_128B / 64B / 32B
}
// byte offset -> swizzled byte offset inside a (8 rows x span) atom region
__device__ __forceinline__ uint32_t swz(uint32_t off, int span) {
    const uint32_t mask = span == 128 ? 7u : span == 64 ? 3u : 1u;
    return off ^ (((off >> 7) & mask) << 4);
}

#define TMEM_LD_32x32b_X32(taddr, r)                                                       \
    asm volatile(                                                                          \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"    \
        "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}," \
        " [%32];"                                                                          \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),          \
          "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),        \
          "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),    \
          "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),    \
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),    \
          "=r"(r[30]), "=r"(r[31])                                                         \
        : "r"(taddr))

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
          const TcParams p, const E *__restrict__ values, const int32_t *__restrict__ adj_o,
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
    // aoff[j * 128 + r]: byte offset (inside an A stage) of nonzero j of CTA row r
    uint16_t *aoff = reinterpret_cast<uint16_t *>(w_buf + p.nw * p.w_stage_bytes);
    int32_t *adj_s = reinterpret_cast<int32_t *>(
        (reinterpret_cast<uintptr_t>(aoff + kBlockM * p.d_t) + 15) & ~uintptr_t(15));
    uint64_t *bars = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(adj_s + (p.adj_smem ? p.u_i * p.d_i : 0)) + 7) & ~uintptr_t(7));
    // one ring of ns = na = nb stages, each holding an A tile and an I slab:
    // full[st] completes on the TMA transaction bytes + 4 densify-warp arrivals,
    // empty[st] on the MMA commit (one wait and one commit per step for the MMA warp)
    uint64_t *full_b = bars, *empty_b = full_b + p.nb;
    uint64_t *full_a = full_b, *empty_a = empty_b;
    uint64_t *full_w = empty_b + p.nb, *empty_w = full_w + p.nw;
    uint64_t *tmem_full = empty_w + p.nw;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) trace(p.debug, 6, 3);
    const int64_t n0 = int64_t(blockIdx.x) * p.tn;
    const int64_t m0 = int64_t(blockIdx.y) * p.rows_valid;  // first W row of this CTA
    const int64_t tbm = m0 / p.tm;
    const int row_in_tile0 = int(m0 - tbm * p.tm);
    // split-K: this CTA runs steps [s_begin, s_begin + nsteps) of the tile-row
    const int kslice = blockIdx.z;
    const int s_begin = kslice * p.sps;
    const int nsteps = min(p.d_o, s_begin + p.sps) - s_begin;

    // TMEM first: the allocation latency overlaps the table build below
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(uint32_t(p.tmem_cols)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        if (lane == 0) trace(p.debug, 6, 5);
    }
    // ---- one-time setup: zero the A ring, scatter-offset table, barriers, TMEM.
    // The in-tile pattern is the same for every step, so the (row, j) -> A
    // position map is computed once here and the per-step densify is a pure
    // table-driven scatter (reference index map: sdmm.py:183-186).  Zeros
    // written now are never overwritten: every step fills the same positions.
    {
        uint4 z = make_uint4(0, 0, 0, 0);
        uint4 *a4 = reinterpret_cast<uint4 *>(a_buf);
        for (int i = threadIdx.x; i < p.na * p.a_stage_bytes / 16; i += kThreads) a4[i] = z;
        const int32_t *adj = adj_i;
        if (p.adj_smem && threadIdx.x < kBlockM && p.prep == nullptr) {
            // one coalesced copy instead of d_t dependent global loads per row; only the
            // four table-building warps synchronise on it (named barrier 1)
            for (int i = threadIdx.x; i < p.u_i * p.d_i; i += kBlockM) adj_s[i] = adj_i[i];
            asm volatile("bar.sync 1, 128;" ::: "memory");
            adj = adj_s;
        }
        if (threadIdx.x < kBlockM && p.prep == nullptr)
            row_offsets<kElt>(p, adj, row_in_tile0, threadIdx.x, aoff + threadIdx.x, kBlockM);
        else if (p.prep != nullptr) {
            // prepared map: one coalesced 16-byte copy into the shared table
            const uint4 *src = reinterpret_cast<const uint4 *>(
                p.prep + size_t(row_in_tile0 / p.rows_valid) * p.d_t * kBlockM);
            uint4 *dst = reinterpret_cast<uint4 *>(aoff);
            for (int i = threadIdx.x; i < p.d_t * kBlockM / 8; i += kThreads) dst[i] = __ldg(src + i);
        }
    }
    if (threadIdx.x == 0) trace(p.debug, 6, 4);
    if (warp == 4 && lane == 0) {
        for (int i = 0; i < p.nb; ++i) { mbar_init(&full_b[i], 1 + 4); mbar_init(&empty_b[i], 1); }
        for (int i = 0; i < p.nw; ++i) { mbar_init(&full_w[i], 1); mbar_init(&empty_w[i], 4); }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&imap)) : "memory");
        if (p.w_tma)
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;
    const int32_t *orow = adj_o + tbm * p.d_o + s_begin;
    if (threadIdx.x == 0) trace(p.debug, 6, 0);

    // Role loops run warp-uniformly (all 32 lanes wait on the barriers); one lane,
    // picked by elect.sync, issues the TMA / tcgen05 instructions.  Issuing from
    // lane-0-only divergent code made the compiler wrap every UTCHMMA/UTMALDG in an
    // elect loop with R2UR conversions (~500 cycles per step, tools/tc_trace.py).
    if (warp == 4) {
        // ================= TMA producer: I slabs (runs ahead by the B ring depth) ==========
        const int atoms = p.tn * kElt / 128;           // 128-byte MN atoms per slab
        const int atom_cols = 128 / kElt;
        const uint32_t atom_bytes = uint32_t(p.tk) * 128;
        for (int s = 0; s < nsteps; ++s) {
            const int st = s % p.nb;
            const uint32_t ph = (s / p.nb) & 1;
            mbar_wait(&empty_b[st], ph ^ 1);
            const int32_t krow = orow[s] * p.tk;
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
                                    tj - p.pad, h0 + ti - p.pad, b0);
                } else if (p.i3d) {
                    // one instruction for the whole slab: (atom cols, K rows, atoms) box
                    tma_load_3d(dst, &imap, &full_b[st], 0, krow, int32_t(n0) / atom_cols);
                } else {
                    for (int a = 0; a < atoms; ++a)
                        tma_load_2d(dst + a * atom_bytes, &imap, &full_b[st],
                                    int32_t(n0) + a * atom_cols, krow);
                }
                trace(p.debug, 0, s);
            }
            __syncwarp();
        }
    } else if (warp == 6) {
        // ================= TMA producer: compressed W tiles (own ring, own pace) ============
        if (p.w_tma) {
            const int wstages = (nsteps + p.ws - 1) / p.ws;
            for (int g = 0; g < wstages; ++g) {
                const int st = g % p.nw;
                const uint32_t ph = (g / p.nw) & 1;
                mbar_wait(&empty_w[st], ph ^ 1);
                if (elect_one()) {
                    mbar_expect_tx(&full_w[st], uint32_t(p.w_stage_bytes));
                    tma_load_2d(w_buf + st * p.w_stage_bytes, &wmap, &full_w[st],
                                (s_begin + g * p.ws) * p.d_t, int32_t(m0));
                    trace(p.debug, 1, g);
                }
                __syncwarp();
            }
        }
    } else if (warp == 5) {
        // ================= MMA issuer =================
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
        unsigned long long seg[3] = {0, 0, 0};
        for (int s = 0; s < nsteps; ++s) {
            const int sb = s % p.nb, sa = s % p.na;
            const unsigned long long c0 = clock64();
            mbar_wait(&full_b[sb], (s / p.nb) & 1);  // I slab landed and A tile densified
            if (lane == 0) trace(p.debug, 7, s);
            tc_fence_after();
            const unsigned long long c1 = clock64();
            if (elect_one()) {
                trace(p.debug, 4, s);
                uint64_t ad = a_desc0 + uint64_t(sa) * a_stage16;
                uint64_t bd = b_desc0 + uint64_t(sb) * b_stage16;
                uint32_t in_atom = 0;
                if (p.a_tmem) {
                    // A tile of this stage sits in TMEM columns [tn + sa*a_tcols, +a_tcols)
                    uint32_t at = tmem_d + uint32_t(p.tn + sa * p.a_tcols);
                    for (int kk = 0; kk < ksteps; ++kk) {
                        if (!(p.debug & 2))
                            tc_mma_ts<kTF32>(tmem_d, at, bd, idesc, (s > 0 || kk > 0) ? 1u : 0u);
                        at += 8;  // 32 bytes of K = 8 TMEM columns
                        bd += b_step16;
                    }
                } else {
                    for (int kk = 0; kk < ksteps; ++kk) {
                        if (!(p.debug & 2)) tc_mma<kTF32>(tmem_d, ad, bd, idesc, (s > 0 || kk > 0) ? 1u : 0u);
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
                }
                tc_commit(&empty_b[sb]);  // frees both the I slab and the A tile of the stage
                trace(p.debug, 5, s);
            }
            __syncwarp();
            const unsigned long long c2 = clock64();
            seg[0] += c1 - c0;
            seg[1] += c2 - c1;
        }
        if (elect_one()) tc_commit(tmem_full);
        __syncwarp();
        if ((p.debug & (8 | 4096)) && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0) {
            g_trace[9][0] = seg[0];
            g_trace[9][1] = seg[1];
        }
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
        const uint32_t wrow = smem_u32(w_buf) + uint32_t(t * p.ws * p.d_t * kElt);
        // TMEM path: per 16-byte K position P of the dense row, code = 8 | chunk index when the
        // row has a nonzero chunk there (positions ascend with the chunks), else 0; 4 bits each
        uint32_t pcode[4] = {0, 0, 0, 0};
        const int npos = p.tk * kElt / 16;
        if (p.a_tmem && active) {
            const int ui = ((row_in_tile0 + t) / p.bm) % p.u_i;
            for (int c = 0; c < p.d_t / V; ++c) {
                const int j = c * V;
                const int k = j % p.bk, q = j / p.bk, ink = q % p.d_i, rk = q / p.d_i;
                const int kcol = (rk * p.v_i + adj_i[ui * p.d_i + ink]) * p.bk + k;
                const int P = kcol * kElt / 16;
                pcode[P / 8] |= uint32_t(8 | c) << (4 * (P % 8));
            }
        }
        for (int s = 0; s < nsteps; ++s) {
            const int sa = s % p.na;
            const int wg = s / p.ws, wsub = s - wg * p.ws;  // W stage and slot inside it
            if (p.w_tma && wsub == 0) {
                mbar_wait(&full_w[wg % p.nw], (wg / p.nw) & 1);
                if (t == 0) trace(p.debug, 8, wg);
            }
            mbar_wait(&empty_a[sa], ((s / p.na) & 1) ^ 1);
            if (t == 0) trace(p.debug, 2, s);
            const uint32_t a = smem_u32(a_buf + sa * p.a_stage_bytes);
            if (p.a_tmem) {
                // assemble the dense row t of A in TMEM lane t: 32 columns (8 positions) per st
                const uint32_t src = wrow + uint32_t((wg % p.nw) * p.w_stage_bytes) +
                                     uint32_t(wsub * p.d_t * kElt);
                uint4 q0 = make_uint4(0, 0, 0, 0), q1 = q0, q2 = q0, q3 = q0;
                const int nch = p.d_t / V;
                if (active && !(p.debug & 1)) {
                    q0 = lds128(src);
                    if (nch > 1) q1 = lds128(src + 16);
                    if (nch > 2) q2 = lds128(src + 32);
                    if (nch > 3) q3 = lds128(src + 48);
                }
                const uint32_t at = tmem_d + (uint32_t(warp * 32) << 16) + uint32_t(p.tn + sa * p.a_tcols);
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    if (g >= npos / 8) break;
                    const uint32_t code = pcode[g];
                    uint32_t r[32];
#pragma unroll
                    for (int pp = 0; pp < 8; ++pp) {
                        const uint32_t bits = (code >> (4 * pp)) & 0xFu;
                        uint4 v = sel4(q0, q1, q2, q3, bits & 3u);
                        if (!(bits & 8u)) v = make_uint4(0, 0, 0, 0);
                        r[4 * pp] = v.x; r[4 * pp + 1] = v.y; r[4 * pp + 2] = v.z; r[4 * pp + 3] = v.w;
                    }
                    TMEM_ST_32x32b_X32(at + uint32_t(g * 32), r);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
            } else if (active && !(p.debug & 1)) {
                if (chunked) {
                    const uint32_t src = wrow + uint32_t((wg % p.nw) * p.w_stage_bytes) +
                                         uint32_t(wsub * p.d_t * kElt);
                    const int nchunks = p.d_t / V;
                    uint4 q[kMaxChunks];
#pragma unroll
                    for (int c = 0; c < kMaxChunks; ++c)
                        if (c < nchunks) q[c] = lds128(src + 16 * c);
#pragma unroll
                    for (int c = 0; c < kMaxChunks; ++c) {
                        if (c < nchunks) {
                            const uint32_t o = (offp[c / 2] >> (16 * (c & 1))) & 0xFFFFu;
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + o),
                                         "r"(q[c].x), "r"(q[c].y), "r"(q[c].z), "r"(q[c].w)
                                         : "memory");
                        }
                    }
                } else if (reg_path) {
                    // compressed row t of this step (TMA-staged): 16-byte shared loads,
                    // all issued before the scatter so their latency overlaps
                    const uint32_t src = wrow + uint32_t((wg % p.nw) * p.w_stage_bytes) +
                                         uint32_t(wsub * p.d_t * kElt);
                    uint4 q[kRegNnz / V];
#pragma unroll
                    for (int c = 0; c < kRegNnz / V; ++c)
                        if (c * V < p.d_t) q[c] = lds128(src + 16 * c);
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
                    const uint32_t src = wrow + uint32_t((wg % p.nw) * p.w_stage_bytes) +
                                         uint32_t(wsub * p.d_t * kElt);
                    for (int j = 0; j < p.d_t; j += V) {
                        uint4 q = lds128(src + j * kElt);
                        const E *qe = reinterpret_cast<const E *>(&q);
#pragma unroll
                        for (int v = 0; v < V; ++v) sts_elem<E>(a + aoff[(j + v) * kBlockM + t], qe[v]);
                    }
                } else {
                    const E *vs = vrow + int64_t(s_begin + s) * p.d_t;
                    for (int j = 0; j < p.d_t; ++j) sts_elem<E>(a + aoff[j * kBlockM + t], vs[j]);
                }
            }
            // make the generic-proxy stores visible to the tensor core, then one
            // release-arrive per warp (full_a counts 4 warps)
            if (!(p.debug & 256)) fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&full_a[sa]);
                if (p.w_tma && (wsub == p.ws - 1 || s == nsteps - 1)) mbar_arrive(&empty_w[wg % p.nw]);
            }
            if (t == 0) trace(p.debug, 3, s);
        }
        // ---- epilogue phase 1: wait for the accumulator; split-K slices > 0 park
        // their fp32 partial tile in the workspace (L2-resident) for the leader
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        if (threadIdx.x == 0) trace(p.debug, 6, 1);
        if (kslice > 0) {
            const int row = warp * 32 + lane;
            const uint32_t lane_base = tmem_d + (uint32_t(warp * 32) << 16);
            float *dst = wsp + (int64_t(kslice - 1) * (int64_t(gridDim.y) * p.rows_valid) + m0 + row) *
                                   p.n_cols;
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
        // ---- epilogue phase 2 (leader): TMEM + partials (fixed slice order) -> output
        const int row = warp * 32 + lane;
        const bool row_ok = row < p.rows_valid;
        const uint32_t lane_base = tmem_d + (uint32_t(warp * 32) << 16);
        const int64_t slice_stride = int64_t(gridDim.y) * p.rows_valid * p.n_cols;
        for (int c = 0; c < p.tn; c += 32) {
            uint32_t r[32];
            TMEM_LD_32x32b_X32(lane_base + uint32_t(c), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int64_t col = n0 + c;
            if (!row_ok || col >= p.n_cols || (p.debug & 4)) continue;
            const bool full = col + 32 <= p.n_cols;
            if (p.ksplit > 1) {
                const float *part = wsp + (m0 + row) * p.n_cols + col;
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
                // NHWC output: pixel (col + q) is a row of c_out = p.ld_out channels
                const int64_t ch = m0 + row;
#pragma unroll 4
                for (int q = 0; q < 32; ++q) {
                    if (col + q >= p.n_cols) break;
                    float v = __uint_as_float(r[q]);
                    if (p.relu) v = fmaxf(v, 0.0f);
                    if constexpr (OUT_BF16)
                        static_cast<__nv_bfloat16 *>(out)[(col + q) * p.ld_out + ch] = __float2bfloat16_rn(v);
                    else
                        static_cast<float *>(out)[(col + q) * p.ld_out + ch] = v;
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
    }
    if (threadIdx.x == 0) trace(p.debug, 6, 2);
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                     "r"(uint32_t(p.tmem_cols)));
    }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
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
    p.tm = c.tm; p.tk = c.tk; p.d_o = c.d_o; p.d_t = c.d_t; p.u_i = c.u_i; p.v_i = c.v_i;
    p.d_i = c.d_i; p.rk = c.rk; p.bm = c.bm; p.bk = c.bk;
    p.rows_valid = c.tm == 64 ? 64 : kBlockM;
    const int kbytes = c.tk * elt;
    p.a_swz = kbytes % 128 == 0 ? 128 : kbytes % 64 == 0 ? 64 : 32;
    p.a_stage_bytes = kBlockM * kbytes;
    // compressed W tiles come in by TMA when a row of one step is whole 16-byte chunks
    p.w_tma = (c.d_t * elt) % 16 == 0 && c.d_t <= 256 ? 1 : 0;
    // W stage: as many consecutive steps as fit one box (<= 256 elements, <= 8 KB)
    p.ws = 1;
    while (p.w_tma && p.ws * 2 <= c.d_o && p.ws * 2 * c.d_t <= 256 &&
           size_t(p.rows_valid) * p.ws * 2 * c.d_t * elt <= 8192)
        p.ws *= 2;
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
    if (const char *env = getenv("RBGP4_TC_TN")) tn = std::max(tn_min, std::min(256, atoi(env)));
    if (force_tn) tn = force_tn;
    p.adj_smem = size_t(c.u_i) * c.d_i * 4 <= 16384 ? 1 : 0;
    // Shared-memory budget, in priority order (one CTA per SM):
    //   1. >= 96 KB of I slabs in flight (TMA latency under load is ~2 us: Little's law),
    //   2. A ring 2..4 deep (densify runs ahead of the MMA),
    //   3. W ring 2 x <= 8 KB,
    //   4. everything left -> more I stages (<= 16).
    for (; tn >= tn_min; tn /= 2) {
        if (force_tn && tn != force_tn) break;
        p.tn = tn;
        p.b_stage_bytes = c.tk * tn * elt;
        p.nw = p.w_tma ? 2 : 1;
        const size_t base = 1024 + size_t(kBlockM) * c.d_t * 2 + 64 +
                            (p.adj_smem ? size_t(c.u_i) * c.d_i * 4 + 16 : 0) + 8 * (2 * 16 + 2 * 2 + 1);
        size_t w_bytes = size_t(p.nw) * p.w_stage_bytes;
        if (getenv("RBGP4_TC_NOA")) p.a_stage_bytes = 0;  // ablation (debug 7 only): no A ring
        // A in TMEM (opt-in, RBGP4_TC_TMEM_A=1): needs 16-byte K runs (bk % V == 0), <= 4 of
        // them per row and <= 32 K positions; shared memory then holds only the I and W rings.
        // Correct, but the register-select row assembly costs ~350 instructions per row per
        // step and measured slower than the shared-memory A ring (34.8 vs 28.8 us, conv10).
        {
            const int V = 16 / elt;
            p.a_tcols = c.tk * elt / 4;
            const bool ok = p.w_tma && c.bk % V == 0 && c.d_t / V <= 4 && c.tk * elt / 16 <= 32 &&
                            tn + 2 * p.a_tcols <= 512 && getenv("RBGP4_TC_TMEM_A") != nullptr;
            p.a_tmem = ok ? 1 : 0;
            if (p.a_tmem) p.a_stage_bytes = 0;
            else p.a_stage_bytes = kBlockM * c.tk * elt;
        }
        const size_t stage = size_t(p.a_stage_bytes) + p.b_stage_bytes;  // A tile + I slab
        if (base + w_bytes + 2 * stage > kSmemCap && p.w_tma) {
            // large compressed tiles: read W straight from global in the densify warps
            p.w_tma = 0;
            p.ws = 1;
            p.nw = 1;
            p.w_stage_bytes = 0;
            p.table_in_regs = 0;
            w_bytes = 0;
        }
        if (base + w_bytes + 2 * stage > kSmemCap) continue;
        const size_t fixed = base + w_bytes;
        int ns = int(std::min<size_t>(16, (kSmemCap - fixed) / stage));
        if (p.a_tmem) ns = std::min(ns, (512 - tn) / p.a_tcols);  // A stages share TMEM with D
        p.na = ns;
        p.nb = ns;
        p.tmem_cols = 32;
        while (p.tmem_cols < (p.a_tmem ? tn + ns * p.a_tcols : tn)) p.tmem_cols *= 2;
        const int64_t tiles = ((c.n_cols + tn - 1) / tn) * blocks_m;
        // split-K in two (a 2-CTA cluster per tile) only when that still fits one wave;
        // deeper splits measured slower (tools/tc_time.py)
        int ks = (tiles * 2 <= kNumSMs && c.d_o >= 2) ? 2 : 1;
        if (const char *env = getenv("RBGP4_TC_KSPLIT")) ks = std::max(1, std::min(8, atoi(env)));
        p.sps = (c.d_o + ks - 1) / ks;
        p.ksplit = (c.d_o + p.sps - 1) / p.sps;  // no empty slices
        out->p = p;
        out->smem = fixed + size_t(ns) * stage;
        out->blocks_m = int(blocks_m);
        return 1;
    }
    set_error("tensor-core path: tile %dx%d does not fit shared memory", c.tm, c.tk);
    return 0;
}

template <typename E, bool OUT_BF16, bool CONV = false>
int launch_typed(const TcPlan &pl, const CUtensorMap &map, const CUtensorMap &wmap,
                 const void *values, const int32_t *adj_o, const int32_t *adj_i, void *out,
                 float *wsp, cudaStream_t stream) {
    auto kern = tc_kernel<E, OUT_BF16, CONV>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(tc): %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    dim3 grid(unsigned((pl.p.n_cols + pl.p.tn - 1) / pl.p.tn), unsigned(pl.blocks_m),
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
    cfg.attrs = attr;
    cfg.numAttrs = pl.p.ksplit > 1 ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kern, map, wmap, pl.p, static_cast<const E *>(values), adj_o, adj_i,
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

size_t tc_prep_size(const ChainDims &c, int compute) {
    TcPlan pl;
    if (!plan_tc(c, compute, &pl)) return 0;
    const int phases = c.tm / pl.p.rows_valid;
    return size_t(phases) * c.d_t * kBlockM * sizeof(uint16_t);
}

int tc_prepare(const ChainDims &c, int compute, const int32_t *adj_i, void *prep, size_t bytes,
               cudaStream_t stream) {
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
    TcPlan pl;
    if (!plan_tc(c, compute, &pl) || pl.p.ksplit <= 1) return 0;
    // (ksplit - 1) fp32 partial copies of the output, row-major (rows, n_cols)
    return size_t(pl.p.ksplit - 1) * size_t(pl.blocks_m) * pl.p.rows_valid * size_t(c.n_cols) * 4;
}

int launch_tc(const ChainDims &c, int compute, int out_dtype, const void *values,
              const int32_t *adj_o, const int32_t *adj_i, const void *prep, const void *inp,
              void *out, void *workspace, size_t workspace_bytes, cudaStream_t stream) {
    if (c.n_cols == 0) return RBGP4_OK;
    TcPlan pl;
    if (!plan_tc(c, compute, &pl)) return RBGP4_EUNSUPPORTED;
    pl.p.prep = static_cast<const uint16_t *>(prep);
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
    if (getenv("RBGP4_TC_2D")) pl.p.i3d = 0;
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (const char *e = getenv("RBGP4_TC_PROMO"))
        promo = atoi(e) == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
              : atoi(e) == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : atoi(e) == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
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
    if (const char *dbg = getenv("RBGP4_TC_DEBUG")) {
        pl.p.debug = atoi(dbg);
        if (pl.p.debug & 8192)
            fprintf(stderr, "[rbgp4 tc plan] tn=%d na=%d nb=%d nw=%d ws=%d w_tma=%d ks=%d smem=%zu a_tmem=%d tmem=%d\n",
                    pl.p.tn, pl.p.na, pl.p.nb, pl.p.nw, pl.p.ws, pl.p.w_tma, pl.p.ksplit, pl.smem,
                    pl.p.a_tmem, pl.p.tmem_cols);
        if (pl.p.debug & 16) { pl.p.w_tma = 0; pl.p.nw = 1; pl.p.ws = 1; pl.p.w_stage_bytes = 0; }
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
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
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
        return obf ? launch_typed<float, true>(pl, map, wmap, values, adj_o, adj_i, out, wsp, stream)
                   : launch_typed<float, false>(pl, map, wmap, values, adj_o, adj_i, out, wsp, stream);
    return obf ? launch_typed<__nv_bfloat16, true>(pl, map, wmap, values, adj_o, adj_i, out, wsp, stream)
               : launch_typed<__nv_bfloat16, false>(pl, map, wmap, values, adj_o, adj_i, out, wsp, stream);
}

// ---------------------------------------------------------------- K3: implicit im2col
namespace {
int conv_tile(const rbgp4_conv_desc &cv, int tn, int *th, int *tb) {
    const int hw = cv.height * cv.width;
    if (tn % cv.width) return 0;
    if (tn <= hw) {
        *th = tn / cv.width;
        *tb = 1;
        return cv.height % *th == 0;
    }
    *th = cv.height;
    *tb = tn / hw;
    return tn % hw == 0 && *tb <= 256;
}
}  // namespace

int conv_plan(const ChainDims &c, const rbgp4_conv_desc *cv, TcPlan *pl) {
    RBGP4_REQUIRE(cv != nullptr, "null conv descriptor");
    RBGP4_REQUIRE(cv->stride == 1 && cv->pad * 2 == cv->kh - 1 && cv->kh == cv->kw,
                  "implicit-im2col path supports stride-1 'same' square convolutions (kh=%d, pad=%d, "
                  "stride=%d)", cv->kh, cv->pad, cv->stride);
    RBGP4_REQUIRE(c.cols == int64_t(cv->kh) * cv->kw * cv->c_in,
                  "chain columns %lld != kh*kw*c_in = %d (tap-major im2col order)", (long long)c.cols,
                  cv->kh * cv->kw * cv->c_in);
    RBGP4_REQUIRE(c.n_cols == int64_t(cv->batch) * cv->height * cv->width,
                  "n_cols %lld != batch*height*width", (long long)c.n_cols);
    RBGP4_REQUIRE(c.tk % 64 == 0 && cv->c_in % c.tk == 0,
                  "conv path needs tk %% 64 == 0 and c_in %% tk == 0 (tk=%d, c_in=%d)", c.tk, cv->c_in);
    RBGP4_REQUIRE(cv->width <= 256 && cv->height <= 256, "feature map too large for one TMA box");
    for (int tn : {128, 64}) {
        int th, tb;
        if (!conv_tile(*cv, tn, &th, &tb)) continue;
        if (!plan_tc(c, RBGP4_COMPUTE_BF16, pl, tn)) continue;
        pl->p.conv = 1;
        pl->p.c_in = cv->c_in;
        pl->p.img_h = cv->height;
        pl->p.img_w = cv->width;
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
    TcPlan pl;
    if (!conv_plan(c, cv, &pl) || pl.p.ksplit <= 1) return 0;
    return size_t(pl.p.ksplit - 1) * size_t(pl.blocks_m) * pl.p.rows_valid * size_t(c.n_cols) * 4;
}

int launch_conv(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, const void *values,
                const int32_t *adj_o, const int32_t *adj_i, const void *prep, const void *x,
                void *out, void *workspace, size_t workspace_bytes, cudaStream_t stream) {
    TcPlan pl;
    if (!conv_plan(c, cv, &pl)) return RBGP4_EUNSUPPORTED;
    if (c.n_cols == 0) return RBGP4_OK;
    pl.p.prep = static_cast<const uint16_t *>(prep);
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
    cuuint32_t box[4] = {64, cuuint32_t(cv->width), cuuint32_t(pl.p.th), cuuint32_t(pl.p.tb)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(x), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled(conv input) failed (%d)", int(r));
        return RBGP4_ECUDA;
    }
    memset(&wmap, 0, sizeof(wmap));
    if (pl.p.w_tma) {
        cuuint64_t wdims[2] = {cuuint64_t(c.row_nnz), cuuint64_t(c.rows)};
        cuuint64_t wstrides[1] = {cuuint64_t(c.row_nnz) * 2};
        cuuint32_t wbox[2] = {cuuint32_t(pl.p.ws * c.d_t), cuuint32_t(pl.p.rows_valid)};
        r = enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(values), wdims,
                wstrides, wbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
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
               ? launch_typed<__nv_bfloat16, true, true>(pl, map, wmap, values, adj_o, adj_i, out, wsp, stream)
               : launch_typed<__nv_bfloat16, false, true>(pl, map, wmap, values, adj_o, adj_i, out, wsp, stream);
}

}  // namespace rbgp4

// debug-only (not part of include/rbgp4.h): copy the CTA-0 trace to the host
extern "C" int rbgp4_debug_trace(unsigned long long *host, int n) {
    if (n > 10 * rbgp4::kTraceSteps) n = 10 * rbgp4::kTraceSteps;
    return cudaMemcpyFromSymbol(host, rbgp4::g_trace, sizeof(unsigned long long) * n) == cudaSuccess
               ? 0 : -3;
}
