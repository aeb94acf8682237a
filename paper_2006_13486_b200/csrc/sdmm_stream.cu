// sdmm_stream.cu -- K5: the RBGP4 SDMM and its implicit-im2col convolution streamed through
// tcgen05, the default compute="bf16" path.
//
// Replaces kronsparse.sdmm._tile_worker (reference sdmm.py:148-205).  Transposed product per
// output tile (tile-row tbm, 128 batch columns / pixels n0..):
//     D^T (128 x rows) += I^T (128 x 16) * W^T (16 x rows)   per K16 slice of a step,
// M = 128 batch columns (the I slab exactly as TMA lands it: MN-major for the SDMM, the K-major
// NHWC pixel x channel box for the conv), the gather being the A descriptor's start address,
// D in TMEM.  Which W rows a slice multiplies is a per-matrix relayout prepared once:
//
// * TC16 (g_r (1,1), g_i (8,8) of degree 2, g_b (16,16): SURVEY §8(d), the bench headline):
//   K4's column-block relayout -- 8 MMAs of N = 32 per step (two row blocks of 16 per column
//   block); for small N, ROW GROUPS -- a unit owns G row blocks of a tile and loads only the
//   16-row pieces of each slab those row blocks read (no split-K exchange).
// * Slices (any g_b that tiles K16: 8 x 8 / 4 x 4 blocks, g_i degree <= 4): slice kb of a step
//   times the union of the rows reading it, zero-padded to N = 32 / 64; each row sums <= 4
//   TMEM partials in the epilogue.
// * Merged tile-row pairs (g_o complete): one unit = two tile-rows, unions twice as wide, the I
//   slab loaded once for both; single-buffered 512-column accumulator.
// * Conv: tap-shifted 4-D NHWC boxes per step, or HALO strips (3x3, stride 1, one channel
//   block): a 16 x 8 output strip stages its 18 x 10 halo once and the nine taps are
//   descriptor row offsets; ReLU and the following 2x2 max pool fused into the epilogue.
//
// Measured design rules (tools/stream_bench.cu, tma_par_bench.cu, umma_bench3.cu, epi_bench.cu;
// DESIGN.md "What bounds the kernels"): a TMA box costs its issuing THREAD ~450 cycles whatever
// its size, so up to six I producer warps take the steps round-robin; an M128 K16 MMA costs ~82
// cycles up to N = 64, so a step is as few, as wide MMAs as the pattern allows; the W producer
// requests the first ring's W before griddepcontrol.wait (weights never depend on the previous
// grid); epilogue warps pack column pairs with one shuffle and store directly under the next
// unit's main loop, the CTA's last unit staged in the idle ring and TMA-stored.
//
// Warps (384 threads): 0-3 epilogue (TMEM lane = batch column), 4 and 7-11 I producers, 6 W
// producer, 5 TMEM allocation + MMA issue (heavy epilogues: warps 8-11 a second epilogue group).
// Deterministic: every unit owns its output rows; fixed step and partial-sum order.
#include "common.cuh"
#include "tc_ptx.cuh"

#include <algorithm>
#include <cstring>
#include <functional>
#include <type_traits>
#include <vector>

namespace rbgp4 {
namespace {

constexpr int kSBatch = 128;                  // MMA M: batch columns per unit
// 12 warps: 0-3 epilogue, 4 and 7-11 I producers (steps round-robin: a TMA box costs its
// issuing thread ~450 cycles, tools/tma_par_bench.cu), 5 MMA, 6 W producer
constexpr int kSThreads = 384;
constexpr int kHaloAtom = (180 * 128 + 1023) & ~1023;  // halo conv: 18 x 10 pixels x 128 B, 1024-aligned
constexpr int kIProd = 6;
constexpr int kProdThreads = 32 * (kIProd + 1);  // the producer warps 4, 6, 7..11 (barrier 3)
constexpr int kMaxDo = 64;                    // steps per tile-row held in producer registers
constexpr int kRgWords = 48;                  // one row-group record (int32 words)
constexpr int kMaxRg = 8;                     // row groups per tile (G = 1)
constexpr int kPieceBytes = 16 * kSBatch * 2; // one slab piece: 16 rows x 128 batch columns, bf16
// record: [0] first g_i column block `lo` of the group's range, [1] range length L (the
// group's row blocks read column blocks lo .. lo+L-1 only), [17 + r * d_i + ink] piece (column
// block - lo) read by MMA (r, ink), [33 + r] output row block of the group's r-th row block
constexpr int kRgLo = 0, kRgLen = 1, kRgMma = 17, kRgRows = 33;

// row groups: one I tensor map per range length L = 1..8 (box = 16 L slab rows x 128 columns)
struct IMaps {
    CUtensorMap m[8];
};

#if RBGP4_DEBUG
// debug builds (option debug bit 512): per-CTA %globaltimer at entry / exit, CTA-0 marks and
// per-step trace (clock64 from entry)
constexpr int kK5Stamps = 4096;
__device__ unsigned long long g_k5_stamp[2][kK5Stamps];
__device__ unsigned long long g_k5_mark[16];
// bit 2048: launch slots (host counter mod 16) -- every CTA's entry / exit %globaltimer and CTA 0's
// marks [first I issued, first full, last accumulator ready, last stores issued], for a whole
// graph of launches (tools/step_timeline.py)
__device__ unsigned long long g_k5_seq[16][3][160];  // [slot][entry | exit | first I issued][CTA]
__device__ unsigned long long g_k5_smark[16][4];
__device__ unsigned long long g_k5_trace[3][64];  // [0] I producer issued, [1] MMA saw full, [2] MMAs issued
__device__ unsigned long long g_k5_epi[16];       // CTA 0: units 0-3 [epilogue start, end (warp 0), MMA acc_empty wait start, end]
__device__ __forceinline__ unsigned long long k5_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define K5_SMARK(i) do { if (p.slot >= 0 && blockIdx.x == 0) g_k5_smark[p.slot][i] = k5_gtimer(); } while (0)
#else
#define K5_SMARK(i) do { } while (0)
#endif

struct SParams {
    int64_t n_cols, ld_out, n_units;
    int32_t u_o, d_o, tm, tk, u_i, d_i, d_t;
    int32_t ns, stage_bytes, i_bytes;  // ring stages; bytes per stage; I part of a stage
    int32_t wres_bytes, ring_bytes;    // row groups: resident W of a unit; ring size
    int32_t g, n_rg;                   // row-group mode: row blocks per unit, groups per tile
    int32_t acc_cols, tmem_cols;       // TMEM columns per accumulator buffer / allocated
    const int32_t *steps;              // [tbm][s] = adjacency slot j << 16 | K-block
    const int32_t *cols;               // whole tiles: TMEM column of row block ui's ink-th partial
    const int32_t *rg;                 // row groups: n_rg records of kRgWords
    // whole tiles (slice relayout): K16 slices per step, MMA N (rows of a slice's union, padded),
    // W rows per step (nsl * mma_n), entries of the cols table (row blocks x 2 partials)
    int32_t nsl, mma_n, w_rows, n_cols_tab, parts;  // parts: TMEM partials per row block (2 or 4)
    // implicit-im2col convolution (NHWC): input channels, OUTPUT map, kernel width, pad, stride
    int32_t c_in, img_h, img_w, kw, pad, stride, relu;
    // halo conv: stride of a staged 64-channel halo atom (bytes), strips per image (rows, columns)
    int32_t halo_atom, strips_y, strips_x, epi2;  // epi2: warps 8-11 are a second epilogue group
    int32_t nbuf;                      // TMEM accumulator buffers (2: epilogue overlapped; 1: 512 columns)
    int32_t debug, slot;
    // conv (bf16, no pool / residual): each epilogue warp stages 64 channels x its 32 pixels
    // (4 KB, 128B swizzle) at ostage_off + 4 KB * slot and writes them with one TMA store
    int32_t ostage, ostage_off;
    // conv residual epilogue (relu bits 2 / 3): O = round(acc) + res; relu(O) also into out2
    const void *res;
    void *out2;
};

__device__ __forceinline__ void tma_store_3d_g(const CUtensorMap *map, uint32_t src, int32_t x, int32_t y, int32_t z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(src) : "memory");
}
__device__ __forceinline__ void tma_store_2d_g(const CUtensorMap *map, uint32_t src, int32_t x, int32_t y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(src) : "memory");
}

// RG: row-group units (TC16 only); CONV: A = tap-shifted NHWC boxes (K-major), O = NHWC;
// HALO (conv, one channel block, 3x3 stride 1): a unit is a strip of 16 output rows x 8 output
// columns of one image; its 18 x 10 halo is staged ONCE (one 4-D box per 64-channel atom) and
// the nine taps are A-descriptor row offsets into it (SBO = 10 halo pixels), the unit's W (all
// taps) stays resident -- the taps no longer re-read the input from L2 (9x -> 1.4x);
// BM: element-block rows of the chain (16 / 8 / 4) -- the granularity of the epilogue's
// TMEM partial loads
template <bool OUT_BF16, bool RG, bool CONV, int BM, bool HALO = false, bool RES = false>
__global__ void __launch_bounds__(kSThreads, 1)
stream_kernel(const __grid_constant__ CUtensorMap imap, const __grid_constant__ CUtensorMap wmap,
              const __grid_constant__ CUtensorMap omap, const __grid_constant__ IMaps imaps, const SParams p,
              void *__restrict__ out) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ int32_t s_rg[RG ? kMaxRg * kRgWords : 1];
    __shared__ int32_t s_cols[RG ? 1 : 128];
    __shared__ uint32_t s_tap[HALO ? 18 : 1];  // halo: per tap, A row offset / B tile offset (16-byte units)
    // 1024-byte aligned ring (swizzle atoms); pointer arithmetic on smem_raw keeps the shared
    // address space visible to the compiler (plain C++ stores to the staging area stay STS)
    unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    // [barriers, 1 KB][row groups: the unit's resident W][ring]
    uint64_t *full = reinterpret_cast<uint64_t *>(base);
    uint64_t *empty = full + 16;
    uint64_t *acc_full = empty + 16;     // [2] last MMA of a unit committed
    uint64_t *acc_empty = acc_full + 2;  // [2] the epilogue has read the buffer
    uint64_t *wfull = acc_empty + 2;     // row groups: the unit's W landed
    uint64_t *wempty = wfull + 1;        // row groups: the unit's MMAs are done with W
    uint64_t *last_full = wempty + 1;    // the CTA's last unit accumulated (one phase: warps 4-7)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(last_full + 1);
    unsigned char *wres = base + 1024;   // row groups: d_o steps x G*16 rows x d_t slots
    unsigned char *ring = wres + p.wres_bytes;
    // ring geometry: whole tiles -- planned on the host; row groups -- a stage holds the
    // longest column-block range among the groups THIS CTA visits (units first, first + grid,
    // ...: the group index cycles with period n_rg), so a CTA whose units are all one group of
    // range L gets ring / (L pieces) stages (~11 for L = 4 instead of ~5 for the worst group).
    // Every warp derives the same values.
    int NS = p.ns, SB = p.stage_bytes;
    if constexpr (RG) {
        const int li = threadIdx.x % 32;
        const int64_t u_l = int64_t(blockIdx.x) + int64_t(li) * gridDim.x;
        int l = (li < p.n_rg && u_l < p.n_units) ? __ldg(p.rg + int(u_l % p.n_rg) * kRgWords + kRgLen) : 1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l = max(l, __shfl_xor_sync(0xffffffffu, l, o));
        SB = l * kPieceBytes;
        NS = min(16, p.ring_bytes / SB);
    }
    constexpr int kThreads = kSThreads;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t first = blockIdx.x, stride = gridDim.x;
    const int upt = RG ? p.n_rg : 1;  // units per tile
#if RBGP4_DEBUG
    const unsigned long long c_entry = clock64();
    const bool trace = (p.debug & 512) && blockIdx.x == 0;
    if ((p.debug & 512) && threadIdx.x == 0 && blockIdx.x < kK5Stamps) g_k5_stamp[0][blockIdx.x] = k5_gtimer();
    if (p.slot >= 0 && threadIdx.x == 0 && blockIdx.x < 160) g_k5_seq[p.slot][0][blockIdx.x] = k5_gtimer();
#define K5_MARK(i) do { if (trace) g_k5_mark[i] = clock64() - c_entry; } while (0)
#else
#define K5_MARK(i) do { } while (0)
#endif


    // ---- epilogue of one unit, row blocks [rb0, rb1), TMEM lane quarter = warp % 4 ----
    // (TMEM lane = batch column).  Run by warps 0-3 for every unit and, for the CTA's last unit,
    // split with warps 4-7.  `cols` / `rec`: the TMEM column table (whole tiles) / the unit's
    // row-group record, in shared or global memory.
    constexpr int kRowBytes = OUT_BF16 ? 64 : 128;  // staged row of one warp's 32 columns
    auto drain = [&](int64_t u, int64_t it, int rb0, int rb1, const int32_t *cols, const int32_t *rec,
                     bool helper) {
        const int q = warp & 3;
        const int b = p.nbuf == 2 ? int(it & 1) : 0;
        const uint32_t bph = uint32_t((p.nbuf == 2 ? (it >> 1) : it) & 1);  // use count of buffer b
        const int64_t tile = u / upt;
        const int tbm = int(tile % p.u_o);
        const int64_t n0 = (tile / p.u_o) * kSBatch;
        const int64_t m0 = int64_t(tbm) * p.tm;
        const bool last = u + stride >= p.n_units;
        const bool stage_last = last && !CONV;  // conv: direct NHWC stores for every unit
        const int64_t c0 = n0 + q * 32;     // this warp's first column
        const bool ok = HALO || c0 < p.n_cols;  // n_cols % 64 == 0: a warp's 32 columns are all in or out
        // conv: this lane's output pixel (NHWC row); halo strips: (r, c) = (m / 8, m % 8) of the
        // unit's 16 x 8 strip, m = TMEM lane
        int64_t pix = c0 + lane;
        int32_t st_x = int32_t(c0), st_y = 0;  // staged conv store: the warp's box coordinates
        // fused 2x2 max pool (conv flag bit 1): window partners are lanes ^1 (x) and ^ystr (y);
        // the (even x, even y) lane stores the pooled pixel `pix` of the (H/2, W/2) map
        const bool pool = CONV && (p.relu & 2);
        int ystr = 1;
        bool leader = true;
        if constexpr (HALO) {
            const int64_t per_img = int64_t(p.strips_y) * p.strips_x;
            const int64_t bimg = u / per_img;
            const int sy = int((u - bimg * per_img) / p.strips_x), sx = int(u % p.strips_x);
            const int m = q * 32 + lane;
            pix = (bimg * p.img_h + sy * 16 + (m >> 3)) * p.img_w + sx * 8 + (m & 7);
            st_x = sx * 8;  // the warp's 4 strip rows x 8 pixels
            st_y = int32_t(bimg * p.img_h + sy * 16 + q * 4);
            if (pool) {
                ystr = 8;
                leader = !(m & 1) && !(m & 8);
                pix = (bimg * (p.img_h / 2) + (sy * 16 + (m >> 3)) / 2) * (p.img_w / 2) + (sx * 8 + (m & 7)) / 2;
                st_x = sx * 4;  // pooled: the warp's 2 rows x 4 pixels
                st_y = int32_t((bimg * p.img_h + sy * 16 + q * 4) / 2);
            }
        } else if (pool) {
            const int64_t hw = int64_t(p.img_h) * p.img_w;
            const int64_t bimg = pix / hw;
            const int rem = int(pix - bimg * hw), y = rem / p.img_w, x = rem - y * p.img_w;
            ystr = p.img_w;
            leader = !(x & 1) && !(y & 1);
            pix = (bimg * (p.img_h / 2) + y / 2) * (p.img_w / 2) + x / 2;
            // maps up to 16 wide: a warp's leaders are 8 consecutive pooled pixels from lane 0's
            st_x = int32_t(__shfl_sync(0xffffffffu, pix, 0));
        }
        const int nrows = RG ? p.g * 16 : p.tm;
        // staged conv stores: whole 64-channel groups only (a range of 4k row blocks from 4k)
        // (pooled: the warp's 8 pooled pixels, 1 KB; the staging row of a leader lane is its pooled
        // pixel's index among them)
        const bool ost = CONV && !RES && OUT_BF16 && p.ostage && !helper && (rb0 % 4) == 0 &&
                         ((rb1 - rb0) % 4) == 0;
        const uint32_t ostg = smem_u32(base) + uint32_t(p.ostage_off) +
                              uint32_t(((warp & 3) + (warp >= 8 ? 4 : 0)) * (pool ? 1024 : 4096));
        const int orow = !pool ? lane : HALO ? ((lane >> 4) * 4 + ((lane & 7) >> 1)) : int(pix - st_x);
        unsigned char *wstage_p = ring + q * nrows * kRowBytes;  // [row][kRowBytes] for columns c0..
        const uint32_t wstage = smem_u32(wstage_p);
        const int k2 = lane >> 1, odd = lane & 1;  // bf16: lane pair (2k, 2k+1) -> columns 2k, 2k+1
        // warps 0-3 follow acc_full[b] unit by unit; the helpers (warps 4-7) may be many phases
        // behind it, so they wait on the single-phase last_full instead
        // residual epilogue: pull this lane's pixel row of R into L2 while the MMAs still run
        const bool resid = CONV && RES && ok;
        if (resid) {
            const char *ra = static_cast<const char *>(p.res) + (pix * p.ld_out + m0) * (OUT_BF16 ? 2 : 4);
            for (int o = 0; o < nrows * (OUT_BF16 ? 2 : 4); o += 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(ra + o));
        }
        if (helper) mbar_wait_parked(last_full, 0u);
        else mbar_wait_parked(&acc_full[b], bph);
        tc_fence_after();
        if (last && threadIdx.x == 0) { K5_MARK(3); K5_SMARK(2); }
#if RBGP4_DEBUG
        if (trace && threadIdx.x == 0 && !helper && it < 4) g_k5_epi[4 * it] = clock64() - c_entry;
#endif
        const uint32_t tmem_d = *tmem_slot;
        const uint32_t lane_base = tmem_d + (uint32_t(q * 32) << 16) + uint32_t(b * p.acc_cols);
        // 16 fp32 rows (row block rb, staging slot rs) of this lane's column -> bf16 pairs packed
        // across the lane pair / f32 as is; staged (last unit) or stored directly.  Kept compact
        // (a loop over row blocks, not unrolled): the epilogue runs cold in the instruction cache.
        // residual row block i (16 output channels of this lane's pixel) into registers, one row
        // block ahead of its use (the loads would otherwise serialise the row-block loop)
        auto rload = [&](int i, uint4 (&r)[4]) {
            if constexpr (CONV && RES) {
                if (resid) {
                    const uint4 *src = reinterpret_cast<const uint4 *>(
                        static_cast<const char *>(p.res) + (pix * p.ld_out + m0 + int64_t(i) * 16) * (OUT_BF16 ? 2 : 4));
#pragma unroll
                    for (int h = 0; h < (OUT_BF16 ? 2 : 4); ++h) r[h] = src[h];
                }
            }
        };
        auto put16 = [&](int rs, int rb, const uint32_t (&va)[16], const uint32_t (&vb)[16], bool two,
                         const uint4 (&rr)[4]) {
            const int64_t grow0 = m0 + int64_t(rb) * 16;
            if constexpr (CONV) {
                // NHWC: this lane's pixel c0 + lane holds output channels grow0 .. grow0 + 15
                // contiguously -> 32 (bf16) / 64 (f32) bytes of 16-byte stores, ReLU fused
                float x[16];
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    x[m] = __uint_as_float(va[m]) + (two ? __uint_as_float(vb[m]) : 0.0f);
                    if (p.relu & 1) x[m] = fmaxf(x[m], 0.0f);
                }
                if (pool) {
#pragma unroll
                    for (int m = 0; m < 16; ++m) {
                        x[m] = fmaxf(x[m], __shfl_xor_sync(0xffffffffu, x[m], 1));
                        x[m] = fmaxf(x[m], __shfl_xor_sync(0xffffffffu, x[m], ystr));
                    }
                    if (!leader && !ost) return;
                }
                if (!ok) return;
#if RBGP4_DEBUG
                if (p.debug & 4096) return;  // ablation: no conv output stores (tools/conv_store_ab.py)
#endif
                const int64_t off = pix * p.ld_out + grow0;
                if constexpr (RES) {
                    // residual (the WRN block tail): O = round(conv) + R, rounded once more on
                    // the store -- what the unfused conv then bf16 / f32 add computes
                    if constexpr (OUT_BF16) {
                        const uint32_t rw[8] = {rr[0].x, rr[0].y, rr[0].z, rr[0].w, rr[1].x, rr[1].y, rr[1].z, rr[1].w};
#pragma unroll
                        for (int h = 0; h < 8; ++h) {
                            const float2 rf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&rw[h]));
                            const float2 cf = __bfloat1622float2(__floats2bfloat162_rn(x[2 * h], x[2 * h + 1]));
                            x[2 * h] = cf.x + rf.x;
                            x[2 * h + 1] = cf.y + rf.y;
                        }
                    } else {
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const float4 v = make_float4(__uint_as_float(rr[h].x), __uint_as_float(rr[h].y),
                                                         __uint_as_float(rr[h].z), __uint_as_float(rr[h].w));
                            x[4 * h] += v.x; x[4 * h + 1] += v.y; x[4 * h + 2] += v.z; x[4 * h + 3] += v.w;
                        }
                    }
                }
                if constexpr (OUT_BF16) {
                    uint32_t w[8];
#pragma unroll
                    for (int h = 0; h < 8; ++h) {
                        const __nv_bfloat162 v2 = __floats2bfloat162_rn(x[2 * h], x[2 * h + 1]);
                        w[h] = *reinterpret_cast<const uint32_t *>(&v2);
                    }
                    if (ost) {
                        // row block rb = channels 16 (rb % 4) .. of the warp's 64-channel group:
                        // chunks 2 (rb % 4), +1 of this lane's 128-byte row, 128B swizzle
                        const int g4 = rb & 3;
                        if (g4 == 0) {  // the previous group's TMA store has read the staging
                            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                            __syncwarp();
                        }
                        if (leader) {
                            const uint32_t row = ostg + uint32_t(orow) * 128u;
                            sts128(row + ((uint32_t(2 * g4) ^ uint32_t(orow & 7)) << 4), w[0], w[1], w[2], w[3]);
                            sts128(row + ((uint32_t(2 * g4 + 1) ^ uint32_t(orow & 7)) << 4), w[4], w[5], w[6], w[7]);
                        }
                        if (g4 == 3) {
                            fence_async_smem();
                            __syncwarp();
                            if (lane == 0) {
                                const int32_t ch0 = int32_t(grow0 - 48);
                                if constexpr (HALO) tma_store_3d_g(&omap, ostg, ch0, st_x, st_y);
                                else tma_store_2d_g(&omap, ostg, ch0, st_x);
                                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                            }
                        }
                        return;
                    }
                    uint4 *g = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(out) + off);
                    g[0] = make_uint4(w[0], w[1], w[2], w[3]);
                    g[1] = make_uint4(w[4], w[5], w[6], w[7]);
                    if (RES && (p.relu & 8)) {  // relu(O): max(0, .) of the rounded pair, sign-exact
#pragma unroll
                        for (int h = 0; h < 8; ++h) {
                            const __nv_bfloat162 v2 = __hmax2(*reinterpret_cast<const __nv_bfloat162 *>(&w[h]),
                                                              __float2bfloat162_rn(0.0f));
                            w[h] = *reinterpret_cast<const uint32_t *>(&v2);
                        }
                        uint4 *g2 = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(p.out2) + off);
                        g2[0] = make_uint4(w[0], w[1], w[2], w[3]);
                        g2[1] = make_uint4(w[4], w[5], w[6], w[7]);
                    }
                } else {
                    float4 *g = reinterpret_cast<float4 *>(static_cast<float *>(out) + off);
#pragma unroll
                    for (int h = 0; h < 4; ++h) g[h] = make_float4(x[4 * h], x[4 * h + 1], x[4 * h + 2], x[4 * h + 3]);
                    if (RES && (p.relu & 8)) {
                        float4 *g2 = reinterpret_cast<float4 *>(static_cast<float *>(p.out2) + off);
#pragma unroll
                        for (int h = 0; h < 4; ++h)
                            g2[h] = make_float4(fmaxf(x[4 * h], 0.0f), fmaxf(x[4 * h + 1], 0.0f),
                                                fmaxf(x[4 * h + 2], 0.0f), fmaxf(x[4 * h + 3], 0.0f));
                    }
                }
            } else if constexpr (OUT_BF16) {
                // all 8 shuffles first, then the stores (plain C++ stores: a volatile asm store with
                // a memory clobber serialised every pair behind its shuffle, ~90 cycles each)
                uint32_t words[8];
#pragma unroll
                for (int h = 0; h < 8; ++h) {
                    const int m = 2 * h;
                    const float x0 = __uint_as_float(va[m]) + (two ? __uint_as_float(vb[m]) : 0.0f);
                    const float x1 = __uint_as_float(va[m + 1]) + (two ? __uint_as_float(vb[m + 1]) : 0.0f);
                    // even lane sends row m+1, odd lane row m; each gets its pair's other column
                    const float recv = __shfl_xor_sync(0xffffffffu, odd ? x0 : x1, 1);
                    const __nv_bfloat162 v2 = odd ? __floats2bfloat162_rn(recv, x1) : __floats2bfloat162_rn(x0, recv);
                    words[h] = *reinterpret_cast<const uint32_t *>(&v2);
                }
                if (stage_last) {
                    // [row][64 B], 64B swizzle: 16-byte chunk ^ (row / 2) % 4 (row = m + odd)
                    unsigned char *sb = wstage_p + rs * 16 * 64 + (k2 & 3) * 4 + odd * 64;
#pragma unroll
                    for (int h = 0; h < 8; ++h)
                        *reinterpret_cast<uint32_t *>(sb + h * 128 + ((((k2 >> 2) ^ (h & 3))) << 4)) = words[h];
                } else if (ok) {
                    uint32_t *gbase = reinterpret_cast<uint32_t *>(static_cast<__nv_bfloat16 *>(out) +
                                                                  (grow0 + odd) * p.ld_out + c0 + 2 * k2);
#pragma unroll
                    for (int h = 0; h < 8; ++h) gbase[int64_t(2 * h) * (p.ld_out / 2)] = words[h];
                }
            } else {
                float x[16];
#pragma unroll
                for (int m = 0; m < 16; ++m) x[m] = __uint_as_float(va[m]) + (two ? __uint_as_float(vb[m]) : 0.0f);
                if (stage_last) {
                    // [row][128 B], 128B swizzle: chunk ^ row % 8
                    unsigned char *sb = wstage_p + rs * 16 * 128 + (lane & 3) * 4;
#pragma unroll
                    for (int m = 0; m < 16; ++m)
                        *reinterpret_cast<float *>(sb + m * 128 + ((((lane >> 2) ^ (m & 7))) << 4)) = x[m];
                } else if (ok) {
                    float *gbase = static_cast<float *>(out) + grow0 * p.ld_out + c0 + lane;
#pragma unroll
                    for (int m = 0; m < 16; ++m) gbase[int64_t(m) * p.ld_out] = x[m];
                }
            }
        };
        // rows 16 i .. 16 i + 15: row groups -> TMEM columns 16 i (one partial); whole tiles ->
        // per element-row block rb of BM rows inside them, its (up to) two partials at TMEM
        // columns cols[2 rb], cols[2 rb + 1] of the slice relayout (-1: no such partial)
        // rows 16 i .. 16 i + 15 of partial pair pp (p.parts = 2: pp = 0; 4: pp = 0, 1).  The first
        // partial of a row block always exists; only the others may be -1.  (The two-partial
        // path keeps the unconditional first load: guarding it doubled the halo conv epilogue.)
        const int nparts = RG ? 1 : p.parts;
        auto tload = [&](int i, uint32_t (&va)[16], uint32_t (&vb)[16], int pp) {
            if constexpr (RG) {
                TMEM_LD_32x32b_X16(lane_base + uint32_t(i * 16), va);
            } else {
#pragma unroll
                for (int j = 0; j < 16 / BM; ++j) {
                    const int rb = i * (16 / BM) + j;
                    const int ca = cols[rb * nparts + 2 * pp], cb = cols[rb * nparts + 2 * pp + 1];
                    uint32_t *pa = va + j * BM, *pb = vb + j * BM;
                    if (pp == 0) {
                        if constexpr (BM == 16) TMEM_LD_32x32b_X16(lane_base + uint32_t(ca), va);
                        else if constexpr (BM == 8) TMEM_LD_32x32b_X8(lane_base + uint32_t(ca), pa);
                        else TMEM_LD_32x32b_X4(lane_base + uint32_t(ca), pa);
                    } else if (ca >= 0) {
                        if constexpr (BM == 16) TMEM_LD_32x32b_X16(lane_base + uint32_t(ca), va);
                        else if constexpr (BM == 8) TMEM_LD_32x32b_X8(lane_base + uint32_t(ca), pa);
                        else TMEM_LD_32x32b_X4(lane_base + uint32_t(ca), pa);
                    } else {
#pragma unroll
                        for (int m = 0; m < BM; ++m) pa[m] = 0u;
                    }
                    if (cb >= 0) {
                        if constexpr (BM == 16) TMEM_LD_32x32b_X16(lane_base + uint32_t(cb), vb);
                        else if constexpr (BM == 8) TMEM_LD_32x32b_X8(lane_base + uint32_t(cb), pb);
                        else TMEM_LD_32x32b_X4(lane_base + uint32_t(cb), pb);
                    } else {
#pragma unroll
                        for (int m = 0; m < BM; ++m) pb[m] = 0u;
                    }
                }
            }
        };
        // software pipeline over row blocks: row block i+1's TMEM loads are in flight while row
        // block i is converted and stored (tcgen05.wait::ld waits for all of them)
        uint32_t a0[16], b0[16], a1[16], b1[16];
        uint4 rA[4], rB[4];  // residual row blocks (conv residual epilogue only)
        if (nparts > 2) {
            // four partials per row (g_i degree 4): both pairs of a row block, then
            // (p0 + p2) + (p1 + p3) in a fixed order -- not pipelined across row blocks
#pragma unroll 1
            for (int i = rb0; i < rb1; ++i) {
                tload(i, a0, b0, 0);
                tload(i, a1, b1, 1);
                rload(i, rA);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    a0[m] = __float_as_uint(__uint_as_float(a0[m]) + __uint_as_float(a1[m]));
                    b0[m] = __float_as_uint(__uint_as_float(b0[m]) + __uint_as_float(b1[m]));
                }
                put16(i, i, a0, b0, true, rA);
            }
        } else {
        tload(rb0, a0, b0, 0);
        rload(rb0, rA);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll 1
        for (int i = rb0; i < rb1; i += 2) {
            if (i + 1 < rb1) { tload(i + 1, a1, b1, 0); rload(i + 1, rB); }
            put16(i, RG ? rec[kRgRows + i] : i, a0, b0, !RG, rA);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (i + 1 >= rb1) break;
            if (i + 2 < rb1) { tload(i + 2, a0, b0, 0); rload(i + 2, rA); }
            put16(i + 1, RG ? rec[kRgRows + i + 1] : i + 1, a1, b1, !RG, rB);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        }
        if (!helper) {
            // all TMEM reads of this buffer are done: the MMA warp may reuse it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[b]);
#if RBGP4_DEBUG
            if (trace && threadIdx.x == 0 && it < 4) g_k5_epi[4 * it + 1] = clock64() - c_entry;
#endif
        }
        if (stage_last) {
            // the ring is idle (this CTA's last MMA has completed): this warp's rows go out by its
            // own TMA stores (32 columns x 16 rows per row block (groups) / x tm/2 rows (tiles))
            fence_async_smem();
            __syncwarp();
            if (threadIdx.x == 0) K5_MARK(11);
            if (ok && elect_one()) {
                if constexpr (RG) {
                    for (int r = rb0; r < rb1; ++r)
                        tma_store_2d_g(&omap, wstage + uint32_t(r * 16 * kRowBytes), int32_t(c0),
                                       int32_t(m0) + rec[kRgRows + r] * 16);
                } else {
                    for (int r = rb0; r < rb1; r += p.tm / 32)
                        tma_store_2d_g(&omap, wstage + uint32_t(r * 16 * kRowBytes), int32_t(c0), int32_t(m0) + r * 16);
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                if (warp == 0) { K5_MARK(4); K5_SMARK(3); }
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
        }
    };

    // a heavy epilogue (p.epi2: the halo conv's 128 rows of 4 x 4 blocks, ~1.5x the unit's MMA
    // time; a single-buffered accumulator, whose epilogue is not overlapped): warps 8-11 are a
    // second epilogue group (the unit's second half of rows) and 4 / 7 the only I producers
    const bool kEpiB = p.epi2 != 0;
    const bool epi_b = kEpiB && warp >= 8;
    if (warp == 4 || (warp >= 6 && !epi_b)) {
        // ========================== TMA producers ==========================
        // warp 6: expect_tx + the W box of every step (before griddepcontrol.wait for the first
        // ring's worth: weights are never the previous grid's output); warp 4: barrier init, then
        // after griddepcontrol.wait the I box of every step -- a whole slab, or (row groups) the
        // 16 L rows of the group's column-block range.  Two boxes per step: a TMA box costs its
        // engine ~150-300 cycles whatever its size (tools/tma_issue_bench.cu).
        const bool wprod = warp == 6;
        // the I boxes of consecutive steps alternate between warps 4 and 7: a box costs its
        // issuing thread ~300-450 cycles, which bounds one issuer at ~35-60 B/clk
        // (tools/stream_bench.cu); two issuers keep the row-group ranges (~16 KB boxes) and
        // the whole slabs ahead of the MMAs
        // producer index of this warp among the I producers 4, 7, 8, .. (steps round-robin).  At
        // most NS producers take part: a producer's next step must be at most one ring round
        // ahead of its last, or its parity wait on `empty` could pass two phases early.
        const int iparity = warp == 4 ? 0 : warp - 6;
        const int n_ip = min(kEpiB ? 2 : kIProd, NS);
        // lane l holds the step words l and l + 32 of the current tile-row (shuffled out)
        int32_t e0 = 0, e1 = 0, rl = 0;
        auto load_steps = [&](int tbm) {
            const int32_t *row = p.steps + int64_t(tbm) * p.d_o;
            e0 = lane < p.d_o ? __ldg(row + lane) : 0;
            e1 = lane + 32 < p.d_o ? __ldg(row + lane + 32) : 0;
        };
        // row groups: lanes 0 / 1 hold the record's lo / L
        auto load_rec = [&](int rgi) { rl = lane < 2 ? __ldg(p.rg + rgi * kRgWords + lane) : 0; };
        int tbm_cur = int((first / upt) % p.u_o);
        int rg_cur = RG ? int(first % p.n_rg) : 0;
        load_steps(tbm_cur);
        if (RG) load_rec(rg_cur);
#if RBGP4_DEBUG
        if (trace && warp == 4 && (e0 == 0x7fffffff || rl == 0x7fffffff)) g_k5_mark[15] = 1;  // wait for the loads
        if (warp == 4 && lane == 0) K5_MARK(6);
#endif
        if (warp == 4 && lane == 0) {
            for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
            for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], kEpiB ? 8 : 4); }
            mbar_init(wfull, 1);
            mbar_init(wempty, 1);
            mbar_init(last_full, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            K5_MARK(7);
        }
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(wprod ? &wmap : &imap)) : "memory");
        }
        __syncwarp();
        // barrier 3 (warps 4, 6, 7): the barrier init is visible to warps 6 and 7; barrier 1
        // (setup, all warps): arrive only -- producers never wait for TMEM or the tables
        const int bar3 = kEpiB ? 96 : kProdThreads;  // the producer warps
        if (warp == 4) asm volatile("barrier.arrive 3, %0;" ::"r"(bar3) : "memory");
        else asm volatile("barrier.sync 3, %0;" ::"r"(bar3) : "memory");
        asm volatile("barrier.arrive 1, %0;" ::"n"(kThreads) : "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        auto step_word = [&](int s) -> int32_t {
            const int32_t a = __shfl_sync(0xffffffffu, e0, s & 31);
            const int32_t b = __shfl_sync(0xffffffffu, e1, s & 31);
            return s < 32 ? a : b;
        };
        const int w_rows = p.w_rows;  // whole tiles: slice-relayout W tile of a step (nsl x mma_n rows)
        // whole tiles: expect_tx (I slab + W tile) and the W box of a step, by warp 6
        auto issue_w = [&](int st, int tbm, int32_t word) {
            const int j = word >> 16;
            if (elect_one()) {
                mbar_expect_tx(&full[st], uint32_t(SB));
                // (merged tile-rows: 512 rows = two boxes; a TMA box spans at most 256 rows)
                for (int r0 = 0; r0 < w_rows; r0 += 256)
                    tma_load_2d(ring + size_t(st) * SB + p.i_bytes + r0 * 32, &wmap, &full[st], 0,
                                (tbm * p.d_o + j) * w_rows + r0);
            }
            __syncwarp();
        };
        // row groups: the unit's whole W (group rgi's rows of the d_o tiles (tbm, j)), one 3-D box
        auto issue_wres = [&](int tbm, int rgi, int64_t it) {
            mbar_wait(wempty, uint32_t(it & 1) ^ 1u);
            if (elect_one()) {
                mbar_expect_tx(wfull, uint32_t(p.wres_bytes));
                tma_load_3d(wres, &wmap, wfull, 0, rgi * p.g * 16, tbm * p.d_o);
            }
            __syncwarp();
        };
        if constexpr (HALO) {
            // W: the tile-row's d_o tap tiles, resident, loaded once (never the previous grid's output)
            if (wprod) {
                if (first < p.n_units && elect_one()) {
                    mbar_expect_tx(wfull, uint32_t(p.d_o * w_rows * 32));
                    for (int j = 0; j < p.d_o; ++j)
                        for (int r0 = 0; r0 < w_rows; r0 += 256)
                            tma_load_2d(wres + (size_t(j) * w_rows + r0) * 32, &wmap, wfull, 0, j * w_rows + r0);
                }
                __syncwarp();
            } else {
                asm volatile("griddepcontrol.wait;" ::: "memory");
                // I: one halo box set per unit, units round-robin over the I producers
                int st = 0, ipu = 0;
                uint32_t ph = 0;
                const int n_iu = min(2, NS);
                const int64_t per_img = int64_t(p.strips_y) * p.strips_x;
                const uint32_t hbytes = uint32_t(p.tk / 64) * 180u * 128u;
                for (int64_t u = first, gu = 0; u < p.n_units; u += stride, ++gu) {
                    const int cst = st;
                    const uint32_t cph = ph;
                    if (++st == NS) { st = 0; ph ^= 1u; }
                    const int mine = ipu;
                    if (++ipu == n_iu) ipu = 0;
                    if (mine != iparity) continue;
                    if (gu >= NS) mbar_wait(&empty[cst], cph ^ 1u);
                    const int64_t bimg = u / per_img;
                    const int sy = int((u - bimg * per_img) / p.strips_x), sx = int(u % p.strips_x);
                    if (elect_one()) {
                        mbar_expect_tx(&full[cst], hbytes);
                        for (int a = 0; a < p.tk / 64; ++a)
                            tma_load_4d(ring + size_t(cst) * SB + size_t(a) * p.halo_atom, &imap, &full[cst], 64 * a,
                                        sx * 8 - 1, sy * 16 - 1, int32_t(bimg));
                    }
                    if (RES && lane < 16) {
                        // residual epilogue: the strip's 16 rows of 8 pixels of R into L2, a unit
                        // ahead of the epilogue that reads them
                        const int64_t px = (bimg * p.img_h + sy * 16 + lane) * p.img_w + sx * 8;
                        const uint32_t rb = uint32_t(8 * p.ld_out * (OUT_BF16 ? 2 : 4));
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                         static_cast<const char *>(p.res) + px * rb / 8), "r"(rb) : "memory");
                    }
                    __syncwarp();
#if RBGP4_DEBUG
                    if (trace && lane == 0 && gu < 64) g_k5_trace[0][gu] = clock64() - c_entry;
#endif
                }
            }
        } else {
        const int pre = min(NS, p.d_o);
        if (wprod && first < p.n_units) {
            if constexpr (RG) issue_wres(tbm_cur, rg_cur, 0);
            else for (int s = 0; s < pre; ++s) issue_w(s, tbm_cur, step_word(s));
            K5_MARK(0);
        }
        if (!wprod) asm volatile("griddepcontrol.wait;" ::: "memory");
        if (warp == 4 && lane == 0) K5_MARK(8);
        int64_t g = 0, it = 0;
        int rs_st = 0, ip = 0;  // ring slot, producer of the current step (g mod kIProd)
        uint32_t rs_ph = 0;
        for (int64_t u = first; u < p.n_units; u += stride, ++it) {
            const int64_t tile = u / upt;
            const int tbm = int(tile % p.u_o);
            const int rgi = RG ? int(u % p.n_rg) : 0;
            const int64_t n0 = (tile / p.u_o) * kSBatch;
            // conv: the unit's 128 output pixels = image b0, output rows h0.. (or whole images)
            int cb0 = 0, ch0 = 0;
            if constexpr (CONV) {
                const int64_t hw = int64_t(p.img_h) * p.img_w;
                cb0 = int(n0 / hw);
                ch0 = int(n0 - int64_t(cb0) * hw) / p.img_w;
            }
            if (tbm != tbm_cur) { load_steps(tbm); tbm_cur = tbm; }
            if (RG && rgi != rg_cur) { load_rec(rgi); rg_cur = rgi; }
            const int lo = RG ? __shfl_sync(0xffffffffu, rl, kRgLo) : 0;
            const int len = RG ? __shfl_sync(0xffffffffu, rl, kRgLen) : 8;
            if (RG && wprod) {
                if (it > 0) issue_wres(tbm, rgi, it);
                continue;  // row groups: W is resident, warp 6 has nothing per step
            }
            for (int s = 0; s < p.d_o; ++s, ++g) {
                // ring position by increments (a 64-bit g % NS is a software division per step)
                const int st = rs_st;
                const uint32_t ph = rs_ph;
                if (++rs_st == NS) { rs_st = 0; rs_ph ^= 1u; }
                const int ipc = ip;
                if (++ip == n_ip) ip = 0;
                const int32_t word = step_word(s);
                if (wprod) {
                    if constexpr (CONV) {
                        if (RES && s == 0 && elect_one()) {
                            // residual epilogue: the unit's 128 pixel rows of R into L2 while its
                            // main loop runs
                            const int64_t npix = min(int64_t(kSBatch), p.n_cols - n0);
                            const int64_t pb = p.ld_out * (OUT_BF16 ? 2 : 4);
                            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                             static_cast<const char *>(p.res) + n0 * pb), "r"(uint32_t(npix * pb)) : "memory");
                        }
                        __syncwarp();
                    }
                    if (g >= NS) mbar_wait(&empty[st], ph ^ 1u);
                    if (g >= pre) issue_w(st, tbm, word);
                } else if (ipc == iparity) {
                    if (g >= NS) mbar_wait(&empty[st], ph ^ 1u);
                    const int32_t krow = (word & 0xFFFF) * p.tk;
                    if (elect_one()) {
                        if constexpr (RG) {
                            mbar_expect_tx(&full[st], uint32_t(len * kPieceBytes));
                            tma_load_3d(ring + size_t(st) * SB, &imaps.m[len - 1], &full[st], 0,
                                        krow + lo * 16, int32_t(n0 / 64));
                        } else if constexpr (CONV) {
                            // K rows [krow, krow + tk) = tap (ti, tj), channels [c0, c0 + tk): per
                            // 64-channel atom one 4-D box of the 128 tap-shifted pixels (OOB = padding)
                            const int tap = krow / p.c_in, c0 = krow - tap * p.c_in;
                            const int ti = tap / p.kw, tj = tap - ti * p.kw;
                            for (int a = 0; a < p.tk / 64; ++a)
                                tma_load_4d(ring + size_t(st) * SB + a * (kSBatch * 128), &imap, &full[st], c0 + 64 * a,
                                            tj - p.pad, ch0 * p.stride + ti - p.pad, cb0);
                        } else {
                            tma_load_3d(ring + size_t(st) * SB, &imap, &full[st], 0, krow, int32_t(n0 / 64));
                        }
                    }
                    __syncwarp();
#if RBGP4_DEBUG
                    if (trace && lane == 0 && g < 64) g_k5_trace[0][g] = clock64() - c_entry;
#endif
                    if (g == 0 && lane == 0) {
                        K5_MARK(1);
                        K5_SMARK(0);
#if RBGP4_DEBUG
                        if (p.slot >= 0 && blockIdx.x < 160) g_k5_seq[p.slot][2][blockIdx.x] = k5_gtimer();
#endif
                    }
                }
            }
        }
        }  // !HALO
    } else if (warp == 5) {
        // ========================= TMEM allocation + MMA issue =========================
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)), "r"(uint32_t(p.tmem_cols)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        tc_fence_before();
        asm volatile("barrier.sync 1, %0;" ::"n"(kThreads) : "memory");
        tc_fence_after();
        const uint32_t tmem_d = *tmem_slot;
        // D f32, A/B bf16, A MN-major (SDMM: I slab) or K-major (conv: NHWC pixel x channel
        // box), B K-major (W rows), N = 16 (row groups) / the slice union (whole tiles), M = 128
        const uint32_t kN = RG ? 16u : uint32_t(p.mma_n);
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((CONV ? 0u : 1u) << 15) | (0u << 16) |
                               ((kN >> 3) << 17) | (uint32_t(kSBatch >> 4) << 24);
        const uint32_t ring_a = smem_u32(ring);
        // A: SDMM -- MN-major, 128B swizzle: 64-column atoms spaced by the rows staged per atom (a
        // whole slab, or one 16-row piece), 8-row groups 1024 B apart; conv -- K-major, 128B
        // swizzle, [64-channel atom][128 pixels][128 B]
        const uint64_t a_desc_t = CONV ? smem_desc(ring_a, 0, 1024, 2u) : smem_desc(ring_a, uint32_t(p.tk) * 128u, 1024, 2u);
        // whole tiles: B offset of slice kb (mma_n rows of 32 B), D column of slice kb
        const uint32_t b_slice16 = uint32_t(p.mma_n * 32) >> 4, d_slice = uint32_t(p.mma_n);
        const int nsl = p.nsl;
        // B: K-major W rows (row groups: d_t slots per row; whole tiles: 16-slot relayout rows)
        constexpr uint32_t w_row = RG ? 64u : 32u;  // d_t = 32 slots (stream_shape_ok)
        const uint64_t b_desc0 = RG ? smem_desc(smem_u32(wres), 0, 8 * w_row, swizzle_layout_code(int(w_row)))
                                    : smem_desc(ring_a + uint32_t(p.i_bytes), 0, 8 * w_row, swizzle_layout_code(int(w_row)));
        // row groups: the adjacency slot j of each step picks the step's W in the resident copy.
        // The group size is a compile-time constant of the loop (G = 1, 2, 4) so a unit's piece
        // offsets are hoisted into registers and a step is 2G back-to-back UTCHMMA after uniform
        // adds (loading them from the record every step cost ~200 cycles per step).
        auto mma_loop = [&](auto gc) {
            constexpr int G = decltype(gc)::value;  // 0: whole tiles
            int32_t e0 = 0, e1 = 0;
            int tbm_cur = -1;
            int64_t g = 0, it = 0;
            int rs_st = 0;
            uint32_t rs_ph = 0;
            for (int64_t u = first; u < p.n_units; u += stride, ++it) {
                const int b = p.nbuf == 2 ? int(it & 1) : 0;
                const uint32_t bph = uint32_t((p.nbuf == 2 ? (it >> 1) : it) & 1);
                uint64_t a_desc0 = a_desc_t;
                uint32_t aoff[G > 0 ? 2 * G : 1];
                if constexpr (G > 0) {
                    const int32_t *rec = s_rg + int(u % p.n_rg) * kRgWords;
                    // the staged range holds L pieces of 16 rows per 64-column atom
                    a_desc0 = smem_desc(ring_a, uint32_t(rec[kRgLen]) * 2048u, 1024, 2u);
#pragma unroll
                    for (int i = 0; i < 2 * G; ++i) aoff[i] = uint32_t(rec[kRgMma + i]) * uint32_t(2048 >> 4);
                    const int tbm = int((u / upt) % p.u_o);
                    if (tbm != tbm_cur) {
                        const int32_t *row = p.steps + int64_t(tbm) * p.d_o;
                        e0 = lane < p.d_o ? __ldg(row + lane) : 0;
                        e1 = lane + 32 < p.d_o ? __ldg(row + lane + 32) : 0;
                        tbm_cur = tbm;
                    }
                    mbar_wait(wfull, uint32_t(it & 1));
                }
#if RBGP4_DEBUG
                if (trace && lane == 0 && it < 4) g_k5_epi[4 * it + 2] = clock64() - c_entry;
#endif
                mbar_wait(&acc_empty[b], bph ^ 1u);
#if RBGP4_DEBUG
                if (trace && lane == 0 && it < 4) g_k5_epi[4 * it + 3] = clock64() - c_entry;
#endif
                tc_fence_after();
                const uint32_t d_base = tmem_d + uint32_t(b * p.acc_cols);
                for (int s = 0; s < p.d_o; ++s, ++g) {
                    const int st = rs_st;
                    const uint32_t ph = rs_ph;
                    if (++rs_st == NS) { rs_st = 0; rs_ph ^= 1u; }
                    int32_t wj = 0;
                    if constexpr (G > 0) {
                        const int32_t a = __shfl_sync(0xffffffffu, e0, s & 31), bb = __shfl_sync(0xffffffffu, e1, s & 31);
                        wj = (s < 32 ? a : bb) >> 16;
                    }
                    mbar_wait(&full[st], ph);
                    tc_fence_after();
#if RBGP4_DEBUG
                    if (trace && lane == 0 && g < 64) g_k5_trace[1][g] = clock64() - c_entry;
#endif
                    if (g == 0 && lane == 0) { K5_MARK(2); K5_SMARK(1); }
                    if (elect_one()) {
                        const uint32_t st16 = uint32_t(st * SB) >> 4;
                        const uint64_t a_st = a_desc0 + st16;
                        if constexpr (G > 0) {
                            const uint64_t b_st = b_desc0 + uint32_t(wj * ((G * 16 * int(w_row)) >> 4));
#pragma unroll
                            for (int r = 0; r < G; ++r)
#pragma unroll
                                for (int ink = 0; ink < 2; ++ink)
                                    tc_mma<false>(d_base + uint32_t(r * 16), a_st + aoff[r * 2 + ink],
                                                  b_st + uint32_t(r * ((16 * w_row) >> 4) + ink * 2), idesc,
                                                  (s > 0 || ink > 0) ? 1u : 0u);
                        } else {
                            // slice relayout: K16 slice kb of the step (16 slab rows / 16 channels)
                            // times the union of the rows reading it, one N = mma_n MMA each (TC16:
                            // 8 column blocks of 16, N = 32)
                            const uint64_t b_st = b_desc0 + st16;
                            const uint32_t acc = s > 0 ? 1u : 0u;
#pragma unroll
                            for (int kb = 0; kb < 8; ++kb) {
                                if (kb >= nsl) break;
                                const uint32_t a16 = CONV ? uint32_t(kb / 4) * uint32_t(kSBatch * 128 / 16) + uint32_t(kb % 4) * 2u
                                                          : uint32_t(kb * 16 * 8);
                                tc_mma<false>(d_base + uint32_t(kb) * d_slice, a_st + a16,
                                              b_st + uint32_t(kb) * b_slice16, idesc, acc);
                            }
                        }
                        tc_commit(&empty[st]);
                        if (s == p.d_o - 1) {
                            tc_commit(&acc_full[b]);
                            if (G > 0) tc_commit(wempty);
                            if (u + stride >= p.n_units) tc_commit(last_full);
                        }
#if RBGP4_DEBUG
                        if (trace && g < 64) g_k5_trace[2][g] = clock64() - c_entry;
#endif
                    }
                    __syncwarp();
                }
            }
        };
        // halo conv: one ring stage per unit; the nine taps (step words: adjacency slot j << 16 | tap)
        // are row offsets ti * 10 + tj into the staged 18 x 10 halo (SW128 K-major rows of 128 B,
        // 8-pixel groups 10 rows apart), the tap's W tile the resident slot j
        auto halo_loop = [&]() {
            constexpr int kTaps = 9;
            // per tap (in 16-byte units): the A start row ti * 10 + tj inside the halo, the B tile of
            // its adjacency slot j in the resident W (kept in shared memory: 18 values held in
            // registers across the unit loop were spilled and reloaded per MMA)
            if (lane < kTaps) {
                const int32_t w = __ldg(p.steps + lane);  // u_o = 1: tile-row 0
                const int t = w & 0xFFFF;
                s_tap[lane] = uint32_t((t / 3) * 10 + t % 3) * (128u >> 4);
                s_tap[kTaps + lane] = uint32_t(w >> 16) * (uint32_t(p.w_rows * 32) >> 4);
            }
            __syncwarp();
            const uint64_t a_halo = smem_desc(ring_a, 0, 10 * 128, 2u);
            const uint64_t b_res = smem_desc(smem_u32(wres), 0, 8 * 32, swizzle_layout_code(32));
            mbar_wait(wfull, 0u);
            int st = 0;
            uint32_t ph = 0;
            int64_t it = 0;
            for (int64_t u = first; u < p.n_units; u += stride, ++it) {
                const int b = p.nbuf == 2 ? int(it & 1) : 0;
                const uint32_t bph = uint32_t((p.nbuf == 2 ? (it >> 1) : it) & 1);
                const int cst = st;
                const uint32_t cph = ph;
                if (++st == NS) { st = 0; ph ^= 1u; }
                mbar_wait(&acc_empty[b], bph ^ 1u);
                mbar_wait(&full[cst], cph);
                tc_fence_after();
#if RBGP4_DEBUG
                if (trace && lane == 0 && it < 64) g_k5_trace[1][it] = clock64() - c_entry;
#endif
                if (elect_one()) {
                    const uint32_t d_base = tmem_d + uint32_t(b * p.acc_cols);
                    const uint32_t stage16 = uint32_t(cst * SB) >> 4;
#pragma unroll 1
                    for (int s = 0; s < kTaps; ++s) {
                        const uint64_t a_s = a_halo + stage16 + s_tap[s];
                        const uint64_t b_s = b_res + s_tap[kTaps + s];
                        const uint32_t acc = s > 0 ? 1u : 0u;
#pragma unroll
                        for (int kb = 0; kb < 8; ++kb) {
                            if (kb >= nsl) break;
                            // (base offset 0: the 128B swizzle acts on the absolute address bits,
                            // so a start shifted by any number of 128-byte rows reads the rows
                            // exactly as TMA swizzled them -- tests/test_slices.py)
                            tc_mma<false>(d_base + uint32_t(kb) * d_slice,
                                          a_s + uint32_t((kb / 4) * (kHaloAtom >> 4) + (kb % 4) * 2),
                                          b_s + uint32_t(kb) * b_slice16, idesc, acc);
                        }
                    }
                    tc_commit(&empty[cst]);
                    tc_commit(&acc_full[b]);
                    if (u + stride >= p.n_units) tc_commit(last_full);
#if RBGP4_DEBUG
                    if (trace && it < 64) g_k5_trace[2][it] = clock64() - c_entry;
#endif
                }
                __syncwarp();
            }
        };
        if constexpr (HALO) {
            halo_loop();
        } else if constexpr (RG) {
            if (p.g == 1) mma_loop(std::integral_constant<int, 1>{});
            else if (p.g == 2) mma_loop(std::integral_constant<int, 2>{});
            else mma_loop(std::integral_constant<int, 4>{});
        } else {
            mma_loop(std::integral_constant<int, 0>{});
        }
    } else {
        // ============================ epilogue (warps 0-3; halo: + 8-11) ============================
        if (warp < 4) {
            if constexpr (RG) {
                for (int i = threadIdx.x; i < p.n_rg * kRgWords; i += 128) s_rg[i] = p.rg[i];
            } else {
                for (int i = threadIdx.x; i < p.n_cols_tab; i += 128) s_cols[i] = p.cols[i];
            }
        }
        asm volatile("barrier.sync 1, %0;" ::"n"(kThreads) : "memory");
        tc_fence_after();
        int64_t it = 0;
        for (int64_t u = first; u < p.n_units; u += stride, ++it) {
            const int nrb = RG ? p.g : p.tm / 16;
            if (kEpiB) {
                // halo: two groups split every unit's rows (its epilogue is ~1.5x its MMA time)
                drain(u, it, epi_b ? nrb / 2 : 0, epi_b ? nrb : nrb / 2, s_cols, nullptr, false);
                continue;
            }
            // the CTA's last unit is the only exposed epilogue: warps 4-7 (idle by then) take
            // the second half of its row blocks
            const bool last = u + stride >= p.n_units;
            const int split = (last && nrb >= 2) ? nrb / 2 : nrb;
            drain(u, it, 0, split, s_cols, RG ? s_rg + int(u % p.n_rg) * kRgWords : nullptr, false);
        }
        // staged conv stores: all of this warp's TMA stores done before the CTA retires
        if (CONV && p.ostage && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    if (!kEpiB && warp >= 4 && warp < 8) {
        // warps 4-7 after their roles: the second half of the last unit's row blocks (tables
        // read from global memory: these warps never synchronised on the epilogue's copies)
        const int64_t n_mine = (p.n_units - first + stride - 1) / stride;
        const int64_t u = first + (n_mine - 1) * stride;
        const int nrb = RG ? p.g : p.tm / 16;
        if (n_mine > 0 && nrb >= 2) {
            drain(u, n_mine - 1, nrb / 2, nrb, p.cols, RG ? p.rg + int(u % p.n_rg) * kRgWords : nullptr, true);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot),
                     "r"(uint32_t(p.tmem_cols)));
    }
#if RBGP4_DEBUG
    if (threadIdx.x == 0) K5_MARK(5);
    if ((p.debug & 512) && threadIdx.x == 0 && blockIdx.x < kK5Stamps) g_k5_stamp[1][blockIdx.x] = k5_gtimer();
    if (p.slot >= 0 && threadIdx.x == 0 && blockIdx.x < 160) g_k5_seq[p.slot][1][blockIdx.x] = k5_gtimer();
#endif
#undef K5_MARK
#undef K5_SMARK
}

// row-permuted copy of the values for the row-group mode: tile (tbm, j) of W (tm rows x d_t
// slots, sorted-column order, reference rcubs.py:79-98) with its row blocks in group order
// perm[k] -- the same bytes, so a group's rows of a step are one contiguous box
__global__ void rg_values_kernel(const __nv_bfloat16 *__restrict__ values, int64_t row_nnz, int tm, int d_t,
                                 int d_o, const int32_t *__restrict__ perm, int64_t total,
                                 __nv_bfloat16 *__restrict__ outv) {
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int slot = int(idx % d_t);
        const int64_t row = idx / d_t;  // row of the permuted copy: ((tbm * d_o + j) * tm + k * 16 + m)
        const int m = int(row % 16), k = int((row / 16) % (tm / 16));
        const int64_t tj = row / tm;
        const int64_t tbm = tj / d_o, j = tj % d_o;
        outv[idx] = values[(tbm * tm + perm[k] * 16 + m) * row_nnz + j * d_t + slot];
    }
}

// K5 section of the prepared buffer: [steps i32 u_o x d_o][records: G = 1, 2, 4][perm i32 8]
// [row-permuted values bf16 (rows x row_nnz)]
int rg_groups(int g) { return 8 / g; }
size_t rg_offset_words(int g) { return g == 1 ? 0 : g == 2 ? size_t(8) * kRgWords : size_t(12) * kRgWords; }
size_t a16w(size_t words) { return (words + 3) & ~size_t(3); }
size_t tables_words(const ChainDims &c) { return a16w(size_t(c.u_o) * c.d_o) + a16w(size_t(14) * kRgWords + 8); }

}  // namespace

// TC16 shape: g_r (1,1), 16 x 16 element blocks, g_i (8,8) of degree 2 (its relayout exists,
// sdmm_gather.cu), 128 x 128 tiles, at most 64 steps per tile-row -- whole tiles on K4's
// relayout, or row groups.
int stream_shape_ok(const ChainDims &c) {
    return c.rm == 1 && c.rk == 1 && c.bm == 16 && c.bk == 16 && c.u_i == 8 && c.v_i == 8 && c.d_i == 2 &&
           c.tm == 128 && c.tk == 128 && c.d_t == 32 && c.d_o <= kMaxDo && c.v_o < (1 << 16) &&
           gather_relayout_ok(c);
}

namespace {
// Slice relayout (any other g_b that tiles K16, e.g. the 8 x 8 / 4 x 4 element blocks of the
// small-channel VGG / WRN layers and the `tc` factorisation): a step's K range is cut into
// K16 slices; slice kb multiplies the 16 slab rows (channels) [16 kb, 16 kb + 16) by the union
// of the tile's rows that have a nonzero there -- a per-matrix constant, since g_r (x) g_i (x)
// g_b repeats in every tile -- padded to `mma_n` rows with zeros.  The prepared values hold,
// per W tile (tbm, j), the [slice][union row][16 k] dense K-major operand (zeros where a union
// row's block does not cover a k); each output row has at most two partials (the slices its
// d_i column blocks fall in), summed in the epilogue.  MMA work per step is tk/16 MMAs of
// N = mma_n, whatever the block size (TC16 is the special case union = d_r blocks of 16).
struct SliceDims {
    int nsl, mma_n, d_r, r;  // r: tile-rows merged into one unit (see merged())
    int parts;               // partial accumulators per row block: 2, or 4 (g_i degree 4)
};
bool slice_dims(const ChainDims &c, SliceDims *sd, int max_cols = 256) {
    if (opts().relayout == 0) return false;  // option relayout=0: no value relayout of any kind
    if (c.rm != 1 || c.rk != 1) return false;
    if ((c.tm != 64 && c.tm != 128 && c.tm != 256) || (c.tk != 64 && c.tk != 128)) return false;
    if (c.bm != 4 && c.bm != 8 && c.bm != 16) return false;
    if (!(c.bk <= 16 ? 16 % c.bk == 0 : c.bk % 16 == 0)) return false;
    const int parts = c.d_i * std::max(1, c.bk / 16) <= 2 ? 2 : 4;
    if (c.d_i * std::max(1, c.bk / 16) > 4) return false;  // <= 4 partials per row
    if (c.d_t != c.d_i * c.bk || c.d_o > kMaxDo || c.v_o >= (1 << 16)) return false;
    if ((int64_t(c.u_i) * c.d_i) % c.v_i) return false;
    const int d_r = c.u_i * c.d_i / c.v_i;
    const int per = (c.bk < 16 ? 16 / c.bk : 1) * d_r * c.bm;
    const int n = (std::min(per, c.tm) + 15) & ~15;
    if (n > 256 || (c.tk / 16) * n > max_cols) return false;
    if (c.tm / c.bm * parts > 128) return false;  // cols table
    sd->nsl = c.tk / 16;
    sd->mma_n = n;
    sd->d_r = d_r;
    sd->r = 1;
    sd->parts = parts;
    return true;
}

// Tile-row merging: when g_o is complete (every tile-row reads every K-block, in the same
// order), R = 2 consecutive tile-rows form one unit -- a virtual tile of 2 tm rows whose slice
// unions are twice as wide (N = 64 for TC16 / 8 x 8 blocks).  Each I slab is then loaded once
// for both tile-rows (half the L2 -> SM bytes) and a step is tk/16 MMAs of twice the N (an
// M128 K16 MMA costs ~82 cycles up to N = 64 and ~95 at N = 128: tools/umma_bench3.cu), for a
// single-buffered 512-column accumulator (the epilogue is no longer overlapped).
ChainDims merged(const ChainDims &c, int r) {
    ChainDims m = c;
    m.tm = c.tm * r;
    m.u_i = c.u_i * r;
    m.u_o = c.u_o / r;
    return m;
}
int merge_factor(const ChainDims &c) {
    if (opts().merge == 0 || c.tm != 128 || c.u_o % 2 || c.d_o != c.v_o) return 1;
    SliceDims sd;
    return slice_dims(merged(c, 2), &sd, 512) ? 2 : 1;
}
// K5 mode of a chain: 0 none, 1 TC16 on K4's relayout (row groups possible), 2 slice relayout
// on the effective (possibly merged) dims `eff`
int k5_mode(const ChainDims &c, ChainDims *eff, SliceDims *sd) {
    *eff = c;
    const int r = merge_factor(c);
    if (r > 1) {
        *eff = merged(c, r);
        slice_dims(*eff, sd, 512);
        sd->r = r;
        return 2;
    }
    if (stream_shape_ok(c)) {
        *sd = SliceDims{8, 32, 2, 1, 2};
        return 1;
    }
    // (512 accumulator columns -- g_i degree 4 -- run single-buffered)
    return slice_dims(c, sd, 512) ? 2 : 0;
}
// slice section of the prepared buffer: [steps i32 u_o x d_o][cols i32 (tm/bm) x 2][map rows i32
// nsl x mma_n][map k-offsets i16 nsl x mma_n x 16][values bf16 u_o x d_o x nsl x mma_n x 16]
struct SliceLayout {
    size_t steps, cols, rows, offs, vals, total;  // word offsets (vals: byte offset), bytes
};
SliceLayout slice_layout(const ChainDims &c, const SliceDims &sd) {
    SliceLayout l;
    const size_t w = size_t(sd.nsl) * sd.mma_n;
    l.steps = 0;
    l.cols = a16w(size_t(c.u_o) * c.d_o);
    l.rows = l.cols + a16w(size_t(c.tm / c.bm) * sd.parts);
    l.offs = l.rows + a16w(w);
    l.vals = 4 * (l.offs + a16w(w * 8));
    l.total = l.vals + size_t(c.u_o) * c.d_o * w * 16 * 2;
    return l;
}

__global__ void slice_values_kernel(const __nv_bfloat16 *__restrict__ values, int64_t row_nnz, int tm, int d_t,
                                    int d_o, int nsl, int mma_n, const int32_t *__restrict__ mrows,
                                    const int16_t *__restrict__ moffs, int64_t total,
                                    __nv_bfloat16 *__restrict__ outv) {
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int kk = int(idx % 16);
        const int64_t r = idx / 16;                  // (tile, slice, union row)
        const int n = int(r % (int64_t(nsl) * mma_n));  // slice * mma_n + union row
        const int64_t tj = r / (int64_t(nsl) * mma_n);  // W tile (tbm, j)
        const int64_t tbm = tj / d_o, j = tj % d_o;
        const int row = mrows[n], off = moffs[n * 16 + kk];
        __nv_bfloat16 v = __float2bfloat16_rn(0.0f);
        if (row >= 0 && off >= 0) v = values[(tbm * tm + row) * row_nnz + j * d_t + off];
        outv[idx] = v;
    }
}

// step words [tbm][s] = adjacency slot j << 16 | K-block (the schedule order of the steps)
void step_words(const ChainDims &c, const int32_t *adj_o_host, const int32_t *sched_host, int32_t *tab) {
    for (int u = 0; u < c.u_o; ++u)
        for (int s = 0; s < c.d_o; ++s) {
            const int j = sched_host ? sched_host[size_t(u) * c.d_o + s] : s;
            tab[size_t(u) * c.d_o + s] = (j << 16) | adj_o_host[size_t(u) * c.d_o + j];
        }
}

int slice_prepare(const ChainDims &c, const SliceDims &sd, const void *values, const int32_t *adj_o_host,
                  const int32_t *sched_host, const int32_t *adj_i_host, void *k5, cudaStream_t stream) {
    const SliceLayout l = slice_layout(c, sd);
    std::vector<int32_t> tab(l.vals / 4, -1);
    step_words(c, adj_o_host, sched_host, tab.data());
    const int n_rb = c.tm / c.bm, w = sd.nsl * sd.mma_n;
    // does row block rb read slab column k (relative to the tile)?  -> its slot offset, else -1
    auto offset_of = [&](int rb, int k) {
        const int cb = k / c.bk;
        int rank = 0;
        bool hit = false;
        for (int ink = 0; ink < c.d_i; ++ink) {
            const int nb = adj_i_host[rb * c.d_i + ink];
            if (nb == cb) hit = true;
            else if (nb < cb) ++rank;
        }
        return hit ? rank * c.bk + k % c.bk : -1;
    };
    int32_t *cols = tab.data() + l.cols, *mrows = tab.data() + l.rows;
    int16_t *moffs = reinterpret_cast<int16_t *>(tab.data() + l.offs);
    std::vector<int> nparts(n_rb, 0);
    for (int kb = 0; kb < sd.nsl; ++kb) {
        int pos = 0;
        for (int rb = 0; rb < n_rb; ++rb) {
            bool touches = false;
            for (int k = 16 * kb; k < 16 * kb + 16 && !touches; ++k) touches = offset_of(rb, k) >= 0;
            if (!touches) continue;
            if ((pos + 1) * c.bm > sd.mma_n || nparts[rb] >= sd.parts) {
                set_error("rbgp4_prepare: slice %d needs more than %d rows / row block %d more than %d partials", kb,
                          sd.mma_n, rb, sd.parts);
                return RBGP4_EUNSUPPORTED;
            }
            cols[rb * sd.parts + nparts[rb]++] = kb * sd.mma_n + pos * c.bm;
            for (int m = 0; m < c.bm; ++m) {
                const int n = kb * sd.mma_n + pos * c.bm + m;
                mrows[n] = rb * c.bm + m;
                for (int kk = 0; kk < 16; ++kk) moffs[n * 16 + kk] = int16_t(offset_of(rb, 16 * kb + kk));
            }
            ++pos;
        }
        for (int n = kb * sd.mma_n + pos * c.bm; n < (kb + 1) * sd.mma_n; ++n)
            for (int kk = 0; kk < 16; ++kk) moffs[n * 16 + kk] = -1;
    }
    for (int rb = 0; rb < n_rb; ++rb)
        if (nparts[rb] == 0) {
            set_error("rbgp4_prepare: row block %d has no nonzero", rb);
            return RBGP4_EUNSUPPORTED;
        }
    (void)w;
    cudaError_t e = cudaMemcpyAsync(k5, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) {
        const int32_t *mr = static_cast<const int32_t *>(k5) + l.rows;
        const int16_t *mo = reinterpret_cast<const int16_t *>(static_cast<const int32_t *>(k5) + l.offs);
        __nv_bfloat16 *outv = reinterpret_cast<__nv_bfloat16 *>(static_cast<char *>(k5) + l.vals);
        const int64_t total = int64_t(c.u_o) * c.d_o * sd.nsl * sd.mma_n * 16;
        slice_values_kernel<<<int(std::min<int64_t>((total + 255) / 256, 8 * kNumSMs)), 256, 0, stream>>>(
            static_cast<const __nv_bfloat16 *>(values), c.row_nnz, c.tm, c.d_t, c.d_o, sd.nsl, sd.mma_n, mr, mo,
            total, outv);
        e = cudaGetLastError();
        if (e == cudaSuccess) note_launch();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // `tab` is a host temporary
    if (e != cudaSuccess) {
        set_error("rbgp4_prepare: writing the K5 slice relayout: %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    return RBGP4_OK;
}
}  // namespace

size_t stream_prep_bytes(const ChainDims &c) {
    ChainDims e;
    SliceDims sd;
    const int mode = k5_mode(c, &e, &sd);
    if (mode == 1) return 4 * tables_words(c) + size_t(c.rows) * c.row_nnz * 2;
    if (mode == 2) return slice_layout(e, sd).total;
    return 0;
}

static int tc16_prepare(const ChainDims &c, const void *values, const int32_t *adj_o_host, const int32_t *sched_host,
                        const int32_t *adj_i_host, void *k5, cudaStream_t stream) {
    const size_t n_steps = size_t(c.u_o) * c.d_o;
    std::vector<int32_t> tab(tables_words(c), 0);
    for (int u = 0; u < c.u_o; ++u)
        for (int s = 0; s < c.d_o; ++s) {
            const int j = sched_host ? sched_host[size_t(u) * c.d_o + s] : s;
            tab[size_t(u) * c.d_o + s] = (j << 16) | adj_o_host[size_t(u) * c.d_o + j];
        }
    // Row-block order for the row groups: a unit of G row blocks loads the contiguous range of
    // g_i column blocks its row blocks read (one TMA box per step), so the pairs (G = 2) are the
    // perfect matching of the 8 row blocks with the smallest total range (all 105 matchings
    // tried), the quads (G = 4) the best pairing of those pairs; every group is a run of `perm`.
    auto nb = [&](int r, int ink) { return adj_i_host[r * c.d_i + ink]; };
    auto range_of = [&](const std::vector<int> &rows, int *lo) {
        int a = c.v_i, b = -1;
        for (int r : rows)
            for (int ink = 0; ink < c.d_i; ++ink) { a = std::min(a, nb(r, ink)); b = std::max(b, nb(r, ink)); }
        if (lo) *lo = a;
        return b - a + 1;
    };
    std::vector<std::pair<int, int>> best_pairs, cur;
    int best_cost = 1 << 30;
    std::vector<char> used(c.u_i, 0);
    std::function<void(int)> match = [&](int cost) {
        int a = 0;
        while (a < c.u_i && used[a]) ++a;
        if (a == c.u_i) {
            if (cost < best_cost) { best_cost = cost; best_pairs = cur; }
            return;
        }
        used[a] = 1;
        for (int b = a + 1; b < c.u_i; ++b) {
            if (used[b]) continue;
            used[b] = 1;
            cur.push_back({a, b});
            match(cost + range_of({a, b}, nullptr));
            cur.pop_back();
            used[b] = 0;
        }
        used[a] = 0;
    };
    match(0);
    // pairs of pairs: 3 ways to split 4 pairs into 2 quads
    const int split[3][4] = {{0, 1, 2, 3}, {0, 2, 1, 3}, {0, 3, 1, 2}};
    int bs = 0, bcost = 1 << 30;
    for (int k = 0; k < 3; ++k) {
        int cost = 0;
        for (int h = 0; h < 2; ++h) {
            const auto &x = best_pairs[split[k][2 * h]], &y = best_pairs[split[k][2 * h + 1]];
            cost += range_of({x.first, x.second, y.first, y.second}, nullptr);
        }
        if (cost < bcost) { bcost = cost; bs = k; }
    }
    std::vector<int32_t> perm;
    for (int k = 0; k < 4; ++k) {
        const auto &x = best_pairs[split[bs][k]];
        perm.push_back(x.first);
        perm.push_back(x.second);
    }
    int32_t *recs = tab.data() + a16w(n_steps);
    for (int g : {1, 2, 4}) {
        for (int gi = 0; gi < rg_groups(g); ++gi) {
            int32_t *rec = recs + rg_offset_words(g) + size_t(gi) * kRgWords;
            std::vector<int> rows(perm.begin() + gi * g, perm.begin() + (gi + 1) * g);
            int lo = 0;
            const int len = range_of(rows, &lo);
            rec[kRgLo] = lo;
            rec[kRgLen] = len;
            for (int r = 0; r < g; ++r) {
                rec[kRgRows + r] = rows[r];
                for (int ink = 0; ink < c.d_i; ++ink) rec[kRgMma + r * c.d_i + ink] = nb(rows[r], ink) - lo;
            }
        }
    }
    int32_t *perm_t = recs + size_t(14) * kRgWords;
    std::copy(perm.begin(), perm.end(), perm_t);
    cudaError_t e = cudaMemcpyAsync(k5, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) {
        const int32_t *perm_d = static_cast<const int32_t *>(k5) + a16w(n_steps) + size_t(14) * kRgWords;
        __nv_bfloat16 *outv = reinterpret_cast<__nv_bfloat16 *>(static_cast<char *>(k5) + 4 * tables_words(c));
        const int64_t total = c.rows * c.row_nnz;
        rg_values_kernel<<<int(std::min<int64_t>((total + 255) / 256, 4 * kNumSMs)), 256, 0, stream>>>(
            static_cast<const __nv_bfloat16 *>(values), c.row_nnz, c.tm, c.d_t, c.d_o, perm_d, total, outv);
        e = cudaGetLastError();
        if (e == cudaSuccess) note_launch();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // `tab` is a host temporary
    if (e != cudaSuccess) {
        set_error("rbgp4_prepare: writing the K5 tables: %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    return RBGP4_OK;
}

// values-only refresh (training): the tables of stream_prepare stay; the value copies are
// rebuilt on the device from the new values (stream-ordered, no host work, graph-capturable)
int stream_prepare_values(const ChainDims &c, const void *values, void *k5, cudaStream_t stream) {
    const int64_t total = c.rows * c.row_nnz;
    const int blocks = int(std::min<int64_t>((total + 255) / 256, 8 * kNumSMs));
    ChainDims e;
    SliceDims sd;
    const int mode = k5_mode(c, &e, &sd);
    if (mode == 1) {
        const int32_t *perm_d = static_cast<const int32_t *>(k5) + a16w(size_t(c.u_o) * c.d_o) + size_t(14) * kRgWords;
        __nv_bfloat16 *outv = reinterpret_cast<__nv_bfloat16 *>(static_cast<char *>(k5) + 4 * tables_words(c));
        rg_values_kernel<<<blocks, 256, 0, stream>>>(static_cast<const __nv_bfloat16 *>(values), c.row_nnz, c.tm,
                                                     c.d_t, c.d_o, perm_d, total, outv);
        RBGP4_CHECK_LAUNCH("rg_values_kernel launch");
        return RBGP4_OK;
    }
    if (mode != 2) return RBGP4_OK;  // no K5 section
    const SliceLayout l = slice_layout(e, sd);
    const int32_t *mr = static_cast<const int32_t *>(k5) + l.rows;
    const int16_t *mo = reinterpret_cast<const int16_t *>(static_cast<const int32_t *>(k5) + l.offs);
    __nv_bfloat16 *outv = reinterpret_cast<__nv_bfloat16 *>(static_cast<char *>(k5) + l.vals);
    const int64_t tot = int64_t(e.u_o) * e.d_o * sd.nsl * sd.mma_n * 16;
    slice_values_kernel<<<int(std::min<int64_t>((tot + 255) / 256, 8 * kNumSMs)), 256, 0, stream>>>(
        static_cast<const __nv_bfloat16 *>(values), e.row_nnz, e.tm, e.d_t, e.d_o, sd.nsl, sd.mma_n, mr, mo, tot, outv);
    RBGP4_CHECK_LAUNCH("slice_values_kernel launch");
    return RBGP4_OK;
}

int stream_prepare(const ChainDims &c, const void *values, const int32_t *adj_o_host, const int32_t *sched_host,
                   const int32_t *adj_i_host, void *k5, cudaStream_t stream) {
    ChainDims e;
    SliceDims sd;
    const int mode = k5_mode(c, &e, &sd);
    if (mode == 1) return tc16_prepare(c, values, adj_o_host, sched_host, adj_i_host, k5, stream);
    if (mode != 2) return RBGP4_EUNSUPPORTED;
    if (sd.r == 1) return slice_prepare(c, sd, values, adj_o_host, sched_host, adj_i_host, k5, stream);
    // merged tile-rows: the virtual tile-row t is tile-row t * r (g_o complete: every tile-row has
    // the same adjacency and slot j <-> K-block j); its row blocks repeat g_i r times
    std::vector<int32_t> ao(size_t(e.u_o) * c.d_o), sc(ao.size()), ai(size_t(e.u_i) * c.d_i);
    for (int t = 0; t < e.u_o; ++t)
        for (int s2 = 0; s2 < c.d_o; ++s2) {
            ao[size_t(t) * c.d_o + s2] = adj_o_host[size_t(t) * sd.r * c.d_o + s2];
            sc[size_t(t) * c.d_o + s2] = sched_host ? sched_host[size_t(t) * sd.r * c.d_o + s2] : s2;
        }
    for (int rb = 0; rb < e.u_i; ++rb)
        for (int ink = 0; ink < c.d_i; ++ink) ai[size_t(rb) * c.d_i + ink] = adj_i_host[(rb % c.u_i) * c.d_i + ink];
    return slice_prepare(e, sd, values, ao.data(), sc.data(), ai.data(), k5, stream);
}

namespace {
struct SPlan {
    SParams p;
    size_t smem;
    unsigned grid;
    bool rg, halo;
    ChainDims eff;  // effective dims (merged tile-rows)
};


// the halo strip conv: 3 x 3 stride 1 'same', one channel block (c_in == tk), u_o = 1, output
// maps cut into 16 x 8 strips
bool halo_ok(const ChainDims &c, const rbgp4_conv_desc *cv) {
    return cv != nullptr && opts().halo != 0 && c.u_o == 1 && c.d_o == 9 && cv->c_in == c.tk && cv->kh == 3 &&
           cv->kw == 3 && cv->stride == 1 && cv->pad == 1 && cv->height % 16 == 0 && cv->width % 8 == 0 &&
           c.n_cols == int64_t(cv->batch) * cv->height * cv->width;
}

constexpr size_t kSSmemCap = 227 * 1024;

int stream_plan(const ChainDims &c_in, int out_dtype, bool conv, SPlan *pl, const rbgp4_conv_desc *cv = nullptr) {
    if (opts().stream == 0) return 0;
    ChainDims c;  // the effective dims: merged tile-rows count as one tile-row of 2 tm rows
    SliceDims sd{};
    const int mode = k5_mode(c_in, &c, &sd);
    if (mode == 0) return 0;
    const bool tc16 = mode == 1;
    // (a warp's 32 columns / pixels are all in or out; conv: OOB images of the last tile load as zeros)
    if (c.n_cols % (conv ? 32 : 64) != 0) return 0;
    const int oelt = out_dtype == RBGP4_BF16 ? 2 : 4;
    SParams p{};
    p.n_cols = c.n_cols;
    p.ld_out = c.ld_out;
    p.u_o = c.u_o; p.d_o = c.d_o; p.tm = c.tm; p.tk = c.tk; p.u_i = c.u_i; p.d_i = c.d_i; p.d_t = c.d_t;
    p.nsl = sd.nsl;
    p.mma_n = sd.mma_n;
    p.w_rows = sd.nsl * sd.mma_n;
    p.n_cols_tab = c.tm / c.bm * sd.parts;
    p.parts = sd.parts;
    const int64_t tiles = c.u_o * ((c.n_cols + kSBatch - 1) / kSBatch);
    // whole tiles when they fill ~2/3 of the SMs, else (TC16 SDMM) the largest row group that does
    int g = 8;
    if (tc16 && !conv) {
        if (opts().stream_g > 0) g = opts().stream_g;
        else if (tiles < 96) g = tiles * 2 >= 96 ? 4 : tiles * 4 >= 96 ? 2 : 1;
        if (g != 1 && g != 2 && g != 4 && g != 8) return 0;
    }
    const bool rg = g < 8;
    const bool halo = conv && sd.r == 1 && halo_ok(c, cv);
    p.g = rg ? g : c.tm / 16;
    p.n_rg = rg ? 8 / g : 1;
    p.n_units = tiles * p.n_rg;
    if (halo) {
        p.strips_y = cv->height / 16;
        p.strips_x = cv->width / 8;
        p.n_units = int64_t(cv->batch) * p.strips_y * p.strips_x;
        p.halo_atom = kHaloAtom;
        p.epi2 = c.tm / c.bm >= 32 ? 1 : 0;
    }
    // row groups: stage = the longest possible column-block range (8 pieces) + the group's W rows
    p.i_bytes = rg ? 8 * kPieceBytes : c.tk * kSBatch * 2;
    // whole tiles: a stage = I slab (conv: pixel x channel box) + the step's relayout W tile;
    // row groups: the I range only, the unit's W resident (d_o steps x G*16 rows x d_t slots)
    const int w_bytes = rg || halo ? 0 : p.w_rows * 32;
    p.stage_bytes = int((size_t(p.i_bytes) + w_bytes + 1023) & ~size_t(1023));
    p.wres_bytes = rg ? int((size_t(c.d_o) * g * 16 * c.d_t * 2 + 1023) & ~size_t(1023)) : 0;
    if (halo) {
        // a stage = the unit's halo (one atom per 64 channels); W of all nine taps resident
        p.stage_bytes = (c.tk / 64) * kHaloAtom;
        p.wres_bytes = int((size_t(c.d_o) * p.w_rows * 32 + 1023) & ~size_t(1023));
    }
    p.acc_cols = rg ? g * 16 : p.w_rows;
    const int cap = opts().stream_ctas > 0 ? std::min(opts().stream_ctas, kNumSMs) : kNumSMs;
    const unsigned grid = unsigned(std::min<int64_t>(p.n_units, cap));
    const bool multi = p.n_units > int64_t(grid);
    // two accumulator buffers when they fit (epilogue of unit i under the MMAs of unit i+1)
    p.nbuf = (multi && p.acc_cols * 2 <= 512) ? 2 : 1;
    if (p.nbuf == 1 && multi && !rg) p.epi2 = 1;
    int tcols = 32;
    while (tcols < p.acc_cols * p.nbuf) tcols *= 2;
    if (tcols > 512) return 0;
    p.tmem_cols = tcols;
    // the last unit is staged in the ring (SDMM): 4 warps x nrows x 32 columns of the output
    const size_t staging = conv ? 0 : size_t(rg ? g * 16 : c.tm) * kSBatch * oelt;
    const size_t statics = (rg ? size_t(kMaxRg) * kRgWords * 4 : 512) + 64;
    const size_t fixed = 1024 + 1024;  // alignment slack + barrier block
    // conv (bf16, no pool / residual): 4 KB of output staging per epilogue warp (TMA stores).
    // Not for halo strips: their stages are 23-46 KB and the staging would cost one (128 ch @16x16
    // 1.37 -> 1.46 ms), while the tap-shifted convs gain 11-17 % (tools/conv_store_ab.py)
    // Pooled epilogues stage only the warp's 8 pooled pixels (1 KB); not for halo strips either
    // (64 ch @32x32 + pool: 4.67 -> 4.87 ms staged).
    const bool pooled = cv != nullptr && (cv->relu & 2);
    const bool ost = conv && !halo && opts().conv_ostage != 0 && out_dtype == RBGP4_BF16 &&
                     cv != nullptr && conv_epilogue().res == nullptr && c.tm % 64 == 0;
    const size_t ost_bytes = ost ? size_t(p.epi2 ? 8 : 4) * (pooled ? 1024 : 4096) : 0;
    if (fixed + statics + p.wres_bytes + ost_bytes + 2 * size_t(p.stage_bytes) > kSSmemCap) return 0;
    int ns = int(std::min<size_t>(16, (kSSmemCap - fixed - statics - p.wres_bytes - ost_bytes) / p.stage_bytes));
    // row groups: the kernel re-cuts the ring into stages of the longest range actually used
    p.ring_bytes = int(kSSmemCap - fixed - statics - p.wres_bytes) & ~1023;
    if (opts().stages > 0) ns = std::max(2, std::min(ns, int(opts().stages)));
    if (ns < 2 || size_t(ns) * p.stage_bytes < staging) return 0;
    p.ns = ns;
    p.debug = DBG(opts().debug);
    p.slot = -1;
    pl->p = p;
    pl->smem = (rg ? fixed + size_t(p.ring_bytes) : fixed + size_t(ns) * p.stage_bytes) + p.wres_bytes;
    if (ost) {  // after the ring (1024-aligned: stages and the W block are multiples of 1 KB)
        p.ostage = 1;
        p.ostage_off = int(1024 + p.wres_bytes + size_t(ns) * p.stage_bytes);
        pl->p.ostage = 1;
        pl->p.ostage_off = p.ostage_off;
        pl->smem += ost_bytes;
    }
    pl->grid = grid;
    pl->rg = rg;
    pl->halo = halo;
    pl->eff = c;
    return 1;
}

using StreamKernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, IMaps, SParams, void *);

template <bool OB>
StreamKernel pick_kernel(bool rg, bool conv, int bm, bool halo) {
    if (rg) return stream_kernel<OB, true, false, 16>;
    if (halo) return bm == 16 ? stream_kernel<OB, false, true, 16, true> : bm == 8 ? stream_kernel<OB, false, true, 8, true>
                                                                             : stream_kernel<OB, false, true, 4, true>;
    if (conv) return bm == 16 ? stream_kernel<OB, false, true, 16> : bm == 8 ? stream_kernel<OB, false, true, 8>
                                                                             : stream_kernel<OB, false, true, 4>;
    return bm == 16 ? stream_kernel<OB, false, false, 16> : bm == 8 ? stream_kernel<OB, false, false, 8>
                                                                    : stream_kernel<OB, false, false, 4>;
}

// the residual epilogue (bf16 conv only): its own instantiations, so the other convs keep their
// register allocation (the runtime-flag version spilled and cost VGG19 19.3 -> 25.3 ms)
StreamKernel pick_res_kernel(int bm, bool halo) {
    if (halo) return bm == 16 ? stream_kernel<true, false, true, 16, true, true>
                              : bm == 8 ? stream_kernel<true, false, true, 8, true, true>
                                        : stream_kernel<true, false, true, 4, true, true>;
    return bm == 16 ? stream_kernel<true, false, true, 16, false, true>
                    : bm == 8 ? stream_kernel<true, false, true, 8, false, true> : stream_kernel<true, false, true, 4, false, true>;
}

// the whole-tile W map: slice-relayout rows of 16 k (32 B), box = one step's nsl x mma_n rows
int encode_slice_w(CUtensorMap *wmap, const ChainDims &c, const SParams &p, const void *vals) {
    auto enc = encode_fn();
    cuuint64_t wdims[2] = {16, cuuint64_t(c.u_o) * c.d_o * p.w_rows};
    cuuint64_t wstrides[1] = {32};
    cuuint32_t wbox[2] = {16, cuuint32_t(std::min(p.w_rows, 256))};
    cuuint32_t e2[2] = {1, 1};
    CUresult r = enc(wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(vals), wdims, wstrides, wbox, e2,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled(K5 W) failed (%d)", int(r));
        return RBGP4_ECUDA;
    }
    return RBGP4_OK;
}

// (cols table, relayout values) of the whole-tile path: K4's relayout for TC16, else the slices
void whole_tile_views(const ChainDims &c, const void *k4, const void *k5, const int32_t **cols, const void **vals) {
    ChainDims e;
    SliceDims sd;
    if (k5_mode(c, &e, &sd) == 1) {
        gather_prep_views(c, k4, cols, vals);
        return;
    }
    const SliceLayout l = slice_layout(e, sd);
    *cols = static_cast<const int32_t *>(k5) + l.cols;
    *vals = static_cast<const char *>(k5) + l.vals;
}

int launch_planned(SPlan &pl, int oelt, bool conv, int bm, const CUtensorMap &imap, const CUtensorMap &wmap,
                   const CUtensorMap &omap, const IMaps &imaps, void *out, cudaStream_t stream) {
    StreamKernel kern = (conv && (pl.p.relu & 4)) ? pick_res_kernel(bm, pl.halo)
                      : oelt == 2 ? pick_kernel<true>(pl.rg, conv, bm, pl.halo) : pick_kernel<false>(pl.rg, conv, bm, pl.halo);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(K5): %s", cudaGetErrorString(e));
        (void)cudaGetLastError();
        return RBGP4_ECUDA;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(pl.grid);
    cfg.blockDim = dim3(kSThreads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = opts().pdl ? 1 : 0;
    if (!conv) note_kernel(pl.rg ? "K5 rows" : "K5 stream");
    else if (pl.halo) note_kernel((pl.p.relu & 2) ? "K5 halo+pool" : (pl.p.relu & 4) ? "K5 halo+res" : "K5 halo");
    e = cudaLaunchKernelEx(&cfg, kern, imap, wmap, omap, imaps, pl.p, out);
    if (e != cudaSuccess) {
        set_error("stream_kernel launch (%u CTAs, smem %zu): %s", pl.grid, pl.smem, cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    RBGP4_CHECK_LAUNCH("stream_kernel launch");
    return RBGP4_OK;
}
}  // namespace

int stream_supported(const ChainDims &c, int out_dtype) {
    SPlan pl;
    return stream_plan(c, out_dtype, false, &pl);
}

int launch_stream(const ChainDims &c, int out_dtype, const void *k4, const void *k5, const void *inp, void *out,
                  cudaStream_t stream) {
    SPlan pl;
    if (!stream_plan(c, out_dtype, false, &pl) || k5 == nullptr || (stream_shape_ok(c) && k4 == nullptr))
        return RBGP4_EUNSUPPORTED;
    const ChainDims &e = pl.eff;
    if (c.n_cols == 0) return RBGP4_OK;
    const int oelt = out_dtype == RBGP4_BF16 ? 2 : 4;
    const int32_t *cols;
    const void *rvals;
    whole_tile_views(c, k4, k5, &cols, &rvals);
    SParams &p = pl.p;
    static int launch_seq = 0;  // debug builds: launch slots for tools/step_timeline.py
    if (p.debug & 2048) p.slot = launch_seq++ & 15;
    p.cols = cols;
    p.steps = static_cast<const int32_t *>(k5);
    p.rg = p.steps + a16w(size_t(c.u_o) * c.d_o) + rg_offset_words(pl.rg ? p.g : 1);
    const void *rgvals = static_cast<const char *>(k5) + 4 * tables_words(c);
    RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(inp) % 16 == 0 && (c.ld_in * 2) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(out) % 16 == 0 && (c.ld_out * oelt) % 16 == 0,
                  "K5 needs 16-byte aligned I / O rows");
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    CUtensorMap imap, wmap, omap;
    IMaps imaps;
    memset(&imaps, 0, sizeof(imaps));
    // I as (64 cols, K rows, N/64 atoms): a whole slab (tk rows) per box; row groups: one map
    // per column-block range length L (16 L rows per box)
    for (int len = pl.rg ? 1 : 8; len <= 8; ++len) {
        cuuint64_t dims[3] = {64, cuuint64_t(c.cols), cuuint64_t(c.n_cols / 64)};
        cuuint64_t strides[2] = {cuuint64_t(c.ld_in) * 2, 128};
        cuuint32_t box[3] = {64, cuuint32_t(pl.rg ? 16 * len : c.tk), 2};
        cuuint32_t e3[3] = {1, 1, 1};
        CUtensorMap *m = pl.rg ? &imaps.m[len - 1] : &imap;
        CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(inp), dims, strides, box,
                         e3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(K5 I) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    if (pl.rg) imap = imaps.m[7];
    if (pl.rg) {
        // row-permuted values as (d_t slots, tm rows, u_o * d_o tiles (tbm, j)); box = a
        // group's G*16 rows of all d_o tiles of its tile-row: the unit's whole W, one load
        cuuint64_t d3[3] = {cuuint64_t(c.d_t), cuuint64_t(c.tm), cuuint64_t(c.u_o) * c.d_o};
        cuuint64_t s3[2] = {cuuint64_t(c.d_t) * 2, cuuint64_t(c.tm) * c.d_t * 2};
        cuuint32_t b3[3] = {cuuint32_t(c.d_t), cuuint32_t(pl.p.g * 16), cuuint32_t(c.d_o)};
        cuuint32_t e3[3] = {1, 1, 1};
        CUresult r = enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(rgvals), d3, s3, b3, e3,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,  // d_t = 32: 64-byte rows
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(K5 W) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    } else if (int rc = encode_slice_w(&wmap, e, p, rvals)) {
        return rc;
    }
    {
        // O (n_cols, rows) row-major; box = one epilogue warp's 32 columns x (16 | tm/2) rows
        cuuint64_t odims[2] = {cuuint64_t(c.n_cols), cuuint64_t(c.rows)};
        cuuint64_t ostrides[1] = {cuuint64_t(c.ld_out) * oelt};
        cuuint32_t obox[2] = {32, cuuint32_t(pl.rg ? 16 : e.tm / 2)};
        cuuint32_t e2[2] = {1, 1};
        CUresult r = enc(&omap, oelt == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out,
                         odims, ostrides, obox, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         oelt == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(K5 O) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    return launch_planned(pl, oelt, false, c.bm, imap, wmap, omap, imaps, out, stream);
}

// Implicit-im2col convolution on K5 (whole tiles): a unit = 128 output pixels (whole output
// rows of one image, or whole images) x one tile-row of output channels; the I slab of a step
// is the tap-shifted NHWC box of those pixels (one 4-D TMA box per 64-channel atom, OOB =
// zero padding, element strides for stride 2), O is NHWC with ReLU fused.
namespace {
bool conv_tiles_ok(const ChainDims &c, const rbgp4_conv_desc *cv, int oelt) {
    const int oh = (cv->height + 2 * cv->pad - cv->kh) / cv->stride + 1;
    const int ow = (cv->width + 2 * cv->pad - cv->kw) / cv->stride + 1;
    const int64_t hw = int64_t(oh) * ow;
    const bool tiles = (kSBatch <= hw) ? (hw % kSBatch == 0 && kSBatch % ow == 0) : (kSBatch % hw == 0);
    const int th = kSBatch <= hw ? kSBatch / ow : oh;
    const int tb = kSBatch <= hw ? 1 : int(kSBatch / hw);
    return tiles && cv->c_in % 64 == 0 && cv->c_in % c.tk == 0 && (cv->stride == 1 || cv->stride == 2) &&
           ow * cv->stride <= 256 && th * cv->stride <= 256 && tb <= 256 && cv->kh == cv->kw &&
           c.n_cols % 32 == 0 && (int64_t(c.rows) * oelt) % 16 == 0;
}
}  // namespace

// the fused 2x2 pool needs whole windows inside a warp's 32 pixels: halo strips (rows ^8), or
// output maps of width 2..16 (a power of two; rows ^ow) with an even height
bool pool_ok(const SPlan &pl, const rbgp4_conv_desc *cv, int out_dtype) {
    if (!(cv->relu & 2)) return true;
    if (out_dtype != RBGP4_BF16) return false;
    const int oh = (cv->height + 2 * cv->pad - cv->kh) / cv->stride + 1;
    const int ow = (cv->width + 2 * cv->pad - cv->kw) / cv->stride + 1;
    if (oh % 2 || ow % 2) return false;
    return pl.halo || (ow <= 16 && (ow & (ow - 1)) == 0);
}

int stream_conv_supported(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype) {
    SPlan pl;
    const int oelt = out_dtype == RBGP4_BF16 ? 2 : 4;
    return cv != nullptr && stream_plan(c, out_dtype, true, &pl, cv) && (pl.halo || conv_tiles_ok(c, cv, oelt)) &&
           pool_ok(pl, cv, out_dtype);
}

int launch_stream_conv(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, const void *k4, const void *k5,
                       const void *x, void *out, cudaStream_t stream) {
    SPlan pl;
    const int oelt = out_dtype == RBGP4_BF16 ? 2 : 4;
    if (!stream_plan(c, out_dtype, true, &pl, cv) || !(pl.halo || conv_tiles_ok(c, cv, oelt)) ||
        !pool_ok(pl, cv, out_dtype) || k5 == nullptr ||
        (stream_shape_ok(c) && k4 == nullptr))
        return RBGP4_EUNSUPPORTED;
    if (c.n_cols == 0) return RBGP4_OK;
    const int32_t *cols;
    const void *rvals;
    whole_tile_views(c, k4, k5, &cols, &rvals);
    SParams &p = pl.p;
    p.cols = cols;
    p.steps = static_cast<const int32_t *>(k5);
    p.rg = nullptr;
    p.ld_out = int64_t(c.rows);  // NHWC: a pixel row holds c_out channels
    note_kernel((cv->relu & 2) ? "K5 conv+pool" : "K5 conv");
    const int oh = (cv->height + 2 * cv->pad - cv->kh) / cv->stride + 1;
    const int ow = (cv->width + 2 * cv->pad - cv->kw) / cv->stride + 1;
    p.c_in = cv->c_in;
    p.img_h = oh;
    p.img_w = ow;
    p.kw = cv->kw;
    p.pad = cv->pad;
    p.stride = cv->stride;
    p.relu = cv->relu;
    RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0,
                  "conv input / output must be 16-byte aligned");
    const ConvEpilogue &ep = conv_epilogue();
    if (ep.res != nullptr) {
        RBGP4_REQUIRE(!(cv->relu & 3), "the residual epilogue adds before any ReLU / pool (conv->relu must be 0)");
        if (out_dtype != RBGP4_BF16) {
            set_error("rbgp4_conv2d_residual: the residual epilogue writes bf16 (this output: add separately)");
            return RBGP4_EUNSUPPORTED;
        }
        RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(ep.res) % 16 == 0 &&
                          reinterpret_cast<uintptr_t>(ep.out2) % 16 == 0,
                      "residual / relu output must be 16-byte aligned");
        p.res = ep.res;
        p.out2 = ep.out2;
        p.relu |= 4 | (ep.out2 != nullptr ? 8 : 0);
        note_kernel("K5 conv+res");  // (launch_planned names the halo variant)
    }
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    const int64_t hw = int64_t(oh) * ow;
    const int th = kSBatch <= hw ? int(kSBatch / ow) : oh;
    const int tb = kSBatch <= hw ? 1 : int(kSBatch / hw);
    CUtensorMap imap, wmap, omap;
    memset(&omap, 0, sizeof(omap));
    IMaps imaps;
    memset(&imaps, 0, sizeof(imaps));
    {
        const cuuint32_t sd = cuuint32_t(cv->stride);
        cuuint32_t estr[4] = {1, sd, sd, 1};  // strided conv: every stride-th input pixel
        const int64_t ihw = int64_t(cv->height) * cv->width;
        cuuint64_t dims[4] = {cuuint64_t(cv->c_in), cuuint64_t(cv->width), cuuint64_t(cv->height),
                              cuuint64_t(cv->batch)};
        cuuint64_t strides[3] = {cuuint64_t(cv->c_in) * 2, cuuint64_t(cv->width) * cv->c_in * 2,
                                 cuuint64_t(ihw) * cv->c_in * 2};
        cuuint32_t box[4] = {64, cuuint32_t(ow) * sd, cuuint32_t(th) * sd, cuuint32_t(tb)};
        if (pl.halo) {  // the 18 x 10 halo of a 16 x 8 output strip
            box[1] = 10;
            box[2] = 18;
            box[3] = 1;
        }
        CUresult r = enc(&imap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(x), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(K5 conv input) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    if (int rc = encode_slice_w(&wmap, pl.eff, p, rvals)) return rc;
    if (p.ostage) {
        // the output for the staged epilogue: NHWC as (channels, pixels) -- box 64 x 32 -- or, for
        // halo strips, (channels, x, batch * rows) -- box 64 x 8 x 4; 128B swizzle like the staging
        // (pooled: the (H/2, W/2) output -- box 64 x 8 pooled pixels, or 64 x 4 x 2 for halo strips)
        const bool pooled = (cv->relu & 2) != 0;
        const cuuint64_t cb = cuuint64_t(c.rows) * 2;
        cuuint64_t dims[3] = {cuuint64_t(c.rows), cuuint64_t(pooled ? c.n_cols / 4 : c.n_cols), 1};
        cuuint64_t strides[2] = {cb, 0};
        cuuint32_t box[3] = {64, pooled ? 8u : 32u, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        cuuint32_t rank = 2;
        if (pl.halo) {
            dims[1] = cuuint64_t(pooled ? ow / 2 : ow);
            dims[2] = cuuint64_t(cv->batch) * (pooled ? oh / 2 : oh);
            strides[1] = cuuint64_t(pooled ? ow / 2 : ow) * cb;
            box[1] = pooled ? 4 : 8;
            box[2] = pooled ? 2 : 4;
            rank = 3;
        }
        CUresult r = enc(&omap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, out, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(K5 conv output) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    return launch_planned(pl, oelt, true, c.bm, imap, wmap, omap, imaps, out, stream);
}

}  // namespace rbgp4

#if RBGP4_DEBUG
// debug builds only (not part of include/rbgp4.h): K5 per-CTA stamps, CTA-0 marks and trace
extern "C" int rbgp4_debug_k5(unsigned long long *stamps, int n, unsigned long long *marks) {
    if (n > 2 * rbgp4::kK5Stamps) n = 2 * rbgp4::kK5Stamps;
    if (cudaMemcpyFromSymbol(stamps, rbgp4::g_k5_stamp, sizeof(unsigned long long) * n) != cudaSuccess) return -3;
    return cudaMemcpyFromSymbol(marks, rbgp4::g_k5_mark, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : -3;
}
extern "C" int rbgp4_debug_k5_seq(unsigned long long *stamps, unsigned long long *marks) {
    if (cudaMemcpyFromSymbol(stamps, rbgp4::g_k5_seq, sizeof(unsigned long long) * 16 * 3 * 160) != cudaSuccess)
        return -3;
    return cudaMemcpyFromSymbol(marks, rbgp4::g_k5_smark, sizeof(unsigned long long) * 64) == cudaSuccess ? 0 : -3;
}
extern "C" int rbgp4_debug_k5_trace(unsigned long long *host) {
    if (cudaMemcpyFromSymbol(host, rbgp4::g_k5_trace, sizeof(unsigned long long) * 192) != cudaSuccess) return -3;
    return cudaMemcpyFromSymbol(host + 192, rbgp4::g_k5_epi, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : -3;
}
#endif  // RBGP4_DEBUG
