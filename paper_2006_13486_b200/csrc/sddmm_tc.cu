// sddmm_tc.cu -- K7: the training direction's weight gradient on the tensor cores (bf16 operands,
// fp32 accumulation), restricted to the RBGP4 pattern (the paper trains with
// fixed masks):
//
//     dW[u, j] = sum_n dO[u, n] * I[c(u, j), n]      for every stored slot j of row u
//
// One CTA per nonzero W tile (tile-row tbm, adjacency slot j of g_o, K-block adj_o[tbm][j]):
//     D (tm x tk) = dO[tbm*tm .., :] x I[K-block rows, :]^T       (K of the MMA = the batch N)
// on tcgen05 -- M = 128 W rows, N = 128 K-block rows, one 64-column batch chunk per ring stage
// (both operands K-major as they lie in memory: rows contiguous along N, TMA 128B swizzle), D in
// TMEM.  The epilogue keeps only the g_i (x) g_b pattern: row u (TMEM lane) of row block ui reads
// D columns [adj_i[ui][ink] * bk, + bk) per neighbour ink -- slots ink*bk + k of step j in the
// (rows, row_nnz) layout of RcubsMatrix.values, so the gradient never leaves the succinct format.
// (The dense tile costs 1/(1 - sp_i) of the pattern's MACs, on tensor cores the cheapest way to
// reduce over a long N.)  Deterministic: each slot is one fixed-order MMA accumulation.
//
// Warps (192 threads): 0-3 epilogue (TMEM lane quarter = warp), 4 TMA producer, 5 MMA issue.
#include "common.cuh"
#include "tc_ptx.cuh"

namespace rbgp4 {
namespace {

constexpr int kTThreads = 192;
constexpr int kChunk = 64;                          // batch columns per stage (128-byte rows)
constexpr int kHalf = 128 * kChunk * 2;             // one operand tile per stage (16 KB)
constexpr int kStage = 2 * kHalf;

struct TParams {
    int64_t n_cols, row_nnz;
    int32_t d_o, tm, tk, u_i, d_i, bm, bk, d_t, ns, n_chunks;
    int32_t split;  // 2: two CTAs per tile, each half of the batch chunks, added into a zeroed grad
    int32_t nmajor; // operands batch-major, dO^T (N x rows) and I^T (N x cols): MN-major MMA operands
};

template <int BK>
__global__ void __launch_bounds__(kTThreads, 1)
sddmm_tc_kernel(const __grid_constant__ CUtensorMap dmap, const __grid_constant__ CUtensorMap imap,
                const TParams p, const int32_t *__restrict__ adj_o, const int32_t *__restrict__ adj_i,
                float *__restrict__ grad) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *full = reinterpret_cast<uint64_t *>(base);
    uint64_t *empty = full + 16;
    uint64_t *acc_full = empty + 16;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_full + 1);
    unsigned char *ring = base + 1024;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int tile = int(blockIdx.x / p.split), half = int(blockIdx.x % p.split);
    const int tbm = tile / p.d_o, j = tile % p.d_o;
    // this CTA's batch chunks [c_lo, c_hi)
    const int c_lo = p.split == 1 ? 0 : (half == 0 ? 0 : p.n_chunks / 2);
    const int c_hi = p.split == 1 ? p.n_chunks : (half == 0 ? p.n_chunks / 2 : p.n_chunks);
    const int n_my = c_hi - c_lo;
    const int kblk = __ldg(adj_o + int64_t(tbm) * p.d_o + j);
    if (warp == 4) {
        if (lane == 0) {
            for (int i = 0; i < p.ns; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
            mbar_init(acc_full, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        asm volatile("barrier.sync 1, %0;" ::"n"(kTThreads) : "memory");
        for (int c = 0; c < n_my; ++c) {
            const int st = c % p.ns;
            if (c >= p.ns) mbar_wait(&empty[st], uint32_t((c / p.ns - 1) & 1));
            if (elect_one()) {
                mbar_expect_tx(&full[st], uint32_t(kStage));
                if (p.nmajor) {
                    // [64-row atom][64 batch rows][64 rows x 2 B]: 3-D boxes (64, 64 batch, 2 atoms)
                    tma_load_3d(ring + size_t(st) * kStage, &dmap, &full[st], 0, (c_lo + c) * kChunk, tbm * p.tm / 64);
                    tma_load_3d(ring + size_t(st) * kStage + kHalf, &imap, &full[st], 0, (c_lo + c) * kChunk,
                                kblk * p.tk / 64);
                } else {
                    tma_load_2d(ring + size_t(st) * kStage, &dmap, &full[st], (c_lo + c) * kChunk, tbm * p.tm);
                    tma_load_2d(ring + size_t(st) * kStage + kHalf, &imap, &full[st], (c_lo + c) * kChunk,
                                kblk * p.tk);
                }
            }
            __syncwarp();
        }
    } else if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(128u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        tc_fence_before();
        asm volatile("barrier.sync 1, %0;" ::"n"(kTThreads) : "memory");
        tc_fence_after();
        const uint32_t tmem_d = *tmem_slot;
        // D f32, A / B bf16, both K-major (rows contiguous along the batch) or both MN-major
        // (batch-major operands: 64-row atoms 8 KB apart = LBO, 8-batch-row groups 1 KB apart),
        // N = 128, M = 128
        const uint32_t mn = p.nmajor ? 1u : 0u;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (mn << 15) | (mn << 16) |
                               ((128u >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t lbo = p.nmajor ? uint32_t(kChunk * 128) : 0u;
        const uint64_t a0 = smem_desc(smem_u32(ring), lbo, 1024, 2u);
        const uint64_t b0 = smem_desc(smem_u32(ring) + kHalf, lbo, 1024, 2u);
        // the next K16 of the batch: 32 bytes along K-major rows, 16 rows of 128 B in MN-major atoms
        const uint32_t kstep = p.nmajor ? uint32_t(16 * 128) >> 4 : 2u;
        for (int c = 0; c < n_my; ++c) {
            const int st = c % p.ns;
            mbar_wait(&full[st], uint32_t((c / p.ns) & 1));
            tc_fence_after();
            if (elect_one()) {
                const uint32_t off = uint32_t(st * kStage) >> 4;
#pragma unroll
                for (int k = 0; k < kChunk / 16; ++k)  // 32 bytes of the 128-byte rows per K16
                    tc_mma<false>(tmem_d, a0 + off + uint32_t(k) * kstep, b0 + off + uint32_t(k) * kstep, idesc,
                                  (c > 0 || k > 0) ? 1u : 0u);
                tc_commit(&empty[st]);
                if (c == n_my - 1) tc_commit(acc_full);
            }
            __syncwarp();
        }
    } else {
        asm volatile("barrier.sync 1, %0;" ::"n"(kTThreads) : "memory");
        mbar_wait_parked(acc_full, 0u);
        tc_fence_after();
        const uint32_t lane_base = *tmem_slot + (uint32_t(warp * 32) << 16);
        const int r = warp * 32 + lane;        // W row inside the tile (TMEM lane)
        float *grow = grad + (int64_t(tbm) * p.tm + r) * p.row_nnz + int64_t(j) * p.d_t;
        // every row block of this warp's 32 rows: its d_i neighbours' D columns (warp-uniform
        // TMEM addresses; lanes of other row blocks discard the load)
        for (int rb = (warp * 32) / p.bm; rb < (warp * 32 + 32) / p.bm; ++rb) {
            const bool mine = r / p.bm == rb;
            for (int ink = 0; ink < p.d_i; ++ink) {
                const uint32_t col = uint32_t(__ldg(adj_i + rb * p.d_i + ink) * BK);
                uint32_t v[BK];
                if constexpr (BK == 16) TMEM_LD_32x32b_X16(lane_base + col, v);
                else if constexpr (BK == 8) TMEM_LD_32x32b_X8(lane_base + col, v);
                else TMEM_LD_32x32b_X4(lane_base + col, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (mine && p.split == 1) {
                    float4 *g = reinterpret_cast<float4 *>(grow + ink * BK);
#pragma unroll
                    for (int q = 0; q < BK / 4; ++q)
                        g[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                           __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
                } else if (mine) {
                    // two halves into a zeroed gradient: 0 + a + b == 0 + b + a exactly (fp32 addition
                    // commutes), so the result is deterministic whichever half lands first
#pragma unroll
                    for (int q = 0; q < BK; ++q) atomicAdd(grow + ink * BK + q, __uint_as_float(v[q]));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(128u));
    }
}

}  // namespace

// 128 x 128 tiles of g_r = (1,1) chains whose blocks tile 32 TMEM lanes and 16-byte rows
int sddmm_tc_supported(const ChainDims &c) {
    return c.rm == 1 && c.rk == 1 && c.tm == 128 && c.tk == 128 && (c.bk == 4 || c.bk == 8 || c.bk == 16) &&
           c.bm <= 32 && 32 % c.bm == 0 && c.row_nnz % 4 == 0 && c.d_t % 4 == 0;
}

int launch_sddmm_tc(const ChainDims &c, const int32_t *adj_o, const int32_t *adj_i, const void *d_out,
                    int64_t ld_do, const void *inp, int64_t ld_in, float *grad, cudaStream_t stream, bool nmajor) {
    if (!sddmm_tc_supported(c)) {
        set_error("rbgp4_sddmm(bf16): the tensor-core gradient needs 128 x 128 tiles, g_r = (1,1), "
                  "bk in {4, 8, 16}, bm | 32");
        return RBGP4_EUNSUPPORTED;
    }
    RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(d_out) % 16 == 0 && reinterpret_cast<uintptr_t>(inp) % 16 == 0 &&
                      (ld_do * 2) % 16 == 0 && (ld_in * 2) % 16 == 0 && reinterpret_cast<uintptr_t>(grad) % 16 == 0,
                  "rbgp4_sddmm(bf16): 16-byte aligned operands and rows");
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    CUtensorMap dmap, imap;
    auto make = [&](CUtensorMap *m, const void *ptr, int64_t rows, int64_t ld) {
        if (nmajor) {  // (N x rows), row stride ld: (64 rows, N batch rows, rows / 64 atoms)
            cuuint64_t d3[3] = {64, cuuint64_t(c.n_cols), cuuint64_t(rows / 64)};
            cuuint64_t s3[2] = {cuuint64_t(ld) * 2, 128};
            cuuint32_t b3[3] = {64, kChunk, 2};
            cuuint32_t e3[3] = {1, 1, 1};
            return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(ptr), d3, s3, b3, e3,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        cuuint64_t dims[2] = {cuuint64_t(c.n_cols), cuuint64_t(rows)};
        cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
        cuuint32_t box[2] = {kChunk, 128};
        cuuint32_t e2[2] = {1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, e2,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    if (make(&dmap, d_out, c.rows, ld_do) != CUDA_SUCCESS || make(&imap, inp, c.cols, ld_in) != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled(sddmm) failed");
        return RBGP4_ECUDA;
    }
    TParams p{};
    p.n_cols = c.n_cols; p.row_nnz = c.row_nnz; p.d_o = c.d_o; p.tm = c.tm; p.tk = c.tk; p.u_i = c.u_i;
    p.d_i = c.d_i; p.bm = c.bm; p.bk = c.bk; p.d_t = c.d_t;
    p.nmajor = nmajor ? 1 : 0;
    p.n_chunks = int((c.n_cols + kChunk - 1) / kChunk);
    p.ns = 6;
    // fewer tiles than SMs: split each tile's batch over two CTAs (deterministic, see the epilogue)
    const int64_t tiles = int64_t(c.u_o) * c.d_o;
    p.split = (tiles <= kNumSMs && p.n_chunks >= 8) ? 2 : 1;
    const size_t smem = 1024 + 1024 + size_t(p.ns) * kStage;
    void (*kern)(CUtensorMap, CUtensorMap, TParams, const int32_t *, const int32_t *, float *) =
        c.bk == 16 ? sddmm_tc_kernel<16> : c.bk == 8 ? sddmm_tc_kernel<8> : sddmm_tc_kernel<4>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(sddmm_tc): %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    if (c.n_cols == 0) {
        // empty batch: the gradient is zero
        e = cudaMemsetAsync(grad, 0, size_t(c.rows) * c.row_nnz * 4, stream);
        return e == cudaSuccess ? RBGP4_OK : RBGP4_ECUDA;
    }
    if (p.split == 2) {
        e = cudaMemsetAsync(grad, 0, size_t(c.rows) * c.row_nnz * 4, stream);
        if (e != cudaSuccess) {
            set_error("sddmm_tc: zeroing the gradient: %s", cudaGetErrorString(e));
            return RBGP4_ECUDA;
        }
    }
    note_kernel("K7 sddmm");
    kern<<<unsigned(tiles * p.split), kTThreads, smem, stream>>>(dmap, imap, p, adj_o, adj_i, grad);
    RBGP4_CHECK_LAUNCH("sddmm_tc_kernel launch");
    return RBGP4_OK;
}

}  // namespace rbgp4
