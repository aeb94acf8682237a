// dense_conv.cu -- K8: the dense first convolution of the VGG19 model (SURVEY §8(f) row 2:
// the paper keeps conv1 dense), 3x3 'same', 3 input channels -> 64, ReLU, NHWC
// bf16 in and out, on tcgen05.
//
// The layer reads 6 B per pixel and writes 128 B per pixel (64 bf16 channels): at batch 32768
// that is 0.2 GB in and 4.3 GB out, an HBM-write-bound layer (~0.7 ms at the measured copy
// bandwidth) that cuDNN ran in 2.6-3.6 ms.  Implicit GEMM per 128-pixel tile:
//     D (128 pixels x 64) = A (128 x K32) * W^T (K32 x 64),  K = the 27 taps x channels + 5 zeros,
// A built by the threads (one pixel each: its 27 input values, gathered through L1 from the
// NHWC input, packed into one 64-byte K-major row, 64B swizzle), W resident in shared memory,
// D double-buffered in TMEM (the MMA of tile i+1 runs under the epilogue of tile i), the
// epilogue reading one pixel's 64 channels per lane (tcgen05.ld) and storing them as one
// contiguous 128-byte NHWC row with the ReLU fused -- into a 128B-swizzled shared-memory staging
// tile (conflict-free), from which each warp's 32 pixels (4 KB, contiguous in NHWC) leave as ONE
// TMA store: 16-byte stores straight from the lanes touched 32 lines per instruction (1.94 ms), a
// linear staging tile with a lane-rotated chunk order and a plain bulk copy still had 2-way bank
// conflicts (1.06 ms); swizzled + TMA store: 0.83 ms, 0.82 of the HBM floor.  The next tile's input loads are issued before the
// epilogue, so their latency hides under it.  Four CTAs per SM.
#include "common.cuh"
#include "tc_ptx.cuh"

namespace rbgp4 {
namespace {

constexpr int kC3Out = 64;                // output channels (the VGG19 / CIFAR conv1)
constexpr int kC3Pix = 128;               // MMA M: pixels per tile
constexpr int kC3Row = 64;                // bytes per K-major row (32 bf16: 27 used)
constexpr int kC3OutRow = kC3Out * 2;     // bytes of one output pixel (NHWC)

__global__ void __launch_bounds__(kC3Pix, 4)
dense_c3_kernel(const __grid_constant__ CUtensorMap omap, const __nv_bfloat16 *__restrict__ x,
                const __nv_bfloat16 *__restrict__ w,
                __nv_bfloat16 *__restrict__ out, int height, int width, int64_t npix) {
    __shared__ __align__(1024) unsigned char s_a[2][kC3Pix * kC3Row];
    __shared__ __align__(1024) unsigned char s_b[kC3Out * kC3Row];
    __shared__ uint64_t done[2];
    __shared__ uint32_t tmem_slot;
    extern __shared__ __align__(128) unsigned char s_out[];  // [2][128 pixels][128 B] output staging
    // 1024-aligned (the 128B swizzle pattern repeats every 8 rows of 128 B)
    unsigned char *s_out1k = s_out + ((1024u - (smem_u32(s_out) & 1023u)) & 1023u);
    const int tid = threadIdx.x, warp = tid / 32;
    // W: [64 rows][32 bf16] as given (k = (ti * 3 + tj) * 3 + c, zero-padded), 64B swizzle
    for (int i = tid; i < kC3Out * 4; i += kC3Pix) {
        const uint4 v = reinterpret_cast<const uint4 *>(w)[i];
        sts128(smem_u32(s_b) + swz(uint32_t(i) * 16u, 64), v.x, v.y, v.z, v.w);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                     "r"(uint32_t(2 * kC3Out)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&done[0], 1);
        mbar_init(&done[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    // D f32, A / B bf16, both K-major, N = 64, M = 128
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kC3Out >> 3) << 17) |
                           (uint32_t(kC3Pix >> 4) << 24);
    const uint64_t b_desc = smem_desc(smem_u32(s_b), 0, 8 * kC3Row, swizzle_layout_code(kC3Row));
    const int64_t hw = int64_t(height) * width;
    const int64_t ntiles = (npix + kC3Pix - 1) / kC3Pix;

    // this thread's pixel of a tile: its 27 input values (OOB taps and pixels = 0)
    uint16_t v[27];
    auto gather = [&](int64_t tile) {
        const int64_t pix = tile * kC3Pix + tid;
        int64_t n = 0;
        int y = 0, xx = 0;
        const bool in = pix < npix;
        if (in) {
            n = pix / hw;
            const int rem = int(pix - n * hw);
            y = rem / width;
            xx = rem - y * width;
        }
        const uint16_t *xs = reinterpret_cast<const uint16_t *>(x);
#pragma unroll
        for (int ti = 0; ti < 3; ++ti)
#pragma unroll
            for (int tj = 0; tj < 3; ++tj) {
                const int yy = y + ti - 1, xc = xx + tj - 1;
                const bool ok = in && yy >= 0 && yy < height && xc >= 0 && xc < width;
                const uint16_t *src = xs + ((n * height + yy) * width + xc) * 3;
#pragma unroll
                for (int c = 0; c < 3; ++c) v[(ti * 3 + tj) * 3 + c] = ok ? __ldg(src + c) : uint16_t(0);
            }
    };
    const int lane = tid % 32;
    auto epilogue = [&](int64_t tile, int64_t it_e) {
        const int b = int(it_e & 1);
        mbar_wait(&done[b], uint32_t((it_e >> 1) & 1));
        tc_fence_after();
        const int64_t wpix0 = tile * kC3Pix + warp * 32;  // this warp's first pixel
        // staging buffer b of this warp: 32 pixel rows of 128 B; its previous bulk store (tile
        // it_e - 2) must have finished reading it
        unsigned char *stg = s_out1k + size_t(b) * kC3Pix * kC3OutRow + size_t(warp) * 32 * kC3OutRow;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16) + uint32_t(b * kC3Out);
        const uint32_t srow = smem_u32(stg) + uint32_t(lane) * kC3OutRow;
        uint32_t r[32];
#pragma unroll
        for (int h = 0; h < kC3Out / 32; ++h) {
            TMEM_LD_32x32b_X32(taddr + uint32_t(h * 32), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            uint32_t o[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const __nv_bfloat162 p2 = __floats2bfloat162_rn(fmaxf(__uint_as_float(r[2 * k]), 0.0f),
                                                                 fmaxf(__uint_as_float(r[2 * k + 1]), 0.0f));
                o[k] = *reinterpret_cast<const uint32_t *>(&p2);
            }
            // chunk (h * 4 + k) of this pixel's 128-byte row, 128B swizzle (chunk ^ row % 8): the 8
            // lanes of a wavefront hit 8 different bank quads; the TMA store undoes the swizzle
#pragma unroll
            for (int k = 0; k < 4; ++k)
                sts128(srow + (uint32_t((h * 4 + k) ^ (lane & 7)) << 4), o[4 * k], o[4 * k + 1], o[4 * k + 2],
                       o[4 * k + 3]);
        }
        tc_fence_before();
        fence_async_smem();
        __syncwarp();
        if (lane == 0 && wpix0 < npix) {  // box 64 channels x 32 pixels, clipped at npix
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&omap)), "r"(0), "r"(int32_t(wpix0)), "r"(smem_u32(stg))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    };

    int64_t it = 0;
    const int64_t first = blockIdx.x;
    if (first < ntiles) gather(first);
    for (int64_t tile = first; tile < ntiles; tile += gridDim.x, ++it) {
        const int b = int(it & 1);
        // A row of this pixel: 27 values + 5 zeros, 16 packed words, 64B-swizzled K-major row.
        // Buffer b was last read by the MMA of tile it-2, whose commit the epilogue of it-2
        // (previous iteration) waited for.
        uint32_t wd[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t lo = 2 * k < 27 ? v[2 * k] : 0u, hi = 2 * k + 1 < 27 ? v[2 * k + 1] : 0u;
            wd[k] = lo | (hi << 16);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
            sts128(smem_u32(s_a[b]) + swz(uint32_t(tid) * kC3Row + uint32_t(c) * 16u, 64), wd[4 * c], wd[4 * c + 1],
                   wd[4 * c + 2], wd[4 * c + 3]);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint64_t a_desc = smem_desc(smem_u32(s_a[b]), 0, 8 * kC3Row, swizzle_layout_code(kC3Row));
            // K = 32 as two K16 MMAs: the second starts 32 B into the swizzled rows
#pragma unroll
            for (int kb = 0; kb < 2; ++kb)
                tc_mma<false>(tmem + uint32_t(b * kC3Out), a_desc + uint64_t(kb * 2), b_desc + uint64_t(kb * 2), idesc,
                              uint32_t(kb));
            tc_commit(&done[b]);
        }
        // the next tile's input loads fly under this epilogue
        if (tile + gridDim.x < ntiles) gather(tile + gridDim.x);
        if (it > 0) epilogue(tile - gridDim.x, it - 1);
    }
    if (it > 0) epilogue(first + (it - 1) * gridDim.x, it - 1);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(uint32_t(2 * kC3Out)));
    }
}

}  // namespace
}  // namespace rbgp4

extern "C" int rbgp4_dense_conv3x3_c3(const void *x, const void *w, void *out, int batch, int height, int width,
                                      int c_out, void *stream) {
    using namespace rbgp4;
    RBGP4_REQUIRE(c_out == kC3Out, "dense_conv3x3_c3: 64 output channels");
    RBGP4_REQUIRE(batch >= 0 && height > 0 && width > 0, "dense_conv3x3_c3: bad sizes");
    RBGP4_REQUIRE(x && w && out, "null device pointer");
    RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(w) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(out) % 16 == 0,
                  "dense_conv3x3_c3: x / w / out must be 16-byte aligned");
    const int64_t npix = int64_t(batch) * height * width;
    if (npix == 0) return RBGP4_OK;
    const int64_t ntiles = (npix + kC3Pix - 1) / kC3Pix;
    const unsigned grid = unsigned(std::min<int64_t>(ntiles, int64_t(kNumSMs) * 4));
    note_kernel("K8 dense c3");
    // output staging, dynamic 33 KB: with the 20 KB static A / W buffers above the 48 KB default,
    // so the opt-in is set on every call (per device, cheap)
    const int smem = 2 * kC3Pix * kC3OutRow + 1024;
    cudaError_t e = cudaFuncSetAttribute(dense_c3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(dense_c3): %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    // the output as (64 channels, npix pixels): box 64 x 32 (a warp's pixels), 128B swizzle
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    CUtensorMap omap;
    {
        const cuuint64_t dims[2] = {cuuint64_t(kC3Out), cuuint64_t(npix)};
        const cuuint64_t strides[1] = {cuuint64_t(kC3OutRow)};
        const cuuint32_t box[2] = {cuuint32_t(kC3Out), 32};
        const cuuint32_t estr[2] = {1, 1};
        CUresult r = enc(&omap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(K8 output) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    dense_c3_kernel<<<grid, kC3Pix, smem, static_cast<cudaStream_t>(stream)>>>(omap, 
        static_cast<const __nv_bfloat16 *>(x), static_cast<const __nv_bfloat16 *>(w),
        static_cast<__nv_bfloat16 *>(out), height, width, npix);
    RBGP4_CHECK_LAUNCH("dense_c3_kernel launch");
    return RBGP4_OK;
}
