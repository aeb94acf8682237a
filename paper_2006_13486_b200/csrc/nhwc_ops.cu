// nhwc_ops.cu -- small NHWC helpers for the sparse-conv network path.
//
// rbgp4_maxpool2x2_nhwc: 2x2 / stride-2 max pooling of a bf16 NHWC tensor, one thread per
// 8 output channels (16-byte loads of the four input pixels).  Bandwidth-bound elementwise
// work; it sits between the conv stages of VGG19, whose ReLU is fused into the conv epilogue.
#include "common.cuh"

namespace rbgp4 {
namespace {

__global__ void maxpool2x2_nhwc_kernel(const __nv_bfloat16 *__restrict__ x, __nv_bfloat16 *__restrict__ y,
                                       int batch, int h, int w, int c) {
    const int oh = h / 2, ow = w / 2, cv = c / 8;
    const int64_t total = int64_t(batch) * oh * ow * cv;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int cc = int(i % cv);
        int64_t r = i / cv;
        const int ox = int(r % ow);
        r /= ow;
        const int oy = int(r % oh);
        const int b = int(r / oh);
        const __nv_bfloat16 *p = x + ((int64_t(b) * h + 2 * oy) * w + 2 * ox) * c + cc * 8;
        uint4 a = *reinterpret_cast<const uint4 *>(p);
        uint4 bq = *reinterpret_cast<const uint4 *>(p + c);
        uint4 cq = *reinterpret_cast<const uint4 *>(p + int64_t(w) * c);
        uint4 dq = *reinterpret_cast<const uint4 *>(p + int64_t(w) * c + c);
        const __nv_bfloat162 *pa = reinterpret_cast<const __nv_bfloat162 *>(&a);
        const __nv_bfloat162 *pb = reinterpret_cast<const __nv_bfloat162 *>(&bq);
        const __nv_bfloat162 *pc = reinterpret_cast<const __nv_bfloat162 *>(&cq);
        const __nv_bfloat162 *pd = reinterpret_cast<const __nv_bfloat162 *>(&dq);
        uint4 o;
        __nv_bfloat162 *po = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
        for (int k = 0; k < 4; ++k) po[k] = __hmax2(__hmax2(pa[k], pb[k]), __hmax2(pc[k], pd[k]));
        *reinterpret_cast<uint4 *>(y + ((int64_t(b) * oh + oy) * ow + ox) * c + cc * 8) = o;
    }
}

}  // namespace
}  // namespace rbgp4

extern "C" int rbgp4_maxpool2x2_nhwc(const void *x, void *y, int batch, int height, int width,
                                     int channels, void *stream) {
    using namespace rbgp4;
    RBGP4_REQUIRE(batch >= 0 && height % 2 == 0 && width % 2 == 0 && channels % 8 == 0,
                  "maxpool2x2: need even H/W and channels %% 8 == 0 (%d x %d x %d)", height, width,
                  channels);
    RBGP4_REQUIRE(reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0,
                  "maxpool2x2: 16-byte aligned tensors required");
    const int64_t total = int64_t(batch) * (height / 2) * (width / 2) * (channels / 8);
    if (total == 0) return RBGP4_OK;
    const int threads = 256;
    const int blocks = int(std::min<int64_t>((total + threads - 1) / threads, 148 * 32));
    maxpool2x2_nhwc_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16 *>(x), static_cast<__nv_bfloat16 *>(y), batch, height, width,
        channels);
    RBGP4_CHECK_LAUNCH("maxpool2x2_nhwc launch");
    return RBGP4_OK;
}

// ---------------------------------------------------------------- im2col / layout transposes
// For the layers the implicit-im2col conv does not take (the fp32 FFMA path of WRN-40-4 and its
// 16-channel bf16 layers): im2col of an NHWC tensor into the chain's tap-major (k*k*C, B*H'*W')
// operand in ONE pass (32 x 32 shared-memory transposes per tap: coalesced channel reads, coalesced
// pixel writes; OOB taps = the zero padding), and the (C, N) -> NHWC (N, C) transpose of the
// product's output with the ReLU fused.  (torch's pad / stack / permute / contiguous chain took
// ~3 ms per 64-channel 32x32 layer at batch 512; the product itself 0.42 ms.)
namespace rbgp4 {
namespace {

constexpr int kColPix = 128;  // output pixels per im2col block (32 channels x 128 pixels)

template <typename T>
__global__ void __launch_bounds__(256) im2col_nhwc_kernel(const T *__restrict__ x, T *__restrict__ cols, int b,
                                                          int h, int w, int c, int k, int stride, int oh, int ow) {
    __shared__ T tile[kColPix][33];
    const int64_t n_pix = int64_t(b) * oh * ow;
    const int tap = blockIdx.z, ti = tap / k, tj = tap % k, pad = (k - 1) / 2;
    const int64_t p0 = int64_t(blockIdx.x) * kColPix;  // first output pixel
    const int c0 = blockIdx.y * 32;                     // first channel
    const int ch = c0 + threadIdx.x;
    if (sizeof(T) == 4 && c % 4 == 0 && n_pix < (int64_t(1) << 31)) {
        // f32: 16-byte loads, 8 lanes x 4 channels per pixel, 4 pixels per warp instruction
        // (the scalar loop below was instruction-bound: 69 % issue, 2.8 TB/s)
        const int tid = threadIdx.y * 32 + threadIdx.x;
        const int cq = tid & 7, pr = tid >> 3;  // channel quad, pixel row (0..31)
        const int chq = c0 + 4 * cq;
        for (int r = pr; r < kColPix; r += 32) {
            const int pix = int(p0) + r;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (pix < n_pix && chq < c) {
                const int ox = pix % ow, t = pix / ow, oy = t % oh, bi = t / oh;
                const int iy = oy * stride + ti - pad, ix = ox * stride + tj - pad;
                if (iy >= 0 && iy < h && ix >= 0 && ix < w)
                    v = *reinterpret_cast<const float4 *>(x + ((int64_t(bi) * h + iy) * w + ix) * c + chq);
            }
            tile[r][4 * cq] = T(v.x);
            tile[r][4 * cq + 1] = T(v.y);
            tile[r][4 * cq + 2] = T(v.z);
            tile[r][4 * cq + 3] = T(v.w);
        }
    } else {
    // read: kColPix pixels x 32 channels, lanes along channels (coalesced NHWC rows); the
    // pixel coordinates are decomposed once and stepped (64-bit divisions per element made
    // this kernel integer-bound)
    int64_t pix = p0 + threadIdx.y;
    int ox = int(pix % ow), oy, bi;
    {
        const int64_t t = pix / ow;
        oy = int(t % oh);
        bi = int(t / oh);
    }
    for (int r = threadIdx.y; r < kColPix; r += blockDim.y) {
        T v = T(0.0f);
        if (pix < n_pix && ch < c) {
            const int iy = oy * stride + ti - pad, ix = ox * stride + tj - pad;
            if (iy >= 0 && iy < h && ix >= 0 && ix < w) v = x[((int64_t(bi) * h + iy) * w + ix) * c + ch];
        }
        tile[r][threadIdx.x] = v;
        pix += blockDim.y;
        ox += blockDim.y;
        while (ox >= ow) {
            ox -= ow;
            if (++oy == oh) { oy = 0; ++bi; }
        }
    }
    }
    __syncthreads();
    // write: 32 channel rows x kColPix pixels, each lane 4 consecutive pixels (one row of cols
    // per warp instruction when the rows are 16-byte aligned)
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int chr = c0 + r;
        if (chr >= c) break;
        T *dst = cols + (int64_t(tap) * c + chr) * n_pix + p0;
#pragma unroll
        for (int half = 0; half < kColPix / 128; ++half) {
            const int px = half * 128 + threadIdx.x * 4;
            if (sizeof(T) == 4 && n_pix % 4 == 0 && p0 + px + 3 < n_pix) {
                float4 v;
                v.x = float(tile[px][r]); v.y = float(tile[px + 1][r]); v.z = float(tile[px + 2][r]); v.w = float(tile[px + 3][r]);
                *reinterpret_cast<float4 *>(dst + px) = v;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (p0 + px + j < n_pix) dst[px + j] = tile[px + j][r];
            }
        }
    }
}

template <typename T>
__global__ void nc_to_nhwc_kernel(const T *__restrict__ src, T *__restrict__ dst, int rows, int64_t n, int relu,
                                  const T *__restrict__ res, T *__restrict__ dst_relu) {
    __shared__ T tile[32][33];
    const int64_t n0 = int64_t(blockIdx.x) * 32;
    const int r0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int row = r0 + r;
        const int64_t col = n0 + threadIdx.x;
        T v = T(0.0f);
        if (row < rows && col < n) v = src[int64_t(row) * n + col];
        tile[r][threadIdx.x] = v;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t col = n0 + r;
        const int row = r0 + threadIdx.x;
        if (row < rows && col < n) {
            T v = tile[threadIdx.x][r];
            if (relu && float(v) < 0.0f) v = T(0.0f);
            // residual (the WRN block tail): v + R rounded like the unfused add; relu copy
            if (res != nullptr) v = T(float(v) + float(res[col * rows + row]));
            dst[col * rows + row] = v;
            if (dst_relu != nullptr) dst_relu[col * rows + row] = float(v) < 0.0f ? T(0.0f) : v;
        }
    }
}

}  // namespace
}  // namespace rbgp4

extern "C" int rbgp4_im2col_nhwc(int dtype, const void *x, void *cols, int batch, int height, int width,
                                 int channels, int k, int stride, void *stream) {
    using namespace rbgp4;
    RBGP4_REQUIRE(dtype == RBGP4_F32 || dtype == RBGP4_BF16, "im2col: F32 or BF16");
    RBGP4_REQUIRE(batch >= 0 && height > 0 && width > 0 && channels > 0 && k % 2 == 1 && (stride == 1 || stride == 2),
                  "im2col: bad geometry");
    const int pad = (k - 1) / 2;
    const int oh = (height + 2 * pad - k) / stride + 1, ow = (width + 2 * pad - k) / stride + 1;
    const int64_t n_pix = int64_t(batch) * oh * ow;
    if (n_pix == 0) return RBGP4_OK;
    dim3 grid(unsigned((n_pix + kColPix - 1) / kColPix), unsigned((channels + 31) / 32), unsigned(k * k));
    dim3 block(32, 8);
    auto s = static_cast<cudaStream_t>(stream);
    if (dtype == RBGP4_F32)
        im2col_nhwc_kernel<float><<<grid, block, 0, s>>>(static_cast<const float *>(x), static_cast<float *>(cols),
                                                         batch, height, width, channels, k, stride, oh, ow);
    else
        im2col_nhwc_kernel<__nv_bfloat16><<<grid, block, 0, s>>>(static_cast<const __nv_bfloat16 *>(x),
                                                                 static_cast<__nv_bfloat16 *>(cols), batch, height,
                                                                 width, channels, k, stride, oh, ow);
    RBGP4_CHECK_LAUNCH("im2col_nhwc launch");
    return RBGP4_OK;
}

namespace {
int nc_to_nhwc_impl(int dtype, const void *src, void *dst, int rows, int64_t n, int relu, const void *res,
                    void *dst_relu, void *stream) {
    using namespace rbgp4;
    RBGP4_REQUIRE(dtype == RBGP4_F32 || dtype == RBGP4_BF16, "nc_to_nhwc: F32 or BF16");
    RBGP4_REQUIRE(rows >= 0 && n >= 0, "nc_to_nhwc: bad sizes");
    if (rows == 0 || n == 0) return RBGP4_OK;
    dim3 grid(unsigned((n + 31) / 32), unsigned((rows + 31) / 32));
    dim3 block(32, 8);
    auto s = static_cast<cudaStream_t>(stream);
    if (dtype == RBGP4_F32)
        nc_to_nhwc_kernel<float><<<grid, block, 0, s>>>(static_cast<const float *>(src), static_cast<float *>(dst),
                                                        rows, n, relu, static_cast<const float *>(res),
                                                        static_cast<float *>(dst_relu));
    else
        nc_to_nhwc_kernel<__nv_bfloat16><<<grid, block, 0, s>>>(
            static_cast<const __nv_bfloat16 *>(src), static_cast<__nv_bfloat16 *>(dst), rows, n, relu,
            static_cast<const __nv_bfloat16 *>(res), static_cast<__nv_bfloat16 *>(dst_relu));
    RBGP4_CHECK_LAUNCH("nc_to_nhwc launch");
    return RBGP4_OK;
}
}  // namespace

extern "C" int rbgp4_nc_to_nhwc(int dtype, const void *src, void *dst, int rows, int64_t n, int relu, void *stream) {
    return nc_to_nhwc_impl(dtype, src, dst, rows, n, relu, nullptr, nullptr, stream);
}

extern "C" int rbgp4_nc_to_nhwc_residual(int dtype, const void *src, const void *residual, void *dst,
                                         void *dst_relu, int rows, int64_t n, void *stream) {
    using namespace rbgp4;
    RBGP4_REQUIRE(residual != nullptr, "nc_to_nhwc_residual: null residual");
    return nc_to_nhwc_impl(dtype, src, dst, rows, n, 0, residual, dst_relu, stream);
}
