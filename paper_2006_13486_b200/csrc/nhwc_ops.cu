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
