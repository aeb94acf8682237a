// tma_issue_bench.cu -- per-box cost of TMA loads issued by one thread per CTA (diagnostic for
// the K5 producer; not product code).  148 CTAs, warm L2: one thread issues `nbox` boxes of a
// shape back to back into distinct shared-memory slots on one mbarrier; reports cycles to issue
// them all and cycles until all bytes landed.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_issue_bench.cu -o tools/tma_issue_bench.bin -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

struct Shape { int dims; int b0, b1, b2; int bytes; };

__global__ void __launch_bounds__(32, 1) issue_kernel(const __grid_constant__ CUtensorMap m, Shape sh, int nbox,
                                                      int krows, int nat, int mode, unsigned long long *out) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x != 0) return;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&m) : "memory");
    for (int rep = 0; rep < 3; ++rep) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(sh.bytes * nbox) : "memory");
        const unsigned long long t0 = clock64();
        for (int i = 0; i < nbox; ++i) {
            unsigned char *dst = buf + size_t(i) * sh.bytes;
            // coordinates vary per box (different rows / atoms), as in the kernel
            const int row = ((blockIdx.x * 7 + i * 13) % (krows / 16)) * 16;
            const int at = (blockIdx.x + i) % nat;
            if (sh.dims == 3)
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(dst)), "l"(&m), "r"(0), "r"(mode ? 0 : row),
                             "r"(at & ~1), "r"(su32(&bar)) : "memory");
            else
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)), "l"(&m), "r"(0), "r"(row),
                             "r"(su32(&bar)) : "memory");
        }
        const unsigned long long t1 = clock64();
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                     ::"r"(su32(&bar)), "r"(rep & 1) : "memory");
        const unsigned long long t2 = clock64();
        if (rep == 2) { out[2 * blockIdx.x] = t1 - t0; out[2 * blockIdx.x + 1] = t2 - t0; }
    }
}

int main() {
    void *fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    const int K = 4608, N = 1024;
    void *dI; cudaMalloc(&dI, size_t(K) * N * 2); cudaMemset(dI, 1, size_t(K) * N * 2);
    unsigned long long *dt; cudaMalloc(&dt, 148 * 16);
    cudaFuncSetAttribute(issue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Case { const char *name; int dims; cuuint32_t box[3]; int swz; int bytes; int nbox; };
    std::vector<Case> cases = {
        {"3D slab (64,128,2) 32KB", 3, {64, 128, 2}, 128, 32768, 5},
        {"3D piece (64,16,2) 4KB", 3, {64, 16, 2}, 128, 4096, 40},
        {"3D piece (64,32,2) 8KB", 3, {64, 32, 2}, 128, 8192, 20},
        {"3D atom (64,16,1) 2KB", 3, {64, 16, 1}, 128, 2048, 80},
        {"2D W relayout (16,256) 8KB", 2, {16, 256, 0}, 32, 8192, 20},
        {"2D W direct (32,16) 1KB", 2, {32, 16, 0}, 64, 1024, 80},
    };
    for (auto &c : cases) {
        CUtensorMap m;
        CUresult r;
        if (c.dims == 3) {
            cuuint64_t d[3] = {64, cuuint64_t(K), cuuint64_t(N / 64)};
            cuuint64_t s[2] = {cuuint64_t(N) * 2, 128};
            cuuint32_t e[3] = {1, 1, 1};
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dI, d, s, c.box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            const int w = c.box[0];
            cuuint64_t d[2] = {cuuint64_t(w), cuuint64_t(K) * N * 2 / (w * 2)};
            cuuint64_t s[1] = {cuuint64_t(w) * 2};
            cuuint32_t e[2] = {1, 1};
            r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dI, d, s, c.box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    c.swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.name, int(r)); continue; }
        Shape sh{c.dims, int(c.box[0]), int(c.box[1]), int(c.box[2]), c.bytes};
        for (int grid : {1, 148}) {
            issue_kernel<<<grid, 32, 200 * 1024>>>(m, sh, c.nbox, K, N / 64, 0, dt);
            issue_kernel<<<grid, 32, 200 * 1024>>>(m, sh, c.nbox, K, N / 64, 0, dt);
            cudaDeviceSynchronize();
            std::vector<unsigned long long> h(2 * grid);
            cudaMemcpy(h.data(), dt, h.size() * 8, cudaMemcpyDeviceToHost);
            std::vector<unsigned long long> a, b;
            for (int i = 0; i < grid; ++i) { a.push_back(h[2 * i]); b.push_back(h[2 * i + 1]); }
            std::sort(a.begin(), a.end()); std::sort(b.begin(), b.end());
            const double ia = double(a[a.size() / 2]) / c.nbox, cb = double(b[b.size() / 2]);
            printf("%-30s grid %3d: issue %6.1f cyc/box  all landed %7.0f cyc  (%5.1f B/clk/CTA, %5.0f cyc/box)\n",
                   c.name, grid, ia, cb, double(c.bytes) * c.nbox / cb, cb / c.nbox);
        }
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
