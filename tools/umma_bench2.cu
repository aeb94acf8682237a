// umma_bench2.cu -- issue cost of the gathered-block kernel's MMA shapes (diagnostic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/umma_bench2.cu -o tools/umma_bench2.bin
// M=128 bf16, A MN-major SW128 (LBO = a_lbo), B K-major with swizzle span b_span, N = n,
// D column advancing by n per MMA (dstep=1) or fixed; cycles per MMA over 1024 MMAs.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout & 7) << 61;
    return d;
}
__global__ void __launch_bounds__(128, 1) k(int n, int b_span, int a_lbo, int dstep, int nblk, int iters, long long *out) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < (65536 + 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(buf)[i] = 0x3c003c00u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    uint32_t el = 0;
    if (threadIdx.x / 32 == 1)
        asm volatile("{\n.reg .pred p;\n.reg .b32 r;\nelect.sync r|p, 0xffffffff;\nselp.b32 %0, 1, 0, p;\n}\n" : "=r"(el));
    if (el) {
        const uint32_t code = b_span == 128 ? 2u : b_span == 64 ? 4u : 6u;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (uint32_t(n >> 3) << 17) | (8u << 24);
        const uint64_t ad = smem_desc(smem_u32(buf), a_lbo, 1024, 2);
        const uint64_t bd = smem_desc(smem_u32(buf + 65536), 0, 8 * b_span, code);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int kb = i % nblk;
            const uint32_t d = tmem + (dstep ? uint32_t(kb * n) : 0u);
            const uint64_t a = ad + uint32_t(kb * 256);           // 16 K rows of 128 B further
            const uint64_t b = bd + uint32_t((kb * n * b_span) >> 4);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                         "l"(a), "l"(b), "r"(idesc), "r"(1));
        }
        long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
        long long t2 = clock64();
        out[0] = t1 - t0; out[1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
// the K4 relayout step: nmma MMAs (N=n) with uniform descriptor arithmetic, commit, wait;
// `steps` times -> cycles per step (issue + commit + completion wait)
__global__ void __launch_bounds__(128, 1) steps_k(int n, int nmma, int steps, long long *out, int bspan = 32, int kcycle = 1, int dsame = 0) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < (65536 + 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(buf)[i] = 0x3c003c00u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x / 32 == 1) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (uint32_t(n >> 3) << 17) | (8u << 24);
        const uint64_t ad = smem_desc(smem_u32(buf), 16384, 1024, 2);
        const uint32_t bcode = bspan == 128 ? 2u : bspan == 64 ? 4u : 6u;
        const uint64_t bd = smem_desc(smem_u32(buf + 65536), 0, 8 * bspan, bcode);
        long long t0 = clock64();
        for (int s = 0; s < steps; ++s) {
            uint32_t el = 0;
            asm volatile("{\n.reg .pred p;\n.reg .b32 r;\nelect.sync r|p, 0xffffffff;\nselp.b32 %0, 1, 0, p;\n}\n" : "=r"(el));
            if (el) {
                uint64_t b = bd;
                uint32_t d = tmem;
                for (int kb = 0; kb < nmma; ++kb) {
                    // kcycle > 1: K offsets inside the B swizzle row cycle like the kernel's ink slots
                    const uint32_t koff = uint32_t((kb % kcycle) * 2);
                    const uint32_t aoff = uint32_t(((kb * 5) % 8) * 128);   // scattered K-blocks
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                                 "l"(ad + aoff), "l"(b + koff), "r"(idesc), "r"(s > 0 ? 1 : 0));
                    if ((kb % kcycle) == kcycle - 1) {
                        b += uint32_t((n * bspan) >> 4);
                        if (!dsame) d += uint32_t(n);
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
            }
            __syncwarp();
            asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)), "r"(s & 1) : "memory");
            asm volatile("tcgen05.fence::after_thread_sync;");
        }
        long long t1 = clock64();
        if (threadIdx.x == 32) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    const int iters = 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 65536 + 16384);
    struct C { int n, span, lbo, dstep, nblk; };
    C cs[] = {{32, 32, 16384, 1, 8}, {32, 32, 16384, 0, 8}, {32, 32, 8192, 1, 8}, {32, 64, 16384, 1, 8},
              {32, 128, 16384, 1, 4}, {16, 32, 16384, 1, 16}, {64, 32, 16384, 1, 4}, {128, 32, 16384, 1, 2},
              {32, 32, 16384, 1, 1}, {256, 32, 16384, 0, 1}};
    for (auto c : cs) {
        k<<<1, 128, 1024 + 65536 + 16384>>>(c.n, c.span, c.lbo, c.dstep, c.nblk, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("N=%3d Bspan=%3d A_LBO=%5d dstep=%d nblk=%2d : issue %6.1f complete %6.1f cyc/MMA %s\n", c.n, c.span,
               c.lbo, c.dstep, c.nblk, double(h[0]) / iters, double(h[1]) / iters, e ? cudaGetErrorString(e) : "");
    }
    cudaFuncSetAttribute(steps_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 65536 + 16384);
    struct S { int n, nm, bspan, kcycle; };
    S ss[] = {{16, 16, 32, 1}, {16, 16, 64, 2}, {16, 16, 128, 4}, {32, 8, 32, 1}, {16, 8, 32, 1}};
    for (auto c : ss) {
        steps_k<<<1, 128, 1024 + 65536 + 16384>>>(c.n, c.nm, 64, d, c.bspan, c.kcycle, 0);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("step of %2d MMAs N=%d Bspan=%3d kcycle=%d + commit + wait: %7.1f cycles/step %s\n", c.nm, c.n,
               c.bspan, c.kcycle, double(h[0]) / 64, e ? cudaGetErrorString(e) : "");
    }
    return 0;
}
