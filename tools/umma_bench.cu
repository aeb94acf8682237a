// umma_bench.cu -- ground-truth costs of the tcgen05 primitives the RBGP4 kernel uses.
// (Diagnostic, not product code.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/umma_bench.cu -o tools/umma_bench.bin
//
// 1. back-to-back tcgen05.mma throughput (cycles per instruction), M=128, N in {128, 256},
//    A K-major SW128, B MN-major SW128 (the kernel's layout) vs B K-major SW128
// 2. tcgen05.commit -> mbarrier completion latency after a burst of MMAs
// 3. mbarrier ping-pong latency between two warps
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout & 7) << 61;
    return d;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 "@!p bra W_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n.reg .pred p;\n.reg .b32 r;\nelect.sync r|p, 0xffffffff;\nselp.b32 %0, 1, 0, p;\n}\n"
                 : "=r"(pred));
    return pred != 0;
}

// mode: 0 = B MN-major, 1 = B K-major
__global__ void __launch_bounds__(128, 1) mma_kernel(int n, int mode, int iters, long long *out) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    // A: 128 rows x 64 bf16 (16 KB), B: 64 x n (n * 128 B)
    for (int i = threadIdx.x; i < (16384 + n * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(buf)[i] = 0x3c003c00u;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (warp == 1) {
        // mode 2 / 3: the gathered-block kernel's shapes -- A MN-major (2 = SDMM) or K-major
        // (3 = conv) SW128, B K-major SW64 (compressed W rows of 64 bytes)
        const uint32_t a_mn = mode == 2 ? 1u : 0u;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (uint32_t(mode == 0) << 16) |
                               (uint32_t(n >> 3) << 17) | (8u << 24);
        const uint64_t ad = mode == 2 ? smem_desc(smem_u32(buf), 64 * 128, 1024, 2) : smem_desc(smem_u32(buf), 0, 1024, 2);
        const uint64_t bd = mode == 0 ? smem_desc(smem_u32(buf + 16384), 64 * 128, 1024, 2)
                          : mode == 1 ? smem_desc(smem_u32(buf + 16384), 0, 1024, 2)
                                      : smem_desc(smem_u32(buf + 16384), 0, 512, 4);
        long long t0 = 0, t1 = 0, t2 = 0;
        if (elect_one()) {
            // warm
            for (int i = 0; i < 16; ++i) mma(tmem, ad + (mode == 2 ? 128 * (i & 3) : 2 * (i & 3)), bd + (mode == 0 ? 128 * (i & 3) : mode >= 2 ? 2 * (i & 1) : 2 * (i & 3)), idesc, 1);
            tc_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        if (elect_one()) {
            t0 = clock64();
            for (int i = 0; i < iters; ++i)
                mma(tmem, ad + (mode == 2 ? 128 * (i & 3) : 2 * (i & 3)), bd + (mode == 0 ? 128 * (i & 3) : mode >= 2 ? 2 * (i & 1) : 2 * (i & 3)), idesc, 1);
            t1 = clock64();
            tc_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 1);
        t2 = clock64();
        if (elect_one() && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// commit latency: issue k MMAs, commit, wait; also an empty commit
__global__ void __launch_bounds__(64, 1) commit_kernel(long long *out) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(buf)[i] = 0;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (16u << 17) | (8u << 24);
    const uint64_t ad = smem_desc(smem_u32(buf), 0, 1024, 2);
    const uint64_t bd = smem_desc(smem_u32(buf + 16384), 64 * 128, 1024, 2);
    if (threadIdx.x < 32) {
        uint32_t ph = 0;
        for (int k : {0, 1, 4, 8}) {
            long long best = 1ll << 40;
            for (int rep = 0; rep < 8; ++rep) {
                long long t0 = 0;
                if (elect_one()) {
                    t0 = clock64();
                    for (int i = 0; i < k; ++i) mma(tmem, ad, bd, idesc, 1);
                    tc_commit(&bar);
                }
                __syncwarp();
                mbar_wait(&bar, ph);
                ph ^= 1;
                long long t1 = clock64();
                if (elect_one()) best = min(best, t1 - t0);
                __syncwarp();
            }
            if (elect_one() && blockIdx.x == 0) out[k] = best;
            __syncwarp();
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

// ping-pong: warp 0 arrives on a, waits b; warp 1 waits a, arrives b
__global__ void __launch_bounds__(64, 1) pingpong_kernel(int iters, long long *out) {
    __shared__ uint64_t a, b;
    if (threadIdx.x == 0) { mbar_init(&a, 1); mbar_init(&b, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const int warp = threadIdx.x / 32;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (warp == 0) {
            if (elect_one()) mbar_arrive(&a);
            __syncwarp();
            mbar_wait(&b, i & 1);
        } else {
            mbar_wait(&a, i & 1);
            if (elect_one()) mbar_arrive(&b);
            __syncwarp();
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
    long long *d, h[16];
    cudaMalloc(&d, 16 * sizeof(long long));
    const int iters = 1024;
    for (int n : {16, 32, 64, 128, 256}) {
        for (int mode : {0, 1, 2, 3}) {
            if (mode < 2 && n < 64) continue;
            const size_t smem = 1024 + 16384 + n * 128;
            cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
            mma_kernel<<<1, 128, smem>>>(n, mode, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
            printf("MMA M128 N%-3d K16 B %s : issue %6.1f cyc/instr, complete %6.1f cyc/instr (floor %d) %s\n",
                   n, mode == 0 ? "MN-major" : mode == 1 ? "K-major " : mode == 2 ? "A-MN/B-K64" : "A-K/B-K64", double(h[0]) / iters, double(h[1]) / iters,
                   128 * n / 256, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    // 148 CTAs concurrently, N=128 MN-major
    {
        const size_t smem = 1024 + 16384 + 128 * 128;
        mma_kernel<<<148, 128, smem>>>(128, 0, iters, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 2 * sizeof(long long), cudaMemcpyDeviceToHost);
        printf("MMA N128 MN-major, 148 CTAs: complete %6.1f cyc/instr\n", double(h[1]) / iters);
    }
    cudaFuncSetAttribute(commit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    commit_kernel<<<1, 64, 40000>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 9 * sizeof(long long), cudaMemcpyDeviceToHost);
    printf("commit->wait latency: 0 MMA %lld, 1 MMA %lld, 4 MMA %lld, 8 MMA %lld cycles %s\n", h[0], h[1], h[4], h[8],
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    pingpong_kernel<<<1, 64>>>(10000, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long), cudaMemcpyDeviceToHost);
    printf("mbarrier ping-pong round trip between two warps: %lld cycles\n", h[0]);
    return 0;
}
