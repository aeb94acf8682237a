// umma_bench3.cu -- tcgen05 MMA step cost under the K4 kernel's occupancy (diagnostic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/umma_bench3.cu -o tools/umma_bench3.bin
// Every CTA (grid = 148 or 296, 1 or 2 per SM by dynamic shared memory) issues `steps` steps of
// `nmma` M128 x N x K16 bf16 MMAs (scattered K blocks of an MN- or K-major A, B K-major span 32),
// one commit per step; wait=1 waits for each step's completion (issue + drain), wait=0 only at
// the end (issue throughput).  Prints the mean cycles per step over CTAs.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
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
__global__ void __launch_bounds__(128, 1) steps3(int n, int nmma, int steps, int amn, int wait, long long *out, int dspan = 128, int seqa = 0, int dpair = 0) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < (32768 + 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(buf)[i] = 0x3c003c00u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(dspan));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (threadIdx.x / 32 == 1) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(amn) << 15) | (uint32_t(n >> 3) << 17) | (8u << 24);
        const uint64_t ad = amn ? smem_desc(smem_u32(buf), 16384, 1024, 2) : smem_desc(smem_u32(buf), 16, 1024, 2);
        const uint64_t bd = smem_desc(smem_u32(buf + 32768), 0, 8 * 32, 6u);
        long long t0 = clock64();
        int phase = 0;
        for (int s = 0; s < steps; ++s) {
            uint32_t el = 0;
            asm volatile("{\n.reg .pred p;\n.reg .b32 r;\nelect.sync r|p, 0xffffffff;\nselp.b32 %0, 1, 0, p;\n}\n" : "=r"(el));
            if (el) {
                uint64_t b = bd;
                uint32_t d = tmem;
                for (int kb = 0; kb < nmma; ++kb) {
                    const int blk = seqa ? kb % 8 : (kb * 5) % 8;
                    const uint32_t aoff = amn ? uint32_t(blk * 128)                                   // 16 rows of 128 B
                                              : uint32_t(((blk / 4) * 16384 + (blk % 4) * 32) >> 4);  // atom, K offset
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                                 "l"(ad + aoff), "l"(b), "r"(idesc), "r"(s > 0 ? 1 : 0));
                    b += uint32_t((n * 32) >> 4);
                    if (!dpair || (kb & 1)) d += uint32_t(n);
                    if (d >= tmem + uint32_t(dspan)) d = tmem;
                    if (b >= bd + (16384 >> 4)) b = bd;
                }
                if (wait || s == steps - 1)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
            }
            __syncwarp();
            if (wait || s == steps - 1) {
                asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)), "r"(phase) : "memory");
                phase ^= 1;
                asm volatile("tcgen05.fence::after_thread_sync;");
            }
        }
        long long t1 = clock64();
        if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(dspan));
}

int main() {
    long long *d;
    cudaMalloc(&d, 8 * 1024);
    const int steps = 256;
    struct C { int n, nmma, amn, grid, smem_kb, wait, dspan = 128, seqa = 0, dpair = 0; };
    std::vector<C> cs;
    // MMA cost vs N at 1 CTA/SM (8 MMAs per step, MN-major A, D over 512 TMEM columns)
    for (int n : {16, 32, 64, 128, 256}) cs.push_back({n, 8, 1, 148, 150, 0, 512, 1, 0});
    for (int n : {32, 64, 128, 256}) cs.push_back({n, 8, 0, 148, 150, 0, 512, 1, 0});
    // in-kernel patterns at 2 CTAs/SM, issue only: direct mode (16 x N16, pairs into one D),
    // relayout (8 x N32 over 256 D columns, sequential A)
    for (int dspan : {128, 256})
        for (int seqa = 0; seqa <= 1; ++seqa)
            for (int dpair = 0; dpair <= 1; ++dpair) {
                cs.push_back({16, 16, 1, 296, 100, 0, dspan, seqa, dpair});
                cs.push_back({32, 8, 1, 296, 100, 0, dspan, seqa, dpair});
            }
    for (int amn = 1; amn >= 1; --amn)
        for (int w = 0; w <= 0; ++w)
            for (auto g : {std::make_pair(148, 150), std::make_pair(296, 100)}) {
                cs.push_back({16, 16, amn, g.first, g.second, w});
                cs.push_back({32, 8, amn, g.first, g.second, w});
                cs.push_back({64, 4, amn, g.first, g.second, w});
                cs.push_back({16, 8, amn, g.first, g.second, w});
            }
    cudaFuncSetAttribute(steps3, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    for (auto c : cs) {
        steps3<<<c.grid, 128, c.smem_kb * 1024>>>(c.n, c.nmma, steps, c.amn, c.wait, d, c.dspan, c.seqa, c.dpair);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h(c.grid);
        cudaMemcpy(h.data(), d, 8 * c.grid, cudaMemcpyDeviceToHost);
        double m = 0;
        for (auto v : h) m += double(v);
        m /= c.grid * steps;
        printf("dspan %d seqA %d dpair %d | A %s  %d CTA/SM  %2d x N%-3d  %s : %7.1f cycles/step  %6.1f /MMA %s\n", c.dspan, c.seqa, c.dpair, c.amn ? "MN" : "K ",
               c.grid / 148, c.nmma, c.n, c.wait ? "issue+drain" : "issue only ", m, m / c.nmma,
               e ? cudaGetErrorString(e) : "");
    }
    return 0;
}
