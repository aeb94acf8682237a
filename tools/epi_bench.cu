// epi_bench.cu -- cost of the K4 epilogue primitives on B200 (diagnostic, not product code):
//   A  tcgen05.ld throughput (32x32b.x16 / .x32), 4 warps and 1 warp per CTA
//   C  a 128 x 128 bf16 output tile from registers: lanes = columns, 2-byte stores per row
//   D  the same tile through shared memory, 16-byte global stores (rows of 256 B)
//   E  DSMEM push of fp32 partials to the peer CTA of a 2-CTA cluster: 4-byte vs 16-byte stores
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/epi_bench.cu -o tools/epi_bench.bin
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

#define LD16(taddr, r)                                                                     \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11," \
                 "%12,%13,%14,%15}, [%16];"                                                \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), \
                   "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), \
                   "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                      \
                 : "r"(taddr))

// A: every active warp reads `cols` TMEM columns of its 32 lanes, `reps` times
__global__ void __launch_bounds__(128, 1) tmem_read(int warps, int cols, int reps, int wait_every,
                                                    unsigned long long *out, float *sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + (uint32_t(warp * 32) << 16);
    float acc = 0.f;
    float accv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) accv[i] = 0.f;
    unsigned long long t0 = clock64();
    if (warp < warps) {
        for (int r = 0; r < reps; ++r) {
            for (int c = 0; c < cols; c += 16 * wait_every) {
                uint32_t v[4][16];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q < wait_every) LD16(base + uint32_t(c + 16 * q), v[q]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q < wait_every)
#pragma unroll
                        for (int i = 0; i < 16; ++i) accv[i] += __uint_as_float(v[q][i]);
            }
        }
    }
    unsigned long long t1 = clock64();
#pragma unroll
    for (int i = 0; i < 16; ++i) acc += accv[i];
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 1234.5f) sink[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

// C / D: CTA b writes the 128 x 128 bf16 tile (tile-row b % 4, column block b / 4) of a
// (512, N) row-major output; thread t = column, 128 fp32 rows in registers (synthetic)
__global__ void __launch_bounds__(128, 1) tile_store(__nv_bfloat16 *out, int64_t ld, int mode, int reps,
                                                     unsigned long long *tout) {
    __shared__ __align__(16) __nv_bfloat16 stage[128 * 128];
    const int t = threadIdx.x;
    const int64_t m0 = (blockIdx.x % 4) * 128, n0 = (blockIdx.x / 4) * 128;
    float r[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) r[q] = float(t * 32 + q);
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        for (int c = 0; c < 128; c += 32) {
            if (mode == 0) {
#pragma unroll
                for (int q = 0; q < 32; ++q) out[(m0 + c + q) * ld + n0 + t] = __float2bfloat16_rn(r[q] + c);
            } else {
                // column t of rows c..c+31 into the staged tile [row][128 cols], then 16-byte rows
#pragma unroll
                for (int q = 0; q < 32; ++q) stage[(c + q) * 128 + (((t >> 3) ^ (q & 7)) << 3) + (t & 7)] = __float2bfloat16_rn(r[q] + c);
            }
        }
        if (mode == 1) {
            __syncthreads();
            // 128 rows x 16 chunks of 16 B: thread t -> chunk t % 16 of rows t / 16 + 8 i
            for (int i = 0; i < 16; ++i) {
                const int row = t / 16 + 8 * i, ch = t % 16;
                const uint4 v = *reinterpret_cast<const uint4 *>(&stage[row * 128 + ((ch ^ (row & 7)) << 3)]);
                *reinterpret_cast<uint4 *>(&out[(m0 + row) * ld + n0 + ch * 8]) = v;
            }
            __syncthreads();
        }
    }
    unsigned long long t1 = clock64();
    if (t == 0) tout[blockIdx.x] = t1 - t0;
}

// E: each CTA of a 2-CTA cluster pushes `kb` KB of fp32 to its peer's shared memory
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
dsmem_push(int kb, int vec, unsigned long long *tout) {
    extern __shared__ __align__(16) float buf[];
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const int n = kb * 256;  // floats
    float *peer;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(peer) : "l"(buf), "r"(rank ^ 1));
    unsigned long long t0 = clock64();
    if (vec) {
        float4 *p4 = reinterpret_cast<float4 *>(peer);
        for (int i = threadIdx.x; i < n / 4; i += 128) p4[i] = make_float4(float(i), 1.f, 2.f, 3.f);
    } else {
        for (int i = threadIdx.x; i < n; i += 128) peer[i] = float(i);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) tout[blockIdx.x] = t1 - t0;
}


// F: the 128 x 128 bf16 tile staged in shared memory (2 atoms of 64 cols x 128 rows, 128B
// swizzle) and written by two TMA tensor stores; cycles to wait_group.read and to wait_group
__global__ void __launch_bounds__(128, 1) tile_tma_store(const __grid_constant__ CUtensorMap omap, int reps,
                                                         unsigned long long *tout) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *stage = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    const int t = threadIdx.x;
    for (int i = t; i < 128 * 128 / 8; i += 128) reinterpret_cast<uint4 *>(stage)[i] = make_uint4(i, i, i, i);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int m0 = (blockIdx.x % 4) * 128, n0 = (blockIdx.x / 4) * 128;
    unsigned long long t0 = clock64(), tr = 0;
    if (t == 0) {
        for (int rep = 0; rep < reps; ++rep) {
            for (int a = 0; a < 2; ++a)
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&omap),
                             "r"(n0 + 64 * a), "r"(m0), "r"(su32(stage + a * 16384)) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        tr = clock64();
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    unsigned long long t1 = clock64();
    if (t == 0) { tout[2 * blockIdx.x] = tr - t0; tout[2 * blockIdx.x + 1] = t1 - t0; }
}

// G: bulk copy (cp.async.bulk shared::cta -> shared::cluster) of `kb` KB into the peer CTA,
// completing on the peer's mbarrier; H: the peer pulls with ld.shared::cluster.v4
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
dsmem_bulk(int kb, int mode, unsigned long long *tout, float *sink) {
    extern __shared__ __align__(16) float bbuf_f[];
    unsigned char *buf = reinterpret_cast<unsigned char *>(bbuf_f);
    __shared__ __align__(8) uint64_t bar;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int bytes = kb * 1024;
    unsigned char *src = buf, *dst = buf + bytes;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
    }
    for (int i = threadIdx.x; i < bytes / 16; i += 128) reinterpret_cast<uint4 *>(src)[i] = make_uint4(i, 1, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    unsigned long long t0 = clock64();
    float acc = 0.f;
    if (mode == 0) {
        if (threadIdx.x == 0) {
            uint32_t pdst, pbar;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(pdst) : "r"(su32(dst)), "r"(rank ^ 1));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(pbar) : "r"(su32(&bar)), "r"(rank ^ 1));
            for (int c = 0; c < bytes; c += 8192)
                asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(pdst + c), "r"(su32(src + c)), "r"(min(8192, bytes - c)), "r"(pbar) : "memory");
            asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n"
                         ::"r"(su32(&bar)) : "memory");
        }
    } else {
        uint32_t psrc;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(psrc) : "r"(su32(src)), "r"(rank ^ 1));
        float4 a4 = make_float4(0, 0, 0, 0);
        for (int i = threadIdx.x; i < bytes / 16; i += 128) {
            float4 v;
            asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(psrc + 16 * i));
            a4.x += v.x; a4.y += v.y; a4.z += v.z; a4.w += v.w;
        }
        acc = a4.x + a4.y + a4.z + a4.w;
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) tout[blockIdx.x] = t1 - t0;
    if (acc == 1.5f) sink[0] = acc;
}

static double median(std::vector<unsigned long long> v) {
    std::sort(v.begin(), v.end());
    return double(v[v.size() / 2]);
}

int main() {
    unsigned long long *dt; float *sink;
    cudaMalloc(&dt, 4096 * 8); cudaMalloc(&sink, 64);
    std::vector<unsigned long long> h(148);
    // ---- A
    for (int warps : {1, 4})
        for (int we : {1, 2, 4}) {
            const int cols = 512, reps = 8;
            tmem_read<<<148, 128>>>(warps, cols, reps, we, dt, sink);
            tmem_read<<<148, 128>>>(warps, cols, reps, we, dt, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(h.data(), dt, 148 * 8, cudaMemcpyDeviceToHost);
            const double cyc = median(h);
            const double bytes = double(warps) * 32 * 4 * cols * reps;
            printf("A tmem read: %d warp(s), %d x16 loads per wait: %8.0f cyc  %6.1f B/clk/SM\n", warps, we, cyc,
                   bytes / cyc);
        }
    // ---- C / D
    {
        const int64_t N = 4096;
        __nv_bfloat16 *o; cudaMalloc(&o, size_t(512) * N * 2);
        for (int mode : {0, 1}) {
            const int reps = 4;
            tile_store<<<128, 128>>>(o, N, mode, reps, dt);
            tile_store<<<128, 128>>>(o, N, mode, reps, dt);
            cudaDeviceSynchronize();
            std::vector<unsigned long long> hh(128);
            cudaMemcpy(hh.data(), dt, 128 * 8, cudaMemcpyDeviceToHost);
            printf("%s 128x128 bf16 tile store: %8.0f cyc per tile (128 CTAs)\n",
                   mode ? "D smem-staged 16B" : "C direct 2B/lane", median(hh) / reps);
        }
        cudaFree(o);
    }
    // ---- E
    cudaFuncSetAttribute(dsmem_push, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int vec : {0, 1}) {
        const int kb = 48;
        dsmem_push<<<148, 128, 64 * 1024>>>(kb, vec, dt);
        dsmem_push<<<148, 128, 64 * 1024>>>(kb, vec, dt);
        cudaDeviceSynchronize();
        cudaMemcpy(h.data(), dt, 148 * 8, cudaMemcpyDeviceToHost);
        const double cyc = median(h);
        printf("E dsmem push %d KB, %s stores: %8.0f cyc  %6.1f B/clk\n", kb, vec ? "16-byte" : "4-byte", cyc,
               kb * 1024.0 / cyc);
    }

    // ---- F
    {
        const int64_t N = 4096;
        void *o; cudaMalloc(&o, size_t(512) * N * 2);
        void *fnp = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
        CUtensorMap m;
        cuuint64_t d[2] = {cuuint64_t(N), 512};
        cuuint64_t s[1] = {cuuint64_t(N) * 2};
        cuuint32_t b[2] = {64, 128}, e[2] = {1, 1};
        enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, o, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(tile_tma_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
        for (int reps : {1, 4}) {
            tile_tma_store<<<128, 128, 40 * 1024>>>(m, reps, dt);
            tile_tma_store<<<128, 128, 40 * 1024>>>(m, reps, dt);
            cudaDeviceSynchronize();
            std::vector<unsigned long long> hh(256), r0, r1;
            cudaMemcpy(hh.data(), dt, 256 * 8, cudaMemcpyDeviceToHost);
            for (int i = 0; i < 128; ++i) { r0.push_back(hh[2 * i]); r1.push_back(hh[2 * i + 1]); }
            printf("F TMA store 128x128 bf16 x%d: read-done %8.0f cyc  write-done %8.0f cyc (per launch, 128 CTAs)\n",
                   reps, median(r0), median(r1));
        }
        cudaFree(o);
    }
    // ---- G / H
    cudaFuncSetAttribute(dsmem_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int mode : {0, 1}) {
        const int kb = 48;
        dsmem_bulk<<<148, 128, 2 * kb * 1024>>>(kb, mode, dt, sink);
        dsmem_bulk<<<148, 128, 2 * kb * 1024>>>(kb, mode, dt, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h.data(), dt, 148 * 8, cudaMemcpyDeviceToHost);
        const double cyc = median(h);
        printf("%s %d KB: %8.0f cyc  %6.1f B/clk\n", mode ? "H dsmem pull ld.shared::cluster.v4" : "G dsmem bulk copy (8 KB chunks)",
               kb, cyc, kb * 1024.0 / cyc);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
