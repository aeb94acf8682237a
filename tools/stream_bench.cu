// stream_bench.cu -- how fast can the SMs pull I slabs from L2 / HBM with TMA?  Diagnostic
// for the K4 SDMM main loop (not product code).  One elected thread per CTA streams a list of
// (row, atom) boxes of a (64 cols, K rows, N/64 atoms) bf16 tensor map through a ring of
// `depth` stages; optional 2-CTA clusters fetch one atom each and multicast it to both.
// Reports event time and the in-kernel span (first CTA start .. last CTA end, %globaltimer).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/stream_bench.cu -o /tmp/sb
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

__device__ __forceinline__ uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void wait_bar(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(su32(b)), "r"(ph) : "memory");
}

struct Cfg {
    int rows, atoms, depth, steps, mc;
    const int2 *list;  // [grid][steps] (krow, atom0)
    unsigned long long *stamps;
};

__global__ void __launch_bounds__(32, 1) stream_kernel(const __grid_constant__ CUtensorMap m, Cfg c) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int stage = c.rows * 128 * c.atoms;
    uint64_t *full = reinterpret_cast<uint64_t *>(buf + c.depth * stage);
    uint64_t *empty = full + c.depth;
    const int cid = blockIdx.x;
    if (threadIdx.x == 0) {
        c.stamps[2 * cid] = gtimer();
        for (int i = 0; i < c.depth; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(su32(&empty[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t rank = 0;
    if (c.mc) {
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        const int2 *L = c.list + size_t(c.mc ? cid / 2 : cid) * c.steps;
        auto issue = [&](int s) {
            const int st = s % c.depth;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(stage) : "memory");
            const int2 e = L[s];
            if (c.mc) {
                unsigned char *dst = buf + st * stage + rank * (c.rows * 128);
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                             " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(su32(dst)), "l"(&m), "r"(0), "r"(e.x),
                             "r"(e.y + int(rank)), "r"(su32(&full[st])), "h"(uint16_t(3)) : "memory");
            } else {
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(buf + st * stage)), "l"(&m), "r"(0),
                             "r"(e.x), "r"(e.y), "r"(su32(&full[st])) : "memory");
            }
        };
        for (int s = 0; s < c.depth && s < c.steps; ++s) issue(s);
        for (int s = 0; s < c.steps; ++s) {
            const int st = s % c.depth;
            wait_bar(&full[st], (s / c.depth) & 1);
            // release slot st: here and (multicast) in the peer, whose box half lands here too
            if (c.mc) {
                uint32_t peer;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer) : "r"(su32(&empty[st])), "r"(rank ^ 1));
                asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(peer) : "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[st])) : "memory");
            }
            const int sn = s + c.depth;
            if (sn < c.steps) {
                wait_bar(&empty[st], (s / c.depth) & 1);
                issue(sn);
            }
        }
        c.stamps[2 * cid + 1] = gtimer();
    }
    if (c.mc) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void ldg_kernel(const uint4 *p, size_t n, unsigned long long *sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) acc ^= p[i].x;
    if (acc == 0x12345678u) sink[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

struct Result { double ev_us, span_us; };

static Result run(const CUtensorMap &m, int rows, int atoms, int depth, int grid, int steps, int mc,
                  const std::vector<int2> &list, const uint4 *flush, size_t flush_n, unsigned long long *sink,
                  int reps) {
    int2 *dl; unsigned long long *st;
    cudaMalloc(&dl, list.size() * sizeof(int2));
    cudaMemcpy(dl, list.data(), list.size() * sizeof(int2), cudaMemcpyHostToDevice);
    cudaMalloc(&st, size_t(grid) * 2 * 8);
    Cfg c{rows, atoms, depth, steps, mc, dl, st};
    const size_t smem = 1024 + size_t(depth) * rows * 128 * atoms + 16 * depth;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = mc ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = mc ? 1 : 0;
    Result r{0, 0};
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    std::vector<unsigned long long> h(size_t(grid) * 2);
    for (int w = -1; w < reps; ++w) {
        if (flush) ldg_kernel<<<148 * 4, 512>>>(flush, flush_n, sink);
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, stream_kernel, m, c);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (w < 0) continue;
        float t; cudaEventElapsedTime(&t, a, b);
        cudaMemcpy(h.data(), st, h.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long lo = ~0ull, hi = 0;
        for (int i = 0; i < grid; ++i) { lo = std::min(lo, h[2 * i]); hi = std::max(hi, h[2 * i + 1]); }
        r.ev_us += t * 1e3 / reps;
        r.span_us += (hi - lo) * 1e-3 / reps;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  error: %s\n", cudaGetErrorString(e));
    cudaFree(dl); cudaFree(st);
    return r;
}

int main() {
    void *fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    const int K = 4608, N = 4096;
    void *dI; cudaMalloc(&dI, size_t(K) * N * 2); cudaMemset(dI, 1, size_t(K) * N * 2);
    const size_t fb = size_t(512) << 20;
    void *fl; cudaMalloc(&fl, fb); cudaMemset(fl, 0, fb);
    unsigned long long *sink; cudaMalloc(&sink, 64);
    auto mkmap = [&](int rows, int atoms) {
        CUtensorMap m;
        cuuint64_t d3[3] = {64, cuuint64_t(K), cuuint64_t(N / 64)};
        cuuint64_t s3[2] = {cuuint64_t(N) * 2, 128};
        cuuint32_t b3[3] = {64, cuuint32_t(rows), cuuint32_t(atoms)};
        cuuint32_t e3[3] = {1, 1, 1};
        enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dI, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        return m;
    };
    const uint4 *flush = static_cast<const uint4 *>(fl);
    const size_t fn = fb / 16;
    std::mt19937 rng(3);
    const double clk = 1.965e9;
    auto report = [&](const char *what, Result r, double bytes, int grid) {
        printf("%-58s ev %7.2f us  span %7.2f us  %7.1f GB/s(span)  %5.1f B/clk/CTA\n", what, r.ev_us, r.span_us,
               bytes / (r.span_us * 1e-6) / 1e9, bytes / grid / (r.span_us * 1e-6) / clk);
    };
    // ---- A/B: warm L2 (the matrix is 37.7 MB, resident after the first pass), random boxes
    for (int rows : {128, 64}) {
        for (int depth : {2, 3, 4, 6, 8, 12}) {
            const int atoms = 2, stage = rows * 128 * atoms;
            if (size_t(depth) * stage > 200 * 1024) continue;
            for (int grid : {148, 296}) {
                if (grid == 296 && size_t(depth) * stage > 100 * 1024) continue;
                const int steps = 96 * (128 / rows) * 148 / grid;
                std::vector<int2> L(size_t(grid) * steps);
                for (auto &e : L) e = make_int2(int(rng() % (K / rows)) * rows, int(rng() % (N / 128)) * 2);
                CUtensorMap m = mkmap(rows, atoms);
                Result r = run(m, rows, atoms, depth, grid, steps, 0, L, nullptr, 0, sink, 5);
                char w[128];
                snprintf(w, sizeof w, "warm  box %3dx2 (%2d KB) depth %2d grid %d", rows, stage / 1024, depth, grid);
                report(w, r, double(L.size()) * stage, grid);
            }
        }
    }
    // ---- C: warm, multicast pairs (each CTA fetches one atom for both)
    for (int depth : {3, 4, 6}) {
        const int rows = 128, grid = 148, steps = 96;
        std::vector<int2> L(size_t(grid / 2) * steps);
        for (auto &e : L) e = make_int2(int(rng() % (K / rows)) * rows, int(rng() % (N / 128)) * 2);
        CUtensorMap m = mkmap(rows, 1);
        Result r = run(m, rows, 2, depth, grid, steps, 1, L, nullptr, 0, sink, 5);
        char w[128];
        snprintf(w, sizeof w, "warm  multicast pairs box 128x2 depth %d grid %d", depth, grid);
        report(w, r, double(grid) * steps * rows * 256, grid);
    }
    // ---- D: cold, conv10 distinct slabs (1152 boxes of 128 rows x 128 cols) over G CTAs
    for (int grid : {128, 148}) {
        for (int depth : {4, 6}) {
            const int rows = 128;
            const int boxes = (K / rows) * (N / 128);
            const int steps = (boxes + grid - 1) / grid;
            std::vector<int2> L(size_t(grid) * steps);
            for (int g = 0; g < grid; ++g)
                for (int s = 0; s < steps; ++s) {
                    int b = std::min(boxes - 1, g + s * grid);
                    L[size_t(g) * steps + s] = make_int2((b % (K / rows)) * rows, (b / (K / rows)) * 2);
                }
            CUtensorMap m = mkmap(rows, 2);
            Result r = run(m, rows, 2, depth, grid, steps, 0, L, flush, fn, sink, 5);
            char w[128];
            snprintf(w, sizeof w, "cold  conv10 distinct depth %d grid %d (%d steps)", depth, grid, steps);
            report(w, r, double(K) * N * 2, grid);
        }
    }
    // ---- E: cold, conv10 pair pattern (4 tile-rows x 32 col blocks, 18 slabs each, every slab read
    // by two tile-rows at the same step: matchings {01,23} {02,13} {03,12}, 6 steps each)
    {
        const int rows = 128, grid = 128, steps = 18;
        std::vector<int2> L(size_t(grid) * steps);
        const int pairs[3][4] = {{1, 0, 3, 2}, {2, 3, 0, 1}, {3, 2, 1, 0}};
        for (int cb = 0; cb < 32; ++cb)
            for (int t = 0; t < 4; ++t)
                for (int s = 0; s < steps; ++s) {
                    const int mt = s / 6, partner = pairs[mt][t];
                    const int lo = std::min(t, partner);  // slab id unique per (matching, pair, step)
                    const int slab = mt * 12 + (lo == 0 ? 0 : 6) + s % 6;
                    L[size_t(cb * 4 + t) * steps + s] = make_int2(slab * rows, cb * 2);
                }
        for (int depth : {4, 5, 6}) {
            CUtensorMap m = mkmap(rows, 2);
            Result r = run(m, rows, 2, depth, grid, steps, 0, L, flush, fn, sink, 5);
            char w[128];
            snprintf(w, sizeof w, "cold  conv10 pair pattern depth %d grid %d", depth, grid);
            report(w, r, double(K) * N * 2, grid);
        }
    }
    // ---- G: cold LDG.128 read of the same 37.7 MB
    for (int blocks : {296, 592, 1184}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        float tot = 0;
        for (int w = 0; w < 5; ++w) {
            ldg_kernel<<<148 * 4, 512>>>(flush, fn, sink);
            cudaEventRecord(a);
            ldg_kernel<<<blocks, 512>>>(static_cast<const uint4 *>(dI), size_t(K) * N * 2 / 16, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float t; cudaEventElapsedTime(&t, a, b); tot += t;
        }
        printf("cold  LDG.128 37.7 MB, %4d blocks x 512: ev %7.2f us  %7.1f GB/s\n", blocks, tot * 1e3 / 5,
               double(K) * N * 2 / (tot * 1e-3 / 5) / 1e9);
    }
    // ---- H: warm LDG.128 read of the same 37.7 MB (per-SM L2 read ceiling for plain loads)
    for (int blocks : {296, 592}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        ldg_kernel<<<blocks, 512>>>(static_cast<const uint4 *>(dI), size_t(K) * N * 2 / 16, sink);
        cudaEventRecord(a);
        for (int w = 0; w < 10; ++w)
            ldg_kernel<<<blocks, 512>>>(static_cast<const uint4 *>(dI), size_t(K) * N * 2 / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float t; cudaEventElapsedTime(&t, a, b);
        printf("warm  LDG.128 37.7 MB, %4d blocks x 512: ev %7.2f us  %7.1f GB/s\n", blocks, t * 1e3 / 10,
               double(K) * N * 2 / (t * 1e-3 / 10) / 1e9);
    }
    return 0;
}
