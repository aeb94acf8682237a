// tma_bench.cu -- how fast can one CTA per SM stream a K x N bf16 matrix into
// shared memory with TMA, as a function of box shape / boxes per stage / ring
// depth?  (Diagnostic for the I-slab stream of sdmm_tc.cu; not product code.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_bench.cu -o /tmp/tma_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct Cfg {
    int rows_per_box;   // box outer extent (K rows)
    int atoms;          // 128-byte column atoms per stage (tn = 64 * atoms)
    int depth;          // ring depth
    int steps;          // stages per CTA
    int use3d;          // one 3-D box per stage instead of `atoms` 2-D boxes
    int col_blocks;     // column blocks (CTAs along N)
    int k_groups;       // CTAs along K (different row ranges)
    const int *slabs;   // optional (k_groups x steps) slab index list: row = slab * rows_per_box
};

__global__ void __launch_bounds__(32, 1)
stream_kernel(const __grid_constant__ CUtensorMap map2, const __grid_constant__ CUtensorMap map3,
              Cfg c, unsigned long long *sink) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int stage_bytes = c.rows_per_box * 128 * c.atoms;
    uint64_t *bars = reinterpret_cast<uint64_t *>(buf + c.depth * stage_bytes);
    if (threadIdx.x != 0) return;
    for (int i = 0; i < c.depth; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int cb = blockIdx.x % c.col_blocks, kg = blockIdx.x / c.col_blocks;
    const int n0 = cb * 64 * c.atoms;
    const int k0 = kg * c.steps * c.rows_per_box;
    auto issue = [&](int s) {
        const int st = s % c.depth;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[st])),
                     "r"(stage_bytes) : "memory");
        unsigned char *dst = buf + st * stage_bytes;
        const int krow = c.slabs ? c.slabs[kg * c.steps + s] * c.rows_per_box : k0 + s * c.rows_per_box;
        if (c.use3d) {
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
                         "l"(reinterpret_cast<uint64_t>(&map3)), "r"(0), "r"(krow), "r"(n0 / 64),
                         "r"(smem_u32(&bars[st])) : "memory");
        } else {
            for (int a = 0; a < c.atoms; ++a)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst + a * c.rows_per_box * 128)),
                             "l"(reinterpret_cast<uint64_t>(&map2)), "r"(n0 + a * 64), "r"(krow),
                             "r"(smem_u32(&bars[st])) : "memory");
        }
    };
    for (int s = 0; s < c.depth && s < c.steps; ++s) issue(s);
    unsigned long long acc = 0;
    for (int s = 0; s < c.steps; ++s) {
        const int st = s % c.depth;
        const uint32_t ph = (s / c.depth) & 1;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                     "@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bars[st])), "r"(ph) : "memory");
        acc += buf[st * stage_bytes + (s & 127)];
        if (s + c.depth < c.steps) issue(s + c.depth);
    }
    sink[blockIdx.x] = acc;
}

// read-only L2 flush: leaves L2 full of clean lines (no write-back traffic afterwards)
__global__ void flush_read(const uint4 *p, size_t n, unsigned long long *sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        acc ^= p[i].x;
    if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char **argv) {
    const int K = 4608, N = 4096;
    void *dI;
    cudaMalloc(&dI, size_t(K) * N * 2);
    cudaMemset(dI, 1, size_t(K) * N * 2);
    const size_t flush_bytes = size_t(512) << 20;
    void *flush;
    cudaMalloc(&flush, flush_bytes);
    cudaMemset(flush, 0, flush_bytes);
    unsigned long long *sink;
    cudaMalloc(&sink, 4096 * 8);
    void *fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    struct Case { int rpb, atoms, depth, use3d, kgroups; };
    std::vector<Case> cases = {
        {64, 2, 7, 0, 1}, {64, 2, 7, 1, 1}, {64, 2, 12, 0, 1}, {128, 2, 6, 0, 1},
        {256, 2, 3, 0, 1}, {64, 4, 6, 0, 1}, {64, 4, 6, 1, 1}, {256, 1, 6, 0, 1},
        {64, 2, 7, 0, 4}, {128, 4, 3, 1, 4}, {32, 2, 12, 0, 1}, {64, 1, 12, 0, 2},
    };
    // the conv10 RBGP4 pattern: 4 tile-rows, 36 of 72 slabs each, every slab used twice
    std::vector<int> slab_list;
    {
        srand(7);
        for (int tr = 0; tr < 4; ++tr) {
            std::vector<int> all(72);
            for (int i = 0; i < 72; ++i) all[i] = i;
            // pairs of tile-rows share complementary halves: (0,1) take odd/even halves etc.
            for (int i = 0; i < 72; ++i) if ((i / 2 + tr) % 2 == 0) slab_list.push_back(i);
        }
    }
    // random variant: a random biregular (4 x 72, d=36) pattern, each slab used by 2 tile-rows
    std::vector<int> rnd_list;
    {
        srand(11);
        std::vector<int> owners;  // 72 slabs x 2 owners
        for (int attempt = 0; attempt < 1000; ++attempt) {
            std::vector<std::vector<int>> rows(4);
            std::vector<int> stubs;
            for (int sl = 0; sl < 72; ++sl) { stubs.push_back(sl); stubs.push_back(sl); }
            for (int i = int(stubs.size()) - 1; i > 0; --i) std::swap(stubs[i], stubs[rand() % (i + 1)]);
            bool ok = true;
            for (int tr = 0; tr < 4 && ok; ++tr) {
                for (int j = 0; j < 36; ++j) rows[tr].push_back(stubs[tr * 36 + j]);
                std::sort(rows[tr].begin(), rows[tr].end());
                for (int j = 1; j < 36; ++j) if (rows[tr][j] == rows[tr][j - 1]) ok = false;
            }
            if (!ok) continue;
            for (int tr = 0; tr < 4; ++tr) rnd_list.insert(rnd_list.end(), rows[tr].begin(), rows[tr].end());
            break;
        }
    }
    int *d_rnd;
    cudaMalloc(&d_rnd, rnd_list.size() * sizeof(int));
    cudaMemcpy(d_rnd, rnd_list.data(), rnd_list.size() * sizeof(int), cudaMemcpyHostToDevice);
    int *d_slabs;
    cudaMalloc(&d_slabs, slab_list.size() * sizeof(int));
    cudaMemcpy(d_slabs, slab_list.data(), slab_list.size() * sizeof(int), cudaMemcpyHostToDevice);
    // full-row boxes: 3-D box covering all 64 column atoms of `rpb` rows (contiguous DRAM)
    cases.push_back({2, 64, 6, 1, 128});
    cases.push_back({4, 64, 4, 1, 128});
    cases.push_back({2, 32, 8, 1, 64});
    cases.push_back({8, 16, 6, 1, 32});
    cases.push_back({64, 2, 8, 1, -4});
    cases.push_back({64, 4, 4, 1, -4});
    cases.push_back({64, 2, 8, 0, -4});
    cases.push_back({64, 2, 8, 1, -104});   // random slab lists
    cases.push_back({64, 4, 4, 1, -104});
    // steady-state read bandwidth: LDG.128 over the 512 MB flush buffer
    for (int blocks : {592, 1184, 2368}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        flush_read<<<blocks, 512>>>(static_cast<const uint4 *>(flush), flush_bytes / 16, sink + 4000);
        cudaEventRecord(a);
        for (int w = 0; w < 5; ++w)
            flush_read<<<blocks, 512>>>(static_cast<const uint4 *>(flush), flush_bytes / 16, sink + 4000);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float t; cudaEventElapsedTime(&t, a, b);
        printf("LDG.128 read 512 MB x5, %d blocks: %8.2f us per pass %7.1f GB/s\n", blocks, t * 1e3 / 5,
               double(flush_bytes) * 5 / (t * 1e-3) / 1e9);
    }
    // baseline: plain LDG.128 streaming of the same matrix by many warps, cold L2
    for (int blocks : {148, 296, 592, 1184}) {
        float tot = 0;
        for (int w = 0; w < 10; ++w) {
            flush_read<<<148 * 4, 512>>>(static_cast<const uint4 *>(flush), flush_bytes / 16, sink + 4000);
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            flush_read<<<blocks, 512>>>(static_cast<const uint4 *>(dI), size_t(K) * N * 2 / 16, sink + 4001);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float t; cudaEventElapsedTime(&t, a, b); tot += t;
        }
        const double us = tot * 1e3 / 10;
        printf("LDG.128 read, %d blocks x 512 thr: %8.2f us %7.1f GB/s\n", blocks, us,
               double(K) * N * 2 / (us * 1e-6) / 1e9);
    }
    for (auto cs : cases) {
        CUtensorMap m2, m3;
        cuuint64_t d2[2] = {cuuint64_t(N), cuuint64_t(K)};
        cuuint64_t s2[1] = {cuuint64_t(N) * 2};
        cuuint32_t b2[2] = {64, cuuint32_t(cs.rpb)};
        cuuint32_t e2[3] = {1, 1, 1};
        enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dI, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        // 3-D view: (64 cols inner, K rows, N/64 atoms) -> box (64, rows, atoms) lands atom-major
        cuuint64_t d3[3] = {64, cuuint64_t(K), cuuint64_t(N / 64)};
        cuuint64_t s3[2] = {cuuint64_t(N) * 2, 128};
        cuuint32_t b3[3] = {64, cuuint32_t(cs.rpb), cuuint32_t(cs.atoms)};
        CUresult r3 = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dI, d3, s3, b3, e2,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cs.use3d && r3 != CUDA_SUCCESS) { printf("3d map failed %d\n", int(r3)); continue; }
        Cfg c;
        c.rows_per_box = cs.rpb; c.atoms = cs.atoms; c.depth = cs.depth; c.use3d = cs.use3d;
        c.col_blocks = N / (64 * cs.atoms);
        c.slabs = nullptr;
        if (cs.kgroups < 0) {   // slab-list mode
            c.k_groups = (-cs.kgroups) % 100;
            c.steps = 36;
            c.slabs = cs.kgroups < -100 ? d_rnd : d_slabs;
        } else {
            c.k_groups = cs.kgroups;
            c.steps = K / cs.rpb / cs.kgroups;
        }
        const int grid = c.col_blocks * c.k_groups;
        const size_t smem = 1024 + size_t(c.depth) * cs.rpb * 128 * cs.atoms + 8 * c.depth;
        cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        for (int w = 0; w < 3; ++w) stream_kernel<<<grid, 32, smem>>>(m2, m3, c, sink);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        const int reps = 10;
        float ms = 0;
        for (int w = 0; w < reps; ++w) {
            flush_read<<<148 * 4, 512>>>(static_cast<const uint4 *>(flush), flush_bytes / 16, sink + 4000);
            cudaEventRecord(a);
            stream_kernel<<<grid, 32, smem>>>(m2, m3, c, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float t;
            cudaEventElapsedTime(&t, a, b);
            ms += t;
        }
        cudaError_t e = cudaGetLastError();
        const double us = ms * 1e3 / reps;
        printf("rows/box %3d atoms %d depth %2d 3d %d kgroups %d grid %4d smem %6zu : %8.2f us  %7.1f GB/s %s\n",
               cs.rpb, cs.atoms, cs.depth, cs.use3d, cs.kgroups, grid, smem, us,
               double(grid) * c.steps * cs.rpb * 128 * cs.atoms / (us * 1e-6) / 1e9,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
