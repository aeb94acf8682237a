// tma_par_bench.cu -- does TMA load throughput per SM grow with the number of issuing threads
// or CTAs?  Diagnostic for the K5 producers (not product code).  Warm L2 (a 37.7 MB bf16
// tensor, resident after the first pass); every CTA has `nw` issuing warps, each streaming
// random boxes through its own ring of `depth` stages (wait for the oldest box to land, reuse
// its slot).  Reports B/clk per SM for 1 or 2 CTAs per SM and 3-D / 2-D box shapes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_par_bench.cu -o tools/tma_par_bench.bin -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

struct Cfg {
    int dims, rows, atoms, bytes, depth, steps, krows, nat;
    const int2 *list;  // [grid * nw][steps] (krow, atom)
};

__global__ void par_kernel(const __grid_constant__ CUtensorMap m, Cfg c) {
    extern __shared__ unsigned char raw[];
    unsigned char *buf = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int w = threadIdx.x / 32, nw = blockDim.x / 32;
    uint64_t *bars = reinterpret_cast<uint64_t *>(buf + size_t(nw) * c.depth * c.bytes);
    uint64_t *full = bars + w * c.depth;
    unsigned char *ring = buf + size_t(w) * c.depth * c.bytes;
    if (threadIdx.x % 32 != 0) return;
    for (int i = 0; i < c.depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int2 *L = c.list + (size_t(blockIdx.x) * nw + w) * c.steps;
    auto issue = [&](int s) {
        const int st = s % c.depth;
        const uint32_t dst = su32(ring + size_t(st) * c.bytes);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(c.bytes) : "memory");
        const int2 e = L[s];
        if (c.dims == 4)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(dst), "l"(&m), "r"(0), "r"((e.x & 3) - 1), "r"(e.x >> 2), "r"(e.y), "r"(su32(&full[st])) : "memory");
        else if (c.dims == 3)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(dst), "l"(&m), "r"(0), "r"(e.x), "r"(e.y), "r"(su32(&full[st])) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(dst), "l"(&m), "r"(e.y * 64), "r"(e.x), "r"(su32(&full[st])) : "memory");
    };
    for (int s = 0; s < c.depth && s < c.steps; ++s) issue(s);
    for (int s = 0; s < c.steps; ++s) {
        const int st = s % c.depth;
        const uint32_t ph = (s / c.depth) & 1;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                     ::"r"(su32(&full[st])), "r"(ph) : "memory");
        if (s + c.depth < c.steps) issue(s + c.depth);
    }
}

int main() {
    void *fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    const int K = 4608, N = 4096;
    void *dI;
    cudaMalloc(&dI, size_t(K) * N * 2);
    cudaMemset(dI, 1, size_t(K) * N * 2);
    std::mt19937 rng(7);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double clk = clk_khz * 1e3;
    struct Shape { const char *name; int dims, rows, atoms; };
    // dims 4: NHWC conv boxes over a (64 ch, W, W, B) bf16 tensor: rows = W (map width), atoms =
    // image rows per box (W x atoms x (128 / (W x atoms)) images = 128 pixels)
    const Shape shapes[] = {{"4d conv 32x32 box 32x4x1", 4, 32, 4}, {"4d conv 8x8 box 8x8x2", 4, 8, 8},
                            {"4d conv 4x4 box 4x4x8", 4, 4, 4},{"3d 64x128x2 (32 KB)", 3, 128, 2}, {"3d 64x64x2 (16 KB)", 3, 64, 2},
                            {"3d 64x32x2 (8 KB)", 3, 32, 2}, {"2d 64x128 (16 KB)", 2, 128, 1},
                            {"2d 64x256 (32 KB)", 2, 256, 1}};
    for (const Shape &sh : shapes) {
        CUtensorMap m;
        const int bytes = sh.dims == 4 ? 128 * 128 : sh.rows * 128 * sh.atoms;
        int nimg = 0;
        if (sh.dims == 4) {
            const int W = sh.rows, hb = sh.atoms, tb = 128 / (W * hb);
            nimg = int((size_t(K) * N * 2) / (size_t(W) * W * 128));
            cuuint64_t d4[4] = {64, cuuint64_t(W), cuuint64_t(W), cuuint64_t(nimg)};
            cuuint64_t s4[3] = {128, cuuint64_t(W) * 128, cuuint64_t(W) * W * 128};
            cuuint32_t b4[4] = {64, cuuint32_t(W), cuuint32_t(hb > W ? W : hb), cuuint32_t(tb)};
            cuuint32_t e4[4] = {1, 1, 1, 1};
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dI, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else if (sh.dims == 3) {
            cuuint64_t d3[3] = {64, cuuint64_t(K), cuuint64_t(N / 64)};
            cuuint64_t s3[2] = {cuuint64_t(N) * 2, 128};
            cuuint32_t b3[3] = {64, cuuint32_t(sh.rows), cuuint32_t(sh.atoms)};
            cuuint32_t e3[3] = {1, 1, 1};
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dI, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t d2[2] = {cuuint64_t(N), cuuint64_t(K)};
            cuuint64_t s2[1] = {cuuint64_t(N) * 2};
            cuuint32_t b2[2] = {64, cuuint32_t(sh.rows)};
            cuuint32_t e2[2] = {1, 1};
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dI, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        for (int cps : {1, 2}) {
            for (int nw : {1, 2, 4}) {
                const size_t budget = (cps == 1 ? 200 : 100) * 1024;
                int depth = int(budget / (size_t(nw) * bytes));
                if (depth > 8) depth = 8;
                if (depth < 2) continue;
                const int grid = 148 * cps;
                const int steps = int((size_t(768) << 20) / (size_t(grid) * nw * bytes));  // ~768 MB moved
                std::vector<int2> L(size_t(grid) * nw * steps);
                if (sh.dims == 4) {
                    const int W = sh.rows, hb = sh.atoms > W ? W : sh.atoms, tb = 128 / (W * hb);
                    // e.x = (output row h0 + tap row) << 2 | tap col (0..2); e.y = first image
                    for (auto &e : L)
                        e = make_int2((int(rng() % (W / hb)) * hb + int(rng() % 3) - 1) * 4 + int(rng() % 3),
                                      int(rng() % (nimg / tb)) * tb);
                } else {
                    for (auto &e : L) e = make_int2(int(rng() % (K / sh.rows)) * sh.rows, int(rng() % (N / 64 / sh.atoms)) * sh.atoms);
                }
                int2 *dl;
                cudaMalloc(&dl, L.size() * sizeof(int2));
                cudaMemcpy(dl, L.data(), L.size() * sizeof(int2), cudaMemcpyHostToDevice);
                Cfg c{sh.dims, sh.rows, sh.atoms, bytes, depth, steps, K, N / 64, dl};
                const size_t smem = 1024 + size_t(nw) * depth * (bytes + 8);
                cudaFuncSetAttribute(par_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                par_kernel<<<grid, 32 * nw, smem>>>(m, c);  // warm-up (fills L2)
                cudaEventRecord(a);
                for (int r = 0; r < 5; ++r) par_kernel<<<grid, 32 * nw, smem>>>(m, c);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float t;
                cudaEventElapsedTime(&t, a, b);
                const double sec = t * 1e-3 / 5;
                const double total = double(grid) * nw * steps * bytes;
                printf("%-22s CTAs/SM %d warps %d depth %d: %7.1f us  %7.1f GB/s  %5.1f B/clk/SM\n", sh.name, cps, nw,
                       depth, sec * 1e6, total / sec / 1e9, total / sec / 148 / clk);
                cudaFree(dl);
            }
        }
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
