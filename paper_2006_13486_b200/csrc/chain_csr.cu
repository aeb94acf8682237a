// chain_csr.cu -- general K-factor chain product in sdmm_reference's order.
//
// Replaces kronsparse.sdmm._csr_rows as driven by sdmm_reference
// (reference sdmm.py:297-330) without materialising the CSR export: the
// column of nonzero j of row u is enumerated in closed form from the factor
// adjacency lists, row-major mixed radix over the factors (rcubs.py:57-76).
// One CTA owns one row u and a 256-column slice; it builds the row's sorted
// column list and values in shared memory once, then every thread runs the
// reference's single accumulation chain  o = fl(o + fl(v_j * x_j))  over
// ascending j for its own column -- bit-identical to the reference in f32
// and f64.  This is the unstructured path (any K, no tiling); the tiled
// kernels of sdmm_simt.cu / sdmm_tc.cu are the fast path for K = 4.
#include "common.cuh"

namespace rbgp4 {
namespace {

constexpr int kMaxFactors = 16;
constexpr int kThreads = 256;

struct ChainParams {
    int32_t k;
    int32_t num_left[kMaxFactors], num_right[kMaxFactors], degree[kMaxFactors];
    int64_t adj_offset[kMaxFactors];
    int64_t rows, row_nnz, n_cols, ld_in, ld_out;
};

template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void __launch_bounds__(kThreads)
chain_row_kernel(const ChainParams p, const int32_t *__restrict__ adjacency,
                 const T *__restrict__ values, const T *__restrict__ inp, T *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *vals = reinterpret_cast<T *>(smem_raw);
    int64_t *cols = reinterpret_cast<int64_t *>(vals + ((p.row_nnz + 1) & ~int64_t(1)));
    const int64_t u = blockIdx.x;

    // left digit of u for every factor (row-major mixed radix)
    __shared__ int32_t digit[kMaxFactors];
    if (threadIdx.x == 0) {
        int64_t rem = u;
        for (int f = p.k - 1; f >= 0; --f) {
            digit[f] = int32_t(rem % p.num_left[f]);
            rem /= p.num_left[f];
        }
    }
    __syncthreads();
    for (int64_t j = threadIdx.x; j < p.row_nnz; j += kThreads) {
        // j in mixed radix over degrees (most significant factor first)
        int64_t rem = j, col = 0, scale = 1;
        for (int f = p.k - 1; f >= 0; --f) {
            int32_t jf = int32_t(rem % p.degree[f]);
            rem /= p.degree[f];
            col += int64_t(adjacency[p.adj_offset[f] + int64_t(digit[f]) * p.degree[f] + jf]) * scale;
            scale *= p.num_right[f];
        }
        cols[j] = col;
        vals[j] = values[u * p.row_nnz + j];
    }
    __syncthreads();
    const int64_t n = int64_t(blockIdx.y) * kThreads + threadIdx.x;
    if (n >= p.n_cols) return;
    T o = T(0);
    for (int64_t j = 0; j < p.row_nnz; ++j) o = add_rn(o, mul_rn(vals[j], inp[cols[j] * p.ld_in + n]));
    out[u * p.ld_out + n] = o;
}

}  // namespace
}  // namespace rbgp4

extern "C" int rbgp4_chain_sdmm(int k, const int32_t *num_left, const int32_t *num_right,
                                const int32_t *degree, const int64_t *adj_offset,
                                const int32_t *adjacency, int dtype, const void *values,
                                const void *inp, void *out, int64_t n_cols, int64_t ld_in,
                                int64_t ld_out, void *stream) {
    using namespace rbgp4;
    RBGP4_REQUIRE(k >= 1 && k <= kMaxFactors, "chain length %d outside [1, %d]", k, kMaxFactors);
    RBGP4_REQUIRE(dtype == RBGP4_F32 || dtype == RBGP4_F64, "chain product supports f32/f64");
    ChainParams p{};
    p.k = k;
    p.rows = 1;
    p.row_nnz = 1;
    for (int f = 0; f < k; ++f) {
        RBGP4_REQUIRE(num_left[f] >= 1 && num_right[f] >= 1 && degree[f] >= 1 &&
                          degree[f] <= num_right[f],
                      "factor %d has invalid sizes (%d, %d, d=%d)", f, num_left[f], num_right[f],
                      degree[f]);
        p.num_left[f] = num_left[f];
        p.num_right[f] = num_right[f];
        p.degree[f] = degree[f];
        p.adj_offset[f] = adj_offset[f];
        p.rows *= num_left[f];
        p.row_nnz *= degree[f];
    }
    RBGP4_REQUIRE(ld_in >= n_cols && ld_out >= n_cols, "leading dimensions smaller than n_cols");
    RBGP4_REQUIRE(p.rows <= 2147483647LL, "too many rows for the grid (%lld)", (long long)p.rows);
    RBGP4_REQUIRE((n_cols + kThreads - 1) / kThreads <= 65535, "too many columns (%lld)",
                  (long long)n_cols);
    p.n_cols = n_cols;
    p.ld_in = ld_in;
    p.ld_out = ld_out;
    if (n_cols == 0 || p.rows == 0) return RBGP4_OK;
    const size_t esz = dtype == RBGP4_F64 ? 8 : 4;
    const size_t smem = ((p.row_nnz + 1) & ~int64_t(1)) * esz + p.row_nnz * sizeof(int64_t);
    RBGP4_REQUIRE(smem <= 227 * 1024, "row_nnz %lld too large for the chain kernel",
                  (long long)p.row_nnz);
    dim3 grid(unsigned(p.rows), unsigned((n_cols + kThreads - 1) / kThreads));
    auto s = static_cast<cudaStream_t>(stream);
    note_kernel("chain");
    if (dtype == RBGP4_F32) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(chain_row_kernel<float>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        chain_row_kernel<float><<<grid, kThreads, smem, s>>>(
            p, adjacency, static_cast<const float *>(values), static_cast<const float *>(inp),
            static_cast<float *>(out));
    } else {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(chain_row_kernel<double>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        chain_row_kernel<double><<<grid, kThreads, smem, s>>>(
            p, adjacency, static_cast<const double *>(values), static_cast<const double *>(inp),
            static_cast<double *>(out));
    }
    RBGP4_CHECK_LAUNCH("chain_row_kernel launch");
    return RBGP4_OK;
}

// Raw CSR triple (sdmm_reference(CsrMatrix), reference sdmm.py:307-330): same
// single ascending chain per output, explicit indices instead of the closed form.
namespace rbgp4 {
namespace {
template <typename T>
__global__ void __launch_bounds__(kThreads)
csr_row_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
               const T *__restrict__ values, const T *__restrict__ inp, T *__restrict__ out,
               int64_t n_cols, int64_t ld_in, int64_t ld_out) {
    const int64_t u = blockIdx.x;
    const int64_t n = int64_t(blockIdx.y) * kThreads + threadIdx.x;
    if (n >= n_cols) return;
    T o = T(0);
    for (int64_t p = indptr[u]; p < indptr[u + 1]; ++p)
        o = add_rn(o, mul_rn(values[p], inp[int64_t(indices[p]) * ld_in + n]));
    out[u * ld_out + n] = o;
}
}  // namespace
}  // namespace rbgp4

extern "C" int rbgp4_csr_sdmm(int64_t rows, const int64_t *indptr, const int32_t *indices,
                              int dtype, const void *values, const void *inp, void *out,
                              int64_t n_cols, int64_t ld_in, int64_t ld_out, void *stream) {
    using namespace rbgp4;
    RBGP4_REQUIRE(dtype == RBGP4_F32 || dtype == RBGP4_F64, "CSR product supports f32/f64");
    RBGP4_REQUIRE(rows >= 0 && rows <= 2147483647LL, "bad row count %lld", (long long)rows);
    RBGP4_REQUIRE(ld_in >= n_cols && ld_out >= n_cols, "leading dimensions smaller than n_cols");
    RBGP4_REQUIRE((n_cols + kThreads - 1) / kThreads <= 65535, "too many columns");
    if (rows == 0 || n_cols == 0) return RBGP4_OK;
    dim3 grid(unsigned(rows), unsigned((n_cols + kThreads - 1) / kThreads));
    auto s = static_cast<cudaStream_t>(stream);
    note_kernel("csr");
    if (dtype == RBGP4_F32)
        csr_row_kernel<float><<<grid, kThreads, 0, s>>>(
            indptr, indices, static_cast<const float *>(values), static_cast<const float *>(inp),
            static_cast<float *>(out), n_cols, ld_in, ld_out);
    else
        csr_row_kernel<double><<<grid, kThreads, 0, s>>>(
            indptr, indices, static_cast<const double *>(values), static_cast<const double *>(inp),
            static_cast<double *>(out), n_cols, ld_in, ld_out);
    RBGP4_CHECK_LAUNCH("csr_row_kernel launch");
    return RBGP4_OK;
}
