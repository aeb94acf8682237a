// sddmm.cu -- the training direction's weight gradient restricted to the RBGP4 pattern
// (the paper trains with fixed masks):
//
//     dW[u, j] = sum_n dO[u, n] * I[c(u, j), n]      for every stored slot j of row u
//
// with the closed-form column map c(u, j) of sdmm.py:173-184.  The result has
// the layout of RcubsMatrix.values (rows, row_nnz) -- the gradient never leaves the succinct
// format.  One CTA per row u stages dO[u, :] in shared memory; each warp owns a stored slot j
// at a time and reduces over n with coalesced 16-byte loads of I's row c(u, j) and a warp
// shuffle tree.  Accumulation is fp32 for f32 operands and fp64 for f64 (FFMA).
#include "common.cuh"

namespace rbgp4 {
namespace {

constexpr int kSThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kSThreads)
sddmm_kernel(const ChainDims c, const int32_t *__restrict__ adj_o, const int32_t *__restrict__ adj_i,
             const T *__restrict__ dout, int64_t ld_do, const T *__restrict__ inp, int64_t ld_in,
             T *__restrict__ grad, int64_t n_chunk) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *drow = reinterpret_cast<T *>(smem_raw);
    const int64_t u = blockIdx.x;
    // row digits (uo, rm, ui, m): u = ((uo*rm + r)*u_i + ui)*bm + m  (sdmm.py:186,197)
    const int m = int(u % c.bm);
    const int ui = int((u / c.bm) % c.u_i);
    const int uo = int(u / (int64_t(c.bm) * c.u_i * c.rm));
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    constexpr int kWarps = kSThreads / 32;
    (void)m;
    for (int64_t j0 = 0; j0 < c.row_nnz; j0 += kWarps) {
        // (the dO row is re-staged per chunk of n when N exceeds the shared buffer)
        const int64_t j = j0 + warp;
        int64_t col = 0;
        if (j < c.row_nnz) {
            // slot j <-> (s, rk, ink, k), column ((adj_o[uo][s]*rk + r)*v_i + adj_i[ui][ink])*bk + k
            const int k = int(j % c.bk);
            const int64_t q = j / c.bk;
            const int ink = int(q % c.d_i);
            const int64_t q2 = q / c.d_i;
            const int r = int(q2 % c.rk);
            const int s = int(q2 / c.rk);
            col = ((int64_t(adj_o[int64_t(uo) * c.d_o + s]) * c.rk + r) * c.v_i + adj_i[ui * c.d_i + ink]) * c.bk + k;
        }
        T acc = T(0);
        for (int64_t n0 = 0; n0 < c.n_cols; n0 += n_chunk) {
            const int64_t nn = min(n_chunk, c.n_cols - n0);
            __syncthreads();
            for (int64_t i = threadIdx.x; i < nn; i += kSThreads) drow[i] = dout[u * ld_do + n0 + i];
            __syncthreads();
            if (j < c.row_nnz) {
                const T *irow = inp + col * ld_in + n0;
                for (int64_t i = lane; i < nn; i += 32) acc = fma(drow[i], irow[i], acc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o /= 2) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (j < c.row_nnz && lane == 0) grad[u * c.row_nnz + j] = acc;
    }
}

}  // namespace
}  // namespace rbgp4

extern "C" int rbgp4_sddmm(const rbgp4_desc *desc, int dtype, const int32_t *adj_o, const int32_t *adj_i,
                           const void *d_out, int64_t ld_do, const void *inp, int64_t ld_in, void *grad_values,
                           void *stream) {
    using namespace rbgp4;
    ChainDims c;
    rbgp4_desc d = *desc;
    // the descriptor's ld_in/ld_out are those of the forward product; SDDMM takes its own
    d.ld_in = d.ld_out = d.n_cols;
    int rc = validate_desc(&d, &c);
    if (rc != RBGP4_OK) return rc;
    RBGP4_REQUIRE(dtype == RBGP4_F32 || dtype == RBGP4_F64 || dtype == RBGP4_BF16,
                  "rbgp4_sddmm: F32, F64 or BF16 operands");
    RBGP4_REQUIRE(ld_do >= c.n_cols && ld_in >= c.n_cols, "rbgp4_sddmm: leading dimensions < n_cols");
    RBGP4_REQUIRE(adj_o && adj_i && grad_values && (c.n_cols == 0 || (d_out && inp)), "rbgp4_sddmm: null pointer");
    if (c.rows == 0) return RBGP4_OK;
    if (dtype == RBGP4_BF16)  // tensor cores (sddmm_tc.cu): bf16 dO / I, f32 gradient
        return launch_sddmm_tc(c, adj_o, adj_i, d_out, ld_do, inp, ld_in, static_cast<float *>(grad_values),
                               static_cast<cudaStream_t>(stream));
    const int esz = dtype == RBGP4_F32 ? 4 : 8;
    const int64_t n_chunk = std::max<int64_t>(1, std::min<int64_t>(c.n_cols, (32 * 1024) / esz));
    const size_t smem = size_t(n_chunk) * esz;
    auto s = static_cast<cudaStream_t>(stream);
    if (dtype == RBGP4_F32)
        sddmm_kernel<float><<<unsigned(c.rows), kSThreads, smem, s>>>(
            c, adj_o, adj_i, static_cast<const float *>(d_out), ld_do, static_cast<const float *>(inp), ld_in,
            static_cast<float *>(grad_values), n_chunk);
    else
        sddmm_kernel<double><<<unsigned(c.rows), kSThreads, smem, s>>>(
            c, adj_o, adj_i, static_cast<const double *>(d_out), ld_do, static_cast<const double *>(inp), ld_in,
            static_cast<double *>(grad_values), n_chunk);
    RBGP4_CHECK_LAUNCH("sddmm_kernel launch");
    return RBGP4_OK;
}

// the nn.Linear layout: d_out_nk (n_cols x rows, row stride ld_do) = dO^T, inp_nk (n_cols x cols,
// row stride ld_in) = I^T, bf16 only (K7 with MN-major operands): no transposed copies
extern "C" int rbgp4_sddmm_nk(const rbgp4_desc *desc, const int32_t *adj_o, const int32_t *adj_i,
                              const void *d_out_nk, int64_t ld_do, const void *inp_nk, int64_t ld_in,
                              void *grad_values, void *stream) {
    using namespace rbgp4;
    ChainDims c;
    rbgp4_desc d = *desc;
    d.ld_in = d.ld_out = d.n_cols;
    int rc = validate_desc(&d, &c);
    if (rc != RBGP4_OK) return rc;
    RBGP4_REQUIRE(ld_do >= c.rows && ld_in >= c.cols, "rbgp4_sddmm_nk: leading dimensions < rows / cols");
    RBGP4_REQUIRE(adj_o && adj_i && grad_values && (c.n_cols == 0 || (d_out_nk && inp_nk)),
                  "rbgp4_sddmm_nk: null pointer");
    if (c.rows == 0) return RBGP4_OK;
    return launch_sddmm_tc(c, adj_o, adj_i, d_out_nk, ld_do, inp_nk, ld_in, static_cast<float *>(grad_values),
                           static_cast<cudaStream_t>(stream), true);
}
