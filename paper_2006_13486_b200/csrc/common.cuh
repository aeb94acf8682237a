// common.cuh -- shared plumbing of the RBGP4 CUDA library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <algorithm>

#include "../../include/rbgp4.h"

namespace rbgp4 {

// thread-local last-error text behind rbgp4_last_error()
void set_error(const char *fmt, ...);
// count a kernel launch for rbgp4_launch_count()
void note_launch(int n = 1);

#define RBGP4_CHECK_LAUNCH(what)                                                   \
    do {                                                                           \
        cudaError_t e__ = cudaGetLastError();                                      \
        if (e__ != cudaSuccess) {                                                  \
            ::rbgp4::set_error("%s: %s", what, cudaGetErrorString(e__));           \
            return RBGP4_ECUDA;                                                    \
        }                                                                          \
        ::rbgp4::note_launch();                                                    \
    } while (0)

#define RBGP4_REQUIRE(cond, ...)                                                   \
    do {                                                                           \
        if (!(cond)) {                                                             \
            ::rbgp4::set_error(__VA_ARGS__);                                       \
            return RBGP4_EINVAL;                                                   \
        }                                                                          \
    } while (0)

constexpr int kNumSMs = 148;

// Derived sizes of a four-factor chain (SURVEY §8 notation).
struct ChainDims {
    int64_t rows, cols, n_cols, ld_in, ld_out;
    int32_t u_o, v_o, d_o, rm, rk, u_i, v_i, d_i, bm, bk;
    int32_t tm, tk, d_t, g;  // W tile rows/cols, nonzeros per tile row, row-group size
    int64_t row_nnz;
};

int validate_desc(const rbgp4_desc *d, ChainDims *out);

// SIMT launchers (sdmm_simt.cu)
int launch_simt(const ChainDims &c, int compute, int dtype, const void *values,
                const int32_t *adj_o, const int32_t *adj_i, const void *inp, void *out,
                cudaStream_t stream);
int simt_supported(const ChainDims &c, int dtype);

// tcgen05 launchers (sdmm_tc.cu)
int launch_tc(const ChainDims &c, int compute, int out_dtype, const void *values,
              const int32_t *adj_o, const int32_t *adj_i, const void *prep, const void *inp,
              void *out, void *workspace, size_t workspace_bytes, cudaStream_t stream);
size_t tc_prep_size(const ChainDims &c, int compute);
int tc_prepare(const ChainDims &c, int compute, const void *values, const int32_t *adj_o, const int32_t *adj_i,
               void *prep, size_t bytes,
               cudaStream_t stream);
int tc_supported(const ChainDims &c, int compute, int out_dtype);
size_t conv_workspace_size(const ChainDims &c, const rbgp4_conv_desc *cv);
int launch_conv(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, const void *values,
                const int32_t *adj_o, const int32_t *adj_i, const void *prep, const void *x,
                void *out, void *workspace, size_t workspace_bytes, cudaStream_t stream);
size_t tc_workspace_size(const ChainDims &c, int compute);

// K4: gathered-block tcgen05 launchers (sdmm_gather.cu); `k4` = the prepared relayout
// section of rbgp4_prepare (null: direct mode on RcubsMatrix.values as stored)
int gather_relayout_ok(const ChainDims &c);
int gather_supported(const ChainDims &c, int compute, int out_dtype, bool relayout);
int launch_gather(const ChainDims &c, int out_dtype, const void *values, const int32_t *adj_o,
                  const int32_t *adj_i, const int32_t *sched, const int32_t *pair, const void *k4,
                  const void *inp, void *out, cudaStream_t stream);
int gather_conv_supported(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, bool relayout);
int launch_gather_conv(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, const void *values,
                       const int32_t *adj_o, const int32_t *adj_i, const int32_t *sched, const int32_t *pair,
                       const void *k4, const void *x, void *out, cudaStream_t stream);
size_t gather_prep_bytes(const ChainDims &c);
int gather_prepare(const ChainDims &c, const void *values, const int32_t *adj_i_host, void *k4,
                   cudaStream_t stream);

}  // namespace rbgp4
