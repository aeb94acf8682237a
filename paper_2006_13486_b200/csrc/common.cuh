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
// record the kernel family of the current launch for rbgp4_last_kernel() (static string)
void note_kernel(const char *name);

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

// Ablation / tracing hooks inside the kernels exist only in debug builds of the library
// (-DRBGP4_DEBUG=1, `python -m paper_2006_13486_b200.build --debug`); in the release library
// DBG(x) is the constant 0 and every such branch is compiled out.
#ifndef RBGP4_DEBUG
#define RBGP4_DEBUG 0
#endif
#define DBG(x) (RBGP4_DEBUG ? (x) : 0)

// Plan overrides (rbgp4_set_option / rbgp4_get_option, include/rbgp4.h).  Thread-local: a
// setting affects only launches planned on the thread that made it, so concurrent callers
// never see each other's A/B switches.  The defaults are the production plan.
struct Options {
    int32_t relayout = -1;    // K4 values relayout: -1 auto, 0 off, 1 wherever admissible
    int32_t dense = 0;        // 1: bf16 always on the densify kernel (K2), never K4
    int32_t persistent = -1;  // persistent tile loop: -1 auto (K4) / off (K2), 0 off, 1 on
    int32_t msplit = 0;       // K4 row-half split over a 2-CTA cluster (opt-in)
    int32_t ksplit = 0;       // split-K slices: 0 auto, else forced (1..8)
    int32_t stages = 0;       // K4 ring stages: 0 auto, else forced (2..16)
    int32_t multicast = -1;   // K4 multicast pairs: -1 auto, 0 off
    int32_t sym = 1;          // K4 symmetric split-K epilogue
    int32_t pdl = 1;          // programmatic dependent launch attribute
    int32_t simt_ct = 0;      // K1 column threads per CTA: 0 auto, else 8 / 16 / 32
    int32_t tc_tn = 0;        // K2 tile columns: 0 auto
    int32_t tc_na = 0;        // K2 A-ring depth: 0 auto
    int32_t tc_nb = 0;        // K2 I-ring depth: 0 auto
    int32_t tc_nw = 0;        // K2 W-ring depth: 0 auto
    int32_t wswz = 1;         // K2 swizzled W staging
    int32_t ostore = 1;       // K2 TMA-store epilogue
    int32_t sched = 1;        // rbgp4_prepare: paired step schedule (0: adjacency order)
    int32_t i3d = 1;          // K2 3-D I boxes
    int32_t promo = -1;       // K2 I-map L2 promotion bytes: -1 auto (256), 0 / 64 / 128 / 256
    int32_t conv_wide = 1;    // K2 conv: 256-pixel tiles for many-wave grids
    int32_t stream = -1;      // K5 (sdmm_stream.cu) for the TC16 SDMM: -1 auto, 0 off (K4)
    int32_t stream_g = 0;     // K5 row blocks per unit: 0 auto, else 1 / 2 / 4 / 8 (whole tiles)
    int32_t halo = -1;        // K5 halo-strip conv where admissible: -1 auto, 0 off
    int32_t simt_wide = -1;   // K1 wide f32 kernel (16 rows x 4 columns per thread): -1 auto, 0 off
    int32_t merge = -1;       // K5: two tile-rows per unit when g_o is complete: -1 auto, 0 off
    int32_t conv_ostage = 1;  // K5 conv: staged TMA-store epilogue (bf16, no pool / residual): 1 on, 0 off
    int32_t simt_ksplit = 0;  // K1 wide ffma step halving over a cluster pair: 0 auto, 1 off, 2 on
    int32_t stream_ctas = 0;  // K5 grid cap: 0 auto (one CTA per SM), else at most this many CTAs
    int32_t debug = 0;        // trace / ablation bits (debug builds only)
};
Options &opts();

// Residual epilogue of the convolution (rbgp4_conv2d_residual, the WRN block tail): set for the
// duration of one call on the calling thread; only the streamed conv (K5) honours it, every other
// conv path refuses a call that sets it.
struct ConvEpilogue {
    const void *res = nullptr;  // O = round(conv) + res  (NHWC, the output's dtype)
    void *out2 = nullptr;       // and relu(O) here
};
ConvEpilogue &conv_epilogue();

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
void gather_prep_views(const ChainDims &c, const void *k4, const int32_t **cols, const void **vals);

// K5: streamed tcgen05 SDMM / conv (sdmm_stream.cu); `k5` = its prepared tables (step words, row
// groups for TC16; slice relayout for other block shapes)
int stream_shape_ok(const ChainDims &c);
size_t stream_prep_bytes(const ChainDims &c);
int stream_prepare(const ChainDims &c, const void *values, const int32_t *adj_o_host, const int32_t *sched_host,
                   const int32_t *adj_i_host, void *k5, cudaStream_t stream);
int stream_supported(const ChainDims &c, int out_dtype);
int launch_stream(const ChainDims &c, int out_dtype, const void *k4, const void *k5, const void *inp, void *out,
                  cudaStream_t stream);
int stream_conv_supported(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype);
int stream_prepare_values(const ChainDims &c, const void *values, void *k5, cudaStream_t stream);
int gather_prepare_values(const ChainDims &c, const void *values, void *k4, cudaStream_t stream);
int tc_prepare_values(const ChainDims &c, int compute, const void *values, void *prep, size_t bytes,
                      cudaStream_t stream);
int launch_stream_conv(const ChainDims &c, const rbgp4_conv_desc *cv, int out_dtype, const void *k4, const void *k5,
                       const void *x, void *out, cudaStream_t stream);
int gather_prepare(const ChainDims &c, const void *values, const int32_t *adj_i_host, void *k4,
                   cudaStream_t stream);
// K7: tensor-core weight gradient (sddmm_tc.cu): bf16 dO / I, f32 gradient in the values layout
int sddmm_tc_supported(const ChainDims &c);
int launch_sddmm_tc(const ChainDims &c, const int32_t *adj_o, const int32_t *adj_i, const void *d_out,
                    int64_t ld_do, const void *inp, int64_t ld_in, float *grad, cudaStream_t stream,
                    bool nmajor = false);

}  // namespace rbgp4
