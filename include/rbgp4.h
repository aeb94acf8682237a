/*
 * rbgp4.h -- C ABI of the B200 RBGP4 sparse x dense product O = W_s x I.
 *
 * Plain pointers and sizes only (no torch, no CUDA types: `stream` is a
 * cudaStream_t passed as void*).  All pointers except `desc` are DEVICE
 * pointers on the current CUDA device.  Every entry point returns 0 on
 * success and a negative RBGP4_E* code on failure; the thread-local
 * rbgp4_last_error() then holds a one-line message.  Launches are
 * stream-ordered and asynchronous; nothing here synchronises the device.
 *
 * Reference interfaces replaced (reference = kronsparse, /root/reference/pkg/src):
 *   rbgp4_sdmm        <- kronsparse.sdmm._tile_worker(values, adj_o, adj_i, inp, out,
 *                        tm, tk, tn, rm, rk, bm, bk, rn, bn, n_ui, n_vi, d_i,
 *                        start, stride)                       sdmm.py:148-205 (args 268-273)
 *   rbgp4_chain_sdmm  <- kronsparse.sdmm._csr_rows(indptr, indices, values, inp, out)
 *                        as called by sdmm_reference             sdmm.py:297-330
 *                        (general K-factor chains; columns enumerated in
 *                        closed form as in rcubs.neighbors, rcubs.py:57-76)
 *   rbgp4_csr_sdmm    <- kronsparse.sdmm._csr_rows on a raw CsrMatrix   sdmm.py:297-330
 *   rbgp4_cast        <- the `.astype(...)` conversions the reference applies
 *                        to operands (bench.py:138-140), on device
 */
#ifndef RBGP4_H_
#define RBGP4_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBGP4_ABI_VERSION 3

/* status codes */
#define RBGP4_OK 0
#define RBGP4_EINVAL (-1)      /* inconsistent descriptor / unsupported shape */
#define RBGP4_EUNSUPPORTED (-2) /* compute mode not available for this shape  */
#define RBGP4_ECUDA (-3)       /* CUDA runtime / launch failure               */
#define RBGP4_EWORKSPACE (-4)  /* workspace missing or too small              */

/* element types */
#define RBGP4_F32 0
#define RBGP4_F64 1
#define RBGP4_BF16 2

/* compute modes of rbgp4_sdmm */
#define RBGP4_COMPUTE_EXACT 0 /* SIMT, reference rounding: bit-identical to rbgp4mm  */
#define RBGP4_COMPUTE_FFMA 1  /* SIMT, same order, fused multiply-add (f32 / f64)    */
#define RBGP4_COMPUTE_TF32 2  /* tcgen05 kind::tf32, f32 operands, fp32 accumulate   */
#define RBGP4_COMPUTE_BF16 3  /* tcgen05 kind::f16 (bf16), fp32 accumulate           */

/*
 * Four-factor chain (g_o, g_r, g_i, g_b) with g_r = K_{rm,rk} and
 * g_b = K_{bm,bk} complete.  W is rows x cols with
 *   rows = u_o*rm*u_i*bm,   cols = v_o*rk*v_i*bk,
 *   row_nnz = d_o*rk*d_i*bk;
 * `values` is the (rows, row_nnz) row-major array of RcubsMatrix.values
 * (sorted-column order, rcubs.py:1-12), adj_o is (u_o, d_o) and adj_i is
 * (u_i, d_i), int32 row-major with ascending rows (graphs.py:87-96).
 * I is cols x n_cols with row stride ld_in; O is rows x n_cols with row
 * stride ld_out (elements).  O is fully overwritten (no accumulation).
 */
typedef struct rbgp4_desc {
    int64_t rows, cols, n_cols;
    int64_t ld_in, ld_out;
    int32_t u_o, v_o, d_o;
    int32_t rm, rk;
    int32_t u_i, v_i, d_i;
    int32_t bm, bk;
} rbgp4_desc;

/*
 * O = W x I.  `in_dtype` is the element type of values and I
 * (F32/F64 for EXACT and FFMA, F32 for TF32, BF16 for BF16); `out_dtype`
 * is F32/F64 (= in_dtype) for the SIMT modes and F32 or BF16 for the
 * tensor-core modes.  `workspace` may be NULL when
 * rbgp4_workspace_size() returns 0.
 */
int rbgp4_sdmm(const rbgp4_desc *desc, int compute, int in_dtype, int out_dtype,
               const void *values, const int32_t *adj_o, const int32_t *adj_i,
               const void *inp, void *out, void *workspace, size_t workspace_bytes,
               void *stream);

/*
 * Per-matrix preparation for the tensor-core modes (optional, cacheable), into a
 * caller-owned device buffer of rbgp4_prepare_size() bytes passed to rbgp4_sdmm_prepared():
 *  - the in-tile scatter map of the densified W tile (depends only on the chain and the
 *    tiling), so CTAs skip rebuilding it;
 *  - the step schedule: the order in which each tile-row walks its g_o neighbours, chosen
 *    so that tile-rows sharing a K-block read its I slab at the same step (one L2 pass
 *    over I instead of d_r(g_o)).  Changes only the fp32 summation order of the steps.
 *  - (bf16, g_b >= 16 x 16) the values re-laid out by g_i column block: a permutation of
 *    `values` (same bytes) in which the row blocks sharing a column block are contiguous,
 *    so the gathered-block kernel covers each column block with one MMA.  `values` are the
 *    device values of the product (bf16 for compute = BF16); other modes ignore them.
 * The schedule is searched on the host from adj_o, so this call synchronises `stream`
 * (once per matrix; it is not on the multiply path).  Returns 0 size for the SIMT modes.
 * ABI v2: values and adj_o added (v1 took adj_i only).
 */
size_t rbgp4_prepare_size(const rbgp4_desc *desc, int compute);
int rbgp4_prepare(const rbgp4_desc *desc, int compute, const void *values, const int32_t *adj_o,
                  const int32_t *adj_i, void *prep, size_t prep_bytes, void *stream);

/* Training: rebuild only the value-dependent sections of a prepared buffer (the relayout
 * copies of `values`) after the values changed; the pattern tables of rbgp4_prepare are kept.
 * Stream-ordered device work only (no host synchronisation; CUDA-graph capturable). */
int rbgp4_prepare_values(const rbgp4_desc *desc, int compute, const void *values, void *prep,
                         size_t prep_bytes, void *stream);

/* rbgp4_sdmm with the prepared buffer of rbgp4_prepare (prep may be NULL). */
int rbgp4_sdmm_prepared(const rbgp4_desc *desc, int compute, int in_dtype, int out_dtype,
                        const void *values, const int32_t *adj_o, const int32_t *adj_i,
                        const void *prep, const void *inp, void *out, void *workspace,
                        size_t workspace_bytes, void *stream);

/*
 * Implicit-im2col sparse convolution: O = W x im2col(X) without ever
 * materialising im2col.  X is NHWC bf16 (batch, height, width, c_in), O is NHWC
 * (batch, height, width, rows) in bf16 or f32, stride 1, "same" padding (pad = (k-1)/2).
 * W is the chain matrix of the layer with rows = c_out and columns in tap-major im2col
 * order, column = (i*kw + j)*c_in + c  (conv weight[c_out, c, i, j]); desc->n_cols must be
 * batch*height*width (ld_in/ld_out are ignored).  `relu` is a flags word: bit 0
 * (RBGP4_CONV_RELU) fuses max(0, .) into the store; bit 1 (RBGP4_CONV_POOL2) fuses the 2x2 /
 * stride-2 max pool that follows a VGG stage, so O is (batch, H'/2, W'/2, rows) -- bf16 output,
 * taken by the streamed kernel where its pixel tiles hold whole 2x2 windows (halo strips, or
 * output maps up to 16 wide); otherwise RBGP4_EUNSUPPORTED (pool separately).
 * Tensor-core bf16 path only (compute = RBGP4_COMPUTE_BF16).
 */
#define RBGP4_CONV_RELU 1
#define RBGP4_CONV_POOL2 2
typedef struct rbgp4_conv_desc {
    int32_t batch, height, width, c_in;
    int32_t kh, kw, pad, stride;
    int32_t relu;
} rbgp4_conv_desc;

size_t rbgp4_conv2d_workspace_size(const rbgp4_desc *desc, const rbgp4_conv_desc *conv);
int rbgp4_conv2d(const rbgp4_desc *desc, const rbgp4_conv_desc *conv, int out_dtype,
                 const void *values, const int32_t *adj_o, const int32_t *adj_i, const void *prep,
                 const void *x, void *out, void *workspace, size_t workspace_bytes, void *stream);

/*
 * The WRN block tail fused into the convolution's epilogue: O = conv(X) + R, R an NHWC tensor
 * shaped and typed like O, rounded as the unfused conv-then-add rounds (bf16: round the conv,
 * add in f32, round again), so the result is bit-identical to rbgp4_conv2d followed by the
 * add; with out_relu != NULL also relu(O) into out_relu (the next block's input).  conv->relu
 * must be 0.  Streamed kernel (K5), bf16 output only: other shapes / an f32 output return
 * RBGP4_EUNSUPPORTED (add separately).
 * Replaces nothing in the reference (its bench lowers convs to rbgp4mm over im2col); it serves
 * the WRN-40-4 model of SURVEY §8(f).
 */
int rbgp4_conv2d_residual(const rbgp4_desc *desc, const rbgp4_conv_desc *conv, int out_dtype,
                          const void *values, const int32_t *adj_o, const int32_t *adj_i, const void *prep,
                          const void *x, const void *residual, void *out, void *out_relu, void *workspace,
                          size_t workspace_bytes, void *stream);

/* The dense first convolution of the VGG19 model (kept dense as in PAPER.md:195-196): 3x3 'same',
 * stride 1, 3 input channels -> c_out = 64, ReLU fused, NHWC bf16 in (batch, height, width, 3) and
 * out (batch, height, width, 64), fp32 accumulation on tcgen05.  w: bf16 [64][32], column
 * k = (i*3 + j)*3 + c for weight[c_out][c][i][j], columns 27..31 zero; 16-byte aligned w / out. */
int rbgp4_dense_conv3x3_c3(const void *x, const void *w, void *out, int batch, int height, int width,
                           int c_out, void *stream);

/* 2x2 / stride-2 max pooling of a bf16 NHWC tensor (the VGG stage boundary);
 * H, W even, channels % 8 == 0, 16-byte aligned. */
int rbgp4_maxpool2x2_nhwc(const void *x, void *y, int batch, int height, int width, int channels,
                          void *stream);

/* Materialised im2col of an NHWC tensor (F32 or BF16) into the chain's tap-major operand
 * cols (k*k*channels, batch*H'*W') ('same' padding, stride 1 or 2), for the layers the
 * implicit-im2col conv does not take (the fp32 FFMA path); one pass, zero padding. */
int rbgp4_im2col_nhwc(int dtype, const void *x, void *cols, int batch, int height, int width, int channels,
                      int k, int stride, void *stream);

/* dst (n, rows) = src (rows, n) transposed (the product's O back to NHWC), ReLU fused if relu. */
int rbgp4_nc_to_nhwc(int dtype, const void *src, void *dst, int rows, int64_t n, int relu, void *stream);
/* The same transpose with the WRN block tail: dst = src^T + residual (residual NHWC like dst,
 * rounded like the unfused add), and relu(dst) into dst_relu when it is not NULL. */
int rbgp4_nc_to_nhwc_residual(int dtype, const void *src, const void *residual, void *dst, void *dst_relu,
                              int rows, int64_t n, void *stream);

/*
 * Training direction: the weight gradient restricted to the pattern,
 *   grad_values[u, j] = sum_n d_out[u, n] * inp[c(u, j), n],
 * in the (rows, row_nnz) layout of `values` (c = the closed-form column map of the chain).
 * d_out is rows x n_cols (row stride ld_do), inp is cols x n_cols (row stride ld_in);
 * desc->n_cols = n_cols (desc->ld_in/ld_out are ignored).  F32 (fp32 FMA), F64, or BF16:
 * bf16 d_out / inp on the tensor cores (128 x 128 tiles, g_r = (1,1), bk in {4, 8, 16}) with an
 * F32 grad_values (fp32 accumulation).
 * The input gradient W^T x dO is rbgp4_sdmm on the transposed chain (a valid RBGP4 chain
 * of the transposed factors; paper_2006_13486_b200.training.transpose builds it).
 */
int rbgp4_sddmm(const rbgp4_desc *desc, int dtype, const int32_t *adj_o, const int32_t *adj_i,
                const void *d_out, int64_t ld_do, const void *inp, int64_t ld_in, void *grad_values,
                void *stream);

/* The same weight gradient with batch-major operands (the nn.Linear layout of a training step):
 * d_out_nk is n_cols x rows (= dO^T, row stride ld_do), inp_nk is n_cols x cols (= I^T, row
 * stride ld_in), bf16 on the tensor cores (K7 with MN-major operands; the rbgp4_sddmm BF16
 * constraints), F32 grad_values.  Bit-identical to rbgp4_sddmm on the transposed operands. */
int rbgp4_sddmm_nk(const rbgp4_desc *desc, const int32_t *adj_o, const int32_t *adj_i, const void *d_out_nk,
                   int64_t ld_do, const void *inp_nk, int64_t ld_in, void *grad_values, void *stream);

/* Bytes of device workspace rbgp4_sdmm needs for (desc, compute, in_dtype). */
size_t rbgp4_workspace_size(const rbgp4_desc *desc, int compute, int in_dtype);

/* 1 if rbgp4_sdmm supports (desc, compute, in_dtype, out_dtype), else 0;
 * the reason for a 0 is left in rbgp4_last_error(). */
int rbgp4_sdmm_supported(const rbgp4_desc *desc, int compute, int in_dtype, int out_dtype);

/*
 * General K-factor chain, reference rounding of sdmm_reference:
 * out[u, n] = fl(... fl(fl(v_0 x_0) + fl(v_1 x_1)) ...) over u's nonzeros in
 * ascending column order.  Factor f has left/right sizes num_left[f],
 * num_right[f], left degree degree[f] and its (num_left[f], degree[f])
 * int32 adjacency at adjacency + adj_offset[f].  Host arrays: num_left,
 * num_right, degree, adj_offset (k entries each).  Device: adjacency,
 * values (rows, row_nnz), inp (cols, ld_in), out (rows, ld_out).
 */
int rbgp4_chain_sdmm(int k, const int32_t *num_left, const int32_t *num_right,
                     const int32_t *degree, const int64_t *adj_offset,
                     const int32_t *adjacency, int dtype, const void *values,
                     const void *inp, void *out, int64_t n_cols, int64_t ld_in,
                     int64_t ld_out, void *stream);

/*
 * Raw CSR triple (sdmm_reference on a CsrMatrix): same rounding, explicit
 * int64 indptr (rows+1) and int32 column indices, all device pointers.
 */
int rbgp4_csr_sdmm(int64_t rows, const int64_t *indptr, const int32_t *indices, int dtype,
                   const void *values, const void *inp, void *out, int64_t n_cols,
                   int64_t ld_in, int64_t ld_out, void *stream);

/* dst[i] = (dst_dtype) src[i] for n elements (F32<->BF16, F64->BF16, F64<->F32). */
int rbgp4_cast(int src_dtype, int dst_dtype, const void *src, void *dst, int64_t n,
               void *stream);

/*
 * Plan overrides (A/B switches for tests and tuning; the defaults are the production plan).
 * Thread-local: a value set on one host thread affects only launches planned on that thread.
 * Names: relayout, dense, persistent, msplit, ksplit, stages, multicast, sym, pdl, simt_ct,
 * tc_tn, tc_na, tc_nb, tc_nw, wswz, ostore, sched, i3d, promo, conv_wide, stream, stream_g,
 * halo, simt_wide, merge, stream_ctas, simt_ksplit, conv_ostage, debug (include the kernels' trace/ablation hooks only in a debug
 * build, see rbgp4_debug_build).  Unknown names and out-of-range values return RBGP4_EINVAL.
 * None of them changes results beyond the fp32 summation order of the tensor-core modes.
 * `relayout` and `merge` change the layout of a prepared buffer: a buffer must be used under the
 * values they had at rbgp4_prepare (rbgp4_prepare_size differs between the layouts, so a cache
 * keyed by the size -- as paper_2006_13486_b200.sdmm.prepared() does -- is safe; `sched` only
 * reorders the steps the buffer records).
 * ABI v3.
 */
int rbgp4_set_option(const char *name, int64_t value);
int rbgp4_get_option(const char *name, int64_t *value);
void rbgp4_reset_options(void);
/* 1 if this library was built with -DRBGP4_DEBUG=1 (trace / ablation hooks), else 0. */
int rbgp4_debug_build(void);

/* Thread-local description of the last failure on this thread. */
const char *rbgp4_last_error(void);

/* RBGP4_ABI_VERSION of the loaded library. */
int rbgp4_abi_version(void);

/* Number of kernels this thread has launched through the ABI (for the
 * benchmark's gpu_launches accounting); reset with rbgp4_reset_launch_count. */
int64_t rbgp4_launch_count(void);
void rbgp4_reset_launch_count(void);

/* Name of the kernel family this thread's last product / convolution launched ("K1 simt",
 * "K2 tc", "K2 conv", "K4 gather", "K4 conv", "K5 stream", "K5 rows", "K5 conv", "csr", ...):
 * which device path a call took, for tests and the benchmark. */
const char *rbgp4_last_kernel(void);

#ifdef __cplusplus
}
#endif

#endif /* RBGP4_H_ */
