// rbgp4_abi.cu -- extern "C" entry points of librbgp4_b200.so (include/rbgp4.h).
//
// The boundary mirrors the reference's native call: the caller owns every
// buffer, the library validates the chain descriptor the way the reference
// validates TilingParams (sdmm.py:208-261) and then queues kernels on the
// caller's stream.  No host synchronisation, no allocation, no fallback: an
// unsupported (shape, compute) pair is an error, never a silent CPU path.
#include "common.cuh"

#include <cstring>
#include <string>

namespace rbgp4 {

namespace {
thread_local char g_last_error[512] = "";
thread_local int64_t g_launches = 0;
thread_local Options g_opts;

struct OptionSlot {
    const char *name;
    int32_t Options::*field;
    int32_t lo, hi;
};
constexpr OptionSlot kOptionSlots[] = {
    {"relayout", &Options::relayout, -1, 1},     {"dense", &Options::dense, 0, 1},
    {"persistent", &Options::persistent, -1, 1}, {"msplit", &Options::msplit, 0, 1},
    {"ksplit", &Options::ksplit, 0, 8},          {"stages", &Options::stages, 0, 16},
    {"multicast", &Options::multicast, -1, 0},   {"sym", &Options::sym, 0, 1},
    {"pdl", &Options::pdl, 0, 1},                {"simt_ct", &Options::simt_ct, 0, 32},
    {"tc_tn", &Options::tc_tn, 0, 256},          {"tc_na", &Options::tc_na, 0, 8},
    {"tc_nb", &Options::tc_nb, 0, 16},           {"tc_nw", &Options::tc_nw, 0, 16},
    {"wswz", &Options::wswz, 0, 1},              {"ostore", &Options::ostore, 0, 1},
    {"sched", &Options::sched, 0, 1},            {"i3d", &Options::i3d, 0, 1},
    {"promo", &Options::promo, -1, 256},         {"conv_wide", &Options::conv_wide, 0, 1},
    {"stream", &Options::stream, -1, 0},         {"stream_g", &Options::stream_g, 0, 8},
    {"halo", &Options::halo, -1, 0},             {"simt_wide", &Options::simt_wide, -1, 0},
    {"merge", &Options::merge, -1, 0},          {"stream_ctas", &Options::stream_ctas, 0, 1024},
    {"simt_ksplit", &Options::simt_ksplit, 0, 2},    {"conv_ostage", &Options::conv_ostage, 0, 1},
    {"debug", &Options::debug, 0, 1 << 30},
};
const OptionSlot *find_option(const char *name) {
    if (name == nullptr) return nullptr;
    for (const auto &s : kOptionSlots)
        if (strcmp(s.name, name) == 0) return &s;
    return nullptr;
}
}  // namespace

Options &opts() { return g_opts; }
thread_local ConvEpilogue g_conv_epi;
ConvEpilogue &conv_epilogue() { return g_conv_epi; }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

void note_launch(int n) { g_launches += n; }
namespace {
thread_local const char *g_last_kernel = "";
}
void note_kernel(const char *name) { g_last_kernel = name; }

int validate_desc(const rbgp4_desc *d, ChainDims *c) {
    RBGP4_REQUIRE(d != nullptr, "null descriptor");
    RBGP4_REQUIRE(d->u_o >= 1 && d->v_o >= 1 && d->d_o >= 1 && d->d_o <= d->v_o,
                  "bad outer factor (u_o=%d, v_o=%d, d_o=%d)", d->u_o, d->v_o, d->d_o);
    RBGP4_REQUIRE(d->u_i >= 1 && d->v_i >= 1 && d->d_i >= 1 && d->d_i <= d->v_i,
                  "bad inner factor (u_i=%d, v_i=%d, d_i=%d)", d->u_i, d->v_i, d->d_i);
    RBGP4_REQUIRE(d->rm >= 1 && d->rk >= 1 && d->bm >= 1 && d->bk >= 1,
                  "bad complete factors (rm=%d, rk=%d, bm=%d, bk=%d)", d->rm, d->rk, d->bm, d->bk);
    c->u_o = d->u_o; c->v_o = d->v_o; c->d_o = d->d_o;
    c->rm = d->rm; c->rk = d->rk; c->u_i = d->u_i; c->v_i = d->v_i; c->d_i = d->d_i;
    c->bm = d->bm; c->bk = d->bk;
    c->tm = d->rm * d->u_i * d->bm;
    c->tk = d->rk * d->v_i * d->bk;
    c->d_t = d->rk * d->d_i * d->bk;
    c->g = d->rm * d->bm;
    c->row_nnz = int64_t(d->d_o) * c->d_t;
    const int64_t rows = int64_t(d->u_o) * c->tm, cols = int64_t(d->v_o) * c->tk;
    RBGP4_REQUIRE(d->rows == rows && d->cols == cols,
                  "descriptor (%lld x %lld) disagrees with the chain (%lld x %lld)",
                  (long long)d->rows, (long long)d->cols, (long long)rows, (long long)cols);
    RBGP4_REQUIRE(d->n_cols >= 0, "negative n_cols");
    RBGP4_REQUIRE(d->ld_in >= d->n_cols && d->ld_out >= d->n_cols,
                  "leading dimensions (%lld, %lld) smaller than n_cols %lld",
                  (long long)d->ld_in, (long long)d->ld_out, (long long)d->n_cols);
    RBGP4_REQUIRE(d->u_o <= 65535, "u_o=%d exceeds the grid's y extent", d->u_o);
    c->rows = rows; c->cols = cols; c->n_cols = d->n_cols;
    c->ld_in = d->ld_in; c->ld_out = d->ld_out;
    return RBGP4_OK;
}

namespace {

__global__ void cast_kernel_f32_bf16(const float *__restrict__ s, __nv_bfloat16 *__restrict__ d,
                                     int64_t n) {
    int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * 4;
    for (; i + 3 < n; i += stride) {
        float4 v = *reinterpret_cast<const float4 *>(s + i);
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t *>(&a);
        pk.y = *reinterpret_cast<uint32_t *>(&b);
        *reinterpret_cast<uint2 *>(d + i) = pk;
    }
    for (; i < n; ++i) d[i] = __float2bfloat16_rn(s[i]);
}

template <typename S, typename D>
__global__ void cast_kernel_scalar(const S *__restrict__ s, D *__restrict__ d, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if constexpr (std::is_same<D, __nv_bfloat16>::value) d[i] = __float2bfloat16_rn(float(s[i]));
        else if constexpr (std::is_same<S, __nv_bfloat16>::value) d[i] = D(__bfloat162float(s[i]));
        else d[i] = D(s[i]);
    }
}

}  // namespace
}  // namespace rbgp4

using namespace rbgp4;

extern "C" {

const char *rbgp4_last_error(void) { return g_last_error; }

int rbgp4_abi_version(void) { return RBGP4_ABI_VERSION; }

int rbgp4_debug_build(void) { return RBGP4_DEBUG; }

int rbgp4_set_option(const char *name, int64_t value) {
    const OptionSlot *s = find_option(name);
    RBGP4_REQUIRE(s != nullptr, "unknown option '%s'", name ? name : "(null)");
    RBGP4_REQUIRE(value >= s->lo && value <= s->hi, "option '%s' = %lld outside [%d, %d]", s->name,
                  (long long)value, s->lo, s->hi);
    RBGP4_REQUIRE(s->field != &Options::debug || value == 0 || RBGP4_DEBUG,
                  "option 'debug' needs a debug build of the library (-DRBGP4_DEBUG=1)");
    g_opts.*(s->field) = int32_t(value);
    return RBGP4_OK;
}

int rbgp4_get_option(const char *name, int64_t *value) {
    const OptionSlot *s = find_option(name);
    RBGP4_REQUIRE(s != nullptr, "unknown option '%s'", name ? name : "(null)");
    RBGP4_REQUIRE(value != nullptr, "null output pointer");
    *value = g_opts.*(s->field);
    return RBGP4_OK;
}

void rbgp4_reset_options(void) { g_opts = Options(); }

int64_t rbgp4_launch_count(void) { return g_launches; }

void rbgp4_reset_launch_count(void) { g_launches = 0; }

const char *rbgp4_last_kernel(void) { return rbgp4::g_last_kernel; }

size_t rbgp4_workspace_size(const rbgp4_desc *desc, int compute, int in_dtype) {
    ChainDims c;
    if (validate_desc(desc, &c) != RBGP4_OK) return 0;
    if (compute == RBGP4_COMPUTE_TF32 || compute == RBGP4_COMPUTE_BF16)
        return tc_workspace_size(c, compute);
    return 0;
}

int rbgp4_sdmm_supported(const rbgp4_desc *desc, int compute, int in_dtype, int out_dtype) {
    ChainDims c;
    if (validate_desc(desc, &c) != RBGP4_OK) return 0;
    switch (compute) {
        case RBGP4_COMPUTE_EXACT:
        case RBGP4_COMPUTE_FFMA:
            if ((in_dtype != RBGP4_F32 && in_dtype != RBGP4_F64) || out_dtype != in_dtype) {
                set_error("SIMT modes need f32/f64 operands and an output of the same type");
                return 0;
            }
            return simt_supported(c, in_dtype);
        case RBGP4_COMPUTE_TF32:
            if (in_dtype != RBGP4_F32) { set_error("tf32 mode consumes f32 operands"); return 0; }
            return tc_supported(c, compute, out_dtype);
        case RBGP4_COMPUTE_BF16:
            if (in_dtype != RBGP4_BF16) { set_error("bf16 mode consumes bf16 operands"); return 0; }
            return tc_supported(c, compute, out_dtype);
        default:
            set_error("unknown compute mode %d", compute);
            return 0;
    }
}

int rbgp4_sdmm_prepared(const rbgp4_desc *desc, int compute, int in_dtype, int out_dtype,
                        const void *values, const int32_t *adj_o, const int32_t *adj_i,
                        const void *prep, const void *inp, void *out, void *workspace,
                        size_t workspace_bytes, void *stream) {
    ChainDims c;
    int rc = validate_desc(desc, &c);
    if (rc != RBGP4_OK) return rc;
    if (!rbgp4_sdmm_supported(desc, compute, in_dtype, out_dtype)) return RBGP4_EUNSUPPORTED;
    if (c.n_cols == 0) return RBGP4_OK;  // empty product: nothing to write
    RBGP4_REQUIRE(values && adj_o && adj_i && inp && out, "null device pointer");
    auto s = static_cast<cudaStream_t>(stream);
    if (compute == RBGP4_COMPUTE_EXACT || compute == RBGP4_COMPUTE_FFMA)
        return launch_simt(c, compute, in_dtype, values, adj_o, adj_i, inp, out, s);
    const size_t need = tc_workspace_size(c, compute);
    if (need > 0 && (workspace == nullptr || workspace_bytes < need)) {
        set_error("tensor-core path needs %zu workspace bytes, got %zu", need, workspace_bytes);
        return RBGP4_EWORKSPACE;
    }
    return launch_tc(c, compute, out_dtype, values, adj_o, adj_i, prep, inp, out, workspace,
                     workspace_bytes, s);
}

int rbgp4_sdmm(const rbgp4_desc *desc, int compute, int in_dtype, int out_dtype,
               const void *values, const int32_t *adj_o, const int32_t *adj_i, const void *inp,
               void *out, void *workspace, size_t workspace_bytes, void *stream) {
    return rbgp4_sdmm_prepared(desc, compute, in_dtype, out_dtype, values, adj_o, adj_i, nullptr,
                               inp, out, workspace, workspace_bytes, stream);
}

size_t rbgp4_prepare_size(const rbgp4_desc *desc, int compute) {
    ChainDims c;
    if (validate_desc(desc, &c) != RBGP4_OK) return 0;
    if (compute == RBGP4_COMPUTE_TF32 || compute == RBGP4_COMPUTE_BF16) return tc_prep_size(c, compute);
    return 0;
}

int rbgp4_prepare(const rbgp4_desc *desc, int compute, const void *values, const int32_t *adj_o,
                  const int32_t *adj_i, void *prep, size_t prep_bytes, void *stream) {
    ChainDims c;
    int rc = validate_desc(desc, &c);
    if (rc != RBGP4_OK) return rc;
    if (compute != RBGP4_COMPUTE_TF32 && compute != RBGP4_COMPUTE_BF16) return RBGP4_OK;
    RBGP4_REQUIRE(adj_o != nullptr && adj_i != nullptr, "null adjacency");
    return tc_prepare(c, compute, values, adj_o, adj_i, prep, prep_bytes, static_cast<cudaStream_t>(stream));
}

int rbgp4_prepare_values(const rbgp4_desc *desc, int compute, const void *values, void *prep, size_t prep_bytes,
                         void *stream) {
    ChainDims c;
    int rc = validate_desc(desc, &c);
    if (rc != RBGP4_OK) return rc;
    if (compute != RBGP4_COMPUTE_TF32 && compute != RBGP4_COMPUTE_BF16) return RBGP4_OK;
    return tc_prepare_values(c, compute, values, prep, prep_bytes, static_cast<cudaStream_t>(stream));
}

size_t rbgp4_conv2d_workspace_size(const rbgp4_desc *desc, const rbgp4_conv_desc *conv) {
    ChainDims c;
    if (validate_desc(desc, &c) != RBGP4_OK) return 0;
    return conv_workspace_size(c, conv);
}

int rbgp4_conv2d(const rbgp4_desc *desc, const rbgp4_conv_desc *conv, int out_dtype,
                 const void *values, const int32_t *adj_o, const int32_t *adj_i, const void *prep,
                 const void *x, void *out, void *workspace, size_t workspace_bytes, void *stream) {
    ChainDims c;
    rbgp4_desc d = *desc;
    d.ld_in = d.ld_out = d.n_cols;  // NHWC operands: leading dimensions are implied
    int rc = validate_desc(&d, &c);
    if (rc != RBGP4_OK) return rc;
    RBGP4_REQUIRE(out_dtype == RBGP4_F32 || out_dtype == RBGP4_BF16, "conv writes f32 or bf16");
    if (c.n_cols == 0) return RBGP4_OK;
    RBGP4_REQUIRE(values && adj_o && adj_i && x && out, "null device pointer");
    return launch_conv(c, conv, out_dtype, values, adj_o, adj_i, prep, x, out, workspace,
                       workspace_bytes, static_cast<cudaStream_t>(stream));
}

int rbgp4_conv2d_residual(const rbgp4_desc *desc, const rbgp4_conv_desc *conv, int out_dtype,
                          const void *values, const int32_t *adj_o, const int32_t *adj_i, const void *prep,
                          const void *x, const void *residual, void *out, void *out_relu, void *workspace,
                          size_t workspace_bytes, void *stream) {
    RBGP4_REQUIRE(residual != nullptr, "rbgp4_conv2d_residual: null residual");
    RBGP4_REQUIRE(conv != nullptr && !(conv->relu & (RBGP4_CONV_RELU | RBGP4_CONV_POOL2)),
                  "rbgp4_conv2d_residual: the residual is added before any ReLU / pool (conv->relu must be 0)");
    ConvEpilogue &ep = conv_epilogue();
    ep.res = residual;
    ep.out2 = out_relu;
    const int rc = rbgp4_conv2d(desc, conv, out_dtype, values, adj_o, adj_i, prep, x, out, workspace,
                                workspace_bytes, stream);
    ep = ConvEpilogue{};
    return rc;
}

int rbgp4_cast(int src_dtype, int dst_dtype, const void *src, void *dst, int64_t n, void *stream) {
    RBGP4_REQUIRE(n >= 0, "negative element count");
    if (n == 0) return RBGP4_OK;
    auto s = static_cast<cudaStream_t>(stream);
    const int threads = 256;
    const int blocks = int(std::min<int64_t>((n + threads * 4 - 1) / (threads * 4), 148 * 16));
    if (src_dtype == RBGP4_F32 && dst_dtype == RBGP4_BF16) {
        if (reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 8 == 0)
            cast_kernel_f32_bf16<<<blocks, threads, 0, s>>>(static_cast<const float *>(src),
                                                            static_cast<__nv_bfloat16 *>(dst), n);
        else
            cast_kernel_scalar<float, __nv_bfloat16><<<blocks, threads, 0, s>>>(
                static_cast<const float *>(src), static_cast<__nv_bfloat16 *>(dst), n);
    } else if (src_dtype == RBGP4_F64 && dst_dtype == RBGP4_BF16) {
        cast_kernel_scalar<double, __nv_bfloat16><<<blocks, threads, 0, s>>>(
            static_cast<const double *>(src), static_cast<__nv_bfloat16 *>(dst), n);
    } else if (src_dtype == RBGP4_BF16 && dst_dtype == RBGP4_F32) {
        cast_kernel_scalar<__nv_bfloat16, float><<<blocks, threads, 0, s>>>(
            static_cast<const __nv_bfloat16 *>(src), static_cast<float *>(dst), n);
    } else if (src_dtype == RBGP4_F64 && dst_dtype == RBGP4_F32) {
        cast_kernel_scalar<double, float><<<blocks, threads, 0, s>>>(
            static_cast<const double *>(src), static_cast<float *>(dst), n);
    } else if (src_dtype == RBGP4_F32 && dst_dtype == RBGP4_F64) {
        cast_kernel_scalar<float, double><<<blocks, threads, 0, s>>>(
            static_cast<const float *>(src), static_cast<double *>(dst), n);
    } else {
        set_error("unsupported cast %d -> %d", src_dtype, dst_dtype);
        return RBGP4_EINVAL;
    }
    RBGP4_CHECK_LAUNCH("cast kernel launch");
    return RBGP4_OK;
}

}  // extern "C"
