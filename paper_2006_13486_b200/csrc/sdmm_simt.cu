// sdmm_simt.cu -- K1: SIMT RBGP4 product with the reference's accumulation order.
//
// Replaces kronsparse.sdmm._tile_worker (reference sdmm.py:148-205).  One CTA
// owns one (tm x tnc) output tile: tile-row tbm of W and a tnc-wide column
// block of I/O.  It walks only g_o's adjacency row (d_o of v_o W tiles; the
// others are structurally zero and skipped), staging per step
//   W tile  values[tbm*tm : +tm, s*d_t : +d_t]      (compressed, dense)
//   I tile  I[adj_o[tbm][s]*tk : +tk, n0 : n0+tnc]
// into a 2-stage cp.async ring in shared memory.  Within the tile the rows
// fall into u_i repetition groups of g = rm*bm rows sharing one set of d_t I
// rows; a per-group row table (computed once per CTA) turns each W column j
// into its I row, so the gather is an indexed shared-memory read.
//
// Each thread owns NCH chunks of RT rows (same group) x 4 columns.  For every
// output element the arithmetic is exactly the reference's:
//   acc = 0;  for s: { c = 0;  for j in d_t: c = c + w*x;  acc = acc + c; }
// EXACT=true rounds every multiply and add separately (__fmul_rn/__fadd_rn,
// never contracted) and is bit-identical to the reference for any tiling;
// EXACT=false uses FFMA in the same order (rel. error ~1e-7, 2x issue rate).
#include "common.cuh"
#include "tc_ptx.cuh"

#include <algorithm>

namespace rbgp4 {
namespace {

struct SimtParams {
    int64_t rows, n_cols, ld_in, ld_out, row_nnz;
    int32_t d_o, tm, tk, rm, rk, bm, bk, u_i, v_i, d_i, d_t, g;
    int32_t tnc, cthreads, wstride, istride;
    int32_t vec_in, vec_out;  // 16-byte paths legal for I loads / O stores
    int32_t nbuf;             // wide variant: TMA ring slots
    int32_t ksplit;           // wide ffma variant: 2 = the steps halved over a (1,1,2) cluster
};

constexpr int kThreads = 256;

template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <typename T> __device__ __forceinline__ T fma_rn(T a, T b, T c);
template <> __device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <> __device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    int n = valid ? 16 : 0;  // zero-fill past the edge
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
template <int B>
__device__ __forceinline__ void cp_async_small(void *smem, const void *gmem, bool valid) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    int n = valid ? B : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(B), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <typename T>
__device__ __forceinline__ void load4(const T *p, T (&x)[4]) {
    if constexpr (sizeof(T) == 4) {
        float4 v = *reinterpret_cast<const float4 *>(p);
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
        double2 a = reinterpret_cast<const double2 *>(p)[0];
        double2 b = reinterpret_cast<const double2 *>(p)[1];
        x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
    }
}

// Stage step s of tile-row tbm into one ring slot.
template <typename T>
__device__ __forceinline__ void stage(const SimtParams &p, const T *__restrict__ values,
                                      const T *__restrict__ inp, int64_t tbm, int64_t oind,
                                      int64_t n0, int s, T *ws, T *is) {
    const int tid = threadIdx.x;
    // compressed W tile: tm rows x d_t contiguous values (scalar copies, odd stride)
    const T *wsrc = values + tbm * p.tm * p.row_nnz + int64_t(s) * p.d_t;
    for (int e = tid; e < p.tm * p.d_t; e += kThreads) {
        int r = e / p.d_t, j = e - r * p.d_t;
        cp_async_small<sizeof(T)>(ws + r * p.wstride + j, wsrc + r * p.row_nnz + j, true);
    }
    // I tile: tk rows x tnc columns, zero-filled beyond n_cols
    const T *isrc = inp + oind * p.tk * p.ld_in + n0;
    if (p.vec_in) {
        constexpr int V = 16 / sizeof(T);
        const int chunks = p.tnc / V;
        for (int e = tid; e < p.tk * chunks; e += kThreads) {
            int r = e / chunks, c = (e - r * chunks) * V;
            bool ok = n0 + c < p.n_cols;  // n_cols % V == 0 on this path
            cp_async16(is + r * p.istride + c, ok ? isrc + r * p.ld_in + c : isrc, ok);
        }
    } else {
        for (int e = tid; e < p.tk * p.tnc; e += kThreads) {
            int r = e / p.tnc, c = e - r * p.tnc;
            bool ok = n0 + c < p.n_cols;
            cp_async_small<sizeof(T)>(is + r * p.istride + c, ok ? isrc + r * p.ld_in + c : isrc, ok);
        }
    }
}

template <typename T, bool EXACT, int RT, int NCH>
__global__ void __launch_bounds__(kThreads)
simt_kernel(const SimtParams p, const T *__restrict__ values, const int32_t *__restrict__ adj_o,
            const int32_t *__restrict__ adj_i, const T *__restrict__ inp, T *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int64_t n0 = int64_t(blockIdx.x) * p.tnc;
    const int64_t tbm = blockIdx.y;
    const int tid = threadIdx.x;

    // smem: [W ring x2][I ring x2][row table]
    T *wring = reinterpret_cast<T *>(smem_raw);
    T *iring = wring + 2 * p.tm * p.wstride;
    int32_t *rowidx = reinterpret_cast<int32_t *>(iring + 2 * p.tk * p.istride);
    const int wslot = p.tm * p.wstride, islot = p.tk * p.istride;

    // I row of W column j for group ui: (rk*v_i + adj_i[ui][ink])*bk + k,
    // with j = (rk*d_i + ink)*bk + k  (reference sdmm.py:183-184)
    for (int e = tid; e < p.u_i * p.d_t; e += kThreads) {
        int ui = e / p.d_t, j = e - ui * p.d_t;
        int k = j % p.bk, q = j / p.bk, ink = q % p.d_i, rk = q / p.d_i;
        rowidx[e] = (rk * p.v_i + adj_i[ui * p.d_i + ink]) * p.bk + k;
    }

    const int tc = tid % p.cthreads;
    const int rthread = tid / p.cthreads;
    const int rthreads = kThreads / p.cthreads;
    const int nchunks = p.tm / RT;

    // rows owned by this thread: chunk q covers group slots [rc*RT, rc*RT+RT)
    int urow[NCH][RT];
    int ugrp[NCH];
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        int rc = rthread + q * rthreads;
        int slot = (rc < nchunks ? rc : 0) * RT;
        int ui = slot / p.g, within = slot - ui * p.g;
        ugrp[q] = ui;
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            int w = within + i, rm = w / p.bm, m = w - rm * p.bm;
            urow[q][i] = (rm * p.u_i + ui) * p.bm + m;
        }
    }

    T acc[NCH][RT][4];
#pragma unroll
    for (int q = 0; q < NCH; ++q)
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[q][i][e] = T(0);

    const int32_t *orow = adj_o + tbm * p.d_o;
    stage<T>(p, values, inp, tbm, orow[0], n0, 0, wring, iring);
    cp_async_commit();

    for (int s = 0; s < p.d_o; ++s) {
        if (s + 1 < p.d_o) {
            const int b = (s + 1) & 1;
            stage<T>(p, values, inp, tbm, orow[s + 1], n0, s + 1, wring + b * wslot,
                     iring + b * islot);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const T *ws = wring + (s & 1) * wslot;
        const T *is = iring + (s & 1) * islot + tc * 4;
#pragma unroll
        for (int q = 0; q < NCH; ++q) {
            if (rthread + q * rthreads >= nchunks) break;
            const int32_t *ridx = rowidx + ugrp[q] * p.d_t;
            T c[RT][4];
#pragma unroll
            for (int i = 0; i < RT; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) c[i][e] = T(0);
            const T *wrow[RT];
#pragma unroll
            for (int i = 0; i < RT; ++i) wrow[i] = ws + urow[q][i] * p.wstride;
#pragma unroll 4
            for (int j = 0; j < p.d_t; ++j) {
                T x[4];
                load4<T>(is + ridx[j] * p.istride, x);
#pragma unroll
                for (int i = 0; i < RT; ++i) {
                    const T w = wrow[i][j];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if constexpr (EXACT) c[i][e] = add_rn(c[i][e], mul_rn(w, x[e]));
                        else c[i][e] = fma_rn(w, x[e], c[i][e]);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < RT; ++i)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[q][i][e] = add_rn(acc[q][i][e], c[i][e]);
        }
        __syncthreads();
    }

    // epilogue: each thread writes RT rows x 4 consecutive columns per chunk
    const int64_t col = n0 + tc * 4;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
        if (rthread + q * rthreads >= nchunks) break;
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            T *dst = out + (tbm * p.tm + urow[q][i]) * p.ld_out + col;
            if (p.vec_out && col + 3 < p.n_cols) {
                if constexpr (sizeof(T) == 4) {
                    *reinterpret_cast<float4 *>(dst) =
                        make_float4(acc[q][i][0], acc[q][i][1], acc[q][i][2], acc[q][i][3]);
                } else {
                    reinterpret_cast<double2 *>(dst)[0] = make_double2(acc[q][i][0], acc[q][i][1]);
                    reinterpret_cast<double2 *>(dst)[1] = make_double2(acc[q][i][2], acc[q][i][3]);
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (col + e < p.n_cols) dst[e] = acc[q][i][e];
            }
        }
    }
}

// ---------------------------------------------------------------- wide f32 variant
// The common f32 shape (repetition groups of >= 16 rows, d_t % 4 == 0, 16-byte aligned rows):
// each thread owns 16 rows of one group x 4 columns, so an I vector (LDS.128) feeds 64 FMAs
// and the W values of 4 consecutive j are one broadcast LDS.128 per row -- about one shared
// wavefront per 8 FFMA instead of one per 2 (the generic kernel is shared-memory bound at
// ~0.22 of the FFMA peak).  Both operands of a step arrive by TMA (one W box of the compressed
// tile-row, tm x d_t, and one I box, tk x tnc, zero-filled past n_cols) into a 2-slot ring
// completed on mbarriers: one thread issues two copies per step, where per-thread cp.async
// address arithmetic was ~40 % of the kernel's instructions and stall samples
// (profiles/r02f_k1wide_conv10_ncu_*).  Same per-element order as the reference
// (sdmm.py:178-204): c = 0; c += w*x over j ascending; acc += c per step.
constexpr int kWideBox = 256;  // TMA box rows per copy

// ROWS rows of one repetition group x COLV float4 column chunks per thread (ROWS * COLV = 16,
// 64 outputs): (16, 1) for groups of >= 16 rows, (8, 2) and (4, 4) for the 8- and 4-row groups
// of the WRN factorisations (G_b (8,8) / (4,4)).  Per 4 consecutive j a thread reads 4 * COLV
// I vectors and ROWS W vectors (LDS.128) for 256 FFMA.  Column chunk k of thread tc sits at
// column 4 * (tc + k * cthreads), so every LDS.128 of a half-warp is one contiguous 256 B row.
template <bool EXACT, int ROWS, int COLV>
__global__ void __launch_bounds__(kThreads)
simt_wide_kernel(const SimtParams p, const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap imap,
                 const int32_t *__restrict__ adj_o, const int32_t *__restrict__ adj_i, float *__restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int64_t n0 = int64_t(blockIdx.x) * p.tnc;
    const int64_t tbm = blockIdx.y;
    const int tid = threadIdx.x;
    const int nbuf = p.nbuf;
    float *ring = reinterpret_cast<float *>(smem_raw);
    const int wslot = p.tm * p.d_t, slot = wslot + p.tk * p.tnc;  // floats per ring slot
    int32_t *rowidx = reinterpret_cast<int32_t *>(ring + nbuf * slot);
    uint64_t *full = reinterpret_cast<uint64_t *>(rowidx + ((p.u_i * p.d_t + 1) & ~1));
    const int32_t *orow = adj_o + tbm * p.d_o;
    const uint32_t step_bytes = uint32_t(slot) * 4u;
    // split steps (ffma only, never EXACT): CTA z of the cluster pair runs steps [s_lo, s_hi)
    const int half = (p.d_o + 1) / 2;
    const int kz = (!EXACT && p.ksplit > 1) ? int(blockIdx.z) : 0;
    const int s_lo = kz ? half : 0, s_hi = (!EXACT && p.ksplit > 1 && kz == 0) ? half : p.d_o;
    auto issue = [&](int s) {  // thread 0: both boxes of step s into slot (s - s_lo) % nbuf
        const int b = (s - s_lo) % nbuf;
        float *ws = ring + b * slot, *is = ws + wslot;
        uint64_t *bar = &full[b];
        mbar_expect_tx(bar, step_bytes);
        const int32_t oind = orow[s];
        for (int r = 0; r < p.tm; r += kWideBox)
            tma_load_2d(ws + r * p.d_t, &wmap, bar, s * p.d_t, int32_t(tbm * p.tm + r));
        for (int r = 0; r < p.tk; r += kWideBox)
            tma_load_2d(is + r * p.tnc, &imap, bar, int32_t(n0), oind * p.tk + r);
    };
    if (tid == 0) {
        for (int b = 0; b < nbuf; ++b) mbar_init(&full[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = s_lo; s < s_lo + nbuf && s < s_hi; ++s) issue(s);
    }
    // row table pre-multiplied by the I row stride (the wanted I row of W column j of group ui)
    for (int e = tid; e < p.u_i * p.d_t; e += int(blockDim.x)) {
        int ui = e / p.d_t, j = e - ui * p.d_t;
        int k = j % p.bk, q = j / p.bk, ink = q % p.d_i, rk = q / p.d_i;
        rowidx[e] = ((rk * p.v_i + adj_i[ui * p.d_i + ink]) * p.bk + k) * p.tnc;
    }
    const int tc = tid % p.cthreads;
    const int slot0 = (tid / p.cthreads) * ROWS;  // this thread's group slots
    const int ui = slot0 / p.g;
    int urow[ROWS];  // W row offsets (floats) inside a slot
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
        const int w = slot0 - ui * p.g + i, rm = w / p.bm, m = w - rm * p.bm;
        urow[i] = ((rm * p.u_i + ui) * p.bm + m) * p.d_t;
    }
    float acc[ROWS][COLV * 4];
#pragma unroll
    for (int i = 0; i < ROWS; ++i)
#pragma unroll
        for (int e = 0; e < COLV * 4; ++e) acc[i][e] = 0.0f;
    __syncthreads();  // row table and barrier init visible
    const int32_t *ridx = rowidx + ui * p.d_t;
    const int cstep = 4 * p.cthreads;  // floats between a thread's column chunks
    for (int s = s_lo; s < s_hi; ++s) {
        const int b = (s - s_lo) % nbuf;
        mbar_wait(&full[b], uint32_t((s - s_lo) / nbuf) & 1u);
        const float *ws = ring + b * slot;
        const float *is = ws + wslot + tc * 4;
        float c[ROWS][COLV * 4];
#pragma unroll
        for (int i = 0; i < ROWS; ++i)
#pragma unroll
            for (int e = 0; e < COLV * 4; ++e) c[i][e] = 0.0f;
#pragma unroll 1
        for (int j = 0; j < p.d_t; j += 4) {
            if constexpr (COLV == 1) {
                float x[4][4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) load4<float>(is + ridx[j + jj], x[jj]);
#pragma unroll
                for (int i = 0; i < ROWS; ++i) {
                    const float4 w4 = *reinterpret_cast<const float4 *>(ws + urow[i] + j);
                    const float w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            if constexpr (EXACT) c[i][e] = __fadd_rn(c[i][e], __fmul_rn(w[jj], x[jj][e]));
                            else c[i][e] = __fmaf_rn(w[jj], x[jj][e], c[i][e]);
                        }
                }
            } else {
                float w[ROWS][4];
#pragma unroll
                for (int i = 0; i < ROWS; ++i) {
                    const float4 w4 = *reinterpret_cast<const float4 *>(ws + urow[i] + j);
                    w[i][0] = w4.x; w[i][1] = w4.y; w[i][2] = w4.z; w[i][3] = w4.w;
                }
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const float *xr = is + ridx[j + jj];
                    float x[COLV * 4];
#pragma unroll
                    for (int k = 0; k < COLV; ++k) {
                        const float4 v = *reinterpret_cast<const float4 *>(xr + k * cstep);
                        x[4 * k] = v.x; x[4 * k + 1] = v.y; x[4 * k + 2] = v.z; x[4 * k + 3] = v.w;
                    }
#pragma unroll
                    for (int i = 0; i < ROWS; ++i)
#pragma unroll
                        for (int e = 0; e < COLV * 4; ++e) {
                            if constexpr (EXACT) c[i][e] = __fadd_rn(c[i][e], __fmul_rn(w[i][jj], x[e]));
                            else c[i][e] = __fmaf_rn(w[i][jj], x[e], c[i][e]);
                        }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < ROWS; ++i)
#pragma unroll
            for (int e = 0; e < COLV * 4; ++e) acc[i][e] = __fadd_rn(acc[i][e], c[i][e]);
        __syncthreads();  // every thread is done with slot b
        if (tid == 0 && s + nbuf < s_hi) issue(s + nbuf);
    }
    if constexpr (!EXACT) {
        if (p.ksplit > 1) {
            // the second half's partial joins the first in CTA 0 of the pair (fixed order: first
            // half + second half, deterministic): its rings are idle after both main loops
            asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            float *xch = ring + tid * (ROWS * COLV * 4);
            if (kz == 1) {
                uint32_t dst;
                asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(dst) : "r"(smem_u32(xch)));
#pragma unroll
                for (int i = 0; i < ROWS; ++i)
#pragma unroll
                    for (int e = 0; e < COLV * 4; e += 4)
                        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                         dst + uint32_t((i * COLV * 4 + e) * 4)),
                                     "f"(acc[i][e]), "f"(acc[i][e + 1]), "f"(acc[i][e + 2]), "f"(acc[i][e + 3])
                                     : "memory");
            }
            asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            if (kz == 1) return;
#pragma unroll
            for (int i = 0; i < ROWS; ++i)
#pragma unroll
                for (int e = 0; e < COLV * 4; ++e) acc[i][e] = __fadd_rn(acc[i][e], xch[i * COLV * 4 + e]);
        }
    }
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
        float *drow = out + (tbm * p.tm + urow[i] / p.d_t) * p.ld_out;
#pragma unroll
        for (int k = 0; k < COLV; ++k) {
            const int64_t col = n0 + tc * 4 + k * cstep;
            float *dst = drow + col;
            if (p.vec_out && col + 3 < p.n_cols) {
                *reinterpret_cast<float4 *>(dst) =
                    make_float4(acc[i][4 * k], acc[i][4 * k + 1], acc[i][4 * k + 2], acc[i][4 * k + 3]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (col + e < p.n_cols) dst[e] = acc[i][4 * k + e];
            }
        }
    }
}

// rows per thread of the wide variant for this chain (0: not eligible)
int wide_rows(const ChainDims &c) {
    for (int r : {16, 8, 4})
        if (c.g % r == 0 && c.tm % r == 0) return r;
    return 0;
}

bool wide_ok(const ChainDims &c, const void *values, const void *inp) {
    if (opts().simt_wide == 0) return false;
    return wide_rows(c) && c.d_t % 4 == 0 && c.d_t <= 256 && c.row_nnz % 4 == 0 &&
           c.ld_in % 4 == 0 && reinterpret_cast<uintptr_t>(values) % 16 == 0 &&
           reinterpret_cast<uintptr_t>(inp) % 16 == 0;
}

template <bool EXACT>
int launch_wide(const ChainDims &c, const float *values, const int32_t *adj_o, const int32_t *adj_i,
                const float *inp, float *out, cudaStream_t stream) {
    SimtParams p{};
    p.rows = c.rows; p.n_cols = c.n_cols; p.ld_in = c.ld_in; p.ld_out = c.ld_out;
    p.row_nnz = c.row_nnz; p.d_o = c.d_o; p.tm = c.tm; p.tk = c.tk; p.rm = c.rm; p.rk = c.rk;
    p.bm = c.bm; p.bk = c.bk; p.u_i = c.u_i; p.v_i = c.v_i; p.d_i = c.d_i; p.d_t = c.d_t; p.g = c.g;
    const int rows = wide_rows(c), colv = 16 / rows;
    const int rthreads = c.tm / rows;
    const int64_t row_blocks = c.rows / c.tm;
    // column threads: 16 (64 columns per CTA at 16 rows per thread; ~220 registers, two CTAs
    // per SM), 8 when 16 would leave SMs without a CTA (conv14, N = 1024: 48 us either way
    // against 62 us on the generic kernel, tools/simt_ab.py); a warp-multiple CTA of <= 256
    // ffma only: a grid short of the SMs halves the steps over (1,1,2) clusters (never EXACT,
    // whose per-element order is the reference's sequential sum over the steps)
    int ksplit = 1;
    if (!EXACT && c.d_o >= 4 && opts().simt_ksplit != 1) {
        const int64_t g16 = (c.n_cols + 4 * colv * 16 - 1) / (4 * colv * 16) * row_blocks;
        const int64_t g8 = (c.n_cols + 4 * colv * 8 - 1) / (4 * colv * 8) * row_blocks;
        if (opts().simt_ksplit == 2 || std::max(g16, g8) < kNumSMs) ksplit = 2;
    }
    int ct = 0;
    if (opts().simt_ct == 8 || opts().simt_ct == 16 || opts().simt_ct == 32) {
        ct = opts().simt_ct;
    } else {
        for (int cand : {16, 8}) {
            if (cand * rthreads > kThreads || (cand * rthreads) % 32) continue;
            ct = cand;
            if ((c.n_cols + 4 * colv * cand - 1) / (4 * colv * cand) * row_blocks * ksplit >= kNumSMs) break;
        }
    }
    if (ct == 0 || ct * rthreads > kThreads || (ct * rthreads) % 32) return RBGP4_EUNSUPPORTED;
    p.cthreads = ct;
    p.tnc = 4 * colv * ct;
    p.wstride = c.d_t;
    p.istride = p.tnc;
    p.vec_out = (c.ld_out % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    // ring depth: as many slots as fit two CTAs per SM (one step in flight is enough when a
    // step is long, e.g. conv10's 48 KB slots; short steps such as WRN's d_t = 8 need more)
    const size_t slot_bytes = (size_t(c.tm) * c.d_t + size_t(c.tk) * p.tnc) * 4;
    const size_t fixed = size_t((c.u_i * c.d_t + 1) & ~1) * 4 + 4 * sizeof(uint64_t);
    int nbuf = int(std::min<size_t>(4, (110 * 1024 - fixed) / slot_bytes));
    if (nbuf < 2) nbuf = 2;
    p.nbuf = nbuf;
    // the pair's exchange reuses CTA 0's ring: 64 floats per thread
    if (size_t(nbuf) * slot_bytes < size_t(rthreads) * ct * 64 * 4) ksplit = 1;
    p.ksplit = ksplit;
    const size_t smem = nbuf * slot_bytes + fixed;
    if (smem > 227 * 1024) return RBGP4_EUNSUPPORTED;
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    CUtensorMap wmap, imap;
    const cuuint32_t estr[2] = {1, 1};
    {   // RcubsMatrix.values as stored: (row_nnz, rows); box d_t x min(tm, 256)
        const cuuint64_t dims[2] = {cuuint64_t(c.row_nnz), cuuint64_t(c.rows)};
        const cuuint64_t strides[1] = {cuuint64_t(c.row_nnz) * 4};
        const cuuint32_t box[2] = {cuuint32_t(c.d_t), cuuint32_t(std::min(c.tm, kWideBox))};
        CUresult r = enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(values), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(simt W) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    {   // I: (n_cols, K) with row stride ld_in; box tnc x min(tk, 256), zero fill past n_cols
        const cuuint64_t dims[2] = {cuuint64_t(c.n_cols), cuuint64_t(c.cols)};
        const cuuint64_t strides[1] = {cuuint64_t(c.ld_in) * 4};
        const cuuint32_t box[2] = {cuuint32_t(p.tnc), cuuint32_t(std::min(c.tk, kWideBox))};
        CUresult r = enc(&imap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(inp), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("cuTensorMapEncodeTiled(simt I) failed (%d)", int(r));
            return RBGP4_ECUDA;
        }
    }
    auto kern = rows == 16 ? simt_wide_kernel<EXACT, 16, 1>
              : rows == 8 ? simt_wide_kernel<EXACT, 8, 2> : simt_wide_kernel<EXACT, 4, 4>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) {
            set_error("cudaFuncSetAttribute(simt wide): %s", cudaGetErrorString(e));
            return RBGP4_ECUDA;
        }
    }
    dim3 grid(unsigned((c.n_cols + p.tnc - 1) / p.tnc), unsigned(c.rows / c.tm), unsigned(ksplit));
    note_kernel(ksplit > 1 ? "K1 simt wide split" : "K1 simt wide");
    if (ksplit > 1) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(unsigned(rthreads * ct));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 2;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p, wmap, imap, adj_o, adj_i, out);
        if (e != cudaSuccess) {
            set_error("simt_wide_kernel (split pair) launch: %s", cudaGetErrorString(e));
            return RBGP4_ECUDA;
        }
    } else {
        kern<<<grid, unsigned(rthreads * ct), smem, stream>>>(p, wmap, imap, adj_o, adj_i, out);
    }
    RBGP4_CHECK_LAUNCH("simt_wide_kernel launch");
    return RBGP4_OK;
}

struct SimtPlan {
    int rt, nch, cthreads;
    size_t smem;
};

template <typename T>
size_t smem_bytes(const ChainDims &c, int cthreads) {
    int tnc = 4 * cthreads;
    int wstride = c.d_t | 1;
    size_t ring = 2 * (size_t(c.tm) * wstride + size_t(c.tk) * tnc) * sizeof(T);
    ring = (ring + 15) & ~size_t(15);
    return ring + size_t(c.u_i) * c.d_t * sizeof(int32_t);
}

template <typename T>
int plan_simt(const ChainDims &c, SimtPlan *plan) {
    int rt = (c.g % 4 == 0) ? 4 : (c.g % 2 == 0) ? 2 : 1;
    const int max_regs_chunks = sizeof(T) == 4 ? 16 : 8;  // NCH*RT bound (register budget)
    const size_t smem_cap = 227 * 1024;
    // Column-block width 4*cthreads: the widest whose grid still covers every SM (one tile per
    // CTA is a serial walk over the d_o steps, so idle SMs cost more than narrower tiles):
    // measured on the VGG shapes, conv13 (N = 1024) 153 -> 64 us at 32 columns per CTA.
    const int ct_opt = opts().simt_ct;
    SimtPlan fallback{};
    bool have = false;
    const int64_t row_blocks = c.rows / c.tm;
    for (int cthreads : {32, 16, 8}) {
        if (ct_opt && ct_opt != cthreads) continue;
        int rthreads = kThreads / cthreads;
        int chunks = c.tm / rt;
        int nch = 1;
        while (nch * rthreads < chunks) nch *= 2;
        if (nch > 8 || nch * rt > max_regs_chunks) continue;
        size_t sm = smem_bytes<T>(c, cthreads);
        if (sm > smem_cap) continue;
        const int64_t grid = (c.n_cols + 4 * cthreads - 1) / (4 * cthreads) * row_blocks;
        fallback = {rt, nch, cthreads, sm};
        have = true;
        if (ct_opt || grid >= kNumSMs) {
            *plan = fallback;
            return 1;
        }
    }
    if (have) {  // no width covers the SMs: the narrowest feasible one
        *plan = fallback;
        return 1;
    }
    set_error("SIMT path: tile %dx%d (d_t=%d, u_i=%d) exceeds register/shared-memory budget",
              c.tm, c.tk, c.d_t, c.u_i);
    return 0;
}

template <typename T, bool EXACT, int RT, int NCH>
int launch_one(const ChainDims &c, const SimtPlan &pl, const T *values, const int32_t *adj_o,
               const int32_t *adj_i, const T *inp, T *out, cudaStream_t stream) {
    SimtParams p{};
    p.rows = c.rows; p.n_cols = c.n_cols; p.ld_in = c.ld_in; p.ld_out = c.ld_out;
    p.row_nnz = c.row_nnz; p.d_o = c.d_o; p.tm = c.tm; p.tk = c.tk; p.rm = c.rm; p.rk = c.rk;
    p.bm = c.bm; p.bk = c.bk; p.u_i = c.u_i; p.v_i = c.v_i; p.d_i = c.d_i; p.d_t = c.d_t;
    p.g = c.g; p.cthreads = pl.cthreads; p.tnc = 4 * pl.cthreads;
    p.wstride = c.d_t | 1; p.istride = p.tnc;
    constexpr int V = 16 / sizeof(T);
    p.vec_in = (c.ld_in % V == 0) && (c.n_cols % V == 0) &&
               (reinterpret_cast<uintptr_t>(inp) % 16 == 0);
    p.vec_out = (c.ld_out % V == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    auto kern = simt_kernel<T, EXACT, RT, NCH>;
    if (pl.smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(pl.smem));
        if (e != cudaSuccess) {
            set_error("cudaFuncSetAttribute(simt): %s", cudaGetErrorString(e));
            return RBGP4_ECUDA;
        }
    }
    dim3 grid(unsigned((c.n_cols + p.tnc - 1) / p.tnc), unsigned(c.rows / c.tm));
    note_kernel("K1 simt");
    kern<<<grid, kThreads, pl.smem, stream>>>(p, values, adj_o, adj_i, inp, out);
    RBGP4_CHECK_LAUNCH("simt_kernel launch");
    return RBGP4_OK;
}

template <typename T, bool EXACT>
int dispatch(const ChainDims &c, const SimtPlan &pl, const void *values, const int32_t *adj_o,
             const int32_t *adj_i, const void *inp, void *out, cudaStream_t s) {
    auto v = static_cast<const T *>(values);
    auto x = static_cast<const T *>(inp);
    auto o = static_cast<T *>(out);
#define RBGP4_SIMT_CASE(RT_, NCH_)                                                        \
    if (pl.rt == RT_ && pl.nch == NCH_)                                                   \
        return launch_one<T, EXACT, RT_, NCH_>(c, pl, v, adj_o, adj_i, x, o, s);
    RBGP4_SIMT_CASE(1, 1) RBGP4_SIMT_CASE(1, 2) RBGP4_SIMT_CASE(1, 4) RBGP4_SIMT_CASE(1, 8)
    RBGP4_SIMT_CASE(2, 1) RBGP4_SIMT_CASE(2, 2) RBGP4_SIMT_CASE(2, 4)
    if constexpr (sizeof(T) == 4) {
        RBGP4_SIMT_CASE(2, 8) RBGP4_SIMT_CASE(4, 1) RBGP4_SIMT_CASE(4, 2) RBGP4_SIMT_CASE(4, 4)
    } else {
        RBGP4_SIMT_CASE(4, 1) RBGP4_SIMT_CASE(4, 2)
    }
#undef RBGP4_SIMT_CASE
    set_error("SIMT path: no kernel instance for RT=%d NCH=%d", pl.rt, pl.nch);
    return RBGP4_EUNSUPPORTED;
}

}  // namespace

int simt_supported(const ChainDims &c, int dtype) {
    SimtPlan pl;
    return dtype == RBGP4_F64 ? plan_simt<double>(c, &pl) : plan_simt<float>(c, &pl);
}

int launch_simt(const ChainDims &c, int compute, int dtype, const void *values,
                const int32_t *adj_o, const int32_t *adj_i, const void *inp, void *out,
                cudaStream_t stream) {
    if (c.n_cols == 0 || c.rows == 0) return RBGP4_OK;
    SimtPlan pl;
    const bool exact = compute == RBGP4_COMPUTE_EXACT;
    if (dtype == RBGP4_F32) {
        if (wide_ok(c, values, inp)) {
            const int rc = exact ? launch_wide<true>(c, static_cast<const float *>(values), adj_o, adj_i,
                                                     static_cast<const float *>(inp), static_cast<float *>(out), stream)
                                 : launch_wide<false>(c, static_cast<const float *>(values), adj_o, adj_i,
                                                      static_cast<const float *>(inp), static_cast<float *>(out), stream);
            if (rc != RBGP4_EUNSUPPORTED) return rc;
        }
        if (!plan_simt<float>(c, &pl)) return RBGP4_EUNSUPPORTED;
        return exact ? dispatch<float, true>(c, pl, values, adj_o, adj_i, inp, out, stream)
                     : dispatch<float, false>(c, pl, values, adj_o, adj_i, inp, out, stream);
    }
    if (dtype == RBGP4_F64) {
        if (!plan_simt<double>(c, &pl)) return RBGP4_EUNSUPPORTED;
        return exact ? dispatch<double, true>(c, pl, values, adj_o, adj_i, inp, out, stream)
                     : dispatch<double, false>(c, pl, values, adj_o, adj_i, inp, out, stream);
    }
    set_error("SIMT path supports f32/f64 operands, got dtype %d", dtype);
    return RBGP4_EINVAL;
}

}  // namespace rbgp4
