// sdmm_tc.cu -- K2: RBGP4 product on the 5th-generation tensor cores (tcgen05).
//
// Replaces kronsparse.sdmm._tile_worker (reference sdmm.py:148-205) for the
// bf16 / tf32 compute modes.  Formulation ("densified tile"):
// a CTA owns 128 rows of one W tile-row (M = 128 MMA rows) and TN <= 256
// output columns.  It walks g_o's adjacency row only (structurally zero
// tiles are skipped, as in the reference), and per step s
//
//   B (I slab)  I[adj_o[tbm][s]*tk : +tk, n0 : n0+TN]  -- TMA, 128B swizzle
//               (32 B atoms for tf32), MN-major UMMA operand (I is row-major,
//               N contiguous, so no transpose is ever materialised)
//   A (W tile)  the 128 x tk dense tile, K-major 32/64/128B swizzle, built in
//               shared memory from the COMPRESSED values (128 x d_t): the
//               in-tile pattern g_r (x) g_i (x) g_b is the same for every
//               step and every tile-row, so the zero positions are written
//               once at kernel start and each step only scatters the d_t
//               nonzeros of each row to their (fixed) positions.
//   D          += A * B   with tk*E/32 tcgen05.mma (M=128, N=TN, K=32 bytes),
//               fp32 accumulation in TMEM (TN columns).
//
// Warp roles (192 threads):  warps 0-3 densify A and run the epilogue
// (tcgen05.ld 32x32b -> registers -> 16-byte global stores; warp w owns TMEM
// lanes 32w..32w+31 = output rows);  warp 4 lane 0 issues the TMA loads;
// warp 5 allocates TMEM and lane 0 issues the MMAs.  An NS-stage mbarrier
// ring links them:  full_b (TMA tx bytes), full_a (128 densify arrivals),
// empty (tcgen05.commit), tmem_full (last commit).
//
// Roofline: bound by HBM for the VGG/WRN layer shapes (compressed W + I +
// O once); the MMA does 1/(1-sp_i) times the useful work, which stays under
// the HBM time while (1-sp_i) * P_tc >= AI * BW (SURVEY §7 hard part 1).
#include "common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

namespace rbgp4 {
namespace {

constexpr int kThreads = 192;
constexpr int kBlockM = 128;

struct TcParams {
    int64_t n_cols, ld_out, row_nnz;
    int32_t tm, tk, d_o, d_t, u_i, v_i, d_i, rk, bm, bk;
    int32_t tn;              // MMA N (columns per CTA), multiple of 16, <= 256
    int32_t rows_valid;      // 128, or 64 when tm == 64 (upper half of A is zero)
    int32_t stages;
    int32_t a_swz;           // K-major swizzle span of A in bytes: 32 / 64 / 128
    int32_t a_stage_bytes, b_stage_bytes;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int32_t x, int32_t y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                     "r"(smem_u32(bar)) : "memory");
}
template <bool TF32>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
    if constexpr (TF32) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
    }
}
// UMMA shared-memory matrix descriptor (sm_100: version 1 at bit 46).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout & 7) << 61;
    return d;
}
__device__ __forceinline__ uint32_t swizzle_layout_code(int span) {
    return span == 128 ? 2u : span == 64 ? 4u : 6u;  // SWIZZLE_128B / 64B / 32B
}
// byte offset -> swizzled byte offset inside a (8 rows x span) atom region
__device__ __forceinline__ uint32_t swz(uint32_t off, int span) {
    const uint32_t mask = span == 128 ? 7u : span == 64 ? 3u : 1u;
    return off ^ (((off >> 7) & mask) << 4);
}

#define TMEM_LD_32x32b_X32(taddr, r)                                                       \
    asm volatile(                                                                          \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"    \
        "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}," \
        " [%32];"                                                                          \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),          \
          "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),        \
          "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),    \
          "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),    \
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),    \
          "=r"(r[30]), "=r"(r[31])                                                         \
        : "r"(taddr))

// ---------------------------------------------------------------- the kernel
template <typename E, bool OUT_BF16>
__global__ void __launch_bounds__(kThreads, 1)
tc_kernel(const __grid_constant__ CUtensorMap imap, const TcParams p, const E *__restrict__ values,
          const int32_t *__restrict__ adj_o, const int32_t *__restrict__ adj_i,
          void *__restrict__ out) {
    constexpr bool kTF32 = sizeof(E) == 4;
    constexpr int kElt = sizeof(E);
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned carve-up: [A stages][B stages][aoff table][barriers][tmem ptr]
    unsigned char *base = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char *a_buf = base;
    unsigned char *b_buf = a_buf + p.stages * p.a_stage_bytes;
    // aoff[j * 128 + r]: byte offset (inside an A stage) of nonzero j of CTA row r
    uint16_t *aoff = reinterpret_cast<uint16_t *>(b_buf + p.stages * p.b_stage_bytes);
    uint64_t *bars = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(aoff + kBlockM * p.d_t) + 7) & ~uintptr_t(7));
    uint64_t *full_b = bars, *full_a = bars + p.stages, *empty = bars + 2 * p.stages;
    uint64_t *tmem_full = bars + 3 * p.stages;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_full + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t n0 = int64_t(blockIdx.x) * p.tn;
    const int64_t m0 = int64_t(blockIdx.y) * p.rows_valid;  // first W row of this CTA
    const int64_t tbm = m0 / p.tm;
    const int row_in_tile0 = int(m0 - tbm * p.tm);

    // ---- one-time setup: zero A stages, scatter-offset table, barriers, TMEM.
    // The in-tile pattern is the same for every step, so the (row, j) -> A
    // position map is computed once here and the per-step densify is a pure
    // table-driven scatter (reference index map: sdmm.py:183-186).
    {
        uint4 z = make_uint4(0, 0, 0, 0);
        uint4 *a4 = reinterpret_cast<uint4 *>(a_buf);
        for (int i = threadIdx.x; i < p.stages * p.a_stage_bytes / 16; i += kThreads) a4[i] = z;
        for (int e = threadIdx.x; e < kBlockM * p.d_t; e += kThreads) {
            const int j = e / kBlockM, r = e - j * kBlockM;
            const int u_loc = row_in_tile0 + r;
            const int ui = (u_loc / p.bm) % p.u_i;
            const int k = j % p.bk, q = j / p.bk, ink = q % p.d_i, rk = q / p.d_i;
            const int kcol = (rk * p.v_i + adj_i[ui * p.d_i + ink]) * p.bk + k;  // local K index
            const uint32_t kb = uint32_t(kcol) * kElt;
            aoff[e] = uint16_t((kb / p.a_swz) * (kBlockM * p.a_swz) +
                               swz(uint32_t(r) * p.a_swz + (kb % p.a_swz), p.a_swz));
        }
    }
    if (warp == 4 && lane == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full_b[s], 1);
            mbar_init(&full_a[s], kBlockM);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&imap)) : "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(uint32_t(p.tn < 32 ? 32 : p.tn)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;
    const int32_t *orow = adj_o + tbm * p.d_o;

    if (warp == 4) {
        // ================= TMA producer: I slabs =================
        if (lane == 0) {
            const int atoms = p.tn * kElt / 128;           // 128-byte MN atoms per slab
            const int atom_cols = 128 / kElt;
            const uint32_t atom_bytes = uint32_t(p.tk) * 128;
            for (int s = 0; s < p.d_o; ++s) {
                const int st = s % p.stages;
                const uint32_t ph = (s / p.stages) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                mbar_expect_tx(&full_b[st], uint32_t(p.b_stage_bytes));
                const int32_t krow = orow[s] * p.tk;
                unsigned char *dst = b_buf + st * p.b_stage_bytes;
                for (int a = 0; a < atoms; ++a)
                    tma_load_2d(dst + a * atom_bytes, &imap, &full_b[st],
                                int32_t(n0) + a * atom_cols, krow);
            }
        }
    } else if (warp == 5) {
        // ================= MMA issuer =================
        if (lane == 0) {
            // instruction descriptor: D f32, A/B bf16|tf32, A K-major, B MN-major, N, M=128
            const uint32_t fmt = kTF32 ? 2u : 1u;
            const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (1u << 16) |
                                   (uint32_t(p.tn >> 3) << 17) | (uint32_t(kBlockM >> 4) << 24);
            const uint32_t a_layout = swizzle_layout_code(p.a_swz);
            const int ksteps = p.tk * kElt / 32;
            for (int s = 0; s < p.d_o; ++s) {
                const int st = s % p.stages;
                const uint32_t ph = (s / p.stages) & 1;
                mbar_wait(&full_b[st], ph);
                mbar_wait(&full_a[st], ph);
                tc_fence_after();
                const uint32_t a0 = smem_u32(a_buf + st * p.a_stage_bytes);
                const uint32_t b0 = smem_u32(b_buf + st * p.b_stage_bytes);
                for (int kk = 0; kk < ksteps; ++kk) {
                    const uint32_t kb = uint32_t(kk) * 32;  // byte offset along K
                    const uint32_t a_addr =
                        a0 + (kb / p.a_swz) * (kBlockM * p.a_swz) + (kb % p.a_swz);
                    const uint64_t ad = smem_desc(a_addr, 0, 8 * p.a_swz, a_layout);
                    const uint32_t b_addr = b0 + (kb / kElt) * 128;  // 32/E K-rows of 128 B
                    // MN-major B: bf16 -> SWIZZLE_128B (8-row K groups, SBO 1024);
                    // tf32 -> SWIZZLE_128B_BASE32B (32 B chunks, 4-row K groups, SBO 512)
                    const uint64_t bd = kTF32 ? smem_desc(b_addr, uint32_t(p.tk) * 128, 512, 1u)
                                              : smem_desc(b_addr, uint32_t(p.tk) * 128, 1024, 2u);
                    tc_mma<kTF32>(tmem_d, ad, bd, idesc, (s > 0 || kk > 0) ? 1u : 0u);
                }
                tc_commit(&empty[st]);
            }
            tc_commit(tmem_full);
        }
    } else {
        // ================= densify (warps 0-3), then epilogue =================
        const int t = threadIdx.x;  // 0..127: this thread densifies CTA row t
        const bool active = t < p.rows_valid;
        const E *vrow = values + (m0 + t) * p.row_nnz;
        constexpr int V = 16 / kElt;  // elements per 16-byte load
        const bool vec = (p.d_t % V == 0) && (p.row_nnz % V == 0) &&
                         (reinterpret_cast<uintptr_t>(values) % 16 == 0);
        for (int s = 0; s < p.d_o; ++s) {
            const int st = s % p.stages;
            const uint32_t ph = (s / p.stages) & 1;
            mbar_wait(&empty[st], ph ^ 1);
            unsigned char *a = a_buf + st * p.a_stage_bytes;
            if (active) {
                const E *vs = vrow + int64_t(s) * p.d_t;
                if (vec) {
                    for (int j = 0; j < p.d_t; j += V) {
                        uint4 q = __ldg(reinterpret_cast<const uint4 *>(vs + j));
                        const E *qe = reinterpret_cast<const E *>(&q);
#pragma unroll
                        for (int v = 0; v < V; ++v)
                            *reinterpret_cast<E *>(a + aoff[(j + v) * kBlockM + t]) = qe[v];
                    }
                } else {
                    for (int j = 0; j < p.d_t; ++j)
                        *reinterpret_cast<E *>(a + aoff[j * kBlockM + t]) = vs[j];
                }
            }
            fence_async_smem();
            mbar_arrive(&full_a[st]);
        }
        // ---- epilogue: TMEM -> registers -> global
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int row = warp * 32 + lane;
        const bool row_ok = row < p.rows_valid;
        const uint32_t lane_base = tmem_d + (uint32_t(warp * 32) << 16);
        for (int c = 0; c < p.tn; c += 32) {
            uint32_t r[32];
            TMEM_LD_32x32b_X32(lane_base + uint32_t(c), r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int64_t col = n0 + c;
            if (!row_ok || col >= p.n_cols) continue;
            const bool full = col + 32 <= p.n_cols;
            if constexpr (OUT_BF16) {
                __nv_bfloat16 *dst = static_cast<__nv_bfloat16 *>(out) + (m0 + row) * p.ld_out + col;
                if (full && (reinterpret_cast<uintptr_t>(dst) % 16 == 0)) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 pk;
                        uint32_t w[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(
                                __uint_as_float(r[q * 8 + 2 * h]), __uint_as_float(r[q * 8 + 2 * h + 1]));
                            w[h] = *reinterpret_cast<uint32_t *>(&b2);
                        }
                        pk = make_uint4(w[0], w[1], w[2], w[3]);
                        reinterpret_cast<uint4 *>(dst)[q] = pk;
                    }
                } else {
                    for (int q = 0; q < 32 && col + q < p.n_cols; ++q)
                        dst[q] = __float2bfloat16_rn(__uint_as_float(r[q]));
                }
            } else {
                float *dst = static_cast<float *>(out) + (m0 + row) * p.ld_out + col;
                if (full && (reinterpret_cast<uintptr_t>(dst) % 16 == 0)) {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<uint4 *>(dst)[q] =
                            make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
                } else {
                    for (int q = 0; q < 32 && col + q < p.n_cols; ++q) dst[q] = __uint_as_float(r[q]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                     "r"(uint32_t(p.tn < 32 ? 32 : p.tn)));
    }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

struct TcPlan {
    TcParams p;
    size_t smem;
    int blocks_m;
};

constexpr size_t kSmemCap = 227 * 1024;

int plan_tc(const ChainDims &c, int compute, TcPlan *out) {
    const int elt = compute == RBGP4_COMPUTE_TF32 ? 4 : 2;
    if (!(c.tm == 64 || c.tm % kBlockM == 0)) {
        set_error("tensor-core path needs tile rows tm = 64 or a multiple of 128 (tm=%d)", c.tm);
        return 0;
    }
    if ((c.tk * elt) % 32 != 0 || c.tk > 256) {
        set_error("tensor-core path needs tk*%d bytes to be a multiple of 32 and tk <= 256 (tk=%d)",
                  elt, c.tk);
        return 0;
    }
    if (c.d_t > 256 || size_t(kBlockM) * c.tk * elt > 65536) {
        set_error("tensor-core path: d_t=%d / tile %dx%d exceeds the 16-bit scatter table", c.d_t,
                  kBlockM, c.tk);
        return 0;
    }
    TcParams p{};
    p.n_cols = c.n_cols; p.ld_out = c.ld_out; p.row_nnz = c.row_nnz;
    p.tm = c.tm; p.tk = c.tk; p.d_o = c.d_o; p.d_t = c.d_t; p.u_i = c.u_i; p.v_i = c.v_i;
    p.d_i = c.d_i; p.rk = c.rk; p.bm = c.bm; p.bk = c.bk;
    p.rows_valid = c.tm == 64 ? 64 : kBlockM;
    const int kbytes = c.tk * elt;
    p.a_swz = kbytes % 128 == 0 ? 128 : kbytes % 64 == 0 ? 64 : 32;
    p.a_stage_bytes = kBlockM * kbytes;
    // widest N (<= 256) that still leaves >= 2 pipeline stages and enough CTAs
    const int64_t blocks_m = c.rows / p.rows_valid;
    int tn = 256;
    const int tn_min = 128 / elt;  // one 128-byte swizzle atom of B along N
    while (tn > tn_min && ((c.n_cols + tn - 1) / tn) * blocks_m < 2 * kNumSMs) tn /= 2;
    for (; tn >= tn_min; tn /= 2) {
        p.tn = tn;
        p.b_stage_bytes = c.tk * tn * elt;
        const size_t fixed = 1024 + size_t(kBlockM) * c.d_t * 2 + 16 + 8 * (3 * 8 + 1) + 16;
        const size_t per = size_t(p.a_stage_bytes) + p.b_stage_bytes;
        if (fixed + 2 * per > kSmemCap) continue;
        // two CTAs per SM when >= 3 stages fit in half the shared memory
        int stages = int((kSmemCap / 2 - 1024 - fixed) / per);
        if (stages < 3) stages = int((kSmemCap - fixed) / per);
        if (stages > 6) stages = 6;
        p.stages = stages;
        out->p = p;
        out->smem = fixed + per * stages;
        out->blocks_m = int(blocks_m);
        return 1;
    }
    set_error("tensor-core path: tile %dx%d does not fit shared memory", c.tm, c.tk);
    return 0;
}

template <typename E, bool OUT_BF16>
int launch_typed(const TcPlan &pl, const CUtensorMap &map, const void *values,
                 const int32_t *adj_o, const int32_t *adj_i, void *out, cudaStream_t stream) {
    auto kern = tc_kernel<E, OUT_BF16>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(tc): %s", cudaGetErrorString(e));
        return RBGP4_ECUDA;
    }
    dim3 grid(unsigned((pl.p.n_cols + pl.p.tn - 1) / pl.p.tn), unsigned(pl.blocks_m));
    kern<<<grid, kThreads, pl.smem, stream>>>(map, pl.p, static_cast<const E *>(values), adj_o,
                                              adj_i, out);
    RBGP4_CHECK_LAUNCH("tc_kernel launch");
    return RBGP4_OK;
}

}  // namespace

int tc_supported(const ChainDims &c, int compute, int out_dtype) {
    if (out_dtype != RBGP4_F32 && out_dtype != RBGP4_BF16) {
        set_error("tensor-core modes write f32 or bf16 outputs");
        return 0;
    }
    TcPlan pl;
    return plan_tc(c, compute, &pl);
}

size_t tc_workspace_size(const ChainDims &, int) { return 0; }

int launch_tc(const ChainDims &c, int compute, int out_dtype, const void *values,
              const int32_t *adj_o, const int32_t *adj_i, const void *inp, void *out, void *,
              size_t, cudaStream_t stream) {
    if (c.n_cols == 0) return RBGP4_OK;
    TcPlan pl;
    if (!plan_tc(c, compute, &pl)) return RBGP4_EUNSUPPORTED;
    const int elt = compute == RBGP4_COMPUTE_TF32 ? 4 : 2;
    if (reinterpret_cast<uintptr_t>(inp) % 16 != 0 || (c.ld_in * elt) % 16 != 0) {
        set_error("tensor-core path needs a 16-byte aligned I with ld_in*%d %% 16 == 0", elt);
        return RBGP4_EUNSUPPORTED;
    }
    auto enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return RBGP4_ECUDA;
    }
    CUtensorMap map;
    cuuint64_t dims[2] = {cuuint64_t(c.n_cols), cuuint64_t(c.cols)};
    cuuint64_t strides[1] = {cuuint64_t(c.ld_in) * elt};
    cuuint32_t box[2] = {cuuint32_t(128 / elt), cuuint32_t(c.tk)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&map, elt == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                     2, const_cast<void *>(inp), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     elt == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", int(r));
        return RBGP4_ECUDA;
    }
    const bool obf = out_dtype == RBGP4_BF16;
    if (compute == RBGP4_COMPUTE_TF32)
        return obf ? launch_typed<float, true>(pl, map, values, adj_o, adj_i, out, stream)
                   : launch_typed<float, false>(pl, map, values, adj_o, adj_i, out, stream);
    return obf ? launch_typed<__nv_bfloat16, true>(pl, map, values, adj_o, adj_i, out, stream)
               : launch_typed<__nv_bfloat16, false>(pl, map, values, adj_o, adj_i, out, stream);
}

}  // namespace rbgp4
