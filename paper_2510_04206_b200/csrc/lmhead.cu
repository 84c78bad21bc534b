// lmhead.cu -- part 2 of the hot path: token-level PPO-clip loss through the LM head and its
// exact backward (PAPER.md P:1182-1190 token factorisation, P:1230-1241 PPO-clip,
// P:1132-1141 token-level mean / decoupled eps).
//
//   K4 k_gather       compacted rows: H[p] = hidden[idx[p]], target/old/adv per row; rows
//                     [T_eff, pad64) zeroed (they are inside GEMM3's K range)
//   K5 gemm<FWD>      z = s * H W^T on tcgen05; epilogue: per (row, 256-col tile) max m and
//                     l = sum exp(z - m), P~ = exp(z - m) -> bf16 [rows, V], z_y gathered
//   K6 k_merge_g      per row: lse = logsumexp over tiles, logp, rho, PPO-clip term,
//                     c = unclipped ? rho*A/N : 0; rewrites the row in place as
//                     G = bf16(c * (P~ * exp(m_tile - lse) - [v == y]))
//   K7 k_loss_reduce  fixed-order fp64 reduction of the per-row terms -> loss, stats
//   K9 gemm<GRADW>    grad_W = s * G^T H      (A = G MN-major, B = H MN-major, K = T_eff)
//   C3                NCCL all-reduce of grad_W on a side stream, overlapped with K8
//   K8 gemm<GRADH>    grad_hidden[idx] = s * G W  (A = G K-major, B = W MN-major, K = V)
//
// Executed tensor work is 6 * T_eff * V * d FLOP (three GEMMs; no recompute: the bf16 P~
// written by the forward epilogue replaces the second logits GEMM).  See DESIGN.md.
#include <cuda.h>
#include <cuda_runtime.h>

#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "gemm_sm100.cuh"
#include "internal.h"

namespace agentrl {

// ---------------------------------------------------------------------------- tensor maps
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    return fn;
}

// bf16 2-D tensor [outer, inner] (row stride = ld elements), box {box_inner, box_outer},
// SWIZZLE_128B (box_inner * 2 B must be 128), out-of-bounds reads return zeros.
static int make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t ld, uint32_t box_inner, uint32_t box_outer) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return AGENTRL_ERR_CUDA;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? AGENTRL_OK : AGENTRL_ERR_CUDA;
}

// CTA-pair (cta_group::2) GEMMs unless AGENTRL_GEMM_PAIR=0 (1-CTA variant, for A/B runs)
static bool gemm_use_pair() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("AGENTRL_GEMM_PAIR");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// L2 eviction policy per GEMM operand (0 normal, 1 evict_first, 2 evict_last); the defaults
// can be overridden for experiments with AGENTRL_L2POL="fa fb wa wb ha hb" (six digits).
static int l2_policy(int which, int dflt) {
    const char* e = getenv("AGENTRL_L2POL");
    if (!e || (int)strlen(e) < 6) return dflt;
    const int v = e[which] - '0';
    return (v >= 0 && v <= 2) ? v : dflt;
}
static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : dflt;
}
static int gemm_group_m() { return env_int("AGENTRL_GROUP_M", 16); }
static int gemm_group_m_bwd() { return env_int("AGENTRL_GROUP_M_BWD", 8); }
// dynamic tile scheduler (atomic counter, tiles claimed in global order) unless
// AGENTRL_GEMM_SCHED=static (tile = unit + i * units: pairs drift apart over long runs)
static bool gemm_dynamic() {
    const char* e = getenv("AGENTRL_GEMM_SCHED");
    return !(e && strcmp(e, "static") == 0);
}
// persistent grid (one CTA per SM) unless AGENTRL_GEMM_FULLGRID=1 (one CTA per tile)
static bool gemm_full_grid() { return env_int("AGENTRL_GEMM_FULLGRID", 0) == 1; }

// 512-column tiles for the long-K backward GEMMs (CTA pairs only) unless
// AGENTRL_GEMM_NSPLIT=1
static bool gemm_wide_n() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("AGENTRL_GEMM_NSPLIT");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1 && gemm_use_pair();
}

// forward/log-prob GEMMs stage two 64-wide K atoms per k-block unless AGENTRL_FWD_KSUB=1
static bool gemm_fwd_ksub2() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("AGENTRL_FWD_KSUB");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

template <int EPI, bool A_MN, bool B_MN, int NSPLIT, int KSUB = 1>
static int launch_gemm(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& g,
                       int64_t max_tiles, cudaStream_t stream, int reserve_sms = 0) {
    ProfScope ps(EPI == EPI_FWD    ? KID_FWD
                 : EPI == EPI_GRADW ? KID_GRADW
                 : EPI == EPI_LOGP  ? KID_LOGP_GEMM
                                    : KID_GRADH,
                 stream);
    // max_tiles is counted in 128 x 256 tiles (an upper bound of the CTAs worth launching)
    if (gemm_use_pair()) {
        auto kern = gemm_sm100_pair_kernel<EPI, A_MN, B_MN, NSPLIT, KSUB>;
        constexpr int smem = GemmCfg<true, NSPLIT, KSUB>::SMEM +
                             (EPI == EPI_GRADW ? GemmCfg<true, NSPLIT, KSUB>::EPI_STAGE : 0);
        static std::atomic<uint64_t> attr_done{0};  // per instantiation and device
        if (!func_attr_once(attr_done, (const void*)kern, smem)) return AGENTRL_ERR_CUDA;
        int64_t grid = gemm_full_grid()
                           ? 2 * std::max<int64_t>(max_tiles, 1)
                           : std::min<int64_t>((num_sms() - reserve_sms) & ~1,
                                               std::max<int64_t>(max_tiles, 2));
        grid &= ~int64_t(1);
        kern<<<(unsigned)grid, GEMM_THREADS, smem, stream>>>(a, b, g);
    } else {
        auto kern = gemm_sm100_kernel<EPI, A_MN, B_MN>;
        constexpr int smem = GemmCfg<false, 1>::SMEM;
        static std::atomic<uint64_t> attr_done{0};
        if (!func_attr_once(attr_done, (const void*)kern, smem)) return AGENTRL_ERR_CUDA;
        int grid = (int)std::min<int64_t>(num_sms() - reserve_sms, std::max<int64_t>(max_tiles, 1));
        kern<<<grid, GEMM_THREADS, smem, stream>>>(a, b, g);
    }
    count_launch();
    AG_CUDA(cudaGetLastError());
    return AGENTRL_OK;
}

// backward progress-throttle wait episodes per GEMM (0 forward, 1 grad_W, 2 grad_hidden), summed
// over calls: agentrl_debug_throttle_waits() (the tests assert the throttle engages)
__device__ unsigned long long g_throttle_waits[3];
static unsigned long long* throttle_wait_ctr(int which) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_throttle_waits) != cudaSuccess) return nullptr;
    return static_cast<unsigned long long*>(p) + which;
}
int debug_throttle_waits(unsigned long long* host3) {
    return cudaMemcpyFromSymbol(host3, g_throttle_waits, sizeof(unsigned long long) * 3) ==
                   cudaSuccess
               ? AGENTRL_OK
               : AGENTRL_ERR_CUDA;
}

// ---------------------------------------------------------------------------- compaction
// (standalone policy-loss entry: idx from loss_mask alone)
__global__ void __launch_bounds__(CHUNK_THREADS)
    k_mask_count(int64_t T, const uint8_t* __restrict__ mask, int32_t* __restrict__ chunk_cnt) {
    const int64_t t0 = (int64_t)blockIdx.x * CHUNK_TOKENS + threadIdx.x * 16;
    int32_t c = 0;
    for (int i = 0; i < 16; ++i)
        if (t0 + i < T) c += mask[t0 + i] != 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    __shared__ int32_t s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t t = 0;
        for (int w = 0; w < 8; ++w) t += s[w];
        chunk_cnt[blockIdx.x] = t;
    }
}

__global__ void k_chunk_scan(int64_t n_chunks, int32_t* chunk, int64_t* meta) {
    // one thread: n_chunks is T/4096 (<= 32768 at T = 2^27)
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int64_t i = 0; i < n_chunks; ++i) {
            int32_t x = chunk[i];
            chunk[i] = (int32_t)run;
            run += x;
        }
        meta[0] = run;
    }
}

__global__ void __launch_bounds__(CHUNK_THREADS)
    k_compact(int64_t T, const uint8_t* __restrict__ mask, const float* __restrict__ adv_tok,
              const int32_t* __restrict__ chunk_base, int32_t* __restrict__ idx,
              float* __restrict__ adv_c) {
    const int64_t t0 = (int64_t)blockIdx.x * CHUNK_TOKENS + threadIdx.x * 16;
    int32_t c = 0;
    for (int i = 0; i < 16; ++i)
        if (t0 + i < T) c += mask[t0 + i] != 0;
    // block exclusive scan
    __shared__ int32_t s[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s[wid] = x;
    __syncthreads();
    int32_t woff = 0;
    for (int w = 0; w < wid; ++w) woff += s[w];
    int32_t pos = chunk_base[blockIdx.x] + woff + x - c;
    for (int i = 0; i < 16; ++i) {
        const int64_t t = t0 + i;
        if (t < T && mask[t]) {
            idx[pos] = (int32_t)t;
            if (adv_c) adv_c[pos] = adv_tok[t];
            ++pos;
        }
    }
}

// ---------------------------------------------------------------------------- K4 gather
__global__ void __launch_bounds__(256)
    k_gather(const int64_t* __restrict__ rows_dev, int64_t T, int32_t d, int32_t V,
             const __nv_bfloat16* __restrict__ hidden, const int32_t* __restrict__ target,
             const float* __restrict__ old_logp, const int32_t* __restrict__ idx,
             __nv_bfloat16* __restrict__ H, int32_t* __restrict__ tgt_c,
             float* __restrict__ old_c, int32_t* d_status, int64_t v0 = 0,
             int64_t V_total = -1) {
    // vocab-parallel head: this rank holds columns [v0, v0 + V) of V_total; a target outside
    // the shard gets tgt_c = -1 (never matches a column here)
    if (V_total < 0) V_total = V;
    const int64_t rows = *rows_dev;
    const int64_t rows_pad = (rows + 63) / 64 * 64;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    const int chunks = d / 8;  // 16-byte chunks per row
    for (int64_t p = (int64_t)blockIdx.x * 8 + warp; p < rows_pad; p += nwarps) {
        uint4* dst = reinterpret_cast<uint4*>(H + p * d);
        if (p < rows) {
            const int64_t t = idx[p];
            const uint4* src = reinterpret_cast<const uint4*>(hidden + t * d);
            for (int c = lane; c < chunks; c += 32) dst[c] = __ldg(src + c);
            if (lane == 0) {
                int64_t y = target[t];
                if (y < 0 || y >= V_total) {
                    atomicOr(d_status, AGENTRL_ST_BAD_TARGET);
                    y = v0;
                }
                const int64_t yl = y - v0;
                tgt_c[p] = (yl >= 0 && yl < V) ? (int32_t)yl : -1;
                if (old_c) old_c[p] = old_logp[t];
            }
        } else {
            for (int c = lane; c < chunks; c += 32) dst[c] = make_uint4(0, 0, 0, 0);
            if (lane == 0) {
                tgt_c[p] = 0;
                if (old_c) old_c[p] = 0.f;
            }
        }
    }
}

// ---------------------------------------------------------------------------- K6 merge + G
constexpr int MERGE_THREADS = 256;
#ifndef MERGE_MINB
#define MERGE_MINB 0  // 0: no residency hint
#endif
#if MERGE_MINB > 0
#define MERGE_BOUNDS __launch_bounds__(MERGE_THREADS, MERGE_MINB)
#else
#define MERGE_BOUNDS __launch_bounds__(MERGE_THREADS)
#endif

__global__ void MERGE_BOUNDS
    k_merge_g(const int64_t* __restrict__ rows_dev, const int64_t* __restrict__ nglob_dev,
              int32_t V, int32_t n_tiles, const float2* __restrict__ part,
              const float* __restrict__ zy, const int32_t* __restrict__ tgt_c,
              const float* __restrict__ old_c, const float* __restrict__ adv_c,
              const int32_t* __restrict__ idx, float eps_lo, float eps_hi,
              const float* __restrict__ w_c /* per-row weight w_t */,
              const float* __restrict__ ref_c /* per-row ref log-prob or null */,
              float kl_beta, uint16_t* __restrict__ PG /* bf16 P~ in, bf16 G out, [rows, V] */,
              double* __restrict__ row_term /* w (-term + beta KL) */,
              float* __restrict__ row_rho, float* __restrict__ row_logp,
              int32_t* __restrict__ row_clip, float* __restrict__ row_kl,
              float* __restrict__ logp_out,
              const int64_t* __restrict__ rng /* optional row range [r0, r1) */,
              const float2* __restrict__ vpstat = nullptr /* [vp_R][vp_stride] (M_r, L'_r) */,
              int32_t vp_R = 0, int64_t vp_stride = 0) {
    extern __shared__ float s_f[];  // [n_tiles] scale per tile
    __shared__ float s_red[MERGE_THREADS / 32];
    __shared__ int s_jm[MERGE_THREADS / 32];
    __shared__ float s_bc[4];
    const int64_t rows = *rows_dev;
    const int64_t rows_pad = (rows + 63) / 64 * 64;
    const double Nd = (double)*nglob_dev;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const float LOG2E = 1.4426950408889634f;
    // row range of this launch; the one ending at rows also zeroes the padding rows
    const int64_t p_lo = rng ? rng[0] : 0;
    const int64_t p_hi = rng ? (rng[1] >= rows ? rows_pad : rng[1]) : rows_pad;

    for (int64_t p = p_lo + blockIdx.x; p < p_hi; p += gridDim.x) {
        uint4* row4 = reinterpret_cast<uint4*>(PG + p * (int64_t)V);
        const int nvec = V / 8;
        if (p >= rows) {  // padding rows inside GEMM3's K range: zero
            for (int c = threadIdx.x; c < nvec; c += MERGE_THREADS) row4[c] = make_uint4(0, 0, 0, 0);
            continue;
        }
        const float2* pr = part + p * (int64_t)n_tiles;
        // lse over tiles: M = max m_j, L = sum l_j exp(m_j - M)   (fixed order per thread +
        // fixed tree -> deterministic)
        float mloc = -INFINITY;
        for (int j = threadIdx.x; j < n_tiles; j += MERGE_THREADS) mloc = fmaxf(mloc, pr[j].x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
        if (lane == 0) s_red[wid] = mloc;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = s_red[0];
            for (int w = 1; w < MERGE_THREADS / 32; ++w) m = fmaxf(m, s_red[w]);
            s_bc[0] = m;
        }
        __syncthreads();
        const float M = s_bc[0];
        // first tile holding the row max (its l' enters without the leading 1)
        int jloc = 0x7fffffff;
        for (int j = threadIdx.x; j < n_tiles; j += MERGE_THREADS)
            if (pr[j].x == M) jloc = min(jloc, j);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) jloc = min(jloc, __shfl_xor_sync(0xffffffffu, jloc, o));
        __syncthreads();
        if (lane == 0) s_jm[wid] = jloc;
        __syncthreads();
        int jM = s_jm[0];
        for (int w = 1; w < MERGE_THREADS / 32; ++w) jM = min(jM, s_jm[w]);
        // L' = sum_v exp(z_v - M) - 1 = l'_{jM} + sum_{j != jM} (1 + l'_j) exp(m_j - M)
        float lloc = 0.f;
        for (int j = threadIdx.x; j < n_tiles; j += MERGE_THREADS) {
            const float2 ml = pr[j];
            lloc += j == jM ? ml.y : (1.f + ml.y) * ex2_approx((ml.x - M) * LOG2E);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lloc += __shfl_xor_sync(0xffffffffu, lloc, o);
        if (lane == 0) s_red[wid] = lloc;
        __syncthreads();
        float c_t = 0.f;
        if (threadIdx.x == 0) {
            float Lm1 = 0.f;
            for (int w = 0; w < MERGE_THREADS / 32; ++w) Lm1 += s_red[w];
            float Mrow = M;  // the row max over every column of the head
            if (vpstat) {
                // vocab-parallel head: combine the ranks' (M_r, L'_r) like tiles -- the first
                // rank holding the row max enters with L'_r, the others with
                // (1 + L'_r) exp(M_r - M); this rank's own M, L' are those of slot rank
                float Mg = -INFINITY;
                for (int r = 0; r < vp_R; ++r) Mg = fmaxf(Mg, vpstat[r * vp_stride + p].x);
                int rM = 0;
                while (rM < vp_R - 1 && vpstat[rM * vp_stride + p].x != Mg) ++rM;
                float L = 0.f;
                for (int r = 0; r < vp_R; ++r) {
                    const float2 st = vpstat[r * vp_stride + p];
                    L += r == rM ? st.y : (1.f + st.y) * ex2_approx((st.x - Mg) * LOG2E);
                }
                Lm1 = L;
                Mrow = Mg;
            }
            // log p_y = (z_y - M) - log1p(L'), not z_y - lse: lse = M + log1p(L') rounds
            // log1p(L') to the ulp of M (~2e-6 at |z| ~ 24), which is the whole of 1 - p_y when
            // p_y -> 1 (the onehot-cancellation rows)
            const float l1 = log1pf(Lm1);
            const float logp = (zy[p] - Mrow) - l1;
            const float A = adv_c[p];
            const float rho = expf(logp - old_c[p]);
            const float lo = 1.f - eps_lo, hi = 1.f + eps_hi;
            const float rc = fminf(fmaxf(rho, lo), hi);
            const double u = (double)rho * (double)A, cl = (double)rc * (double)A;
            const double term = u < cl ? u : cl;
            const bool clipped = (A > 0.f && rho > hi) || (A < 0.f && rho < lo);
            // weight w_t (1/N token mean by default) and the k3 KL penalty (8(f) variants):
            //   loss_t = w (-term + beta KL),  c_t = w ([unclipped] rho A - beta (1 - e^r))
            const double w = w_c ? (double)w_c[p] : 1.0 / Nd;
            double kl = 0.0, dkl = 0.0;
            if (kl_beta > 0.f && ref_c) {
                const double r = (double)ref_c[p] - (double)logp;
                const double er = exp(r);
                kl = er - r - 1.0;
                dkl = 1.0 - er;
            }
            c_t = (float)(w * ((clipped ? 0.0 : (double)rho * (double)A) - (double)kl_beta * dkl));
            row_term[p] = w * (-term + (double)kl_beta * kl);
            row_rho[p] = rho;
            row_logp[p] = logp;
            row_clip[p] = clipped ? 1 : 0;
            row_kl[p] = (float)kl;
            if (logp_out) logp_out[idx[p]] = logp;
            s_bc[0] = l1;
            s_bc[1] = c_t;
            s_bc[3] = Mrow;
            // target column: c (p_y - 1) = c expm1(z_y - lse), exact where p_y -> 1
            s_bc[2] = c_t * expm1f(logp);
        }
        __syncthreads();
        const float l1 = s_bc[0];
        c_t = s_bc[1];
        const float g_y = s_bc[2];
        const float Mrow = s_bc[3];
        // exp(m_j - lse) = exp((m_j - M) - log1p(L'))
        for (int j = threadIdx.x; j < n_tiles; j += MERGE_THREADS)
            s_f[j] = c_t * ex2_approx(((pr[j].x - Mrow) - l1) * LOG2E);
        __syncthreads();
        const int32_t y = tgt_c[p];
        // 16-byte vectors, MERGE_UNROLL loads in flight per thread before any store
        auto conv = [&](const uint4& in, int v0) -> uint4 {
            const float f = s_f[v0 >> 8];  // 256-column tiles
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&in);
            float g[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 x = __bfloat1622float2(h2[k]);
                g[2 * k] = f * x.x;
                g[2 * k + 1] = f * x.y;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (v0 + k == y) g[k] = g_y;
            uint4 out;
            out.x = pack_bf162(g[0], g[1]);
            out.y = pack_bf162(g[2], g[3]);
            out.z = pack_bf162(g[4], g[5]);
            out.w = pack_bf162(g[6], g[7]);
            return out;
        };
        constexpr int MERGE_UNROLL = 4;
        int c = threadIdx.x;
        for (; c + (MERGE_UNROLL - 1) * MERGE_THREADS < nvec; c += MERGE_UNROLL * MERGE_THREADS) {
            uint4 in[MERGE_UNROLL];
#pragma unroll
            for (int u = 0; u < MERGE_UNROLL; ++u) in[u] = row4[c + u * MERGE_THREADS];
#pragma unroll
            for (int u = 0; u < MERGE_UNROLL; ++u)
                row4[c + u * MERGE_THREADS] = conv(in[u], (c + u * MERGE_THREADS) * 8);
        }
        for (; c < nvec; c += MERGE_THREADS) row4[c] = conv(row4[c], c * 8);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------- K7 reduce
__global__ void __launch_bounds__(1024)
    k_loss_reduce(const int64_t* __restrict__ rows_dev, const int64_t* __restrict__ nglob_dev,
                  const double* __restrict__ row_term, const float* __restrict__ row_rho,
                  const float* __restrict__ row_logp, const int32_t* __restrict__ row_clip,
                  const float* __restrict__ row_kl, double* __restrict__ loss_out,
                  double* __restrict__ stats_out, int32_t* d_status) {
    __shared__ double s[5][32];
    const int64_t rows = *rows_dev;
    const double N = (double)*nglob_dev;
    double a = 0.0, b = 0.0, c = 0.0, e = 0.0, k = 0.0;
    // thread t sums rows t, t + 1024, ... in order (coalesced loads; a fixed order, so the
    // result is deterministic), then a fixed shuffle tree and a fixed warp order
#pragma unroll 4
    for (int64_t p = threadIdx.x; p < rows; p += blockDim.x) {
        a += row_term[p];  // w_t (-term_t + beta KL_t)
        b += (double)row_rho[p];
        c += (double)row_logp[p];
        e += (double)row_clip[p];
        k += (double)row_kl[p];
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
        e += __shfl_down_sync(0xffffffffu, e, o);
        k += __shfl_down_sync(0xffffffffu, k, o);
    }
    if (lane == 0) {
        s[0][wid] = a;
        s[1][wid] = b;
        s[2][wid] = c;
        s[3][wid] = e;
        s[4][wid] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double A = 0, B = 0, Cc = 0, E = 0, K = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            A += s[0][w];
            B += s[1][w];
            Cc += s[2][w];
            E += s[3][w];
            K += s[4][w];
        }
        const double loss = N > 0.0 ? A : 0.0;
        *loss_out = loss;
        // non-finite loss, log-probs or ratios (e.g. a non-finite behaviour log-prob, whose
        // ratio the clamp would otherwise hide from the loss)
        if (!isfinite(loss) || !isfinite(Cc) || !isfinite(B)) atomicOr(d_status, AGENTRL_ST_NONFINITE);
        if (!(N > 0.0)) atomicOr(d_status, AGENTRL_ST_NO_TOKENS);  // S:204 (R16)
        if (stats_out) {
            const double r = rows > 0 ? (double)rows : 1.0;
            stats_out[0] = E / r;
            stats_out[1] = B / r;
            stats_out[2] = Cc / r;
            stats_out[3] = (double)rows;
            stats_out[4] = K / r;
        }
    }
}

// ---------------------------------------------------------------------------- host
LossWs plan_loss(int64_t T, int32_t d, int32_t V, size_t base, int32_t vp_world) {
    WsPlan p;
    p.off = base;
    LossWs w;
    const int64_t rows_cap = ceil_div(std::max<int64_t>(T, 1), GEMM_BM) * GEMM_BM;
    const int64_t n_chunks = ceil_div(T, CHUNK_TOKENS);
    w.n_tiles = (int32_t)ceil_div(V, GEMM_BN);
    w.idx = p.take(sizeof(int32_t) * (size_t)(T + 1));
    w.meta = p.take(sizeof(int64_t) * 4);
    w.chunk_cnt = p.take(sizeof(int32_t) * (size_t)(n_chunks + 1));
    w.chunk_base = w.chunk_cnt;
    w.tgt_c = p.take(sizeof(int32_t) * (size_t)rows_cap);
    w.old_c = p.take(sizeof(float) * (size_t)rows_cap);
    w.adv_c = p.take(sizeof(float) * (size_t)rows_cap);
    w.H = p.take((size_t)rows_cap * d * 2, 1024);
    w.P = p.take((size_t)rows_cap * V * 2, 1024);
    w.part = p.take(sizeof(float2) * (size_t)rows_cap * w.n_tiles);
    w.zy = p.take(sizeof(float) * (size_t)rows_cap);
    w.row_term = p.take(sizeof(double) * (size_t)rows_cap);
    w.row_rho = p.take(sizeof(float) * (size_t)rows_cap);
    w.row_logp = p.take(sizeof(float) * (size_t)rows_cap);
    w.row_clip = p.take(sizeof(int32_t) * (size_t)rows_cap);
    w.row_kl = p.take(sizeof(float) * (size_t)rows_cap);
    w.w_c = p.take(sizeof(float) * (size_t)rows_cap);
    w.ref_c = p.take(sizeof(float) * (size_t)rows_cap);
    w.red = p.take(sizeof(double) * 8);
    w.sched = p.take(sizeof(int) * 32);
    w.fbnd = p.take(sizeof(int64_t) * (MAX_FWD_CHUNKS + 1));
    w.prog = p.take(sizeof(int64_t) * (2 + MAX_FWD_CHUNKS) * PROG_UNITS);
    w.vp_world = vp_world;
    w.vpstat = w.vp_gh = 0;
    if (vp_world > 0) {
        w.vpstat = p.take(sizeof(float2) * (size_t)vp_world * rows_cap);
        w.vp_gh = p.take(sizeof(float) * (size_t)rows_cap * d, 1024);
    }
    w.total = p.off;
    return w;
}

// ---------------------------------------------------------------------------- vocab-parallel
// (W_head sharded by vocabulary rows over the group, every rank holding the
// same token rows).  Per row, this rank's statistics over its columns: M_r = max z,
// L'_r = sum exp(z - M_r) - 1 (the first max left out, as in the tile merge) -> its slot of the
// all-gather buffer (the other slots are zero; a sum all-reduce then fills every slot).
__global__ void __launch_bounds__(256)
    k_vp_row_stats(const int64_t* __restrict__ rows_dev, int32_t n_tiles,
                   const float2* __restrict__ part, float2* __restrict__ slot) {
    const int64_t rows = *rows_dev;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const float LOG2E = 1.4426950408889634f;
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < rows;
         p += nw) {
        const float2* pr = part + p * (int64_t)n_tiles;
        float M = -INFINITY;
        for (int j = lane; j < n_tiles; j += 32) M = fmaxf(M, pr[j].x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        int jm = 0x7fffffff;
        for (int j = lane; j < n_tiles; j += 32)
            if (pr[j].x == M) jm = min(jm, j);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) jm = min(jm, __shfl_xor_sync(0xffffffffu, jm, o));
        float L = 0.f;
        for (int j = lane; j < n_tiles; j += 32) {
            const float2 ml = pr[j];
            L += j == jm ? ml.y : (1.f + ml.y) * ex2_approx((ml.x - M) * LOG2E);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
        if (lane == 0) slot[p] = make_float2(M, L);
    }
}

// grad_hidden[idx[p]] = bf16(the all-reduced fp32 partial row p)
__global__ void __launch_bounds__(256)
    k_vp_scatter(const int64_t* __restrict__ rows_dev, int32_t d, const int32_t* __restrict__ idx,
                 const float* __restrict__ gh32, __nv_bfloat16* __restrict__ gh) {
    const int64_t rows = *rows_dev;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < rows;
         p += nw) {
        const float4* src = reinterpret_cast<const float4*>(gh32 + p * d);
        uint2* dst = reinterpret_cast<uint2*>(gh + (int64_t)idx[p] * d);
        for (int c = lane; c < d / 4; c += 32) {
            const float4 v = src[c];
            dst[c] = make_uint2(pack_bf162(v.x, v.y), pack_bf162(v.z, v.w));
        }
    }
}

// per-row aggregation weight w_t and reference log-prob (objective variants):
//   w_t = tok_weight[t] | 1/(G K_j n_g(t)) (GRPO group mean, reading R7b)
//       | 1/N (token mean)
__global__ void __launch_bounds__(256)
    k_row_weights(const int64_t* __restrict__ rows_dev, const int64_t* __restrict__ nglob_dev,
                  const int32_t* __restrict__ idx, const float* __restrict__ tok_weight,
                  const float* __restrict__ ref_logp, int32_t agg,
                  const int64_t* __restrict__ off, int32_t n_traj,
                  const int32_t* __restrict__ n_g, const int32_t* __restrict__ group_id,
                  const int32_t* __restrict__ grp_cnt, int32_t n_groups,
                  const int64_t* __restrict__ ngrp_dev, float* __restrict__ w_c,
                  float* __restrict__ ref_c, int32_t n_fchunks, float fratio,
                  int64_t* __restrict__ fbnd) {
    const int64_t rows = *rows_dev;
    const double N = (double)*nglob_dev;
    if (blockIdx.x == 0 && threadIdx.x <= n_fchunks) {
        // forward row chunks [fbnd[c], fbnd[c+1]): 256-row aligned, the last ends at rows;
        // geometric sizes (chunk c+1 = fratio x chunk c) keep the merge of the last chunk,
        // the one that cannot overlap a forward chunk, short
        const int c = threadIdx.x;
        double frac;
        if (fratio == 1.f) {
            frac = (double)c / n_fchunks;
        } else {
            const double r = fratio;
            frac = (1.0 - pow(r, (double)c)) / (1.0 - pow(r, (double)n_fchunks));
        }
        const int64_t b = (int64_t)ceil(frac * (double)rows / 256.0) * 256;
        fbnd[c] = c == n_fchunks ? rows : min(rows, b);
    }
    const double G = ngrp_dev ? (double)*ngrp_dev : 0.0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < rows;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = idx[p];
        double w = N > 0.0 ? 1.0 / N : 0.0;
        if (tok_weight) {
            w = tok_weight[t];
        } else if (agg == 1 && off && n_g && group_id && grp_cnt && G > 0.0) {
            int32_t lo = 0, hi = n_traj;  // trajectory of token t
            while (hi - lo > 1) {
                const int32_t mid = (lo + hi) >> 1;
                if (off[mid] <= t) lo = mid;
                else hi = mid;
            }
            const int32_t ng = n_g[lo], j = group_id[lo];
            const int32_t K = (j >= 0 && j < n_groups) ? grp_cnt[j] : 0;
            // E_{i,j} 1/K_{i,j} sum_g (token mean of g): w = 1 / (G K_j n_g)
            w = (ng > 0 && K > 0) ? 1.0 / (G * (double)K * (double)ng) : 0.0;
        }
        w_c[p] = (float)w;
        if (ref_c) ref_c[p] = ref_logp ? ref_logp[t] : 0.f;
    }
}

struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
};
static SideStream& side_stream() {
    static thread_local SideStream per_dev[MAX_DEVICES];  // a stream belongs to one device
    SideStream& ss = per_dev[current_device() & (MAX_DEVICES - 1)];
    if (!ss.s) {
        cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&ss.e0, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ss.e1, cudaEventDisableTiming);
    }
    return ss;
}

// backward-GEMM progress throttle: max lead in k-blocks over the slowest pair
// (AGENTRL_THROTTLE_LEAD, default 96, 0 = off) checked every AGENTRL_THROTTLE_EVERY k-blocks.
// glm9b: grad GEMM HBM reads 144/151 -> 67/64 GB at lead 192, +3% cycles, step 157 -> 150 ms on
// the power-capped part (profiles/r01_throttle.txt); lead 96 then measured 0.6 ms/step faster
// than 192 (less DRAM, higher clock; 2 x 3 interleaved A/B rounds, profiles/r01_ab_lead.txt)
static int throttle_lead() {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("AGENTRL_THROTTLE_LEAD");
        v = e ? atoi(e) : 96;
    }
    return gemm_dynamic() ? v : 0;
}
static int throttle_every() { return env_int("AGENTRL_THROTTLE_EVERY", 8); }
// forward GEMM throttle (AGENTRL_THROTTLE_LEAD_FWD, k-blocks of 128 K; 0 = off)
static int throttle_lead_fwd() {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("AGENTRL_THROTTLE_LEAD_FWD");
        v = e ? atoi(e) : 0;
    }
    return gemm_dynamic() ? v : 0;
}

// SMs left free for NCCL while grad_hidden overlaps C3 (AGENTRL_COMM_SMS, default 16), only
// when the communicator spans more than one rank
static int comm_reserve_sms() {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("AGENTRL_COMM_SMS");
        v = e ? std::max(0, atoi(e)) : 16;
    }
    return std::min(v, num_sms() / 2);
}

// forward row chunks (AGENTRL_FWD_CHUNKS; default 1 = the merge runs after the whole forward).
// With 4 chunks the merge of chunk c overlaps the forward of chunk c+1, but the co-resident
// merge blocks slow the forward GEMM about as much as they hide (live forward 51 vs 47.7 ms at
// glm9b), and the last merge stays exposed: 1 chunk measured 0.7 ms/step faster (3 A/B pairs)
static int fwd_chunks() {
    static int v = -1;
    if (v < 0) v = std::min(env_int("AGENTRL_FWD_CHUNKS", 1), MAX_FWD_CHUNKS);
    return v;
}
// one GPU: grad_hidden and grad_W on two prioritised streams so their tails overlap
// (AGENTRL_BWD_OVERLAP=1; off: measured neutral, 155.75 vs 155.46 ms full size and 20.50 vs
// 20.43 ms at the 1/8 shard, interleaved A/B)
static bool bwd_overlap() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("AGENTRL_BWD_OVERLAP");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}
// size ratio of consecutive forward row chunks (AGENTRL_FWD_RATIO, default 1 = equal; 0.5 and
// 0.35 shorten the last, un-overlapped merge but slow the forward as much: same step time)
static float fwd_ratio() {
    static float v = -1.f;
    if (v < 0.f) {
        const char* e = getenv("AGENTRL_FWD_RATIO");
        const float x = e ? (float)atof(e) : 0.f;
        v = (x > 0.f && x <= 1.f) ? x : 1.f;
    }
    return v;
}
struct ForkStreams {
    cudaStream_t hi = nullptr, lo = nullptr;  // forward chunks / merges
    cudaEvent_t fork = nullptr, join = nullptr, ev[MAX_FWD_CHUNKS] = {};
};
static ForkStreams& fork_streams() {
    static thread_local ForkStreams fs[MAX_DEVICES];  // per device
    ForkStreams& f = fs[current_device() & (MAX_DEVICES - 1)];
    if (!f.hi) {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        cudaStreamCreateWithPriority(&f.hi, cudaStreamNonBlocking, greatest);
        cudaStreamCreateWithPriority(&f.lo, cudaStreamNonBlocking, least);
        cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming);
        for (auto& e : f.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    return f;
}

int launch_policy_loss(const agentrl_loss_args* a, const agentrl_loss_out* o, uint8_t* ws,
                       const LossWs& w, const int32_t* idx_dev, const int64_t* rows_dev,
                       const float* adv_c_dev, const int64_t* nglob_dev, agentrl_comm comm,
                       int32_t* d_status, cudaStream_t stream, const FusedExtras* fx) {
    const int64_t T = a->T;
    const int32_t d = a->d, V = a->V;
    const int64_t rows_cap = ceil_div(std::max<int64_t>(T, 1), GEMM_BM) * GEMM_BM;
    int64_t* meta = reinterpret_cast<int64_t*>(ws + w.meta);
    int32_t* idx = reinterpret_cast<int32_t*>(ws + w.idx);
    float* adv_c = reinterpret_cast<float*>(ws + w.adv_c);
    int32_t* tgt_c = reinterpret_cast<int32_t*>(ws + w.tgt_c);
    float* old_c = reinterpret_cast<float*>(ws + w.old_c);
    __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(ws + w.H);
    uint16_t* PG = reinterpret_cast<uint16_t*>(ws + w.P);
    float2* part = reinterpret_cast<float2*>(ws + w.part);
    float* zy = reinterpret_cast<float*>(ws + w.zy);
    double* row_term = reinterpret_cast<double*>(ws + w.row_term);
    float* row_rho = reinterpret_cast<float*>(ws + w.row_rho);
    float* row_logp = reinterpret_cast<float*>(ws + w.row_logp);
    int32_t* row_clip = reinterpret_cast<int32_t*>(ws + w.row_clip);
    float* row_kl = reinterpret_cast<float*>(ws + w.row_kl);
    float* w_c = reinterpret_cast<float*>(ws + w.w_c);
    float* ref_c = reinterpret_cast<float*>(ws + w.ref_c);
    int* sched = reinterpret_cast<int*>(ws + w.sched);
    int64_t* fbnd = reinterpret_cast<int64_t*>(ws + w.fbnd);
    // vocab-parallel head (grad_W_mode 3): W_head is this rank's vocabulary shard, every rank
    // holds the same rows; the forward runs unchunked (the row statistics are all-gathered
    // between the forward GEMM and the merge)
    const bool vp = a->grad_W_mode == 3 && comm && w.vp_world > 0;
    const int vp_R = vp ? comm_world(comm) : 0;
    const int64_t vp_v0 = vp ? (int64_t)comm_rank(comm) * V : 0;
    const int n_fc = vp ? 1 : fwd_chunks();
    int* ctr_fwd = gemm_dynamic() ? sched + 0 : nullptr;
    int* ctr_gw = gemm_dynamic() ? sched + 4 : nullptr;
    int* ctr_gh = gemm_dynamic() ? sched + 8 : nullptr;
    AG_CUDA(cudaMemsetAsync(sched, 0, 32 * sizeof(int), stream));
    // progress arrays: [0] grad_W, [1] grad_hidden, [2 + c] forward chunk c
    int64_t* prog = reinterpret_cast<int64_t*>(ws + w.prog);
    const int lead = throttle_lead(), lead_fwd = throttle_lead_fwd();
    if (lead > 0 || lead_fwd > 0)
        AG_CUDA(cudaMemsetAsync(prog, 0xff, (2 + MAX_FWD_CHUNKS) * PROG_UNITS * sizeof(int64_t),
                                stream));

    // ---- compaction (standalone) or reuse of part 1's
    if (!idx_dev) {
        const int64_t n_chunks = ceil_div(T, CHUNK_TOKENS);
        int32_t* chunk = reinterpret_cast<int32_t*>(ws + w.chunk_cnt);
        AG_CUDA(cudaMemsetAsync(meta, 0, 4 * sizeof(int64_t), stream));
        if (n_chunks > 0) {
            ProfScope ps(KID_COMPACT, stream);
            k_mask_count<<<(unsigned)n_chunks, CHUNK_THREADS, 0, stream>>>(T, a->loss_mask, chunk);
            k_chunk_scan<<<1, 32, 0, stream>>>(n_chunks, chunk, meta);
            k_compact<<<(unsigned)n_chunks, CHUNK_THREADS, 0, stream>>>(T, a->loss_mask, a->adv_tok,
                                                                         chunk, idx, adv_c);
            count_launch(3);
        }
        idx_dev = idx;
        rows_dev = meta;
        adv_c_dev = adv_c;
        nglob_dev = a->n_mask_global;
    }

    // ---- outputs that are defined everywhere (grad_hidden's zero rows: below, beside the
    // forward when the merge stream exists -- only the grad_hidden GEMM reads it back)
    if (n_fc <= 1 && T > 0) AG_CUDA(cudaMemsetAsync(o->grad_hidden, 0, (size_t)T * d * 2, stream));
    if (o->logp) AG_CUDA(cudaMemsetAsync(o->logp, 0, (size_t)T * sizeof(float), stream));

    // ---- K4 gather
    {
        int grid = num_sms() * 4;
        ProfScope ps(KID_GATHER, stream);
        k_gather<<<grid, 256, 0, stream>>>(rows_dev, T, d, V,
                                           reinterpret_cast<const __nv_bfloat16*>(a->hidden),
                                           a->target, a->old_logp, idx_dev, H, tgt_c, old_c,
                                           d_status, vp_v0, vp ? (int64_t)V * vp_R : V);
        k_row_weights<<<num_sms() * 2, 256, 0, stream>>>(
            rows_dev, nglob_dev, idx_dev, a->tok_weight, a->ref_logp, a->loss_agg,
            fx ? fx->off : nullptr, fx ? fx->n_traj : 0, fx ? fx->n_g : nullptr,
            fx ? fx->group_id : nullptr, fx ? fx->grp_cnt : nullptr, fx ? fx->n_groups : 0,
            fx ? fx->ngrp : nullptr, w_c, ref_c, n_fc, fwd_ratio(), fbnd);
        count_launch(2);
        AG_CUDA(cudaGetLastError());
    }

    // ---- tensor maps
    CUtensorMap mH_K, mH_MN, mW_K, mW_MN, mG_K, mG_MN;
    int rc;
    if ((rc = make_map(&mH_K, H, d, rows_cap, d, 64, 128))) return rc;
    if ((rc = make_map(&mH_MN, H, d, rows_cap, d, 64, 64))) return rc;
    // K-major B box = the B rows one CTA stages (128 in a CTA pair, 256 alone)
    if ((rc = make_map(&mW_K, a->W_head, d, V, d, 64, gemm_use_pair() ? 128 : 256))) return rc;
    if ((rc = make_map(&mW_MN, a->W_head, d, V, d, 64, 64))) return rc;
    if ((rc = make_map(&mG_K, PG, V, rows_cap, V, 64, 128))) return rc;
    if ((rc = make_map(&mG_MN, PG, V, rows_cap, V, 64, 64))) return rc;

    const int64_t max_m_tiles = rows_cap / GEMM_BM;
    // ---- K5 forward GEMM + softmax-statistics epilogue, K6 merge.  With n_fc > 1 row chunks
    // the forward runs chunk by chunk on a high-priority stream and the (HBM-bound) merge of
    // chunk c runs on a low-priority stream beside the (tensor-bound) forward of chunk c+1.
    // vocab-parallel: z_y is written only by the rank whose shard holds y_t; the others keep 0
    // for the sum all-reduce
    if (vp) AG_CUDA(cudaMemsetAsync(zy, 0, sizeof(float) * (size_t)rows_cap, stream));
    ForkStreams* fs = n_fc > 1 ? &fork_streams() : nullptr;
    cudaStream_t s_fwd = stream, s_mrg = stream;
    if (fs) {
        s_fwd = fs->hi;
        s_mrg = fs->lo;
        AG_CUDA(cudaEventRecord(fs->fork, stream));
        AG_CUDA(cudaStreamWaitEvent(s_fwd, fs->fork, 0));
        AG_CUDA(cudaStreamWaitEvent(s_mrg, fs->fork, 0));
        // 2 T d bytes of zeros on the low-priority stream, overlapped with the forward GEMM
        if (T > 0) AG_CUDA(cudaMemsetAsync(o->grad_hidden, 0, (size_t)T * d * 2, s_mrg));
    }
    for (int c = 0; c < n_fc; ++c) {
        GemmArgs g{};
        g.m_range = n_fc > 1 ? fbnd + c : nullptr;
        g.m_dev = rows_dev;
        g.N = V;
        g.K_static = d;
        g.group_m = gemm_group_m();
        g.pol_a = l2_policy(0, 2);  // H rows of the current row group: reused by every column
        g.pol_b = l2_policy(1, 1);  // W: streamed, shared only by the concurrent row tiles
        g.tile_counter = ctr_fwd ? ctr_fwd + 16 * (c > 0) + c : nullptr;
        if (lead_fwd > 0) {
            g.prog = prog + (2 + c) * PROG_UNITS;
            g.prog_every = throttle_every();
            g.prog_lead = lead_fwd;
            g.prog_waits = throttle_wait_ctr(0);
        }
        g.scale = a->logit_scale;
        g.tgt = tgt_c;
        g.P = reinterpret_cast<__nv_bfloat16*>(PG);
        g.ldP = V;
        g.part = part;
        g.n_tiles = w.n_tiles;
        g.zy = zy;
        rc = gemm_fwd_ksub2()
                 ? launch_gemm<EPI_FWD, false, false, 1, 2>(mH_K, mW_K, g, max_m_tiles * w.n_tiles, s_fwd)
                 : launch_gemm<EPI_FWD, false, false, 1, 1>(mH_K, mW_K, g, max_m_tiles * w.n_tiles, s_fwd);
        if (rc) return rc;
        if (fs) {
            AG_CUDA(cudaEventRecord(fs->ev[c], s_fwd));
            AG_CUDA(cudaStreamWaitEvent(s_mrg, fs->ev[c], 0));
        }
        float2* vpstat = vp ? reinterpret_cast<float2*>(ws + w.vpstat) : nullptr;
        if (vp) {  // all-gather of (M_r, L'_r) per row and the owner's z_y (sum all-reduces)
            AG_CUDA(cudaMemsetAsync(vpstat, 0, sizeof(float2) * (size_t)vp_R * rows_cap, stream));
            k_vp_row_stats<<<num_sms() * 4, 256, 0, stream>>>(
                rows_dev, w.n_tiles, part, vpstat + (size_t)comm_rank(comm) * rows_cap);
            count_launch();
            AG_CUDA(cudaGetLastError());
            if ((rc = comm_allreduce_f32(comm, reinterpret_cast<float*>(vpstat),
                                         (size_t)2 * vp_R * rows_cap, stream)))
                return rc;
            if ((rc = comm_allreduce_f32(comm, zy, (size_t)rows_cap, stream))) return rc;
        }
        // merge + loss terms + G (in place) of this chunk; chunks merged beside the next
        // forward chunk keep a small footprint (2 blocks per SM next to the GEMM CTA)
        size_t smem = sizeof(float) * (size_t)w.n_tiles;
        // one wave: every block resident, so the grid-stride row split has no second-wave tail
        // (8 blocks per SM at 40 registers left a quarter of the blocks for a second wave)
        static int merge_occ = 0;
        if (merge_occ <= 0 &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&merge_occ, k_merge_g, MERGE_THREADS,
                                                          sizeof(float) * 4096) != cudaSuccess)
            merge_occ = 4;
        static const int merge_bps = env_int("AGENTRL_MERGE_BPS", 0);  // A/B override
        if (merge_bps > 0) merge_occ = merge_bps;
        int grid = num_sms() * (c + 1 < n_fc ? 2 : std::max(1, merge_occ));
        ProfScope ps(KID_MERGE, s_mrg);
        k_merge_g<<<grid, MERGE_THREADS, smem, s_mrg>>>(
            rows_dev, nglob_dev, V, w.n_tiles, part, zy, tgt_c, old_c, adv_c_dev, idx_dev,
            a->clip_eps_low, a->clip_eps_high, w_c, a->kl_beta > 0.f ? ref_c : nullptr,
            a->kl_beta, PG, row_term, row_rho, row_logp, row_clip, row_kl, o->logp,
            n_fc > 1 ? fbnd + c : nullptr, vpstat, vp_R, rows_cap);
        count_launch();
        AG_CUDA(cudaGetLastError());
    }
    if (fs) {  // join: the last merge waited on the last forward chunk
        AG_CUDA(cudaEventRecord(fs->join, s_mrg));
        AG_CUDA(cudaStreamWaitEvent(stream, fs->join, 0));
    }
    // ---- K7 loss reduction (+ C2)
    {
        ProfScope ps(KID_REDUCE, stream);
        k_loss_reduce<<<1, 1024, 0, stream>>>(rows_dev, nglob_dev, row_term, row_rho, row_logp,
                                              row_clip, row_kl, o->loss, o->loss_stats, d_status);
    }
    count_launch();
    AG_CUDA(cudaGetLastError());
    if (comm && !vp) {  // (vocab-parallel: every rank already holds the whole loss)
        if ((rc = comm_allreduce_f64(comm, o->loss, 1, stream))) return rc;
    }
    // ---- K9 grad_W = s G^T H   (M = V, N = d, K = T_eff); with a peer window (grad_W_mode 2)
    // the epilogue is also C3: each tile goes straight to its owner's window (peer.cu)
    PeerWindow* pw = (comm && a->grad_W_mode == 2) ? comm_peer(comm) : nullptr;
    if (pw && !peer_window_fits(pw, V, d)) pw = nullptr;
    if (pw && (rc = peer_guard(pw, d_status, stream))) return rc;  // owners done with epoch-1
    auto launch_grad_W = [&](cudaStream_t s) -> int {
        GemmArgs g{};
        if (pw) {
            g.peer_out = pw->d_staging;
            g.peer_rows = V / pw->world;
            g.peer_rank = pw->rank;
        }
        g.M_static = V;
        g.N = d;
        g.k_dev = rows_dev;
        g.group_m = gemm_group_m_bwd();
        // G^T column blocks are shared by the d/512 pairs of one row block, which drift apart
        // over the K = T_eff loop: evict_first made the laggards re-read G from HBM (DRAM
        // 160 -> 131 GB at glm9b with evict_normal, profiles/r01_l2pol_dyn.txt)
        g.pol_a = l2_policy(2, 0);
        g.pol_b = l2_policy(3, 0);  // H: re-read by every wave
        g.tile_counter = ctr_gw;
        if (lead > 0) {
            g.prog = prog;
            g.prog_every = throttle_every();
            g.prog_lead = lead;
            g.prog_waits = throttle_wait_ctr(1);
        }
        g.scale = a->logit_scale;
        g.gw = o->grad_W;
        g.ldo = d;
        const int64_t tiles = ceil_div(V, GEMM_BM) * ceil_div(d, GEMM_BN);
        return gemm_wide_n() ? launch_gemm<EPI_GRADW, true, true, 2>(mG_MN, mH_MN, g, tiles, s)
                             : launch_gemm<EPI_GRADW, true, true, 1>(mG_MN, mH_MN, g, tiles, s);
    };
    // ---- K8 grad_hidden = s G W   (M = T_eff, N = d, K = V), scattered to idx rows
    auto launch_grad_hidden = [&](cudaStream_t s, int rsv) -> int {
        GemmArgs g{};
        g.m_dev = rows_dev;
        g.N = d;
        g.K_static = V;
        g.group_m = gemm_group_m_bwd();
        g.pol_a = l2_policy(4, 0);  // G rows: shared by the pairs of one row block (as above)
        g.pol_b = l2_policy(5, 0);  // W: re-read by every wave
        g.tile_counter = ctr_gh;
        if (lead > 0) {
            g.prog = prog + PROG_UNITS;
            g.prog_every = throttle_every();
            g.prog_lead = lead;
            g.prog_waits = throttle_wait_ctr(2);
        }
        g.scale = a->logit_scale;
        g.idx = idx_dev;
        g.gh = reinterpret_cast<__nv_bfloat16*>(o->grad_hidden);
        g.ldo = d;
        const int64_t tiles = max_m_tiles * ceil_div(d, GEMM_BN);
        int r;
        if (vp) {
            // this rank's vocabulary columns give a partial grad_h: fp32 rows (the EPI_GRADW
            // epilogue, row = compacted row), summed over the group, then scattered as bf16
            float* gh32 = reinterpret_cast<float*>(ws + w.vp_gh);
            g.gw = gh32;
            r = gemm_wide_n() ? launch_gemm<EPI_GRADW, false, true, 2>(mG_K, mW_MN, g, tiles, s, 0)
                              : launch_gemm<EPI_GRADW, false, true, 1>(mG_K, mW_MN, g, tiles, s, 0);
            if (r) return r;
            if ((r = comm_allreduce_f32(comm, gh32, (size_t)rows_cap * d, s))) return r;
            k_vp_scatter<<<num_sms() * 4, 256, 0, s>>>(rows_dev, d, idx_dev, gh32,
                                                       reinterpret_cast<__nv_bfloat16*>(o->grad_hidden));
            count_launch();
            AG_CUDA(cudaGetLastError());
            return AGENTRL_OK;
        }
        return gemm_wide_n() ? launch_gemm<EPI_GRADH, false, true, 2>(mG_K, mW_MN, g, tiles, s, rsv)
                             : launch_gemm<EPI_GRADH, false, true, 1>(mG_K, mW_MN, g, tiles, s, rsv);
    };
    SideStream* ss = nullptr;
    if (!comm && bwd_overlap()) {
        // one GPU: grad_hidden (fewer, longer tiles) on the high-priority stream takes every SM
        // first; grad_W on the low-priority stream starts on the SMs grad_hidden's last wave
        // leaves idle, so the two GEMMs' tails overlap
        ForkStreams& f = fork_streams();
        AG_CUDA(cudaEventRecord(f.fork, stream));
        AG_CUDA(cudaStreamWaitEvent(f.hi, f.fork, 0));
        AG_CUDA(cudaStreamWaitEvent(f.lo, f.fork, 0));
        if ((rc = launch_grad_hidden(f.hi, 0))) return rc;
        if ((rc = launch_grad_W(f.lo))) return rc;
        AG_CUDA(cudaEventRecord(f.ev[0], f.hi));
        AG_CUDA(cudaEventRecord(f.ev[1], f.lo));
        AG_CUDA(cudaStreamWaitEvent(stream, f.ev[0], 0));
        AG_CUDA(cudaStreamWaitEvent(stream, f.ev[1], 0));
        return AGENTRL_OK;
    }
    if ((rc = launch_grad_W(stream))) return rc;
    // ---- C3 grad_W all-reduce on a side stream, overlapped with K8
    if (comm && (a->grad_W_mode == 1 || a->grad_W_mode == 2)) {
        ss = &side_stream();
        AG_CUDA(cudaEventRecord(ss->e0, stream));
        AG_CUDA(cudaStreamWaitEvent(ss->s, ss->e0, 0));
        rc = pw ? peer_signal_reduce(pw, o->grad_W, V, d, d_status, ss->s)  // fused C3 tail
             : a->grad_W_mode == 1
                 ? comm_allreduce_f32(comm, o->grad_W, (size_t)V * d, ss->s)
                 : comm_reduce_scatter_f32(comm, o->grad_W, (size_t)V * d, ss->s);  // FSDP shard
        if (rc) return rc;
        AG_CUDA(cudaEventRecord(ss->e1, ss->s));
    }
    // with a collective C3 in flight on the side stream, leave SMs for the NCCL kernel so it
    // overlaps this GEMM instead of queueing behind its persistent CTAs.  The fused P2P C3 has
    // already moved its bytes inside the grad_W GEMM; its side-stream tail (a slot sum of a few
    // dozen blocks) needs no reserved SMs.
    const bool nccl_c3 = ss && !pw && comm_world(comm) > 1;
    if ((rc = launch_grad_hidden(stream, nccl_c3 ? comm_reserve_sms() : 0))) return rc;
    if (ss) AG_CUDA(cudaStreamWaitEvent(stream, ss->e1, 0));
    return AGENTRL_OK;
}

}  // namespace agentrl

// ============================================================================ log-prob forward
// agentrl_logprob_fwd: forward-only token log-probs and entropies (the
// trainer's recomputation of pi_old / pi_ref log-probs, and the entropy that DAPO
// monitors).  Same compaction / gather / forward GEMM as part 2, with the EPI_LOGP
// epilogue (no P~ store: per (row, tile) max m, l' = sum exp(z-m) - 1,
// u = sum exp(z-m) (m - z) >= 0), then one warp per row, with l1 = log1p(L'):
//   logp = (z_y - M) - l1,
//   entropy = -sum_v p_v log p_v = sum_v p_v (lse - z_v)
//           = l1 + sum_j exp((m_j - M) - l1) [(M - m_j)(1 + l'_j) + u_j]
//   (every term >= 0: exact to fp32 rounding even for p_y -> 1 rows).
namespace agentrl {

__global__ void __launch_bounds__(256)
    k_logp_merge(const int64_t* __restrict__ rows_dev, int32_t n_tiles,
                 const float4* __restrict__ part4, const float* __restrict__ zy,
                 const int32_t* __restrict__ idx, float* __restrict__ logp_out,
                 float* __restrict__ ent_out, int32_t* d_status) {
    const int64_t rows = *rows_dev;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float LOG2E = 1.4426950408889634f;
    for (int64_t p = (int64_t)blockIdx.x * 8 + warp; p < rows; p += (int64_t)gridDim.x * 8) {
        const float4* pr = part4 + p * (int64_t)n_tiles;
        float M = -INFINITY;
        for (int j = lane; j < n_tiles; j += 32) M = fmaxf(M, pr[j].x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        int jm = 0x7fffffff;
        for (int j = lane; j < n_tiles; j += 32)
            if (pr[j].x == M) jm = min(jm, j);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) jm = min(jm, __shfl_xor_sync(0xffffffffu, jm, o));
        float Lm1 = 0.f;
        for (int j = lane; j < n_tiles; j += 32) {
            const float4 t = pr[j];
            Lm1 += j == jm ? t.y : (1.f + t.y) * ex2_approx((t.x - M) * LOG2E);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) Lm1 += __shfl_xor_sync(0xffffffffu, Lm1, o);
        const float l1 = log1pf(Lm1);
        float Hs = 0.f;  // sum_j w_j [(M - m_j)(1 + l'_j) + u_j]
        for (int j = lane; j < n_tiles; j += 32) {
            const float4 t = pr[j];
            Hs += expf((t.x - M) - l1) * fmaf(M - t.x, 1.f + t.y, t.z);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) Hs += __shfl_xor_sync(0xffffffffu, Hs, o);
        if (lane == 0) {
            const float logp = (zy[p] - M) - l1;  // see k_merge_g
            const int64_t t = idx[p];
            logp_out[t] = logp;
            if (ent_out) ent_out[t] = l1 + Hs;
            if (!isfinite(logp)) atomicOr(d_status, AGENTRL_ST_NONFINITE);
        }
    }
}

LogpWs plan_logp(int64_t T, int32_t d, int32_t V, size_t base) {
    WsPlan p;
    p.off = base;
    LogpWs w;
    const int64_t rows_cap = ceil_div(std::max<int64_t>(T, 1), GEMM_BM) * GEMM_BM;
    const int64_t n_chunks = ceil_div(T, CHUNK_TOKENS);
    w.n_tiles = (int32_t)ceil_div(V, GEMM_BN);
    w.idx = p.take(sizeof(int32_t) * (size_t)(T + 1));
    w.meta = p.take(sizeof(int64_t) * 4);
    w.chunk = p.take(sizeof(int32_t) * (size_t)(n_chunks + 1));
    w.tgt_c = p.take(sizeof(int32_t) * (size_t)rows_cap);
    w.H = p.take((size_t)rows_cap * d * 2, 1024);
    w.part4 = p.take(sizeof(float4) * (size_t)rows_cap * w.n_tiles);
    w.zy = p.take(sizeof(float) * (size_t)rows_cap);
    w.sched = p.take(sizeof(int) * 16);
    w.total = p.off;
    return w;
}

int launch_logprob(const agentrl_logprob_args* a, float* logp, float* entropy, uint8_t* ws,
                   const LogpWs& w, int32_t* d_status, cudaStream_t stream) {
    const int64_t T = a->T;
    const int32_t d = a->d, V = a->V;
    const int64_t rows_cap = ceil_div(std::max<int64_t>(T, 1), GEMM_BM) * GEMM_BM;
    int64_t* meta = reinterpret_cast<int64_t*>(ws + w.meta);
    int32_t* idx = reinterpret_cast<int32_t*>(ws + w.idx);
    int32_t* chunk = reinterpret_cast<int32_t*>(ws + w.chunk);
    int32_t* tgt_c = reinterpret_cast<int32_t*>(ws + w.tgt_c);
    __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(ws + w.H);
    float4* part4 = reinterpret_cast<float4*>(ws + w.part4);
    float* zy = reinterpret_cast<float*>(ws + w.zy);
    int* sched = reinterpret_cast<int*>(ws + w.sched);
    AG_CUDA(cudaMemsetAsync(meta, 0, 4 * sizeof(int64_t), stream));
    AG_CUDA(cudaMemsetAsync(sched, 0, 16 * sizeof(int), stream));
    AG_CUDA(cudaMemsetAsync(logp, 0, (size_t)T * sizeof(float), stream));
    if (entropy) AG_CUDA(cudaMemsetAsync(entropy, 0, (size_t)T * sizeof(float), stream));
    const int64_t n_chunks = ceil_div(T, CHUNK_TOKENS);
    if (n_chunks > 0) {
        ProfScope ps(KID_COMPACT, stream);
        k_mask_count<<<(unsigned)n_chunks, CHUNK_THREADS, 0, stream>>>(T, a->loss_mask, chunk);
        k_chunk_scan<<<1, 32, 0, stream>>>(n_chunks, chunk, meta);
        k_compact<<<(unsigned)n_chunks, CHUNK_THREADS, 0, stream>>>(T, a->loss_mask, nullptr,
                                                                     chunk, idx, nullptr);
        count_launch(3);
    }
    {
        ProfScope ps(KID_GATHER, stream);
        k_gather<<<num_sms() * 4, 256, 0, stream>>>(
            meta, T, d, V, reinterpret_cast<const __nv_bfloat16*>(a->hidden), a->target, nullptr,
            idx, H, tgt_c, nullptr, d_status);
        count_launch();
        AG_CUDA(cudaGetLastError());
    }
    CUtensorMap mH_K, mW_K;
    int rc;
    if ((rc = make_map(&mH_K, H, d, rows_cap, d, 64, 128))) return rc;
    if ((rc = make_map(&mW_K, a->W_head, d, V, d, 64, gemm_use_pair() ? 128 : 256))) return rc;
    {
        GemmArgs g{};
        g.m_dev = meta;
        g.N = V;
        g.K_static = d;
        g.group_m = gemm_group_m();
        g.pol_a = l2_policy(0, 2);
        g.pol_b = l2_policy(1, 1);
        g.tile_counter = gemm_dynamic() ? sched : nullptr;
        g.scale = a->logit_scale;
        g.tgt = tgt_c;
        g.part4 = part4;
        g.n_tiles = w.n_tiles;
        g.zy = zy;
        const int64_t mt = (rows_cap / GEMM_BM) * w.n_tiles;
        rc = gemm_fwd_ksub2() ? launch_gemm<EPI_LOGP, false, false, 1, 2>(mH_K, mW_K, g, mt, stream)
                              : launch_gemm<EPI_LOGP, false, false, 1, 1>(mH_K, mW_K, g, mt, stream);
        if (rc) return rc;
    }
    {
        ProfScope ps(KID_LOGP_MERGE, stream);
        k_logp_merge<<<num_sms() * 8, 256, 0, stream>>>(meta, w.n_tiles, part4, zy, idx, logp,
                                                        entropy, d_status);
        count_launch();
        AG_CUDA(cudaGetLastError());
    }
    return AGENTRL_OK;
}

}  // namespace agentrl
