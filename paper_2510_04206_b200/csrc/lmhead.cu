// lmhead.cu -- part 2 of the hot path: token-level PPO-clip loss through the LM head and its
// exact backward (PAPER.md P:1182-1190 token factorisation, P:1230-1241 PPO-clip,
// P:1132-1141 token-level mean / decoupled eps).
//
//   K4 k_gather       compacted rows: H[p] = hidden[idx[p]], target/old per row; rows
//                     [T_eff, pad64) zeroed (they are inside grad_W's K range)
//   K5 gemm<FWD>      z = s * H W^T on tcgen05; epilogue: per (row, 256-col tile) max m and
//                     l' = sum exp(z - m) - 1, P~ = exp(z - m) -> bf16 [rows, V], z_y gathered
//   K6 k_row_stats    per row: lse over tiles, logp, rho, PPO-clip term, c = unclipped ? w rho A
//                     : 0; the per-(row, tile) gradient scale f = c exp((m_tile - M) - log1p(L'))
//                     and the target column's G value c expm1(logp)
//   K7 k_loss_reduce  fixed-order fp64 reduction of the per-row terms -> loss, stats
//   K9 gemm<GRADW,XF> grad_W = s * G^T H   (A = P~ MN-major, B = H MN-major, K = T_eff)
//   C3                grad_W all-reduce / reduce-scatter on a side stream, overlapped with K8, or
//                     fused into K9's epilogue as peer stores (peer.cu)
//   K8 gemm<GRADH,XF> grad_hidden[idx] = s * G W  (A = P~ K-major, B = W MN-major, K = V)
// In K8 and K9 (XF) transform warps rewrite each staged P~ tile in shared memory as
// G = bf16(f * P~) (target column replaced) before the MMA reads it: G never exists in HBM.
//
// Executed tensor work is 6 * T_eff * V * d FLOP (three GEMMs; no recompute: the bf16 P~
// written by the forward epilogue replaces the second logits GEMM).  See DESIGN.md.
//
// Schedule and staging choices are compile-time constants (measured defaults; A/B builds pass
// -D overrides through build.py, tests/test_gpu_variants.py keeps them parity-green).
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

// ---------------------------------------------------------------------------- build knobs
// CTA-pair (cta_group::2) GEMMs; 0: the 1-CTA cta_group::1 variant (128 x 256 tiles)
#ifndef AGENTRL_GEMM_PAIR
#define AGENTRL_GEMM_PAIR 1
#endif
// dynamic tile scheduler (atomic counter, tiles claimed in global order); 0: static persistent
// striding (tile = unit + i * units: pairs drift apart over long runs)
#ifndef AGENTRL_GEMM_DYNAMIC
#define AGENTRL_GEMM_DYNAMIC 1
#endif
// 1: one CTA (pair) per tile instead of one per SM
#ifndef AGENTRL_GEMM_FULLGRID
#define AGENTRL_GEMM_FULLGRID 0
#endif
// 512-column tiles for the long-K backward GEMMs (CTA pairs only); 0: 256-column tiles
#ifndef AGENTRL_GEMM_WIDE_N
#define AGENTRL_GEMM_WIDE_N 1
#endif
// forward / log-prob GEMMs stage two 64-wide K atoms per k-block (8 MMAs per barrier round
// trip: 94% vs 89% tensor-pipe active, profiles/r01_fwd_ksub.txt); 1: one atom
#ifndef AGENTRL_FWD_KSUB
#define AGENTRL_FWD_KSUB 2
#endif
// raster: tiles grouped by GROUP_M row blocks, columns fastest inside (forward / backward)
#ifndef AGENTRL_GROUP_M
#define AGENTRL_GROUP_M 16
#endif
#ifndef AGENTRL_GROUP_M_BWD
#define AGENTRL_GROUP_M_BWD 8
#endif
// L2 eviction policy per operand (0 normal, 1 evict_first, 2 evict_last): forward H evict_last
// (reused by every column block of its row group), W evict_first (streamed); backward all
// normal (evict_first on G made the pairs sharing a row block re-read it from HBM,
// profiles/r01_l2pol_dyn.txt)
#ifndef AGENTRL_L2POL_FWD_A
#define AGENTRL_L2POL_FWD_A 2
#endif
#ifndef AGENTRL_L2POL_FWD_B
#define AGENTRL_L2POL_FWD_B 1
#endif
#ifndef AGENTRL_L2POL_BWD
#define AGENTRL_L2POL_BWD 0
#endif
// backward-GEMM progress throttle: max lead in k-blocks over the slowest pair (0 = off),
// checked every THROTTLE_EVERY k-blocks.  glm9b: grad GEMM HBM reads 144/151 -> 67/64 GB at
// lead 192, +3% cycles, step 157 -> 150 ms on the power-capped part (profiles/r01_throttle.txt);
// lead 96 then measured 0.6 ms/step faster than 192 (profiles/r01_ab_lead.txt)
#ifndef AGENTRL_THROTTLE_LEAD
#define AGENTRL_THROTTLE_LEAD 96
#endif
#ifndef AGENTRL_THROTTLE_EVERY
#define AGENTRL_THROTTLE_EVERY 8
#endif
// forward GEMM throttle (k-blocks of 128 K; 0 = off)
#ifndef AGENTRL_THROTTLE_LEAD_FWD
#define AGENTRL_THROTTLE_LEAD_FWD 0
#endif
// grad_hidden split-K: n > 0 forces n (1: never split, the default); 0 = chosen from the
// workspace's row bound (tile-wave tails at small shard sizes).  Measured on the power-capped
// part (profiles/r02_ksplit_ab.txt): the split grad_hidden is 5-7% faster at the 2/4/8-GPU
// shard sizes, but the step is 0.4-1.7% slower -- the partials' round trip and the busier tail
// cost power that the other GEMMs' clock pays for -- so it is off by default.
#ifndef AGENTRL_KSPLIT_FORCE
#define AGENTRL_KSPLIT_FORCE 1
#endif
// SMs left free for an NCCL C3 kernel while grad_hidden overlaps it (multi-rank only)
#ifndef AGENTRL_COMM_SMS
#define AGENTRL_COMM_SMS 16
#endif

constexpr bool kPair = AGENTRL_GEMM_PAIR != 0;
constexpr bool kDynamic = AGENTRL_GEMM_DYNAMIC != 0;
constexpr bool kWideN = AGENTRL_GEMM_WIDE_N != 0 && kPair;
constexpr int kFwdKsub = AGENTRL_FWD_KSUB == 1 ? 1 : 2;
constexpr int kThrottleLead = kDynamic ? AGENTRL_THROTTLE_LEAD : 0;
constexpr int kThrottleLeadFwd = kDynamic ? AGENTRL_THROTTLE_LEAD_FWD : 0;

template <int EPI, bool A_MN, bool B_MN, int NSPLIT, int KSUB = 1, bool XF = false>
static int launch_gemm(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& g,
                       int64_t max_tiles, cudaStream_t stream, int reserve_sms = 0) {
    ProfScope ps(EPI == EPI_FWD    ? KID_FWD
                 : EPI == EPI_GRADW ? (A_MN ? KID_GRADW : KID_GRADH)
                 : EPI == EPI_LOGP  ? KID_LOGP_GEMM
                                    : KID_GRADH,
                 stream);
    constexpr int threads = XF ? GEMM_THREADS_XF : GEMM_THREADS;
    // max_tiles is counted in 128 x 256 tiles (an upper bound of the CTAs worth launching)
    if constexpr (kPair) {
        auto kern = gemm_sm100_pair_kernel<EPI, A_MN, B_MN, NSPLIT, KSUB, XF>;
        constexpr int smem = GemmCfg<true, NSPLIT, KSUB>::SMEM +
                             (EPI == EPI_GRADW ? GemmCfg<true, NSPLIT, KSUB>::EPI_STAGE : 0) +
                             (EPI == EPI_FWD ? GemmCfg<true, NSPLIT, KSUB>::PSTAGE : 0) +
                             (XF ? GemmCfg<true, NSPLIT, KSUB>::STAGES * XIN_STAGE : 0);
        static std::atomic<uint64_t> attr_done{0};  // per instantiation and device
        if (!func_attr_once(attr_done, (const void*)kern, smem)) return AGENTRL_ERR_CUDA;
        int64_t grid = AGENTRL_GEMM_FULLGRID
                           ? 2 * std::max<int64_t>(max_tiles, 1)
                           : std::min<int64_t>((num_sms() - reserve_sms) & ~1,
                                               std::max<int64_t>(max_tiles, 2));
        grid &= ~int64_t(1);
        kern<<<(unsigned)grid, threads, smem, stream>>>(a, b, g);
    } else {
        auto kern = gemm_sm100_kernel<EPI, A_MN, B_MN, XF>;
        constexpr int smem = GemmCfg<false, 1>::SMEM + (XF ? GemmCfg<false, 1>::STAGES * XIN_STAGE : 0) +
                             (EPI == EPI_FWD ? GemmCfg<false, 1>::PSTAGE : 0);
        static std::atomic<uint64_t> attr_done{0};
        if (!func_attr_once(attr_done, (const void*)kern, smem)) return AGENTRL_ERR_CUDA;
        int grid = AGENTRL_GEMM_FULLGRID
                       ? (int)std::max<int64_t>(max_tiles, 1)
                       : (int)std::min<int64_t>(num_sms() - reserve_sms,
                                                std::max<int64_t>(max_tiles, 1));
        kern<<<grid, threads, smem, stream>>>(a, b, g);
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
// rows_eff: the masked rows part 2 processes, min(T_eff, row_limit) (the caller's max_rows;
// more masked tokens than that set AGENTRL_ST_ROWS_OVERFLOW and only the first row_limit are
// processed).  Written here by block 0 for every later kernel of the call.
__global__ void __launch_bounds__(256)
    k_gather(const int64_t* __restrict__ rows_dev, int64_t row_limit, int64_t* rows_eff, int64_t T,
             int32_t d, int32_t V, const __nv_bfloat16* __restrict__ hidden,
             const int32_t* __restrict__ target, const float* __restrict__ old_logp,
             const int32_t* __restrict__ idx, __nv_bfloat16* __restrict__ H,
             int32_t* __restrict__ tgt_c, float* __restrict__ old_c, int32_t* d_status,
             int64_t v0 = 0, int64_t V_total = -1) {
    // vocab-parallel head: this rank holds columns [v0, v0 + V) of V_total; a target outside
    // the shard gets tgt_c = -1 (never matches a column here)
    if (V_total < 0) V_total = V;
    const int64_t rows_all = *rows_dev;
    const int64_t rows = rows_all < row_limit ? rows_all : row_limit;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *rows_eff = rows;
        if (rows_all > row_limit) atomicOr(d_status, AGENTRL_ST_ROWS_OVERFLOW);
    }
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

// ---------------------------------------------------------------------------- K6 row stats
// A block owns RS_ROWS consecutive rows (lane = row, so every access to the tile-major part /
// fscale arrays is 32 consecutive rows); warp w takes the 256-column tiles j = w, w + 8, ...
// Per row, in a fixed order (deterministic): M = max_j m_j and the first tile jM holding it;
// L' = sum_v exp(z_v - M) - 1 = l'_{jM} + sum_{j != jM} (1 + l'_j) exp(m_j - M) (warp partials
// added in warp order); then the loss terms and the gradient scale of every tile,
// f_j = c exp(m_j - lse) = c exp((m_j - M) - log1p(L')).
constexpr int RS_ROWS = 32;
constexpr int RS_WARPS = 8;

// The row statistics over the tiles of this rank's columns, in the fixed order above (shared by
// k_row_stats and the vocab-parallel slot kernel, so a one-rank vocab-parallel head reproduces
// the single-GPU bits): returns M and the first tile jM holding it; warp w's L' partial is left
// in s_l[w][lane] (the caller sums the warps in warp order after a barrier).
__device__ __forceinline__ void rs_max_sum(const float2* __restrict__ part, int64_t ld,
                                           int32_t n_tiles, int64_t p, bool ok,
                                           float (&s_m)[RS_WARPS][RS_ROWS],
                                           int (&s_j)[RS_WARPS][RS_ROWS],
                                           float (&s_l)[RS_WARPS][RS_ROWS], float& M, int& jM) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const float LOG2E = 1.4426950408889634f;
    // ---- row max and the first tile holding it (tiles in increasing order per warp)
    float m = -INFINITY;
    int jm = 0x7fffffff;
    if (ok)
#pragma unroll 4
        for (int j = w; j < n_tiles; j += RS_WARPS) {
            const float x = part[(int64_t)j * ld + p].x;
            if (x > m) {
                m = x;
                jm = j;
            }
        }
    s_m[w][lane] = m;
    s_j[w][lane] = jm;
    __syncthreads();
    M = s_m[0][lane];
    jM = s_j[0][lane];
#pragma unroll
    for (int q = 1; q < RS_WARPS; ++q) {
        const float x = s_m[q][lane];
        const int jq = s_j[q][lane];
        if (x > M || (x == M && jq < jM)) {
            M = x;
            jM = jq;
        }
    }
    // ---- L' partials
    float L = 0.f;
    if (ok)
#pragma unroll 4
        for (int j = w; j < n_tiles; j += RS_WARPS) {
            const float2 ml = part[(int64_t)j * ld + p];
            L += j == jM ? ml.y : (1.f + ml.y) * ex2_approx((ml.x - M) * LOG2E);
        }
    s_l[w][lane] = L;
    __syncthreads();
}

__global__ void __launch_bounds__(RS_ROWS * RS_WARPS)
    k_row_stats(const int64_t* __restrict__ rows_dev, const int64_t* __restrict__ nglob_dev,
                int32_t n_tiles, int64_t ld, const float2* __restrict__ part /* [n_tiles][ld] */,
                const float* __restrict__ zy, const int32_t* __restrict__ tgt_c,
                const float* __restrict__ old_c, const float* __restrict__ adv_c,
                const int32_t* __restrict__ idx, float eps_lo, float eps_hi,
                const float* __restrict__ w_c /* per-row weight w_t */,
                const float* __restrict__ ref_c /* per-row ref log-prob or null */,
                float kl_beta, float* __restrict__ fscale /* [n_tiles][ld] */,
                int2* __restrict__ xrow /* [rows] (target column, G value bits) */,
                double* __restrict__ row_term /* w (-term + beta KL) */,
                float* __restrict__ row_rho, float* __restrict__ row_logp,
                int32_t* __restrict__ row_clip, float* __restrict__ row_kl,
                float* __restrict__ logp_out,
                const float2* __restrict__ vpstat = nullptr /* [vp_R][vp_stride] (M_r, L'_r) */,
                int32_t vp_R = 0, int64_t vp_stride = 0) {
    __shared__ float s_m[RS_WARPS][RS_ROWS];
    __shared__ int s_j[RS_WARPS][RS_ROWS];
    __shared__ float s_l[RS_WARPS][RS_ROWS];
    __shared__ float s_c[RS_ROWS], s_sub[RS_ROWS];
    const int64_t rows = *rows_dev;
    const double Nd = (double)*nglob_dev;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const float LOG2E = 1.4426950408889634f;

    for (int64_t p0 = (int64_t)blockIdx.x * RS_ROWS; p0 < rows; p0 += (int64_t)gridDim.x * RS_ROWS) {
        const int64_t p = p0 + lane;
        const bool ok = p < rows;
        float M;
        int jM;
        rs_max_sum(part, ld, n_tiles, p, ok, s_m, s_j, s_l, M, jM);
        if (w == 0) {
            float Lm1 = 0.f;
#pragma unroll
            for (int q = 0; q < RS_WARPS; ++q) Lm1 += s_l[q][lane];
            float c_t = 0.f;
            if (ok) {
                float Mrow = M;  // the row max over every column of the head
                if (vpstat) {
                    // vocab-parallel head: combine the ranks' (M_r, L'_r) like tiles -- the first
                    // rank holding the row max enters with L'_r, the others with
                    // (1 + L'_r) exp(M_r - M); this rank's own M, L' are those of slot rank
                    float Mg = -INFINITY;
                    for (int r = 0; r < vp_R; ++r) Mg = fmaxf(Mg, vpstat[r * vp_stride + p].x);
                    int rM = 0;
                    while (rM < vp_R - 1 && vpstat[rM * vp_stride + p].x != Mg) ++rM;
                    float Lg = 0.f;
                    for (int r = 0; r < vp_R; ++r) {
                        const float2 st = vpstat[r * vp_stride + p];
                        Lg += r == rM ? st.y : (1.f + st.y) * ex2_approx((st.x - Mg) * LOG2E);
                    }
                    Lm1 = Lg;
                    Mrow = Mg;
                }
                // log p_y = (z_y - M) - log1p(L'), not z_y - lse: lse = M + log1p(L') rounds
                // log1p(L') to the ulp of M (~2e-6 at |z| ~ 24), which is the whole of 1 - p_y
                // when p_y -> 1 (the onehot-cancellation rows)
                const float l1 = log1pf(Lm1);
                const float logp = (zy[p] - Mrow) - l1;
                const float A = adv_c[p];
                const float rho = expf(logp - old_c[p]);
                const float lo = 1.f - eps_lo, hi = 1.f + eps_hi;
                const float rc = fminf(fmaxf(rho, lo), hi);
                const double u = (double)rho * (double)A, cl = (double)rc * (double)A;
                const double term = u < cl ? u : cl;
                const bool clipped = (A > 0.f && rho > hi) || (A < 0.f && rho < lo);
                // weight w_t (1/N token mean by default) and the k3 KL penalty (8(f)):
                //   loss_t = w (-term + beta KL),  c_t = w ([unclipped] rho A - beta (1 - e^r))
                const double wt = w_c ? (double)w_c[p] : 1.0 / Nd;
                double kl = 0.0, dkl = 0.0;
                if (kl_beta > 0.f && ref_c) {
                    const double r = (double)ref_c[p] - (double)logp;
                    const double er = exp(r);
                    kl = er - r - 1.0;
                    dkl = 1.0 - er;
                }
                c_t = (float)(wt * ((clipped ? 0.0 : (double)rho * (double)A) -
                                    (double)kl_beta * dkl));
                row_term[p] = wt * (-term + (double)kl_beta * kl);
                row_rho[p] = rho;
                row_logp[p] = logp;
                row_clip[p] = clipped ? 1 : 0;
                row_kl[p] = (float)kl;
                if (logp_out) logp_out[idx[p]] = logp;
                // target column: c (p_y - 1) = c expm1(z_y - lse), exact where p_y -> 1
                xrow[p] = make_int2(tgt_c[p], __float_as_int(c_t * expm1f(logp)));
                s_sub[lane] = l1;  // f_j = c exp((m_j - M) - l1)
                s_m[0][lane] = Mrow;
            }
            s_c[lane] = c_t;
        }
        __syncthreads();
        // ---- gradient scale of every tile (the backward GEMMs form G = bf16(f * P~))
        if (ok) {
            const float c_t = s_c[lane], l1 = s_sub[lane], Mrow = s_m[0][lane];
#pragma unroll 4
            for (int j = w; j < n_tiles; j += RS_WARPS)
                fscale[(int64_t)j * ld + p] =
                    c_t * ex2_approx(((part[(int64_t)j * ld + p].x - Mrow) - l1) * LOG2E);
        }
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
// rows_cap: the row capacity of the per-row buffers, max_rows (<= 0: T) rounded up to 256
int64_t loss_rows_cap(int64_t T, int64_t max_rows) {
    const int64_t r = (max_rows > 0 && max_rows < T) ? max_rows : T;
    return ceil_div(std::max<int64_t>(r, 1), 2 * GEMM_BM) * (2 * GEMM_BM);  // whole pair tiles
}

// grad_hidden has ceil(rows/256) x ceil(d/512) equal-length tiles for the CTA pairs; when that
// is a few waves with a partial last one, splitting every tile's k-blocks into S ranges (fp32
// partials summed afterwards) fills the idle pairs.  Cost in tile-waves: ceil(tiles S / pairs)
// / S, plus the partials' HBM round trip relative to the GEMM (8 S rows d bytes at ~6 TB/s
// against 2 rows V d FLOP at ~1.3 PF/s: S * 1733 / V of the GEMM).  Needs the row bound.
static int32_t choose_ksplit(int64_t max_rows, int32_t d, int32_t V) {
    if (AGENTRL_KSPLIT_FORCE > 0) return AGENTRL_KSPLIT_FORCE;
    const int pairs = num_sms() / 2;
    if (max_rows <= 0 || pairs <= 0) return 1;
    const int64_t tiles = ceil_div(max_rows, 2 * GEMM_BM) * ceil_div(d, 2 * GEMM_BN);
    const double waves = (double)tiles / pairs;
    // (small problems of less than one wave stay whole: their tiles already run in parallel)
    if (!kWideN || waves < 1.0 || waves >= 16.0) return 1;
    auto cost = [&](int S) {
        return std::ceil((double)tiles * S / pairs) / S + (S > 1 ? waves * S * 1733.0 / V : 0.0);
    };
    int32_t best = 1;
    double bc = cost(1);
    for (int S = 2; S <= 4; ++S)
        if (cost(S) < 0.98 * bc) {
            bc = cost(S);
            best = S;
        }
    return best;
}

LossWs plan_loss(int64_t T, int64_t max_rows, int32_t d, int32_t V, size_t base,
                 int32_t vp_world) {
    WsPlan p;
    p.off = base;
    LossWs w;
    const int64_t rows_cap = loss_rows_cap(T, max_rows);
    const int64_t n_chunks = ceil_div(T, CHUNK_TOKENS);
    w.rows_cap = rows_cap;
    w.n_tiles = (int32_t)ceil_div(V, GEMM_BN);
    w.idx = p.take(sizeof(int32_t) * (size_t)(T + 1));
    w.meta = p.take(sizeof(int64_t) * 4);
    w.chunk_cnt = p.take(sizeof(int32_t) * (size_t)(n_chunks + 1));
    w.chunk_base = w.chunk_cnt;
    w.tgt_c = p.take(sizeof(int32_t) * (size_t)rows_cap);
    w.old_c = p.take(sizeof(float) * (size_t)rows_cap);
    w.adv_c = p.take(sizeof(float) * (size_t)std::max<int64_t>(T, 1));  // standalone compaction
    w.H = p.take((size_t)rows_cap * d * 2, 1024);
    w.P = p.take((size_t)rows_cap * V * 2, 1024);
    w.part = p.take(sizeof(float2) * (size_t)rows_cap * w.n_tiles);
    w.fscale = p.take(sizeof(float) * (size_t)rows_cap * w.n_tiles);
    w.xrow = p.take(sizeof(int2) * (size_t)rows_cap);
    w.zy = p.take(sizeof(float) * (size_t)rows_cap);
    w.row_term = p.take(sizeof(double) * (size_t)rows_cap);
    w.row_rho = p.take(sizeof(float) * (size_t)rows_cap);
    w.row_logp = p.take(sizeof(float) * (size_t)rows_cap);
    w.row_clip = p.take(sizeof(int32_t) * (size_t)rows_cap);
    w.row_kl = p.take(sizeof(float) * (size_t)rows_cap);
    w.w_c = p.take(sizeof(float) * (size_t)rows_cap);
    w.ref_c = p.take(sizeof(float) * (size_t)rows_cap);
    w.rows_eff = p.take(sizeof(int64_t) * 2);
    w.sched = p.take(sizeof(int) * 32);
    w.prog = p.take(sizeof(int64_t) * 3 * PROG_UNITS);
    w.ksplit = vp_world > 0 ? 1 : choose_ksplit(max_rows > 0 && max_rows < T ? max_rows : 0, d, V);
    w.splitk = w.ksplit > 1 ? p.take(sizeof(float) * (size_t)w.ksplit * rows_cap * d, 1024) : 0;
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
// L'_r = sum exp(z - M_r) - 1 (the first max left out, as across tiles) -> its slot of the
// all-gather buffer (the other slots are zero; a sum all-reduce then fills every slot).
__global__ void __launch_bounds__(RS_ROWS * RS_WARPS)
    k_vp_row_stats(const int64_t* __restrict__ rows_dev, int32_t n_tiles, int64_t ld,
                   const float2* __restrict__ part /* [n_tiles][ld] */,
                   float2* __restrict__ slot) {
    __shared__ float s_m[RS_WARPS][RS_ROWS];
    __shared__ int s_j[RS_WARPS][RS_ROWS];
    __shared__ float s_l[RS_WARPS][RS_ROWS];
    const int64_t rows = *rows_dev;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t p0 = (int64_t)blockIdx.x * RS_ROWS; p0 < rows; p0 += (int64_t)gridDim.x * RS_ROWS) {
        const int64_t p = p0 + lane;
        const bool ok = p < rows;
        float M;
        int jM;
        rs_max_sum(part, ld, n_tiles, p, ok, s_m, s_j, s_l, M, jM);
        if (w == 0 && ok) {
            float Lm1 = 0.f;  // warp partials in warp order, as in k_row_stats
#pragma unroll
            for (int q = 0; q < RS_WARPS; ++q) Lm1 += s_l[q][lane];
            slot[p] = make_float2(M, Lm1);
        }
        __syncthreads();
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

// split-K grad_hidden: grad_hidden[idx[p]] = bf16(sum over splits s, in order, of partial s)
__global__ void __launch_bounds__(256)
    k_splitk_scatter(const int64_t* __restrict__ rows_dev, int32_t d, int32_t S, int64_t stride,
                     const int32_t* __restrict__ idx, const float* __restrict__ parts,
                     __nv_bfloat16* __restrict__ gh) {
    const int64_t rows = *rows_dev;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < rows;
         p += nw) {
        const float4* src = reinterpret_cast<const float4*>(parts + p * d);
        uint2* dst = reinterpret_cast<uint2*>(gh + (int64_t)idx[p] * d);
        for (int c = lane; c < d / 4; c += 32) {
            float4 v = src[c];
            for (int s = 1; s < S; ++s) {
                const float4 u = src[s * (stride / 4) + c];
                v.x += u.x;
                v.y += u.y;
                v.z += u.z;
                v.w += u.w;
            }
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
                  float* __restrict__ ref_c) {
    const int64_t rows = *rows_dev;
    const double N = (double)*nglob_dev;
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

int launch_policy_loss(const agentrl_loss_args* a, const agentrl_loss_out* o, uint8_t* ws,
                       const LossWs& w, const int32_t* idx_dev, const int64_t* rows_dev,
                       const float* adv_c_dev, const int64_t* nglob_dev, agentrl_comm comm,
                       int32_t* d_status, cudaStream_t stream, const FusedExtras* fx) {
    const int64_t T = a->T;
    const int32_t d = a->d, V = a->V;
    const int64_t rows_cap = w.rows_cap;
    int64_t* meta = reinterpret_cast<int64_t*>(ws + w.meta);
    int32_t* idx = reinterpret_cast<int32_t*>(ws + w.idx);
    float* adv_c = reinterpret_cast<float*>(ws + w.adv_c);
    int32_t* tgt_c = reinterpret_cast<int32_t*>(ws + w.tgt_c);
    float* old_c = reinterpret_cast<float*>(ws + w.old_c);
    __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(ws + w.H);
    __nv_bfloat16* P = reinterpret_cast<__nv_bfloat16*>(ws + w.P);
    float2* part = reinterpret_cast<float2*>(ws + w.part);
    float* fscale = reinterpret_cast<float*>(ws + w.fscale);
    int2* xrow = reinterpret_cast<int2*>(ws + w.xrow);
    float* zy = reinterpret_cast<float*>(ws + w.zy);
    double* row_term = reinterpret_cast<double*>(ws + w.row_term);
    float* row_rho = reinterpret_cast<float*>(ws + w.row_rho);
    float* row_logp = reinterpret_cast<float*>(ws + w.row_logp);
    int32_t* row_clip = reinterpret_cast<int32_t*>(ws + w.row_clip);
    float* row_kl = reinterpret_cast<float*>(ws + w.row_kl);
    float* w_c = reinterpret_cast<float*>(ws + w.w_c);
    float* ref_c = reinterpret_cast<float*>(ws + w.ref_c);
    int64_t* rows_eff = reinterpret_cast<int64_t*>(ws + w.rows_eff);
    int* sched = reinterpret_cast<int*>(ws + w.sched);
    // vocab-parallel head (grad_W_mode 3): W_head is this rank's vocabulary shard, every rank
    // holds the same rows (the row statistics are all-gathered between the forward GEMM and the
    // row statistics kernel)
    const bool vp = a->grad_W_mode == 3 && comm && w.vp_world > 0;
    const int vp_R = vp ? comm_world(comm) : 0;
    const int64_t vp_v0 = vp ? (int64_t)comm_rank(comm) * V : 0;
    int* ctr_fwd = kDynamic ? sched + 0 : nullptr;
    int* ctr_gw = kDynamic ? sched + 4 : nullptr;
    int* ctr_gh = kDynamic ? sched + 8 : nullptr;
    AG_CUDA(cudaMemsetAsync(sched, 0, 32 * sizeof(int), stream));
    // progress arrays: [0] grad_W, [1] grad_hidden, [2] forward
    int64_t* prog = reinterpret_cast<int64_t*>(ws + w.prog);
    if (kThrottleLead > 0 || kThrottleLeadFwd > 0)
        AG_CUDA(cudaMemsetAsync(prog, 0xff, 3 * PROG_UNITS * sizeof(int64_t), stream));

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

    // ---- outputs that are defined everywhere (grad_hidden's zero rows; only the grad_hidden
    // GEMM writes it back)
    if (T > 0) AG_CUDA(cudaMemsetAsync(o->grad_hidden, 0, (size_t)T * d * 2, stream));
    if (o->logp) AG_CUDA(cudaMemsetAsync(o->logp, 0, (size_t)T * sizeof(float), stream));

    // ---- K4 gather (+ the row count clamped to the workspace's rows_cap -> rows_eff)
    {
        int grid = num_sms() * 4;
        ProfScope ps(KID_GATHER, stream);
        // the caller's bound exactly (rows_cap is it rounded up to GEMM_BM)
        const int64_t row_limit = (a->max_rows > 0 && a->max_rows < T) ? a->max_rows : T;
        k_gather<<<grid, 256, 0, stream>>>(rows_dev, row_limit, rows_eff, T, d, V,
                                           reinterpret_cast<const __nv_bfloat16*>(a->hidden),
                                           a->target, a->old_logp, idx_dev, H, tgt_c, old_c,
                                           d_status, vp_v0, vp ? (int64_t)V * vp_R : V);
        k_row_weights<<<num_sms() * 2, 256, 0, stream>>>(
            rows_eff, nglob_dev, idx_dev, a->tok_weight, a->ref_logp, a->loss_agg,
            fx ? fx->off : nullptr, fx ? fx->n_traj : 0, fx ? fx->n_g : nullptr,
            fx ? fx->group_id : nullptr, fx ? fx->grp_cnt : nullptr, fx ? fx->n_groups : 0,
            fx ? fx->ngrp : nullptr, w_c, ref_c);
        count_launch(2);
        AG_CUDA(cudaGetLastError());
    }
    rows_dev = rows_eff;

    // ---- tensor maps
    CUtensorMap mH_K, mH_MN, mW_K, mW_MN, mP_K, mP_MN;
    int rc;
    if ((rc = make_map(&mH_K, H, d, rows_cap, d, 64, 128))) return rc;
    if ((rc = make_map(&mH_MN, H, d, rows_cap, d, 64, 64))) return rc;
    // K-major B box = the B rows one CTA stages (128 in a CTA pair, 256 alone)
    if ((rc = make_map(&mW_K, a->W_head, d, V, d, 64, kPair ? 128 : 256))) return rc;
    if ((rc = make_map(&mW_MN, a->W_head, d, V, d, 64, 64))) return rc;
    if ((rc = make_map(&mP_K, P, V, rows_cap, V, 64, 128))) return rc;
    if ((rc = make_map(&mP_MN, P, V, rows_cap, V, 64, 64))) return rc;

    const int64_t max_m_tiles = rows_cap / GEMM_BM;
    // ---- K5 forward GEMM + softmax-statistics epilogue.  vocab-parallel: z_y is written only
    // by the rank whose shard holds y_t; the others keep 0 for the sum all-reduce
    if (vp) AG_CUDA(cudaMemsetAsync(zy, 0, sizeof(float) * (size_t)rows_cap, stream));
    {
        GemmArgs g{};
        g.m_dev = rows_dev;
        g.N = V;
        g.K_static = d;
        g.group_m = AGENTRL_GROUP_M;
        g.pol_a = AGENTRL_L2POL_FWD_A;  // H rows of the current row group: reused by every column
        g.pol_b = AGENTRL_L2POL_FWD_B;  // W: streamed, shared only by the concurrent row tiles
        g.tile_counter = ctr_fwd;
        if (kThrottleLeadFwd > 0) {
            g.prog = prog + 2 * PROG_UNITS;
            g.prog_every = AGENTRL_THROTTLE_EVERY;
            g.prog_lead = kThrottleLeadFwd;
            g.prog_waits = throttle_wait_ctr(0);
        }
        g.scale = a->logit_scale;
        g.tgt = tgt_c;
        g.P = P;
        g.ldP = V;
        g.part = part;
        g.ldpart = rows_cap;
        g.n_tiles = w.n_tiles;
        g.zy = zy;
        rc = launch_gemm<EPI_FWD, false, false, 1, kFwdKsub>(mH_K, mW_K, g, max_m_tiles * w.n_tiles,
                                                             stream);
        if (rc) return rc;
    }
    float2* vpstat = vp ? reinterpret_cast<float2*>(ws + w.vpstat) : nullptr;
    if (vp) {  // all-gather of (M_r, L'_r) per row and the owner's z_y (sum all-reduces)
        AG_CUDA(cudaMemsetAsync(vpstat, 0, sizeof(float2) * (size_t)vp_R * rows_cap, stream));
        k_vp_row_stats<<<(unsigned)std::max<int64_t>(ceil_div(rows_cap, RS_ROWS), 1),
                         RS_ROWS * RS_WARPS, 0, stream>>>(
            rows_dev, w.n_tiles, rows_cap, part, vpstat + (size_t)comm_rank(comm) * rows_cap);
        count_launch();
        AG_CUDA(cudaGetLastError());
        if ((rc = comm_allreduce_f32(comm, reinterpret_cast<float*>(vpstat),
                                     (size_t)2 * vp_R * rows_cap, stream)))
            return rc;
        if ((rc = comm_allreduce_f32(comm, zy, (size_t)rows_cap, stream))) return rc;
    }
    // ---- K6 row statistics: loss terms, gradient scales and target columns
    {
        ProfScope ps(KID_ROWSTATS, stream);
        k_row_stats<<<(unsigned)std::max<int64_t>(ceil_div(rows_cap, RS_ROWS), 1),
                      RS_ROWS * RS_WARPS, 0, stream>>>(
            rows_dev, nglob_dev, w.n_tiles, rows_cap, part, zy, tgt_c, old_c, adv_c_dev, idx_dev,
            a->clip_eps_low, a->clip_eps_high, w_c, a->kl_beta > 0.f ? ref_c : nullptr,
            a->kl_beta, fscale, xrow, row_term, row_rho, row_logp, row_clip, row_kl, o->logp,
            vpstat, vp_R, rows_cap);
        count_launch();
        AG_CUDA(cudaGetLastError());
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
    auto xf_args = [&](GemmArgs& g) {
        g.P = P;  // the transform warps' A source (register path)
        g.ldP = V;
        g.xf_scale = fscale;
        g.xf_row = xrow;
        g.xf_rows = rows_dev;
        g.xf_ld = rows_cap;
    };
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
        g.group_m = AGENTRL_GROUP_M_BWD;
        g.pol_a = AGENTRL_L2POL_BWD;  // P~ column blocks, shared by the d/512 pairs of a row block
        g.pol_b = AGENTRL_L2POL_BWD;  // H: re-read by every wave
        g.tile_counter = ctr_gw;
        if (kThrottleLead > 0) {
            g.prog = prog;
            g.prog_every = AGENTRL_THROTTLE_EVERY;
            g.prog_lead = kThrottleLead;
            g.prog_waits = throttle_wait_ctr(1);
        }
        g.scale = a->logit_scale;
        g.gw = o->grad_W;
        g.ldo = d;
        xf_args(g);
        const int64_t tiles = ceil_div(V, GEMM_BM) * ceil_div(d, GEMM_BN);
        return launch_gemm<EPI_GRADW, true, true, kWideN ? 2 : 1, 1, true>(mP_MN, mH_MN, g, tiles, s);
    };
    // ---- K8 grad_hidden = s G W   (M = T_eff, N = d, K = V), scattered to idx rows
    auto launch_grad_hidden = [&](cudaStream_t s, int rsv) -> int {
        GemmArgs g{};
        g.m_dev = rows_dev;
        g.N = d;
        g.K_static = V;
        g.group_m = AGENTRL_GROUP_M_BWD;
        g.pol_a = AGENTRL_L2POL_BWD;  // P~ rows: shared by the pairs of one row block
        g.pol_b = AGENTRL_L2POL_BWD;  // W: re-read by every wave
        g.tile_counter = ctr_gh;
        if (kThrottleLead > 0) {
            g.prog = prog + PROG_UNITS;
            g.prog_every = AGENTRL_THROTTLE_EVERY;
            g.prog_lead = kThrottleLead;
            g.prog_waits = throttle_wait_ctr(2);
        }
        g.scale = a->logit_scale;
        g.idx = idx_dev;
        g.gh = reinterpret_cast<__nv_bfloat16*>(o->grad_hidden);
        g.ldo = d;
        xf_args(g);
        const int64_t tiles = max_m_tiles * ceil_div(d, GEMM_BN);
        int r;
        if (vp) {
            // this rank's vocabulary columns give a partial grad_h: fp32 rows (the EPI_GRADW
            // epilogue, row = compacted row), summed over the group, then scattered as bf16
            float* gh32 = reinterpret_cast<float*>(ws + w.vp_gh);
            g.gw = gh32;
            r = launch_gemm<EPI_GRADW, false, true, kWideN ? 2 : 1, 1, true>(mP_K, mW_MN, g, tiles, s, 0);
            if (r) return r;
            if ((r = comm_allreduce_f32(comm, gh32, (size_t)rows_cap * d, s))) return r;
            k_vp_scatter<<<num_sms() * 4, 256, 0, s>>>(rows_dev, d, idx_dev, gh32,
                                                       reinterpret_cast<__nv_bfloat16*>(o->grad_hidden));
            count_launch();
            AG_CUDA(cudaGetLastError());
            return AGENTRL_OK;
        }
        if (w.ksplit > 1 && kWideN) {
            // split-K: fp32 partials of the ksplit k-ranges (EPI_GRADW rows = compacted rows),
            // then one pass sums them in split order and scatters bf16 rows to idx
            float* parts = reinterpret_cast<float*>(ws + w.splitk);
            g.gw = parts;
            g.gw_split = rows_cap * (int64_t)d;
            g.ksplit = w.ksplit;
            g.prog = nullptr;  // (the throttle assumes every unit walks the same k-blocks)
            r = launch_gemm<EPI_GRADW, false, true, 2, 1, true>(mP_K, mW_MN, g, tiles * w.ksplit, s,
                                                                rsv);
            if (r) return r;
            k_splitk_scatter<<<num_sms() * 4, 256, 0, s>>>(
                rows_dev, d, w.ksplit, rows_cap * (int64_t)d, idx_dev, parts,
                reinterpret_cast<__nv_bfloat16*>(o->grad_hidden));
            count_launch();
            AG_CUDA(cudaGetLastError());
            return AGENTRL_OK;
        }
        return launch_gemm<EPI_GRADH, false, true, kWideN ? 2 : 1, 1, true>(mP_K, mW_MN, g, tiles, s, rsv);
    };
    if ((rc = launch_grad_W(stream))) return rc;
    // ---- C3 grad_W all-reduce / reduce-scatter on a side stream, overlapped with K8
    SideStream* ss = nullptr;
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
    const int rsv = nccl_c3 ? std::min(AGENTRL_COMM_SMS, num_sms() / 2) : 0;
    if ((rc = launch_grad_hidden(stream, rsv))) return rc;
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
            const float logp = (zy[p] - M) - l1;  // see k_row_stats
            const int64_t t = idx[p];
            logp_out[t] = logp;
            if (ent_out) ent_out[t] = l1 + Hs;
            if (!isfinite(logp)) atomicOr(d_status, AGENTRL_ST_NONFINITE);
        }
    }
}

LogpWs plan_logp(int64_t T, int64_t max_rows, int32_t d, int32_t V, size_t base) {
    WsPlan p;
    p.off = base;
    LogpWs w;
    const int64_t rows_cap = loss_rows_cap(T, max_rows);
    const int64_t n_chunks = ceil_div(T, CHUNK_TOKENS);
    w.rows_cap = rows_cap;
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
    const int64_t rows_cap = w.rows_cap;
    int64_t* meta = reinterpret_cast<int64_t*>(ws + w.meta);
    int32_t* idx = reinterpret_cast<int32_t*>(ws + w.idx);
    int32_t* chunk = reinterpret_cast<int32_t*>(ws + w.chunk);
    int32_t* tgt_c = reinterpret_cast<int32_t*>(ws + w.tgt_c);
    __nv_bfloat16* H = reinterpret_cast<__nv_bfloat16*>(ws + w.H);
    float4* part4 = reinterpret_cast<float4*>(ws + w.part4);
    float* zy = reinterpret_cast<float*>(ws + w.zy);
    int* sched = reinterpret_cast<int*>(ws + w.sched);
    int64_t* rows_eff = meta + 2;  // min(T_eff, rows_cap), written by k_gather
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
        const int64_t row_limit = (a->max_rows > 0 && a->max_rows < T) ? a->max_rows : T;
        k_gather<<<num_sms() * 4, 256, 0, stream>>>(
            meta, row_limit, rows_eff, T, d, V, reinterpret_cast<const __nv_bfloat16*>(a->hidden),
            a->target, nullptr, idx, H, tgt_c, nullptr, d_status);
        count_launch();
        AG_CUDA(cudaGetLastError());
    }
    CUtensorMap mH_K, mW_K;
    int rc;
    if ((rc = make_map(&mH_K, H, d, rows_cap, d, 64, 128))) return rc;
    if ((rc = make_map(&mW_K, a->W_head, d, V, d, 64, kPair ? 128 : 256))) return rc;
    {
        GemmArgs g{};
        g.m_dev = rows_eff;
        g.N = V;
        g.K_static = d;
        g.group_m = AGENTRL_GROUP_M;
        g.pol_a = AGENTRL_L2POL_FWD_A;
        g.pol_b = AGENTRL_L2POL_FWD_B;
        g.tile_counter = kDynamic ? sched : nullptr;
        g.scale = a->logit_scale;
        g.tgt = tgt_c;
        g.part4 = part4;
        g.n_tiles = w.n_tiles;
        g.zy = zy;
        const int64_t mt = (rows_cap / GEMM_BM) * w.n_tiles;
        rc = launch_gemm<EPI_LOGP, false, false, 1, kFwdKsub>(mH_K, mW_K, g, mt, stream);
        if (rc) return rc;
    }
    {
        ProfScope ps(KID_LOGP_MERGE, stream);
        k_logp_merge<<<num_sms() * 8, 256, 0, stream>>>(rows_eff, w.n_tiles, part4, zy, idx, logp,
                                                        entropy, d_status);
        count_launch();
        AG_CUDA(cudaGetLastError());
    }
    return AGENTRL_OK;
}

}  // namespace agentrl
