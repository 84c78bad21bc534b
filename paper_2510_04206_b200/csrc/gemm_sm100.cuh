// gemm_sm100.cuh -- persistent, warp-specialised tcgen05 GEMM for sm_100a with the three
// fused epilogues of the LM-head loss path.
//
//   D (fp32, TMEM) = sum_k A * B^T, bf16 operands staged by TMA (SWIZZLE_128B) through a
//   STAGES-deep shared-memory ring; one elected thread issues tcgen05.mma (K=16).
//
//   PAIR = true  (default): a CTA pair (cluster of 2, cta_group::2) computes a 256-row tile.
//                Each CTA stages 128 rows of A and half of B's rows per k-block; the leader
//                CTA issues tcgen05.mma.cta_group::2 (M=256, N=256) and commits to both CTAs'
//                barriers; TMA bytes of both CTAs complete on the leader's full barrier.
//   PAIR = false: one CTA computes a 128-row tile with cta_group::1 (kept for A/B tests).
//
//   NSPLIT = 1: 256-column tiles, two TMEM accumulators (2 x 256 fp32 columns) so the
//               epilogue of tile i overlaps the MMAs of tile i+1 (short-K GEMMs: forward).
//   NSPLIT = 2: 512-column tiles (two N=256 MMAs per K step into one 512-column
//               accumulator).  A third more MMA work per staged byte, half the re-reads of
//               the shared operand; for the long-K backward GEMMs (K = V or T_eff) the
//               un-overlapped epilogue is ~1% of a tile.
//
//   warp 0      : TMA producer (one lane)
//   warp 1      : TMEM allocator + MMA issuer (one lane, leader CTA)
//   warps 2..5  : epilogue; warp w reads TMEM lanes 32*(w%4) .. +31 (row = lane)
//
// Operand majors: A/B either K-major (K contiguous; one TMA box {64, rows}) or MN-major (MN
// contiguous; boxes {64 (MN), 64 (K)} stacked along MN, LBO = 8 KB between 64-wide atoms).
//
// Epilogues (row r = output row; each CTA owns 128 rows of the tile):
//   EPI_FWD   logits z = s*acc: per (row, 256-col tile) max m and l' = sum exp(z-m) - 1 over
//             valid columns (the first max element is left out of the sum: no cancellation
//             later), P~ = exp(z - m) stored as bf16, z_y gathered when the row's target falls
//             in the tile.  The T x V logits never reach HBM in fp32 (P~ is 2 B/entry).
//   EPI_GRADH grad_hidden[idx[r], :] = bf16(s * acc)   (scatter to the original token row)
//   EPI_GRADW grad_W[r, :] = s * acc (fp32); zeros if the (dynamic) K extent is 0.
//
// XF = true (the two backward GEMMs): operand A is the forward's bf16 P~ = exp(z - m_tile), and
// 4 transform warps (warps 6..9) rewrite each staged A tile in shared memory as the softmax
// gradient G = bf16(f * P~) with f = c_t exp((m_tile - M_t) - log1p(L'_t)) per (row, 256-column
// vocabulary tile) and the target column replaced by c_t expm1(log p_t),
// before the MMA may read it.  Every 128-byte line of a SWIZZLE_128B tile belongs to one token
// and one vocabulary tile, so one scale covers a line.  Each CTA's TMA then completes on its own
// full barrier; the transform warps of both CTAs arrive on the leader's `ready` barrier, which
// the MMA issuer waits on instead.  No G tensor exists in HBM.
#pragma once
#include "ptx.cuh"

namespace agentrl {

constexpr int GEMM_BM = 128;  // rows per CTA
constexpr int GEMM_BN = 256;  // columns per MMA (and per FWD statistics tile)
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 192;     // producer, MMA, 4 epilogue warps
constexpr int GEMM_THREADS_XF = 352;  // + 4 transform warps and 1 input-loader warp (XF)
constexpr int XF_WARP0 = 6;
constexpr int XF_LOADER_WARP = XF_WARP0 + 4;
// XF: per-stage side buffer of the transform's inputs, filled by the loader warp: grad_hidden:
// the 128 rows' scales f (512 B); grad_W: the 64 tokens' scales (256 B) and (target column,
// G value) pairs (512 B)
constexpr int XIN_STAGE = 1024;
// backward (XF) GEMMs: the producer also prefetches the operand boxes of k-block kb + this many
// into L2 when it loads kb (0 = off, the default).  Measured at glm9b (profiles/r02_ab_pf.txt):
// 8 or 16 k-blocks ahead made grad_W 29% and grad_hidden 14% slower -- the extra L2 requests of
// 74 pairs prefetching overlapping boxes cost more than the latency they hide
#ifndef AGENTRL_PREFETCH_KB
#define AGENTRL_PREFETCH_KB 0
#endif

// KSUB: 64-wide K atoms per pipeline stage (K-major operands only).  KSUB = 2 stages 128 K
// per k-block: 8 MMAs per barrier round trip instead of 4, for the short-K forward GEMM whose
// 4-MMA k-blocks left the tensor pipe ~12% idle (profiles/r01_fwd_ksub.txt).
template <bool PAIR, int NSPLIT, int KSUB = 1>
struct GemmCfg {
    static_assert(NSPLIT == 1 || (NSPLIT == 2 && PAIR), "512-column tiles need a CTA pair");
    static_assert(KSUB == 1 || KSUB == 2, "one or two K atoms per stage");
    static constexpr int BK = GEMM_BK * KSUB;                    // K per stage
    static constexpr int A_ATOM = GEMM_BM * GEMM_BK * 2;         // 16 KB: 128 rows x 64 K
    static constexpr int A_STAGE = A_ATOM * KSUB;
    static constexpr int B_ROWS = PAIR ? GEMM_BN / 2 : GEMM_BN;  // B rows per CTA per MMA
    static constexpr int B_ATOM = B_ROWS * GEMM_BK * 2;
    static constexpr int B_HALF = B_ATOM * KSUB;                 // bytes per MMA's B slice
    static constexpr int B_STAGE = NSPLIT * B_HALF;
    static constexpr int STAGES = (PAIR ? (NSPLIT == 1 ? 6 : 4) : 4) / KSUB;
    static constexpr int TILE_M = PAIR ? 2 * GEMM_BM : GEMM_BM;  // rows per tile
    static constexpr int TILE_N = GEMM_BN * NSPLIT;              // columns per tile
    static constexpr int ACC_BUFS = NSPLIT == 1 ? 2 : 1;
    // backward tiles: a 32 x 33 fp32 transpose slab per epilogue warp, so the peer-memory
    // epilogue (grad_W fused with its reduce-scatter) writes 128 contiguous bytes per row and
    // warp instruction instead of 16 B from each of 32 rows
#ifndef AGENTRL_EPI_SLAB
#define AGENTRL_EPI_SLAB 1
#endif
    static constexpr int EPI_STAGE = (NSPLIT == 2 && AGENTRL_EPI_SLAB) ? 4 * 32 * 33 * 4 : 0;
    // (EPI_STAGE is added by the launcher for the grad_W GEMM only)
    // forward: a 32-row x 64-byte bf16 staging slot per epilogue warp, so each P~ store
    // instruction writes 8 rows x 64 contiguous bytes (full 32-byte sectors) instead of 16 B
    // from each of 32 rows (added by the launcher for the forward GEMM only)
#ifndef AGENTRL_GRADW_STAGE
#define AGENTRL_GRADW_STAGE 1  // the local grad_W epilogue staged for full-line stores
#endif
#ifndef AGENTRL_FWD_PSTAGE
#define AGENTRL_FWD_PSTAGE 1
#endif
    static constexpr int PSTAGE = AGENTRL_FWD_PSTAGE ? 4 * 32 * 64 : 0;
    static constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) + 1024 + 1024;
    static constexpr int TX_BYTES = (A_STAGE + B_STAGE) * (PAIR ? 2 : 1);
};

// EPI_LOGP: forward-only log-prob/entropy statistics (no P~ store): per (row, tile)
// (m, l', u = sum exp(z - m) z)
enum { EPI_FWD = 0, EPI_GRADH = 1, EPI_GRADW = 2, EPI_LOGP = 3 };

struct GemmArgs {
    // problem: rows M (dynamic if m_dev), cols N, reduction K (dynamic if k_dev)
    int64_t M_static;
    const int64_t* m_dev;
    const int64_t* m_range;  // optional [r0, r1): only rows r0 .. r1-1 (r0 a multiple of 256)
    int32_t N;
    int64_t K_static;
    const int64_t* k_dev;
    int32_t group_m;       // raster: tiles grouped by group_m row-blocks, columns fastest inside
    int32_t pol_a, pol_b;  // L2 policy per operand: 0 normal, 1 evict_first, 2 evict_last
    float scale;           // logit_scale s
    // EPI_FWD
    const int32_t* tgt;  // [rows] target token of each compacted row
    __nv_bfloat16* P;    // [rows, ldP] exp(z - m), bf16: fp32's exponent range, so entries far
                         // below the tile max survive (p_y -> 1 rows)
    int64_t ldP;
    float2* part;   // [n_tiles][ldpart] (m, l'), tile-major  (EPI_FWD)
    int64_t ldpart;
    float4* part4;  // [rows, n_tiles] (m, l', u, 0)       (EPI_LOGP)
    int32_t n_tiles;
    float* zy;  // [rows]
    // EPI_GRADH
    const int32_t* idx;  // [rows] original token index
    __nv_bfloat16* gh;   // [T, ldo]
    // EPI_GRADW
    float* gw;  // [V, ldo]
    int64_t ldo;
    // EPI_GRADW fused with the reduce-scatter (peer.cu): row r goes to owner o = r / peer_rows,
    // into slot peer_rank of o's window: peer_out[o] + (peer_rank * peer_rows + r mod) * ldo
    float* const* peer_out;
    int64_t peer_rows;
    int32_t peer_rank;
    // split-K (grad_hidden at small shard sizes): ksplit > 1 splits every tile's k-blocks into
    // ksplit contiguous ranges (work unit = tile * ksplit + split); the EPI_GRADW epilogue then
    // writes split s's fp32 partial at gw + s * gw_split
    int32_t ksplit;
    int64_t gw_split;
    // dynamic tile scheduler: zeroed int counter (tiles claimed in global order), or null for
    // the static persistent schedule (tile = unit + i * units)
    int* tile_counter;
    // optional progress throttle (dynamic scheduler only): int64 [units], preset to -1.  Each
    // pair leader publishes its position wave * num_kb + kb every prog_every k-blocks and waits
    // while it is more than prog_lead k-blocks ahead of the slowest active pair, so pairs that
    // share operand slices stay within an L2-resident window instead of drifting apart.
    int64_t* prog;
    int32_t prog_every, prog_lead;
    unsigned long long* prog_waits;  // optional: +1 per throttle wait episode (debug counter)
    // XF: operand A is P~ (bf16 [rows, V]); G = bf16(xf_scale[tile * xf_ld + row] * P~)
    // (tile-major: consecutive rows are contiguous), target column (xf_row[row].x, -1 = none)
    // = __int_as_float(xf_row[row].y); rows at or past *xf_rows (the dynamic T_eff) are zero
    const float* xf_scale;
    const int2* xf_row;
    const int64_t* xf_rows;
    int64_t xf_ld;
};

__device__ __forceinline__ void prog_store(int64_t* p, int64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void prog_load2(const int64_t* p, int64_t& a, int64_t& b) {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
// min position over the units that have started and not finished (-1: not started,
// INT64_MAX: finished); 8 loads in flight per round (n_units padded to even by the -1 preset)
__device__ __forceinline__ int64_t prog_min(const int64_t* prog, int64_t n_units) {
    int64_t mn = INT64_MAX;
    for (int64_t u = 0; u < n_units; u += 8) {
        int64_t v[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) prog_load2(prog + u + 2 * i, v[2 * i], v[2 * i + 1]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (u + i < n_units && v[i] >= 0 && v[i] < mn) mn = v[i];
    }
    return mn;
}
// wait until this unit is at most `lead` k-blocks ahead of the slowest active unit.  Positions
// only grow, so a stale minimum is a lower bound: re-read only when it says we may be ahead.
// The slowest unit never waits.
__device__ __forceinline__ void prog_throttle(const int64_t* prog, int64_t n_units, int64_t mine,
                                              int32_t lead, int64_t& cached_min,
                                              unsigned long long* waits) {
    if (mine - cached_min <= (int64_t)lead) return;
    bool counted = false;
    for (;;) {
        cached_min = prog_min(prog, n_units);
        if (mine - cached_min <= (int64_t)lead) return;
        if (waits && !counted) {
            atomicAdd(waits, 1ull);
            counted = true;
        }
        __nanosleep(100);
    }
}

constexpr int QD = 4;  // tile-queue depth (dynamic scheduler)

__device__ __forceinline__ void tile_coords(int64_t tile, int64_t num_m, int64_t num_n,
                                            int32_t group_m, int64_t& m_blk, int64_t& n_blk) {
    const int64_t per_group = (int64_t)group_m * num_n;
    const int64_t g = tile / per_group;
    const int64_t first_m = g * group_m;
    const int64_t gm = min((int64_t)group_m, num_m - first_m);
    const int64_t local = tile - first_m * num_n;
    m_blk = first_m + local % gm;
    n_blk = local / gm;
}

__device__ __forceinline__ uint64_t make_policy(int which) {
    return which == 1 ? policy_evict_first()
                      : (which == 2 ? policy_evict_last() : policy_evict_normal());
}

template <int ACC_BUFS>
__device__ __forceinline__ void advance_acc(int& acc, uint32_t& acc_phase) {
    if constexpr (ACC_BUFS == 2) {
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
    } else {
        acc_phase ^= 1;
    }
}

// TMA loads of one k-block: A (128 rows of this CTA) and B (per MMA half: B_ROWS rows)
// LOCAL_BAR (XF): every CTA's bytes complete on its own full barrier (its transform warps
// wait on it), else a pair's bytes complete on the leader's
template <bool A_MN, bool B_MN, bool PAIR, int NSPLIT, int KSUB, bool LOCAL_BAR>
__device__ __forceinline__ void load_stage(const CUtensorMap& tmA, const CUtensorMap& tmB,
                                           uint64_t* full_bar, uint32_t full_bar_leader,
                                           uint8_t* a_dst, uint8_t* b_dst, int32_t m0,
                                           int32_t n0, int32_t k0, uint64_t pol_a,
                                           uint64_t pol_b) {
    using Cfg = GemmCfg<PAIR, NSPLIT, KSUB>;
    static_assert(KSUB == 1 || (!A_MN && !B_MN), "K atoms are stacked for K-major operands");
    auto ld = [&](const CUtensorMap& m, uint8_t* dst, int32_t x, int32_t y, uint64_t pol) {
        if constexpr (PAIR && !LOCAL_BAR) tma_load_2d_pair(&m, full_bar_leader, dst, x, y, pol);
        else tma_load_2d(&m, full_bar, dst, x, y, pol);
    };
    if constexpr (!A_MN) {
#pragma unroll
        for (int a = 0; a < KSUB; ++a) ld(tmA, a_dst + a * Cfg::A_ATOM, k0 + a * GEMM_BK, m0, pol_a);
    } else {
#pragma unroll
        for (int i = 0; i < GEMM_BM / 64; ++i) ld(tmA, a_dst + i * 8192, m0 + i * 64, k0, pol_a);
    }
#pragma unroll
    for (int h = 0; h < NSPLIT; ++h) {
        const int32_t nh = n0 + h * GEMM_BN;
        uint8_t* bd = b_dst + h * Cfg::B_HALF;
        if constexpr (!B_MN) {
#pragma unroll
            for (int a = 0; a < KSUB; ++a) ld(tmB, bd + a * Cfg::B_ATOM, k0 + a * GEMM_BK, nh, pol_b);
        } else {
#pragma unroll
            for (int i = 0; i < Cfg::B_ROWS / 64; ++i) ld(tmB, bd + i * 8192, nh + i * 64, k0, pol_b);
        }
    }
}

// L2 prefetch of the boxes load_stage would load for k-block k0 (same coordinates)
template <bool A_MN, bool B_MN, bool PAIR, int NSPLIT, int KSUB>
__device__ __forceinline__ void prefetch_stage(const CUtensorMap& tmA, const CUtensorMap& tmB,
                                               int32_t m0, int32_t n0, int32_t k0) {
    using Cfg = GemmCfg<PAIR, NSPLIT, KSUB>;
    if constexpr (!A_MN) {
#pragma unroll
        for (int a = 0; a < KSUB; ++a) tma_prefetch_l2_2d(&tmA, k0 + a * GEMM_BK, m0);
    } else {
#pragma unroll
        for (int i = 0; i < GEMM_BM / 64; ++i) tma_prefetch_l2_2d(&tmA, m0 + i * 64, k0);
    }
#pragma unroll
    for (int h = 0; h < NSPLIT; ++h) {
        const int32_t nh = n0 + h * GEMM_BN;
        if constexpr (!B_MN) {
#pragma unroll
            for (int a = 0; a < KSUB; ++a) tma_prefetch_l2_2d(&tmB, k0 + a * GEMM_BK, nh);
        } else {
#pragma unroll
            for (int i = 0; i < Cfg::B_ROWS / 64; ++i) tma_prefetch_l2_2d(&tmB, nh + i * 64, k0);
        }
    }
}

// XF: one 128-byte line of a SWIZZLE_128B tile (64 bf16 of one token and one vocabulary tile;
// logical 16-byte chunk c sits at physical chunk c ^ (line & 7)), at shared address `line`,
// rewritten in place as G = bf16(f * P~) (each product rounded once in fp32, then to bf16);
// element ycol (0..63, else none) = gy; zero: the whole line is 0
__device__ __forceinline__ void xf_line(uint32_t line, int l, float f, int ycol, float gy,
                                        bool zero) {
    const int sw = l & 7;
    if (zero) {
#pragma unroll
        for (int c = 0; c < 8; ++c) sts128(line + ((c ^ sw) << 4), make_uint4(0u, 0u, 0u, 0u));
        return;
    }
    uint4 v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = lds128(line + ((c ^ sw) << 4));
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            // bf16 pair -> fp32 pair {lo, hi}: the bf16 bits are the fp32's high half
            const uint64_t x = ((uint64_t)(w[k] & 0xffff0000u) << 32) | (uint64_t)(w[k] << 16);
            const uint64_t g = fmul2(x, f);
            o[k] = pack_bf162(__uint_as_float((uint32_t)g), __uint_as_float((uint32_t)(g >> 32)));
        }
        sts128(line + ((c ^ sw) << 4), make_uint4(o[0], o[1], o[2], o[3]));
    }
    if (ycol >= 0) {  // the target column: c (p_y - 1), stored over this thread's own product
        const __nv_bfloat16 b = __float2bfloat16_rn(gy);
        sts16(line + ((((ycol >> 3) ^ sw) << 4) | ((ycol & 7) << 1)),
              *reinterpret_cast<const uint16_t*>(&b));
    }
}

template <int EPI, bool A_MN, bool B_MN, bool PAIR, int NSPLIT, int KSUB, bool XF = false>
__device__ __forceinline__ void gemm_body(const CUtensorMap& tmA, const CUtensorMap& tmB,
                                          const GemmArgs& p) {
    using Cfg = GemmCfg<PAIR, NSPLIT, KSUB>;
    static_assert(!XF || KSUB == 1, "the transform handles one 64-wide K atom per stage");
    static_assert((EPI != EPI_FWD && EPI != EPI_LOGP) || NSPLIT == 1,
                  "forward statistics are per 256-column tile");
    constexpr int STAGES = Cfg::STAGES;
    constexpr int ACC_BUFS = Cfg::ACC_BUFS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * Cfg::A_STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * Cfg::B_STAGE);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* tfull = bars + 2 * STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* tq_full = tempty + 2;   // tile queue (dynamic scheduler): QD slots
    uint64_t* tq_empty = tq_full + QD;
    uint64_t* ready = tq_empty + QD;  // XF: stage transformed (leader's is the one used)
    uint64_t* xin_full = ready + STAGES;  // XF: the stage's transform inputs are in smem
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xin_full + STAGES);
    // XF: the transform inputs of each stage after the 1 KB barrier region (then the grad_W slab)
    uint8_t* xin = reinterpret_cast<uint8_t*>(bars) + 1024;
    const uint32_t xin_base = smem_u32(xin);
    (void)xin_base;
    volatile int32_t* tile_q = reinterpret_cast<volatile int32_t*>(tmem_slot + 4);
    const bool dyn = p.tile_counter != nullptr;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int64_t unit = PAIR ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
    const int64_t n_units = PAIR ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;

    const int64_t r0 = p.m_range ? p.m_range[0] : 0;
    const int64_t M = p.m_range ? p.m_range[1] : (p.m_dev ? *p.m_dev : p.M_static);
    const int64_t K = p.k_dev ? *p.k_dev : p.K_static;
    const int64_t num_m = M > r0 ? (M - r0 + Cfg::TILE_M - 1) / Cfg::TILE_M : 0;
    const int64_t num_n = (p.N + Cfg::TILE_N - 1) / Cfg::TILE_N;
    const int64_t num_tiles = num_m * num_n;
    const int64_t num_kb = (K + Cfg::BK - 1) / Cfg::BK;
    // work units: tile * S + split (S = 1: the tiles themselves)
    const int64_t S = p.ksplit > 1 ? p.ksplit : 1;
    const int64_t num_work = num_tiles * S;
    auto split_unit = [&](int64_t w, int64_t& tt, int64_t& kb_b, int64_t& kb_e, int64_t& sp) {
        tt = w / S;
        sp = w - tt * S;
        kb_b = sp * num_kb / S;
        kb_e = (sp + 1) * num_kb / S;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], PAIR ? 8 : 4);  // one arrive per epilogue warp (x2 CTAs)
        }
        for (int q = 0; q < QD; ++q) {
            mbar_init(&tq_full[q], 1);
            // consumers of a queue slot: leader MMA + 4 epilogue warps (+ 4 transform warps and
            // the input loader) (+ the peer's producer and the same warps); only the leader's
            // tq_empty is used
            constexpr int per_cta = XF ? 9 : 4;
            mbar_init(&tq_empty[q], PAIR ? 2 + 2 * per_cta : 1 + per_cta);
        }
        if constexpr (XF)
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(&ready[s], PAIR ? 8 : 4);
                mbar_init(&xin_full[s], 32);  // every lane of the loader warp
            }
        fence_mbar_init();
        fence_proxy_async_smem();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1) {
        if (PAIR) tmem_alloc_pair(tmem_slot, 512);
        else tmem_alloc(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // peer barriers initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            const uint64_t pol_a = make_policy(p.pol_a);
            const uint64_t pol_b = make_policy(p.pol_b);
            int stage = 0;
            uint32_t phase = 0;
            const bool throttle = dyn && leader && p.prog != nullptr && p.prog_every > 0;
            int64_t prog_cached_min = INT64_MIN / 2;
            for (int64_t it = 0;; ++it) {
                int64_t tile;
                if (!dyn) {
                    tile = unit + it * n_units;
                } else {
                    const int slot = (int)(it & (QD - 1));
                    const uint32_t ph = (uint32_t)(it / QD) & 1u;
                    if (leader) {  // claim the next tile in global order, publish to the pair
                        mbar_wait(&tq_empty[slot], ph ^ 1);
                        tile = atomicAdd(p.tile_counter, 1);
                        tile_q[slot] = (int32_t)tile;
                        mbar_arrive(&tq_full[slot]);
                        if constexpr (PAIR) {
                            const uint32_t pf = mapa_shared(smem_u32(&tq_full[slot]), 1);
                            mbar_arrive_expect_tx_remote(pf, 4);
                            st_async_remote_u32(mapa_shared(smem_u32((const void*)&tile_q[slot]), 1),
                                                (uint32_t)tile, pf);
                        }
                    } else {
                        mbar_wait(&tq_full[slot], ph);
                        tile = tile_q[slot];
                        mbar_arrive_cluster(mapa_shared(smem_u32(&tq_empty[slot]), 0));
                    }
                }
                if (tile >= num_work) {
                    if (throttle) prog_store(p.prog + unit, INT64_MAX);
                    break;
                }
                int64_t tt, kb_b, kb_e, sp;
                split_unit(tile, tt, kb_b, kb_e, sp);
                int64_t m_blk, n_blk;
                tile_coords(tt, num_m, num_n, p.group_m, m_blk, n_blk);
                const int32_t m0 = (int32_t)(r0 + m_blk * Cfg::TILE_M + rank * GEMM_BM);
                const int32_t n0 = (int32_t)(n_blk * Cfg::TILE_N + rank * Cfg::B_ROWS);
                const int64_t wave_pos = (tile / n_units) * num_kb;
                for (int64_t kb = kb_b; kb < kb_e; ++kb) {
                    if (throttle && kb % p.prog_every == 0) {
                        prog_store(p.prog + unit, wave_pos + kb);
                        prog_throttle(p.prog, n_units, wave_pos + kb, p.prog_lead, prog_cached_min,
                                      p.prog_waits);
                    }
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint32_t fb = 0;
                    if constexpr (PAIR && !XF) {
                        fb = mapa_shared(smem_u32(&full[stage]), 0);
                        // leader: arm its own full barrier for both CTAs' bytes (CTA scope; the
                        // peer's TMA completes its bytes on it directly)
                        if (leader) mbar_arrive_expect_tx(&full[stage], Cfg::TX_BYTES);
                    } else {
                        // XF: each CTA's own bytes (tile + the transform's inputs) on its own
                        // barrier (its transform warps wait on it)
                        mbar_arrive_expect_tx(&full[stage], XF && PAIR ? Cfg::TX_BYTES / 2
                                                                       : Cfg::TX_BYTES);
                    }
                    load_stage<A_MN, B_MN, PAIR, NSPLIT, KSUB, XF>(
                        tmA, tmB, &full[stage], fb, sA + stage * Cfg::A_STAGE,
                        sB + stage * Cfg::B_STAGE, m0, n0, (int32_t)(kb * Cfg::BK), pol_a, pol_b);
                    if constexpr (XF && AGENTRL_PREFETCH_KB > 0) {
                        if (kb + AGENTRL_PREFETCH_KB < kb_e)
                            prefetch_stage<A_MN, B_MN, PAIR, NSPLIT, KSUB>(
                                tmA, tmB, m0, n0, (int32_t)((kb + AGENTRL_PREFETCH_KB) * Cfg::BK));
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0 && leader) {
            constexpr uint32_t idesc = umma_idesc_bf16(Cfg::TILE_M, GEMM_BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t it = 0;; ++it) {
                int64_t tile;
                if (!dyn) {
                    tile = unit + it * n_units;
                } else {
                    const int slot = (int)(it & (QD - 1));
                    mbar_wait(&tq_full[slot], (uint32_t)(it / QD) & 1u);
                    tile = tile_q[slot];
                    mbar_arrive(&tq_empty[slot]);
                }
                if (tile >= num_work) break;
                int64_t tt, kb_b, kb_e, sp;
                split_unit(tile, tt, kb_b, kb_e, sp);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * GEMM_BN);
                for (int64_t kb = kb_b; kb < kb_e; ++kb) {
                    mbar_wait(XF ? &ready[stage] : &full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + stage * Cfg::A_STAGE);
                    const uint32_t b_base = smem_u32(sB + stage * Cfg::B_STAGE);
#pragma unroll
                    for (int k = 0; k < Cfg::BK / 16; ++k) {
                        // K-major: atom k/4 (stacked), +32 B per K=16 inside the 128 B row
                        const uint32_t ka = (uint32_t)((k >> 2) * Cfg::A_ATOM + (k & 3) * 32);
                        const uint32_t kb_off = (uint32_t)((k >> 2) * Cfg::B_ATOM + (k & 3) * 32);
                        const uint64_t adesc =
                            A_MN ? umma_desc_sw128(a_base + k * 2048, 8192, 1024)
                                 : umma_desc_sw128(a_base + ka, 16, 1024);
                        const uint32_t accum = (kb > kb_b || k > 0) ? 1u : 0u;
#pragma unroll
                        for (int h = 0; h < NSPLIT; ++h) {
                            const uint32_t bh = b_base + h * Cfg::B_HALF;
                            const uint64_t bdesc =
                                B_MN ? umma_desc_sw128(bh + k * 2048, 8192, 1024)
                                     : umma_desc_sw128(bh + kb_off, 16, 1024);
                            const uint32_t dh = d_tmem + (uint32_t)(h * GEMM_BN);
                            if constexpr (PAIR) tc_mma_f16_pair(dh, adesc, bdesc, idesc, accum);
                            else tc_mma_f16(dh, adesc, bdesc, idesc, accum);
                        }
                    }
                    if constexpr (PAIR) tc_commit_pair_mc(&empty[stage], 0x3);
                    else tc_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if constexpr (PAIR) tc_commit_pair_mc(&tfull[acc], 0x3);
                else tc_commit(&tfull[acc]);
                advance_acc<ACC_BUFS>(acc, acc_phase);
            }
        }
        __syncwarp();
    } else if (XF && warp == XF_LOADER_WARP) {
        // ------------------------------------------------------------ input loader (XF)
        // The transform's per-stage inputs -- grad_hidden: the 128 rows' scales f of the
        // stage's 256-column tile; grad_W: the 64 tokens' scales and (target column, G value)
        // -- loaded with plain loads and stored to xin[stage] as soon as the stage is free (the
        // producer's `empty`), then published with xin_full (release / acquire).  Kept out of
        // the transform warps, whose proxy fence would otherwise wait for these loads.
        if constexpr (XF) {
            const int64_t rows = *p.xf_rows;
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t it = 0;; ++it) {
                int64_t tile;
                if (!dyn) {
                    tile = unit + it * n_units;
                } else {
                    const int slot = (int)(it & (QD - 1));
                    mbar_wait_sleep(&tq_full[slot], (uint32_t)(it / QD) & 1u);
                    tile = tile_q[slot];
                    __syncwarp();
                    if (lane == 0) {
                        if (leader) mbar_arrive(&tq_empty[slot]);
                        else mbar_arrive_cluster(mapa_shared(smem_u32(&tq_empty[slot]), 0));
                    }
                }
                if (tile >= num_work) break;
                int64_t tt, kb_b, kb_e, sp;
                split_unit(tile, tt, kb_b, kb_e, sp);
                int64_t m_blk, n_blk;
                tile_coords(tt, num_m, num_n, p.group_m, m_blk, n_blk);
                const int64_t m0 = r0 + m_blk * Cfg::TILE_M + rank * GEMM_BM;
                for (int64_t kb = kb_b; kb < kb_e; ++kb) {
                    float fv[4];
                    int2 yv[2];
                    // loads first (rows past the valid range are never used: zero lines)
                    if constexpr (!A_MN) {
                        const float* src = p.xf_scale + ((kb * GEMM_BK) >> 8) * p.xf_ld + m0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int64_t r = m0 + q * 32 + lane;
                            fv[q] = r < rows ? __ldg(src + q * 32 + lane) : 0.f;
                        }
                    } else {
                        const int64_t k0 = kb * GEMM_BK;
                        const float* src = p.xf_scale + (m0 >> 8) * p.xf_ld + k0;
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const int64_t r = k0 + q * 32 + lane;
                            fv[q] = r < rows ? __ldg(src + q * 32 + lane) : 0.f;
                            yv[q] = r < rows ? __ldg(p.xf_row + r) : make_int2(-1, 0);
                        }
                    }
                    mbar_wait_sleep(&empty[stage], phase ^ 1);  // the stage's previous use done
                    const uint32_t xs = xin_base + stage * XIN_STAGE;
                    if constexpr (!A_MN) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) sts32f(xs + 4 * (q * 32 + lane), fv[q]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            sts32f(xs + 4 * (q * 32 + lane), fv[q]);
                            sts64i2(xs + 256 + 8 * (q * 32 + lane), yv[q]);
                        }
                    }
                    mbar_arrive(&xin_full[stage]);  // release: the stores above
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (XF && warp >= XF_WARP0) {
        // ------------------------------------------------------------ transform (XF)
        if constexpr (XF) {
            // Thread t owns line t of each staged A tile.  The stage's scales (and, for grad_W,
            // the tokens' target columns) come from xin[stage] (the loader warp), so this loop
            // issues no global loads in steady state: its proxy fence waits only for its own
            // shared-memory stores.
            const int t = threadIdx.x - XF_WARP0 * 32;
            const int64_t rows = *p.xf_rows;
            const uint32_t ready_leader = PAIR ? mapa_shared(smem_u32(&ready[0]), 0) : 0u;
            const int line = A_MN ? (t & 63) : t;
            const uint32_t line_off = smem_u32(sA) + (A_MN ? (t >> 6) * 8192 : 0) + line * 128;
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t it = 0;; ++it) {
                int64_t tile;
                if (!dyn) {
                    tile = unit + it * n_units;
                } else {
                    const int slot = (int)(it & (QD - 1));
                    mbar_wait_sleep(&tq_full[slot], (uint32_t)(it / QD) & 1u);
                    tile = tile_q[slot];
                    __syncwarp();
                    if (lane == 0) {
                        if (leader) mbar_arrive(&tq_empty[slot]);
                        else mbar_arrive_cluster(mapa_shared(smem_u32(&tq_empty[slot]), 0));
                    }
                }
                if (tile >= num_work) break;
                int64_t tt, kb_b, kb_e, sp;
                split_unit(tile, tt, kb_b, kb_e, sp);
                int64_t m_blk, n_blk;
                tile_coords(tt, num_m, num_n, p.group_m, m_blk, n_blk);
                const int64_t m0 = r0 + m_blk * Cfg::TILE_M + rank * GEMM_BM;
                // A_MN = false (grad_hidden): line t = token row m0 + t, K = vocabulary; the
                // row's (target column, G value) is fixed for the tile.
                // A_MN = true (grad_W): line t = token k0 + (t & 63) of the vocabulary atom
                // m0 + 64 (t >> 6), K = tokens.
                int2 yr = make_int2(-1, 0);
                const int64_t tok = m0 + t;
                if (!A_MN && tok < rows) yr = __ldg(p.xf_row + tok);
                const int64_t vcol0 = m0 + 64 * (t >> 6);
                const bool vcol_ok = !A_MN || vcol0 < M;
                for (int64_t kb = kb_b; kb < kb_e; ++kb) {
                    mbar_wait_sleep(&xin_full[stage], phase);  // the stage's scales
                    mbar_wait_sleep(&full[stage], phase);      // the stage's P~ tile
                    const uint32_t xs = xin_base + stage * XIN_STAGE;
                    float f;
                    int ycol = -1;
                    float gy;
                    bool zero;
                    if constexpr (!A_MN) {
                        zero = tok >= rows;
                        f = lds32f(xs + 4 * t);
                        const int64_t yl = (int64_t)yr.x - kb * GEMM_BK;
                        if (yr.x >= 0 && yl >= 0 && yl < 64) ycol = (int)yl;
                        gy = __int_as_float(yr.y);
                    } else {
                        const int64_t tk = kb * GEMM_BK + (t & 63);
                        zero = tk >= rows || !vcol_ok;
                        f = lds32f(xs + 4 * (t & 63));
                        const int2 y2 = lds64i2(xs + 256 + 8 * (t & 63));
                        const int64_t yl = (int64_t)y2.x - vcol0;
                        if (y2.x >= 0 && yl >= 0 && yl < 64) ycol = (int)yl;
                        gy = __int_as_float(y2.y);
                    }
                    xf_line(line_off + stage * Cfg::A_STAGE, line, f, ycol, gy, zero);
                    fence_proxy_async_smem();  // generic smem writes -> the MMA's proxy
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (PAIR) mbar_arrive_cluster(ready_leader + stage * 8);
                        else mbar_arrive(&ready[stage]);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        uint32_t tempty_leader0 = 0u, tempty_leader1 = 0u;
        if constexpr (PAIR) {
            tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
            tempty_leader1 = mapa_shared(smem_u32(&tempty[1]), 0);
        }
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t it = 0;; ++it) {
            int64_t tile;
            if (!dyn) {
                tile = unit + it * n_units;
            } else {
                const int slot = (int)(it & (QD - 1));
                mbar_wait_sleep(&tq_full[slot], (uint32_t)(it / QD) & 1u);
                tile = tile_q[slot];
                __syncwarp();
                if (lane == 0) {
                    if (leader) mbar_arrive(&tq_empty[slot]);
                    else mbar_arrive_cluster(mapa_shared(smem_u32(&tq_empty[slot]), 0));
                }
            }
            if (tile >= num_work) break;
            int64_t tt, kb_b, kb_e, sp;
            split_unit(tile, tt, kb_b, kb_e, sp);
            const bool have_k = kb_e > kb_b;  // (else a zero tile: empty K range)
            int64_t m_blk, n_blk;
            tile_coords(tt, num_m, num_n, p.group_m, m_blk, n_blk);
            const int64_t row = r0 + m_blk * Cfg::TILE_M + rank * GEMM_BM + q * 32 + lane;
            const bool row_ok = row < M;
            mbar_wait_sleep(&tfull[acc], acc_phase);
            tc_fence_after();
            uint32_t r[32];
#pragma unroll 1
            for (int h = 0; h < NSPLIT; ++h) {
                const int32_t col0 = (int32_t)(n_blk * Cfg::TILE_N + h * GEMM_BN);
                const int32_t ncol = min(GEMM_BN, p.N - col0);  // valid columns (may be <= 0)
                const uint32_t taddr =
                    tmem_base + lane_base + (uint32_t)(acc * GEMM_BN + h * GEMM_BN);

                if constexpr (EPI == EPI_FWD || EPI == EPI_LOGP) {
                    constexpr bool kStoreP = EPI == EPI_FWD;  // EPI_LOGP: statistics only
                    const float s = p.scale;
                    const float LOG2E = 1.4426950408889634f;
                    // pass 1: tile max over valid columns
                    float m = -INFINITY;
#pragma unroll 1
                    for (int c = 0; c < GEMM_BN / 32; ++c) {
                        tmem_ld_32x32b_x32(taddr + c * 32, r);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c * 32 + j < ncol) m = fmaxf(m, s * __uint_as_float(r[j]));
                    }
                    // pass 2: P~ = exp(z - m), l' = sum P~ - 1 (the first max element is left
                    // out of the sum instead of subtracting 1 afterwards, so l' keeps full
                    // relative precision when the tile max dominates -- p_y close to 1), z_y
                    const int32_t y = row_ok ? p.tgt[row] : -1;
                    const int32_t yl = y - col0;
                    // u (EPI_LOGP): sum exp(z - m) (m - z) >= 0 -- nonnegative terms, so the
                    // entropy of a peaked row is not a difference of two ~|z| numbers
                    float l = 0.f, u = 0.f;
                    bool max_seen = false;
                    const float mb = m * LOG2E;
                    __nv_bfloat16* prow =
                        kStoreP ? p.P + (row_ok ? row : 0) * p.ldP + col0 : nullptr;
                    // the warp's staging slot (AGENTRL_FWD_PSTAGE): row r's four 16-byte pieces
                    // at r * 4 + (piece ^ ((r >> 1) & 3)) -- conflict-free both ways
                    uint4* pst = reinterpret_cast<uint4*>(xin) + q * (32 * 4);
                    const int64_t row0 = row - lane;
                    (void)pst;
                    (void)row0;
#pragma unroll 1
                    for (int c = 0; c < GEMM_BN / 32; ++c) {
                        tmem_ld_32x32b_x32(taddr + c * 32, r);
                        tmem_ld_wait();
                        float e[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float z = s * __uint_as_float(r[j]);
                            const bool ok = c * 32 + j < ncol;
                            e[j] = ok ? ex2_approx(fmaf(z, LOG2E, -mb)) : 0.f;
                            const bool is_max = ok && !max_seen && z == m;
                            max_seen |= is_max;
                            if (is_max) e[j] = 1.f;
                            l += is_max ? 0.f : e[j];
                            if constexpr (!kStoreP) u = fmaf(e[j], ok ? m - z : 0.f, u);
                            if (c * 32 + j == yl && row_ok) p.zy[row] = z;
                        }
                        if constexpr (kStoreP && Cfg::PSTAGE > 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                uint4 v;
                                v.x = pack_bf162(e[j + 0], e[j + 1]);
                                v.y = pack_bf162(e[j + 2], e[j + 3]);
                                v.z = pack_bf162(e[j + 4], e[j + 5]);
                                v.w = pack_bf162(e[j + 6], e[j + 7]);
                                pst[lane * 4 + ((j >> 3) ^ ((lane >> 1) & 3))] = v;
                            }
                            __syncwarp();
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int rl = i * 8 + (lane >> 2), pc = lane & 3;
                                const uint4 v = pst[rl * 4 + (pc ^ ((rl >> 1) & 3))];
                                const int64_t rg = row0 + rl;
                                if (rg < M && c * 32 + pc * 8 < ncol)
                                    *reinterpret_cast<uint4*>(p.P + rg * p.ldP + col0 + c * 32 +
                                                              pc * 8) = v;
                            }
                            __syncwarp();
                        } else if (kStoreP && row_ok) {
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                if (c * 32 + j < ncol) {
                                    uint4 v;
                                    v.x = pack_bf162(e[j + 0], e[j + 1]);
                                    v.y = pack_bf162(e[j + 2], e[j + 3]);
                                    v.z = pack_bf162(e[j + 4], e[j + 5]);
                                    v.w = pack_bf162(e[j + 6], e[j + 7]);
                                    *reinterpret_cast<uint4*>(prow + c * 32 + j) = v;
                                }
                            }
                        }
                    }
                    if (row_ok) {
                        // tile-major [n_tiles][ldpart]: the 32 lanes (rows) of a warp store 256
                        // contiguous bytes
                        if constexpr (kStoreP) p.part[n_blk * p.ldpart + row] = make_float2(m, l);
                        else p.part4[row * p.n_tiles + n_blk] = make_float4(m, l, u, 0.f);
                    }
                } else if constexpr (EPI == EPI_GRADH) {
                    const float s = p.scale;
                    __nv_bfloat16* orow =
                        p.gh + (row_ok ? (int64_t)p.idx[row] : 0) * p.ldo + col0;
#pragma unroll 1
                    for (int c = 0; c < GEMM_BN / 32; ++c) {
                        tmem_ld_32x32b_x32(taddr + c * 32, r);
                        tmem_ld_wait();
                        if (row_ok) {
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                if (c * 32 + j < ncol) {
                                    uint4 v;
                                    v.x = pack_bf162(s * __uint_as_float(r[j + 0]),
                                                     s * __uint_as_float(r[j + 1]));
                                    v.y = pack_bf162(s * __uint_as_float(r[j + 2]),
                                                     s * __uint_as_float(r[j + 3]));
                                    v.z = pack_bf162(s * __uint_as_float(r[j + 4]),
                                                     s * __uint_as_float(r[j + 5]));
                                    v.w = pack_bf162(s * __uint_as_float(r[j + 6]),
                                                     s * __uint_as_float(r[j + 7]));
                                    *reinterpret_cast<uint4*>(orow + c * 32 + j) = v;
                                }
                            }
                        }
                    }
                } else if (EPI == EPI_GRADW && Cfg::EPI_STAGE > 0 && p.peer_out) {
                    // EPI_GRADW fused with the reduce-scatter: each 32 x 32 chunk goes through
                    // the warp's smem slab; then row i of the warp's 32 rows is written by the
                    // 32 lanes as 128 contiguous bytes straight into its owner's window
                    const float s = have_k ? p.scale : 0.f;
                    float* slab = reinterpret_cast<float*>(xin + (XF ? STAGES * XIN_STAGE : 0)) +
                                  q * (32 * 33);
                    const int64_t row0 = row - lane;
                    const int64_t o0 = row0 / p.peer_rows;  // owner of the warp's first row
#pragma unroll 1
                    for (int c = 0; c < GEMM_BN / 32; ++c) {
                        if (have_k) {
                            tmem_ld_32x32b_x32(taddr + c * 32, r);
                            tmem_ld_wait();
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) r[j] = 0u;
                        }
#pragma unroll
                        for (int j = 0; j < 32; ++j) slab[lane * 33 + j] = s * __uint_as_float(r[j]);
                        __syncwarp();
                        const bool col_ok = c * 32 + lane < ncol;
#pragma unroll 4
                        for (int i = 0; i < 32; ++i) {
                            const int64_t ri = row0 + i;
                            if (ri < M && col_ok) {
                                int64_t o = o0, lr = ri - o0 * p.peer_rows;
                                if (lr >= p.peer_rows) {  // the 32 rows cross an owner boundary
                                    o = ri / p.peer_rows;
                                    lr = ri - o * p.peer_rows;
                                }
                                float* dst = p.peer_out[o] +
                                             ((int64_t)p.peer_rank * p.peer_rows + lr) * p.ldo + col0 +
                                             c * 32 + lane;
                                *dst = slab[i * 33 + lane];
                            }
                        }
                        __syncwarp();
                    }
                } else if (EPI == EPI_GRADW && Cfg::EPI_STAGE > 0 && AGENTRL_GRADW_STAGE) {
                    // local grad_W (also the split-K and vocabulary-parallel fp32 partials): each
                    // 32 x 32 chunk is staged in the warp's slab (row r's eight 16-byte pieces at
                    // r * 8 + (piece ^ (r & 7)): conflict-free both ways), then every store
                    // instruction writes 4 rows x 128 contiguous bytes (full lines) instead of
                    // 16 B from each of 32 rows -- the same instruction count
                    const float s = have_k ? p.scale : 0.f;
                    float4* slab = reinterpret_cast<float4*>(
                                       xin + (XF ? STAGES * XIN_STAGE : 0)) + q * (32 * 8);
                    const int64_t row0 = row - lane;
                    float* obase = p.gw + sp * p.gw_split + col0;
#pragma unroll 1
                    for (int c = 0; c < GEMM_BN / 32; ++c) {
                        if (have_k) {
                            tmem_ld_32x32b_x32(taddr + c * 32, r);
                            tmem_ld_wait();
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) r[j] = 0u;
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            slab[lane * 8 + (j ^ (lane & 7))] =
                                make_float4(s * __uint_as_float(r[4 * j + 0]),
                                            s * __uint_as_float(r[4 * j + 1]),
                                            s * __uint_as_float(r[4 * j + 2]),
                                            s * __uint_as_float(r[4 * j + 3]));
                        __syncwarp();
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int rl = i * 4 + (lane >> 3), pc = lane & 7;
                            const float4 v = slab[rl * 8 + (pc ^ (rl & 7))];
                            const int64_t ri = row0 + rl;
                            if (ri < M && c * 32 + pc * 4 < ncol)
                                *reinterpret_cast<float4*>(obase + ri * p.ldo + c * 32 + pc * 4) = v;
                        }
                        __syncwarp();
                    }
                } else {  // EPI_GRADW
                    const float s = have_k ? p.scale : 0.f;
                    const int64_t rr = row_ok ? row : 0;
                    float* orow;
                    if (p.peer_out) {  // straight into the owner's window (NVLink peer memory)
                        const int64_t o = rr / p.peer_rows;
                        orow = p.peer_out[o] +
                               ((int64_t)p.peer_rank * p.peer_rows + (rr - o * p.peer_rows)) * p.ldo +
                               col0;
                    } else {
                        orow = p.gw + sp * p.gw_split + rr * p.ldo + col0;
                    }
#pragma unroll 1
                    for (int c = 0; c < GEMM_BN / 32; ++c) {
                        if (have_k) {
                            tmem_ld_32x32b_x32(taddr + c * 32, r);
                            tmem_ld_wait();
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) r[j] = 0u;
                        }
                        if (row_ok) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4) {
                                if (c * 32 + j < ncol) {
                                    float4 v = make_float4(s * __uint_as_float(r[j + 0]),
                                                           s * __uint_as_float(r[j + 1]),
                                                           s * __uint_as_float(r[j + 2]),
                                                           s * __uint_as_float(r[j + 3]));
                                    *reinterpret_cast<float4*>(orow + c * 32 + j) = v;
                                }
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
                else mbar_arrive(&tempty[acc]);
            }
            advance_acc<ACC_BUFS>(acc, acc_phase);
        }
        // peer stores visible system-wide before the kernel ends (the signal kernel follows)
        if constexpr (EPI == EPI_GRADW) {
            if (p.peer_out) __threadfence_system();
        }
    }

    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync();  // peer done with TMEM / remote barriers before teardown
    tc_fence_after();
    if (warp == 1) {
        if (PAIR) tmem_dealloc_pair(tmem_base, 512);
        else tmem_dealloc(tmem_base, 512);
    }
}

template <int EPI, bool A_MN, bool B_MN, int NSPLIT, int KSUB, bool XF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(XF ? GEMM_THREADS_XF : GEMM_THREADS, 1)
    gemm_sm100_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmB, const GemmArgs p) {
    gemm_body<EPI, A_MN, B_MN, true, NSPLIT, KSUB, XF>(tmA, tmB, p);
}

template <int EPI, bool A_MN, bool B_MN, bool XF>
__global__ void __launch_bounds__(XF ? GEMM_THREADS_XF : GEMM_THREADS, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, const GemmArgs p) {
    gemm_body<EPI, A_MN, B_MN, false, 1, 1, XF>(tmA, tmB, p);
}

}  // namespace agentrl
