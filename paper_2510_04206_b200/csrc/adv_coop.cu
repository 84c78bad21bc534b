// adv_coop.cu -- part 1 (GRPO group advantage P:1263, then task advantage normalization,
// sec 3.2 Eq.1) as ONE cooperative persistent kernel with grid-wide barriers
// between its phases (two launches around the NCCL all-reduce when a communicator is given).
//
//   phase 0  zero the integer scratch (n_g, K_j, fill counters)
//   phase A  token-parallel (4096-token chunks, 16 B mask loads): n_g via integer atomics,
//            per-chunk masked counts; trajectory-parallel: K_j, offsets validation
//   phase B1 block 0: exclusive scans of chunk counts (-> compaction bases) and K_j
//   phase B2 trajectory-parallel: group member lists (atomic slots)
//   phase B3 group-parallel: sort members (-> deterministic order), exact-equal rule,
//            population std, A_hat_g (fp64); per-group (N, S, Q) = (sum n, sum n A, sum n A^2)
//   phase B4 block 0: per-task (N_i, S_i, Q_i) as a fixed-order sum over groups
//   [C1 NCCL all-reduce of the 3*n_tasks doubles -- second launch starts here]
//   phase C  token-parallel: mu_i = S_i/N_i, sigma_i = sqrt(max(Q_i/N_i - mu_i^2, 0)),
//            adv_tok[t] = mask ? (A_hat_g - mu)/max(sigma, eps) : 0, stable compaction
//            idx[] / adv_c[] for part 2; block 0 writes task_stats and N.
// Every reduction has a fixed order, so results are bitwise run-to-run deterministic.
#include <cooperative_groups.h>
#include <algorithm>
#include <cuda_runtime.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace agentrl {

constexpr int COOP_THREADS = 256;
#ifndef ADV_MIN_BLOCKS
#define ADV_MIN_BLOCKS 3  // resident blocks per SM the register budget is cut for
#endif
constexpr int GMAX_BLOCKS = 2048;  // cap on the cooperative grid (per-block scratch arrays)
constexpr int WCHUNK = 512;        // tokens per warp chunk (32 lanes x 16 tokens)
constexpr int WOFF_CAP = 64;       // trajectory offsets staged per warp chunk
constexpr int NWARPS = COOP_THREADS / 32;
constexpr int TASK_BATCH = 16;  // tasks reduced per barrier in the per-block partials
constexpr int BT_CAP = 2048;    // trajectories a block stages in smem for its token range

// static shared memory of the cooperative kernels (one arena for all phases)
struct CoopSmem {
    int32_t s_w[8];
    int32_t s_pre[GMAX_BLOCKS + 1];
    // the offsets of the trajectories overlapping this block's tokens (or, on the fallback path
    // for blocks spanning more than BT_CAP trajectories, per-warp offset staging)
    int64_t s_boff[BT_CAP + 1];
    int32_t s_aux[BT_CAP];  // phase A: masked count per staged trajectory; C: its A~ (f32 bits)
};

// phase timestamps of the last cooperative launch (block 0, after each grid barrier), read by
// agentrl_debug_adv_phase_ns(); 8 x %globaltimer ns
__device__ unsigned long long g_adv_phase_ns[8];
__device__ __forceinline__ void phase_mark(int i) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_adv_phase_ns[i] = t;
    }
}

struct AdvParams {
    int64_t T;
    int32_t n_traj, n_groups, n_tasks;
    int64_t n_chunks;
    const int64_t* off;
    const int32_t* task_id;
    const int32_t* group_id;
    const float* rewards;
    const uint8_t* mask;
    double eps_std;
    int32_t *n_g, *chunk, *grp_cnt, *grp_start, *grp_fill, *members, *grp_task, *chunk_first;
    int32_t *blk_chunk, *blk_grp;  // per-block masked / member totals
    int32_t* chunk_base;           // [n_chunks] compaction base of each chunk within its block
    double* blk_part;              // per-block per-task (N, S, Q) partials
    double *adv_hat, *grp_nsq, *stats;
    int64_t* meta;
    int32_t* d_status;
    float* adv_tok;
    int32_t* idx;
    float* adv_c;
    double* task_stats_out;
    int64_t* n_mask_global_out;
    int32_t compact;  // write idx[] / adv_c[] (needed by the fused step only)
};

__device__ __forceinline__ int32_t coop_find_traj(const int64_t* __restrict__ off,
                                                  int32_t n_traj, int64_t t) {
    int32_t lo = 0, hi = n_traj;
    while (hi - lo > 1) {
        const int32_t mid = (lo + hi) >> 1;
        if (off[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo < n_traj ? lo : n_traj - 1;
}

// trajectories [bf, bf + n) overlap this block's warp chunks [c_lo, c_hi) (clamped; 0 if none)
__device__ __forceinline__ int32_t block_traj_range(const AdvParams& p, int64_t c_lo, int64_t c_hi,
                                                    int32_t& bf) {
    bf = 0;
    if (p.n_traj <= 0 || c_lo >= c_hi) return 0;
    int32_t f = p.chunk_first[c_lo];
    int32_t l = c_hi < p.n_chunks ? p.chunk_first[c_hi] : p.n_traj - 1;
    f = min(max(f, 0), p.n_traj - 1);
    l = min(max(l, f), p.n_traj - 1);
    bf = f;
    return l - f + 1;
}
// k in [lo, hi) with s[k] <= t < s[k+1] (clamped to lo / hi - 1)
__device__ __forceinline__ int32_t smem_find_in(const int64_t* s, int32_t lo, int32_t hi, int64_t t) {
    while (hi - lo > 1) {
        const int32_t mid = (lo + hi) >> 1;
        if (s[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}
// mask byte i (compile-time after unrolling) of a 16-byte vector, as 0/1
__device__ __forceinline__ int32_t mbit(const uint4& v, int i) {
    const uint32_t w = i < 4 ? v.x : (i < 8 ? v.y : (i < 12 ? v.z : v.w));
    return ((w >> (8 * (i & 3))) & 0xffu) != 0u;
}

__device__ __forceinline__ void coop_mask16(const uint8_t* __restrict__ mask, int64_t T,
                                            int64_t t0, bool any_traj, uint8_t (&m)[16]) {
    if (any_traj && t0 + 16 <= T && (reinterpret_cast<uintptr_t>(mask + t0) & 15) == 0) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(mask + t0));
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
#pragma unroll
        for (int i = 0; i < 16; ++i) m[i] = b[i];
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) m[i] = (any_traj && t0 + i < T) ? mask[t0 + i] : 0;
    }
}

// Token -> trajectory lookup for one 4096-token chunk: the block stages off[first .. last+1]
// of the trajectories that overlap the chunk into shared memory (one coalesced load) and every
// thread binary-searches there, instead of ~log2(n_traj) dependent global loads per phase.
constexpr int SOFF_CAP = 1024;
struct ChunkTraj {
    int32_t first, cnt;  // cnt = number of staged offsets (trajectories + 1); 0 = not staged
};
__device__ __forceinline__ ChunkTraj stage_chunk_offsets(const int64_t* __restrict__ off,
                                                         const int32_t* __restrict__ chunk_first,
                                                         int32_t n_traj, int64_t c,
                                                         int64_t n_chunks, int64_t* s_off) {
    ChunkTraj r{0, 0};
    int32_t f = chunk_first[c];
    int32_t l = (c + 1 < n_chunks) ? chunk_first[c + 1] : n_traj - 1;
    f = min(max(f, 0), n_traj - 1);
    l = min(max(l, f), n_traj - 1);
    const int32_t cnt = l - f + 2;
    r.first = f;
    if (cnt <= SOFF_CAP) {
        for (int32_t i = threadIdx.x; i < cnt; i += blockDim.x) s_off[i] = off[f + i];
        r.cnt = cnt;
    }
    __syncthreads();
    return r;
}
// local index k with s_off[k] <= t < s_off[k+1] (clamped)
__device__ __forceinline__ int32_t smem_find(const int64_t* s_off, int32_t cnt, int64_t t) {
    int32_t lo = 0, hi = cnt - 1;
    while (hi - lo > 1) {
        const int32_t mid = (lo + hi) >> 1;
        if (s_off[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

// warp-level staging of the offsets of the trajectories overlapping warp chunk c; returns the
// number staged (0: too many, use the global binary search)
__device__ __forceinline__ int32_t warp_stage(const int64_t* __restrict__ off,
                                              const int32_t* __restrict__ wfirst, int32_t n_traj,
                                              int64_t c, int64_t n_wchunks, int64_t* s_offw,
                                              int32_t& first) {
    const int lane = threadIdx.x & 31;
    int32_t f = wfirst[c];
    int32_t l = (c + 1 < n_wchunks) ? wfirst[c + 1] : n_traj - 1;
    f = min(max(f, 0), n_traj - 1);
    l = min(max(l, f), n_traj - 1);
    const int32_t cnt = l - f + 2;
    first = f;
    if (cnt > WOFF_CAP) return 0;
    for (int32_t i = lane; i < cnt; i += 32) s_offw[i] = off[f + i];
    __syncwarp();
    return cnt;
}
__device__ __forceinline__ int32_t warp_incl_scan(int32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// ---- software-pipelined chunk inputs: the mask bytes and trajectory range of the NEXT chunk
// are loaded while the current chunk is processed (breaks the per-warp dependent-load chain)
struct ChunkIn {
    uint4 mk;
    int32_t f, l, base;
};
__device__ __forceinline__ ChunkIn chunk_fetch(const AdvParams& p, int64_t c, bool any_traj,
                                               bool want_base) {
    ChunkIn r;
    const int lane = threadIdx.x & 31;
    const int64_t t0 = c * WCHUNK + lane * 16;
    if (any_traj && t0 + 16 <= p.T && (reinterpret_cast<uintptr_t>(p.mask + t0) & 15) == 0) {
        r.mk = __ldg(reinterpret_cast<const uint4*>(p.mask + t0));
    } else {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        for (int i = 0; i < 16; ++i)
            if (any_traj && t0 + i < p.T) w[i >> 2] |= (uint32_t)p.mask[t0 + i] << (8 * (i & 3));
        r.mk = make_uint4(w[0], w[1], w[2], w[3]);
    }
    r.f = any_traj ? p.chunk_first[c] : 0;
    r.l = (any_traj && c + 1 < p.n_chunks) ? p.chunk_first[c + 1] : p.n_traj - 1;
    r.base = want_base ? p.chunk_base[c] : 0;
    return r;
}
__device__ __forceinline__ void unpack16(const uint4& v, uint8_t (&m)[16]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
}
__device__ __forceinline__ int32_t warp_stage_fl(const int64_t* __restrict__ off, int32_t f,
                                                 int32_t l, int32_t n_traj, int64_t* s_offw,
                                                 int32_t& first) {
    const int lane = threadIdx.x & 31;
    f = min(max(f, 0), n_traj - 1);
    l = min(max(l, f), n_traj - 1);
    const int32_t cnt = l - f + 2;
    first = f;
    if (cnt > WOFF_CAP) return 0;
    for (int32_t i = lane; i < cnt; i += 32) s_offw[i] = off[f + i];
    __syncwarp();
    return cnt;
}

// exclusive scan of one int per thread over a 256-thread block (returns prefix; total out)
__device__ __forceinline__ int32_t coop_block_exscan(int32_t v, int32_t* s_w, int32_t& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int32_t w = lane < 8 ? s_w[lane] : 0;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < 8) s_w[lane] = w;
    }
    __syncthreads();
    const int32_t base = wid > 0 ? s_w[wid - 1] : 0;
    total = s_w[7];
    __syncthreads();
    return base + x - v;
}

// in-place exclusive scan of a[0..n) by one block of 256 threads (contiguous per-thread
// segments, then a block scan of segment sums); returns the total
__device__ int64_t coop_block_scan_array(int32_t* a, int64_t n, int64_t* s_seg) {
    const int64_t per = (n + COOP_THREADS - 1) / COOP_THREADS;
    const int64_t lo = min(n, (int64_t)threadIdx.x * per), hi = min(n, lo + per);
    int64_t s = 0;
    for (int64_t i = lo; i < hi; ++i) s += a[i];
    // block scan of 64-bit segment sums
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_seg[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < 8 ? s_seg[lane] : 0;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < 8) s_seg[lane] = w;
    }
    __syncthreads();
    int64_t run = (wid > 0 ? s_seg[wid - 1] : 0) + x - s;
    const int64_t total = s_seg[7];
    for (int64_t i = lo; i < hi; ++i) {
        const int32_t v = a[i];
        a[i] = (int32_t)run;
        run += v;
    }
    __syncthreads();
    return total;
}

__device__ __forceinline__ double coop_block_sum(double v, double* s_red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) s_red[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < COOP_THREADS / 32; ++w) r += s_red[w];
    __syncthreads();
    return r;  // thread 0
}

// ------------------------------------------------------------------ helpers
// balanced contiguous partition of [0, n) over G blocks
__device__ __forceinline__ int64_t part_lo(int64_t n, int64_t b, int64_t G) { return n * b / G; }
// block owning item j under part_lo
__device__ __forceinline__ int64_t part_owner(int64_t n, int64_t j, int64_t G) {
    return ((j + 1) * G + n - 1) / n - 1;
}
// exclusive prefix over blocks of a per-block int array, computed by every block into smem
__device__ void block_prefix_smem(const int32_t* __restrict__ blk, int64_t G, int32_t* s_pre,
                                  int32_t* s_w) {
    // G <= GMAX_BLOCKS; each thread scans a contiguous segment
    const int64_t per = (G + COOP_THREADS - 1) / COOP_THREADS;
    const int64_t lo = min(G, (int64_t)threadIdx.x * per), hi = min(G, lo + per);
    int32_t sum = 0;
    for (int64_t b = lo; b < hi; ++b) sum += blk[b];
    int32_t total;
    int32_t run = coop_block_exscan(sum, s_w, total);
    for (int64_t b = lo; b < hi; ++b) {
        s_pre[b] = run;
        run += blk[b];
    }
    if (threadIdx.x == 0) s_pre[G] = total;
    __syncthreads();
}

// ------------------------------------------------------------------ phases 0 .. B4
__device__ __forceinline__ void coop_stats_phases(const AdvParams& p, cg::grid_group& grid, CoopSmem& sm) {
    static_assert(NWARPS * WOFF_CAP <= BT_CAP + 1, "fallback staging fits the arena");
    int32_t* s_w = sm.s_w;
    int32_t* s_pre = sm.s_pre;
    int64_t* s_off = sm.s_boff;  // fallback path: per-warp staging
    const int64_t G = gridDim.x, B = blockIdx.x;
    const int64_t gtid = B * blockDim.x + threadIdx.x;
    const int64_t gstride = G * blockDim.x;
    int32_t st = 0;
    phase_mark(0);
    const int64_t c_lo = part_lo(p.n_chunks, B, G), c_hi = part_lo(p.n_chunks, B + 1, G);
    const int64_t j_lo = part_lo(p.n_groups, B, G), j_hi = part_lo(p.n_groups, B + 1, G);

    // phase 0: zero scratch; chunk -> first-trajectory table
    if (gtid == 0) p.meta[3] = 0;  // local count of trajectories with masked tokens (n_seq)
    for (int64_t i = gtid; i < p.n_traj; i += gstride) p.n_g[i] = 0;
    for (int64_t i = gtid; i < p.n_groups; i += gstride) {
        p.grp_cnt[i] = 0;
        p.grp_fill[i] = 0;
    }
    for (int64_t g = gtid; g < p.n_traj; g += gstride) {  // chunks whose first token is in g
        const int64_t a = p.off[g], b = p.off[g + 1];
        const int64_t lo = (a + WCHUNK - 1) / WCHUNK;
        const int64_t hi = min((b + WCHUNK - 1) / WCHUNK, p.n_chunks);
        for (int64_t c = max(lo, (int64_t)0); c < hi; ++c) p.chunk_first[c] = (int32_t)g;
    }
    grid.sync();
    phase_mark(1);

    // phase A: this block's contiguous warp chunks (512 tokens each, one warp per chunk):
    // n_g, per-chunk counts, block total.  Fast path: the block stages the offsets of the
    // trajectories its tokens cover once (one coalesced load) and counts per trajectory with
    // shared atomics; the chunk loop then has no dependent global loads.
    const bool any_traj = p.n_traj > 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t bf = 0;
    const int32_t nbt = any_traj ? block_traj_range(p, c_lo, c_hi, bf) : 0;
    const bool staged = nbt > 0 && nbt <= BT_CAP;
    if (staged) {
        for (int32_t k = threadIdx.x; k <= nbt; k += COOP_THREADS) {
            sm.s_boff[k] = p.off[bf + k];
            if (k < nbt) sm.s_aux[k] = 0;
        }
    }
    __syncthreads();
    int64_t* s_offw = s_off + warp * WOFF_CAP;
    int32_t warp_total = 0;
    ChunkIn nxt{};
    if (c_lo + warp < c_hi) nxt = chunk_fetch(p, c_lo + warp, any_traj, false);
    for (int64_t c = c_lo + warp; c < c_hi; c += NWARPS) {
        const ChunkIn cur = nxt;
        if (c + NWARPS < c_hi) nxt = chunk_fetch(p, c + NWARPS, any_traj, false);
        const int64_t t0 = c * WCHUNK + lane * 16;
        int32_t mine = 0;
        if (staged) {
            if (t0 < p.T) {
                const int32_t klo = min(max(cur.f - bf, 0), nbt - 1);
                const int32_t khi = min(max(cur.l - bf + 1, klo + 1), nbt);
                int32_t k = smem_find_in(sm.s_boff, klo, khi, t0);
                int64_t end = sm.s_boff[k + 1];
                int32_t cnt = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int64_t t = t0 + i;
                    while (t >= end && k + 1 < nbt) {
                        if (cnt) atomicAdd(&sm.s_aux[k], cnt);
                        cnt = 0;
                        ++k;
                        end = sm.s_boff[k + 1];
                    }
                    const int32_t bit = mbit(cur.mk, i);  // 0 past T (zero-filled load)
                    cnt += bit;
                    mine += bit;
                }
                if (cnt) atomicAdd(&sm.s_aux[k], cnt);
            }
        } else {
            uint8_t m[16];
            unpack16(cur.mk, m);
            int32_t first = 0, cnt_st = 0;
            if (any_traj) cnt_st = warp_stage_fl(p.off, cur.f, cur.l, p.n_traj, s_offw, first);
            if (t0 < p.T && any_traj) {
                int32_t g, k = 0;
                int64_t end;
                if (cnt_st) {
                    k = smem_find(s_offw, cnt_st, t0);
                    g = first + k;
                    end = s_offw[k + 1];
                } else {
                    g = coop_find_traj(p.off, p.n_traj, t0);
                    end = p.off[g + 1];
                }
                int32_t cnt = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int64_t t = t0 + i;
                    if (t >= p.T) break;
                    while (t >= end && g + 1 < p.n_traj) {
                        if (cnt) atomicAdd(&p.n_g[g], cnt);
                        cnt = 0;
                        ++g;
                        ++k;
                        end = (cnt_st && k + 1 < cnt_st) ? s_offw[k + 1] : p.off[g + 1];
                    }
                    const int32_t bit = m[i] != 0;
                    cnt += bit;
                    mine += bit;
                }
                if (cnt) atomicAdd(&p.n_g[g], cnt);
            }
        }
        const int32_t total = __shfl_sync(0xffffffffu, warp_incl_scan(mine), 31);
        if (lane == 0) p.chunk[c] = total;
        warp_total += total;
        __syncwarp();  // s_offw restaged by this warp's next chunk
    }
    if (staged) {  // per-trajectory block counts -> n_g (integer atomics: exact, order-free)
        __syncthreads();
        for (int32_t k = threadIdx.x; k < nbt; k += COOP_THREADS)
            if (sm.s_aux[k]) atomicAdd(&p.n_g[bf + k], sm.s_aux[k]);
    }
    if (lane == 0) s_w[warp] = warp_total;
    __syncthreads();
    // block-local exclusive scan of this block's chunk counts -> chunk_base (local), so that the
    // apply phase can place every chunk without block-wide exchanges
    {
        const int64_t n = c_hi - c_lo;
        const int64_t per = (n + COOP_THREADS - 1) / COOP_THREADS;
        const int64_t lo = c_lo + min(n, (int64_t)threadIdx.x * per);
        const int64_t hi = min(c_hi, lo + per);
        int32_t sum = 0;
        for (int64_t c = lo; c < hi; ++c) sum += p.chunk[c];
        int32_t total;
        int32_t run = coop_block_exscan(sum, s_w, total);
        for (int64_t c = lo; c < hi; ++c) {
            const int32_t v = p.chunk[c];
            p.chunk_base[c] = run;
            run += v;
        }
        if (threadIdx.x == 0) p.blk_chunk[B] = total;
    }
    for (int64_t g = gtid; g < p.n_traj; g += gstride) {
        const int32_t j = p.group_id[g], i = p.task_id[g];
        if (j < 0 || j >= p.n_groups || i < 0 || i >= p.n_tasks) {
            st |= AGENTRL_ST_GROUP_SPANS_TASKS;
            continue;
        }
        atomicAdd(&p.grp_cnt[j], 1);
        if (p.off[g + 1] < p.off[g]) st |= AGENTRL_ST_BAD_OFFSETS;
    }
    if (gtid == 0 && (p.off[0] != 0 || p.off[p.n_traj] != p.T)) st |= AGENTRL_ST_BAD_OFFSETS;
    grid.sync();
    phase_mark(2);

    // phase B1: local exclusive scan of K_j over this block's groups; block total
    {
        const int64_t n = j_hi - j_lo;
        const int64_t per = (n + COOP_THREADS - 1) / COOP_THREADS;
        const int64_t lo = j_lo + min(n, (int64_t)threadIdx.x * per);
        const int64_t hi = min(j_hi, lo + per);
        int32_t sum = 0;
        for (int64_t j = lo; j < hi; ++j) sum += p.grp_cnt[j];
        int32_t total;
        int32_t run = coop_block_exscan(sum, s_w, total);
        for (int64_t j = lo; j < hi; ++j) {
            p.grp_start[j] = run;  // local start within this block's member range
            run += p.grp_cnt[j];
        }
        if (threadIdx.x == 0) p.blk_grp[B] = total;
    }
    grid.sync();
    phase_mark(3);

    // phase B2: global group starts = block prefix + local; scatter member lists
    block_prefix_smem(p.blk_grp, G, s_pre, s_w);
    for (int64_t g = gtid; g < p.n_traj; g += gstride) {
        const int32_t j = p.group_id[g], i = p.task_id[g];
        if (j < 0 || j >= p.n_groups || i < 0 || i >= p.n_tasks) continue;
        const int64_t owner = part_owner(p.n_groups, j, G);
        const int32_t slot = atomicAdd(&p.grp_fill[j], 1);
        p.members[s_pre[owner] + p.grp_start[j] + slot] = (int32_t)g;
    }
    grid.sync();
    phase_mark(4);

    // phase B3: this block's groups (GRPO advantage; readings R1, R2, R14), then the
    // block's per-task partial (N, S, Q) in a fixed order
    unsigned long long nz = 0;  // trajectories with masked tokens (sequence-mean weights)
    for (int64_t j = j_lo + threadIdx.x; j < j_hi; j += COOP_THREADS) {
        const int32_t K = p.grp_cnt[j];
        int32_t* mb = p.members + s_pre[B] + p.grp_start[j];
        for (int a = 1; a < K; ++a) {
            const int32_t x = mb[a];
            int b = a - 1;
            while (b >= 0 && mb[b] > x) {
                mb[b + 1] = mb[b];
                --b;
            }
            mb[b + 1] = x;
        }
        double N = 0.0, S = 0.0, Q = 0.0;
        int32_t task0 = -1;
        if (K > 0) {
            if (K == 1) st |= AGENTRL_ST_GROUP_TOO_SMALL;
            task0 = p.task_id[mb[0]];
            double sum = 0.0, rmax = p.rewards[mb[0]], rmin = rmax;
            for (int a = 0; a < K; ++a) {
                const double r = p.rewards[mb[a]];
                if (p.task_id[mb[a]] != task0) st |= AGENTRL_ST_GROUP_SPANS_TASKS;
                sum += r;
                rmax = fmax(rmax, r);
                rmin = fmin(rmin, r);
            }
            const bool flat = rmax == rmin;
            const double mean = sum / (double)K;
            double ss = 0.0;
            if (!flat)
                for (int a = 0; a < K; ++a) {
                    const double dlt = (double)p.rewards[mb[a]] - mean;
                    ss += dlt * dlt;
                }
            const double sd = sqrt(ss / (double)K);
            const double den = sd > p.eps_std ? sd : p.eps_std;
            for (int a = 0; a < K; ++a) {
                const int32_t g = mb[a];
                const double ah = flat ? 0.0 : ((double)p.rewards[g] - mean) / den;
                p.adv_hat[g] = ah;
                const double n = (double)p.n_g[g];
                N += n;
                S += n * ah;
                Q += n * ah * ah;
                nz += p.n_g[g] > 0;
            }
        }
        p.grp_task[j] = task0;
        p.grp_nsq[3 * j + 0] = N;
        p.grp_nsq[3 * j + 1] = S;
        p.grp_nsq[3 * j + 2] = Q;
    }
    if (nz) atomicAdd(reinterpret_cast<unsigned long long*>(&p.meta[3]), nz);  // integer: exact
    __syncthreads();
    // per-task partials of this block: warp shuffles (fixed tree) + one barrier, tasks in
    // batches of TASK_BATCH
    {
        __shared__ double s_wp[NWARPS][TASK_BATCH][3];
        const int warp_b = threadIdx.x >> 5, lane_b = threadIdx.x & 31;
        for (int32_t i0 = 0; i0 < p.n_tasks; i0 += TASK_BATCH) {
            const int32_t nb = min(TASK_BATCH, p.n_tasks - i0);
            for (int32_t ii = 0; ii < nb; ++ii) {
                double N = 0.0, S = 0.0, Q = 0.0;
                for (int64_t j = j_lo + threadIdx.x; j < j_hi; j += COOP_THREADS)
                    if (p.grp_task[j] == i0 + ii) {
                        N += p.grp_nsq[3 * j];
                        S += p.grp_nsq[3 * j + 1];
                        Q += p.grp_nsq[3 * j + 2];
                    }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    N += __shfl_down_sync(0xffffffffu, N, o);
                    S += __shfl_down_sync(0xffffffffu, S, o);
                    Q += __shfl_down_sync(0xffffffffu, Q, o);
                }
                if (lane_b == 0) {
                    s_wp[warp_b][ii][0] = N;
                    s_wp[warp_b][ii][1] = S;
                    s_wp[warp_b][ii][2] = Q;
                }
            }
            __syncthreads();
            if (threadIdx.x < 3 * nb) {
                const int ii = threadIdx.x / 3, k = threadIdx.x % 3;
                double v = 0.0;
                for (int w = 0; w < NWARPS; ++w) v += s_wp[w][ii][k];
                p.blk_part[3 * ((int64_t)B * p.n_tasks + i0 + ii) + k] = v;
            }
            __syncthreads();
        }
    }
    if (st) atomicOr(p.d_status, st);
    grid.sync();
    phase_mark(5);

    // phase B4 (block 0): per-task moments over the token set = fixed-order sum
    // of the block partials (warp w handles tasks w, w+8, ...; lanes stride over blocks)
    if (B == 0) {
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int32_t i = wid; i < p.n_tasks; i += COOP_THREADS / 32) {
            double N = 0.0, S = 0.0, Q = 0.0;
            for (int64_t b = lane; b < G; b += 32) {
                const double* bp = p.blk_part + 3 * (b * p.n_tasks + i);
                N += bp[0];
                S += bp[1];
                Q += bp[2];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                N += __shfl_down_sync(0xffffffffu, N, o);
                S += __shfl_down_sync(0xffffffffu, S, o);
                Q += __shfl_down_sync(0xffffffffu, Q, o);
            }
            if (lane == 0) {
                p.stats[3 * i] = N;
                p.stats[3 * i + 1] = S;
                p.stats[3 * i + 2] = Q;
            }
        }
        if (threadIdx.x == 0) p.stats[3 * p.n_tasks] = (double)p.meta[3];  // n_seq (local)
    }
}

// ------------------------------------------------------------------ phase C
// (needs gridDim.x == the stats launch's grid: it owns the same contiguous chunk ranges)
__device__ __forceinline__ void coop_apply_phase(const AdvParams& p, CoopSmem& sm) {
    extern __shared__ double s_task[];  // [2*n_tasks]: mu, max(sigma, eps)
    int32_t* s_w = sm.s_w;
    int32_t* s_pre = sm.s_pre;
    int64_t* s_off = sm.s_boff;  // fallback path: per-warp staging
    const int64_t G = gridDim.x, B = blockIdx.x;
    for (int32_t i = threadIdx.x; i < p.n_tasks; i += blockDim.x) {
        const double N = p.stats[3 * i], S = p.stats[3 * i + 1], Q = p.stats[3 * i + 2];
        const double mu = N > 0.0 ? S / N : 0.0;
        const double sd = N > 0.0 ? sqrt(fmax(Q / N - mu * mu, 0.0)) : 0.0;
        s_task[2 * i] = mu;
        s_task[2 * i + 1] = sd > p.eps_std ? sd : p.eps_std;
        if (B == 0 && p.task_stats_out) {
            p.task_stats_out[3 * i] = N;
            p.task_stats_out[3 * i + 1] = mu;
            p.task_stats_out[3 * i + 2] = sd;
        }
    }
    block_prefix_smem(p.blk_chunk, G, s_pre, s_w);  // also orders s_task writes
    if (B == 0 && threadIdx.x < 32) {
        double nsum = 0.0;
        for (int32_t i = threadIdx.x; i < p.n_tasks; i += 32) nsum += p.stats[3 * i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nsum += __shfl_down_sync(0xffffffffu, nsum, o);
        if (threadIdx.x == 0) {
            const int64_t n = (int64_t)nsum;
            p.meta[0] = s_pre[G];  // local masked rows
            p.meta[1] = n;         // global N
            p.meta[2] = (int64_t)p.stats[3 * p.n_tasks];  // global n_seq
            if (p.n_mask_global_out) *p.n_mask_global_out = n;
            if (n == 0) atomicOr(p.d_status, AGENTRL_ST_NO_TOKENS);
        }
    }
    const bool any_traj = p.n_traj > 0;
    const int64_t c_lo = part_lo(p.n_chunks, B, G), c_hi = part_lo(p.n_chunks, B + 1, G);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t* s_offw = s_off + warp * WOFF_CAP;
    const int32_t blk_base = s_pre[B];
    // compaction staging (dynamic smem after s_task; present only when p.compact)
    int32_t(*s_cidx)[WCHUNK] = reinterpret_cast<int32_t(*)[WCHUNK]>(s_task + 2 * p.n_tasks);
    float(*s_cadv)[WCHUNK] = reinterpret_cast<float(*)[WCHUNK]>(s_task + 2 * p.n_tasks) + NWARPS;
    // Fast path: the block stages the offsets and final values A~_g = (A^_g - mu_i) / max(sigma_i,
    // eps) (Eq.1) of the trajectories its tokens cover; the chunk loop then streams
    // mask -> adv_tok with smem lookups only.
    int32_t bf = 0;
    const int32_t nbt = any_traj ? block_traj_range(p, c_lo, c_hi, bf) : 0;
    const bool staged = nbt > 0 && nbt <= BT_CAP;
    if (staged) {
        for (int32_t k = threadIdx.x; k <= nbt; k += COOP_THREADS) {
            sm.s_boff[k] = p.off[bf + k];
            if (k < nbt) {
                const int32_t ti = p.task_id[bf + k];
                const float at = (ti >= 0 && ti < p.n_tasks)
                                     ? (float)((p.adv_hat[bf + k] - s_task[2 * ti]) / s_task[2 * ti + 1])
                                     : 0.f;
                sm.s_aux[k] = __float_as_int(at);
            }
        }
    }
    __syncthreads();
    // every warp walks its own chunks with no block-wide exchange: the chunk's compaction base
    // is the block prefix plus the local base stored by the counting phase
    ChunkIn nxt{};
    if (c_lo + warp < c_hi) nxt = chunk_fetch(p, c_lo + warp, any_traj, true);
    for (int64_t c = c_lo + warp; c < c_hi; c += NWARPS) {
        const ChunkIn cur = nxt;
        if (c + NWARPS < c_hi) nxt = chunk_fetch(p, c + NWARPS, any_traj, true);
        const int32_t wbase = blk_base + cur.base;
        const int64_t t0 = c * WCHUNK + lane * 16;
        int32_t mine = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) mine += mbit(cur.mk, i);
        const int32_t incl = warp_incl_scan(mine);
        const int32_t wtotal = __shfl_sync(0xffffffffu, incl, 31);
        int32_t pos = incl - mine;  // position within this warp chunk's compacted range
        float outv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) outv[i] = 0.f;
        if (staged) {
            if (t0 < p.T && mine > 0) {
                const int32_t klo = min(max(cur.f - bf, 0), nbt - 1);
                const int32_t khi = min(max(cur.l - bf + 1, klo + 1), nbt);
                int32_t k = smem_find_in(sm.s_boff, klo, khi, t0);
                int64_t end = sm.s_boff[k + 1];
                float at = __int_as_float(sm.s_aux[k]);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int64_t t = t0 + i;
                    while (t >= end && k + 1 < nbt) {
                        ++k;
                        end = sm.s_boff[k + 1];
                        at = __int_as_float(sm.s_aux[k]);
                    }
                    const bool on = mbit(cur.mk, i);
                    outv[i] = on ? at : 0.f;
                    if (p.compact && on) {  // staged in smem, written coalesced below
                        s_cidx[warp][pos] = (int32_t)t;
                        s_cadv[warp][pos] = at;
                        ++pos;
                    }
                }
            }
        } else {  // fallback: per-warp offset staging (warp-collective), global lookups
            int32_t first = 0, cnt_st = 0;
            if (any_traj) cnt_st = warp_stage_fl(p.off, cur.f, cur.l, p.n_traj, s_offw, first);
            if (t0 < p.T && any_traj && mine > 0) {
                int32_t g, k = 0;
                int64_t end;
                if (cnt_st) {
                    k = smem_find(s_offw, cnt_st, t0);
                    g = first + k;
                    end = s_offw[k + 1];
                } else {
                    g = coop_find_traj(p.off, p.n_traj, t0);
                    end = p.off[g + 1];
                }
                int32_t gcur = -1;
                float at = 0.f;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int64_t t = t0 + i;
                    while (t >= end && g + 1 < p.n_traj) {
                        ++g;
                        ++k;
                        end = (cnt_st && k + 1 < cnt_st) ? s_offw[k + 1] : p.off[g + 1];
                    }
                    const bool on = t < p.T && mbit(cur.mk, i);
                    if (on) {
                        if (g != gcur) {  // Eq.1 for this trajectory
                            gcur = g;
                            const int32_t ti = p.task_id[g];
                            at = (ti >= 0 && ti < p.n_tasks)
                                     ? (float)((p.adv_hat[g] - s_task[2 * ti]) / s_task[2 * ti + 1])
                                     : 0.f;
                        }
                        outv[i] = at;
                        if (p.compact) {
                            s_cidx[warp][pos] = (int32_t)t;
                            s_cadv[warp][pos] = at;
                            ++pos;
                        }
                    }
                }
            }
        }
        if (t0 < p.T) {
            if (t0 + 16 <= p.T && (reinterpret_cast<uintptr_t>(p.adv_tok + t0) & 15) == 0) {
                float4* o4 = reinterpret_cast<float4*>(p.adv_tok + t0);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    o4[i] = make_float4(outv[4 * i], outv[4 * i + 1], outv[4 * i + 2], outv[4 * i + 3]);
            } else {
                for (int i = 0; i < 16; ++i)
                    if (t0 + i < p.T) p.adv_tok[t0 + i] = outv[i];
            }
        }
        __syncwarp();  // s_offw restaged by this warp's next chunk; s_c* complete
        if (p.compact) {
            for (int32_t i = lane; i < wtotal; i += 32) {
                p.idx[wbase + i] = s_cidx[warp][i];
                p.adv_c[wbase + i] = s_cadv[warp][i];
            }
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(COOP_THREADS, ADV_MIN_BLOCKS) k_adv_coop_all(const AdvParams p) {
    __shared__ CoopSmem sm;
    cg::grid_group grid = cg::this_grid();
    coop_stats_phases(p, grid, sm);
    grid.sync();
    phase_mark(6);
    coop_apply_phase(p, sm);
    grid.sync();
    phase_mark(7);
}

__global__ void __launch_bounds__(COOP_THREADS, ADV_MIN_BLOCKS) k_adv_coop_stats(const AdvParams p) {
    __shared__ CoopSmem sm;
    cg::grid_group grid = cg::this_grid();
    coop_stats_phases(p, grid, sm);
}

__global__ void __launch_bounds__(COOP_THREADS, ADV_MIN_BLOCKS) k_adv_coop_apply(const AdvParams p) {
    __shared__ CoopSmem sm;
    coop_apply_phase(p, sm);
}

static int coop_grid(const void* kern, size_t smem, int64_t want) {
    // occupancy per (kernel, dynamic smem, device), cached: keeps the per-call host work small
    struct Key {
        const void* k;
        size_t smem;
        int dev;
        int per_sm;
    };
    static thread_local Key cache[8];
    static thread_local int n_cache = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = -1;
    for (int i = 0; i < n_cache; ++i)
        if (cache[i].k == kern && cache[i].smem == smem && cache[i].dev == dev) per_sm = cache[i].per_sm;
    if (per_sm < 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, COOP_THREADS, smem) !=
            cudaSuccess)
            per_sm = 0;
        cache[n_cache % 8] = Key{kern, smem, dev, per_sm};
        n_cache = n_cache < 8 ? n_cache + 1 : 8;
    }
    if (per_sm <= 0) return 0;
    const int64_t cap = (int64_t)per_sm * num_sms();
    return (int)std::max<int64_t>(1, std::min<int64_t>({cap, want, (int64_t)GMAX_BLOCKS}));
}

int launch_adv_norm_coop(const agentrl_batch* b, double eps_std, float* adv_tok,
                         double* task_stats, int64_t* n_mask_global, uint8_t* ws, const AdvWs& w,
                         agentrl_comm comm, int32_t* d_status, cudaStream_t stream, bool compact) {
    static thread_local int coop = -1, coop_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != coop_dev) {
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        coop_dev = dev;
    }
    if (!coop) return AGENTRL_ERR_UNSUPPORTED;
    AdvParams p;
    p.T = b->T;
    p.n_traj = b->n_traj;
    p.n_groups = b->n_groups;
    p.n_tasks = b->n_tasks;
    p.n_chunks = ceil_div(b->T, WCHUNK);
    p.off = b->traj_offsets;
    p.task_id = b->task_id;
    p.group_id = b->group_id;
    p.rewards = b->rewards;
    p.mask = b->loss_mask;
    p.eps_std = eps_std;
    p.n_g = reinterpret_cast<int32_t*>(ws + w.n_g);
    p.chunk = reinterpret_cast<int32_t*>(ws + w.chunk_cnt);
    p.grp_cnt = reinterpret_cast<int32_t*>(ws + w.grp_cnt);
    p.grp_start = reinterpret_cast<int32_t*>(ws + w.grp_start);
    p.grp_fill = reinterpret_cast<int32_t*>(ws + w.grp_fill);
    p.members = reinterpret_cast<int32_t*>(ws + w.members);
    p.grp_task = reinterpret_cast<int32_t*>(ws + w.grp_task);
    p.chunk_first = reinterpret_cast<int32_t*>(ws + w.chunk_first);
    p.blk_chunk = reinterpret_cast<int32_t*>(ws + w.blk_chunk);
    p.chunk_base = reinterpret_cast<int32_t*>(ws + w.wchunk_base);
    p.blk_grp = reinterpret_cast<int32_t*>(ws + w.blk_grp);
    p.blk_part = reinterpret_cast<double*>(ws + w.blk_part);
    p.adv_hat = reinterpret_cast<double*>(ws + w.adv_hat);
    p.grp_nsq = reinterpret_cast<double*>(ws + w.grp_nsq);
    p.stats = reinterpret_cast<double*>(ws + w.stats);
    p.meta = reinterpret_cast<int64_t*>(ws + w.meta);
    p.d_status = d_status;
    p.adv_tok = adv_tok;
    p.idx = reinterpret_cast<int32_t*>(ws + w.idx);
    p.adv_c = reinterpret_cast<float*>(ws + w.adv_c);
    p.task_stats_out = task_stats;
    p.n_mask_global_out = n_mask_global;
    p.compact = compact ? 1 : 0;
    const size_t smem = sizeof(double) * 2 * (size_t)std::max(1, b->n_tasks) +
                        (compact ? (size_t)NWARPS * WCHUNK * 8 : 0);
    if (smem > 96 * 1024) return AGENTRL_ERR_UNSUPPORTED;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute((const void*)k_adv_coop_all,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute((const void*)k_adv_coop_apply,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        attr = true;
    }
    const int64_t want = std::max<int64_t>({ceil_div(p.n_chunks, NWARPS),
                                            ceil_div(p.n_traj, COOP_THREADS),
                                            ceil_div(p.n_groups, COOP_THREADS), 1});
    void* args[] = {&p};
    if (!comm) {
        const int grid = coop_grid((const void*)k_adv_coop_all, smem, want);
        if (!grid) return AGENTRL_ERR_UNSUPPORTED;
        ProfScope ps(KID_STATS, stream);
        AG_CUDA(cudaLaunchCooperativeKernel((const void*)k_adv_coop_all, grid, COOP_THREADS, args,
                                            smem, stream));
        count_launch();
        return AGENTRL_OK;
    }
    const int grid = coop_grid((const void*)k_adv_coop_stats, 0, want);
    if (!grid) return AGENTRL_ERR_UNSUPPORTED;
    {
        ProfScope ps(KID_STATS, stream);
        AG_CUDA(cudaLaunchCooperativeKernel((const void*)k_adv_coop_stats, grid, COOP_THREADS, args,
                                            0, stream));
        count_launch();
    }
    int rc = comm_allreduce_f64(comm, p.stats, (size_t)3 * b->n_tasks + 1, stream);
    if (rc != AGENTRL_OK) return rc;
    ProfScope ps(KID_APPLY, stream);
    // same grid as the stats launch: phase C reuses its contiguous chunk partition
    k_adv_coop_apply<<<grid, COOP_THREADS, smem, stream>>>(p);
    count_launch();
    AG_CUDA(cudaGetLastError());
    return AGENTRL_OK;
}

int debug_adv_phase_ns(unsigned long long* host8) {
    return cudaMemcpyFromSymbol(host8, g_adv_phase_ns, sizeof(unsigned long long) * 8) ==
                   cudaSuccess
               ? AGENTRL_OK
               : AGENTRL_ERR_CUDA;
}

}  // namespace agentrl
