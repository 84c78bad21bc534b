// adv_norm.cu -- part 1 of the hot path: GRPO group advantage followed by
// the task advantage normalization of sec 3.2 Eq.1, on device.
//
//   K1 k_count   token-parallel (4096 tokens / block, 16 B mask loads): masked-token count
//                per trajectory n_g (integer atomics -> exact), per-chunk counts for the
//                compaction, group sizes K_j.
//   K2 k_stats   one block: chunk/group scans, group member lists (sorted -> deterministic),
//                A_hat_g in fp64 (exact-equal rule, population std, eps floor), validation,
//                per-task (N_i, S_i = sum n_g A_hat_g, Q_i = sum n_g A_hat_g^2) with a fixed-order
//                block reduction.
//   C1           all-reduce of the 3*n_tasks doubles over NCCL (multi-GPU only).
//   K3 k_apply   token-parallel: mu_i = S_i/N_i, sigma_i = sqrt(max(Q_i/N_i - mu_i^2, 0)),
//                A_tilde = (A_hat - mu)/max(sigma, eps) -> adv_tok[t] (0 on unmasked tokens),
//                stable compaction idx[] and compacted advantages adv_c[] for part 2.
//
// HBM traffic per token: 1 B mask (read twice: K1, K3) + 4 B adv + 4+4 B compaction writes on
// masked tokens; per trajectory ~40 B.  The kernels are launch-latency bound at the paper's
// batch sizes.
#include <cuda_runtime.h>
#include <stdlib.h>

#include <algorithm>

#include "internal.h"

// the cooperative kernels (adv_coop.cu) unless built with -DAGENTRL_ADV_COOP=0; the 3-kernel path
// below also serves devices without cooperative launch
#ifndef AGENTRL_ADV_COOP
#define AGENTRL_ADV_COOP 1
#endif

namespace agentrl {

__device__ __forceinline__ int32_t find_traj(const int64_t* __restrict__ off, int32_t n_traj,
                                             int64_t t) {
    // last g with off[g] <= t  (upper_bound(t) - 1), clamped into [0, n_traj-1]
    int32_t lo = 0, hi = n_traj;  // search in off[0..n_traj]
    while (hi - lo > 1) {
        int32_t mid = (lo + hi) >> 1;
        if (off[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo < n_traj ? lo : n_traj - 1;
}

__device__ __forceinline__ void load_mask16(const uint8_t* __restrict__ mask, int64_t T,
                                            int64_t t0, uint8_t (&m)[16]) {
    if (t0 + 16 <= T && (reinterpret_cast<uintptr_t>(mask + t0) & 15) == 0) {
        uint4 v = __ldg(reinterpret_cast<const uint4*>(mask + t0));
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
#pragma unroll
        for (int i = 0; i < 16; ++i) m[i] = b[i];
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) m[i] = (t0 + i < T) ? mask[t0 + i] : 0;
    }
}

// exclusive block scan of one int per thread (blockDim.x = 256); returns the block total
__device__ int32_t block_exscan_256(int32_t v, int32_t* s_warp, int32_t& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int32_t w = lane < 8 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < 8) s_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const int32_t warp_off = wid > 0 ? s_warp[wid - 1] : 0;
    total = s_warp[7];
    __syncthreads();
    return warp_off + x - v;
}

// ---------------------------------------------------------------------------- K1
__global__ void __launch_bounds__(CHUNK_THREADS)
    k_count(int64_t T, int32_t n_traj, int32_t n_groups, int32_t n_tasks,
            const int64_t* __restrict__ off, const int32_t* __restrict__ group_id,
            const int32_t* __restrict__ task_id, const uint8_t* __restrict__ mask,
            int32_t* __restrict__ n_g, int32_t* __restrict__ chunk_cnt,
            int32_t* __restrict__ grp_cnt) {
    __shared__ int32_t s_warp[8];
    const int64_t t0 = (int64_t)blockIdx.x * CHUNK_TOKENS + threadIdx.x * 16;
    uint8_t m[16];
    load_mask16(mask, T, t0, m);
    int32_t mine = 0;
    if (t0 < T && n_traj > 0) {
        int32_t g = find_traj(off, n_traj, t0);
        int64_t end = off[g + 1];
        int32_t c = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int64_t t = t0 + i;
            if (t >= T) break;
            while (t >= end && g + 1 < n_traj) {
                if (c) atomicAdd(&n_g[g], c);
                c = 0;
                ++g;
                end = off[g + 1];
            }
            const int32_t b = m[i] != 0;
            c += b;
            mine += b;
        }
        if (c) atomicAdd(&n_g[g], c);
    }
    int32_t total;
    block_exscan_256(mine, s_warp, total);
    if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = total;
    // group sizes K_j (grid-stride over trajectories); a member with an invalid group or task
    // id is left out exactly as k_stats leaves it out of the member lists (else K_j would count
    // member slots k_stats never fills)
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_traj;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = group_id[g], i = task_id[g];
        if (j >= 0 && j < n_groups && i >= 0 && i < n_tasks) atomicAdd(&grp_cnt[j], 1);
    }
}

// ---------------------------------------------------------------------------- K2
constexpr int STATS_THREADS = 1024;

__device__ __forceinline__ double block_sum_f64(double v, double* s_red) {
    // fixed-order reduction: warp tree, then warp 0 over the 32 warp sums
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) s_red[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < (int)(blockDim.x >> 5) ? s_red[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

__device__ int64_t block_exscan_i32_inplace(int32_t* a, int64_t n, int64_t* s_tmp) {
    // exclusive scan of a[0..n) in place by one block; returns total.  Sequential per-thread
    // segments + scan of segment sums (deterministic).
    const int64_t per = (n + blockDim.x - 1) / blockDim.x;
    const int64_t lo = min(n, (int64_t)threadIdx.x * per), hi = min(n, lo + per);
    int64_t s = 0;
    for (int64_t i = lo; i < hi; ++i) s += a[i];
    s_tmp[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t run = 0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
            int64_t x = s_tmp[i];
            s_tmp[i] = run;
            run += x;
        }
        s_tmp[blockDim.x] = run;
    }
    __syncthreads();
    int64_t run = s_tmp[threadIdx.x];
    for (int64_t i = lo; i < hi; ++i) {
        int32_t x = a[i];
        a[i] = (int32_t)run;
        run += x;
    }
    const int64_t total = s_tmp[blockDim.x];
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(STATS_THREADS)
    k_stats(int64_t T, int32_t n_traj, int32_t n_groups, int32_t n_tasks, int64_t n_chunks,
            const int64_t* __restrict__ off, const int32_t* __restrict__ task_id,
            const int32_t* __restrict__ group_id, const float* __restrict__ rewards,
            double eps_std, const int32_t* __restrict__ n_g, int32_t* chunk_cnt /*->base*/,
            int32_t* grp_cnt, int32_t* grp_start, int32_t* grp_fill, int32_t* members,
            double* __restrict__ adv_hat, double* __restrict__ stats, int64_t* meta,
            int32_t* d_status) {
    __shared__ int64_t s_tmp[STATS_THREADS + 1];
    __shared__ double s_red[32];
    __shared__ int32_t s_status;
    if (threadIdx.x == 0) s_status = 0;
    __syncthreads();

    // 1. chunk counts -> exclusive bases; local masked count
    const int64_t n_mask_local = block_exscan_i32_inplace(chunk_cnt, n_chunks, s_tmp);
    // 2. group starts
    for (int64_t j = threadIdx.x; j < n_groups; j += blockDim.x) grp_start[j] = grp_cnt[j];
    __syncthreads();
    block_exscan_i32_inplace(grp_start, n_groups, s_tmp);
    // 3. scatter members (slot order is racy; sorted below)
    int32_t st = 0;
    for (int64_t g = threadIdx.x; g < n_traj; g += blockDim.x) {
        const int32_t j = group_id[g];
        const int32_t i = task_id[g];
        if (j < 0 || j >= n_groups || i < 0 || i >= n_tasks) {
            st |= AGENTRL_ST_GROUP_SPANS_TASKS;
            continue;
        }
        const int32_t slot = atomicAdd(&grp_fill[j], 1);
        members[grp_start[j] + slot] = (int32_t)g;
    }
    // offsets validation
    if (threadIdx.x == 0 && n_traj >= 0 && (off[0] != 0 || off[n_traj] != T))
        st |= AGENTRL_ST_BAD_OFFSETS;
    for (int64_t g = threadIdx.x; g < n_traj; g += blockDim.x)
        if (off[g + 1] < off[g]) st |= AGENTRL_ST_BAD_OFFSETS;
    __syncthreads();
    // 4. per group: sort members, GRPO advantage (R1 population std, R2 exact rule)
    for (int64_t j = threadIdx.x; j < n_groups; j += blockDim.x) {
        const int32_t s0 = grp_start[j], K = grp_cnt[j];
        int32_t* mb = members + s0;
        for (int a = 1; a < K; ++a) {  // insertion sort -> trajectory order
            int32_t x = mb[a];
            int b = a - 1;
            while (b >= 0 && mb[b] > x) {
                mb[b + 1] = mb[b];
                --b;
            }
            mb[b + 1] = x;
        }
        if (K == 0) continue;
        if (K == 1) st |= AGENTRL_ST_GROUP_TOO_SMALL;
        const int32_t task0 = task_id[mb[0]];
        double sum = 0.0, rmax = rewards[mb[0]], rmin = rmax;
        for (int a = 0; a < K; ++a) {
            const double r = rewards[mb[a]];
            if (task_id[mb[a]] != task0) st |= AGENTRL_ST_GROUP_SPANS_TASKS;
            sum += r;
            rmax = fmax(rmax, r);
            rmin = fmin(rmin, r);
        }
        if (rmax == rmin) {
            for (int a = 0; a < K; ++a) adv_hat[mb[a]] = 0.0;
            continue;
        }
        const double mean = sum / (double)K;
        double ss = 0.0;
        for (int a = 0; a < K; ++a) {
            const double dlt = (double)rewards[mb[a]] - mean;
            ss += dlt * dlt;
        }
        const double sd = sqrt(ss / (double)K);
        const double den = sd > eps_std ? sd : eps_std;
        for (int a = 0; a < K; ++a) adv_hat[mb[a]] = ((double)rewards[mb[a]] - mean) / den;
    }
    if (st) atomicOr(&s_status, st);
    __syncthreads();
    // 5. per-task raw moments over the token set: N_i, S_i, Q_i
    for (int32_t i = 0; i < n_tasks; ++i) {
        double N = 0.0, S = 0.0, Q = 0.0;
        for (int64_t g = threadIdx.x; g < n_traj; g += blockDim.x) {
            if (task_id[g] != i) continue;
            const double n = (double)n_g[g];
            const double a = adv_hat[g];
            N += n;
            S += n * a;
            Q += n * a * a;
        }
        N = block_sum_f64(N, s_red);
        S = block_sum_f64(S, s_red);
        Q = block_sum_f64(Q, s_red);
        if (threadIdx.x == 0) {
            stats[3 * i + 0] = N;
            stats[3 * i + 1] = S;
            stats[3 * i + 2] = Q;
        }
    }
    {  // groups with members (G of the GRPO group mean), local
        double nz = 0.0;
        for (int64_t j = threadIdx.x; j < n_groups; j += blockDim.x) nz += grp_cnt[j] > 0 ? 1.0 : 0.0;
        nz = block_sum_f64(nz, s_red);
        if (threadIdx.x == 0) stats[3 * n_tasks] = nz;
    }
    if (threadIdx.x == 0) {
        meta[0] = n_mask_local;
        if (s_status) atomicOr(d_status, s_status);
    }
}

// ---------------------------------------------------------------------------- K3
__global__ void __launch_bounds__(CHUNK_THREADS)
    k_apply(int64_t T, int32_t n_traj, int32_t n_tasks, const int64_t* __restrict__ off,
            const int32_t* __restrict__ task_id, const uint8_t* __restrict__ mask,
            const double* __restrict__ adv_hat, const double* __restrict__ stats, double eps_std,
            const int32_t* __restrict__ chunk_base, float* __restrict__ adv_tok,
            int32_t* __restrict__ idx, float* __restrict__ adv_c, double* task_stats_out,
            int64_t* n_mask_global_out, int64_t* meta, int32_t* d_status) {
    __shared__ int32_t s_warp[8];
    const int64_t t0 = (int64_t)blockIdx.x * CHUNK_TOKENS + threadIdx.x * 16;
    uint8_t m[16];
    load_mask16(mask, T, t0, m);
    int32_t mine = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) mine += m[i] != 0;
    int32_t total;
    const int32_t pos0 = chunk_base[blockIdx.x] + block_exscan_256(mine, s_warp, total);

    if (t0 < T && n_traj > 0) {
        int32_t g = find_traj(off, n_traj, t0);
        int64_t end = off[g + 1];
        int32_t cur_g = -1;
        float at = 0.f;
        int32_t pos = pos0;
        float outv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int64_t t = t0 + i;
            outv[i] = 0.f;
            if (t >= T) continue;
            while (t >= end && g + 1 < n_traj) {
                ++g;
                end = off[g + 1];
            }
            if (m[i]) {
                if (g != cur_g) {  // Eq.1 for this trajectory
                    cur_g = g;
                    const int32_t ti = task_id[g];
                    double a = 0.0;
                    if (ti >= 0 && ti < n_tasks) {
                        const double N = stats[3 * ti], S = stats[3 * ti + 1],
                                     Q = stats[3 * ti + 2];
                        const double mu = N > 0.0 ? S / N : 0.0;
                        const double var = N > 0.0 ? fmax(Q / N - mu * mu, 0.0) : 0.0;
                        const double sd = sqrt(var);
                        a = (adv_hat[g] - mu) / (sd > eps_std ? sd : eps_std);
                    }
                    at = (float)a;
                }
                outv[i] = at;
                idx[pos] = (int32_t)t;
                adv_c[pos] = at;
                ++pos;
            }
        }
        if (t0 + 16 <= T && (reinterpret_cast<uintptr_t>(adv_tok + t0) & 15) == 0) {
            float4* o4 = reinterpret_cast<float4*>(adv_tok + t0);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                o4[i] = make_float4(outv[4 * i], outv[4 * i + 1], outv[4 * i + 2],
                                    outv[4 * i + 3]);
        } else {
            for (int i = 0; i < 16; ++i)
                if (t0 + i < T) adv_tok[t0 + i] = outv[i];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        // global outputs: task_stats (N, mu, sigma) and N = sum_i N_i
        double nsum = 0.0;
        for (int32_t i = threadIdx.x; i < n_tasks; i += 32) {
            const double N = stats[3 * i], S = stats[3 * i + 1], Q = stats[3 * i + 2];
            const double mu = N > 0.0 ? S / N : 0.0;
            const double sd = N > 0.0 ? sqrt(fmax(Q / N - mu * mu, 0.0)) : 0.0;
            if (task_stats_out) {
                task_stats_out[3 * i] = N;
                task_stats_out[3 * i + 1] = mu;
                task_stats_out[3 * i + 2] = sd;
            }
            nsum += N;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nsum += __shfl_down_sync(0xffffffffu, nsum, o);
        if (threadIdx.x == 0) {
            const int64_t n = (int64_t)nsum;
            meta[1] = n;
            meta[2] = (int64_t)stats[3 * n_tasks];
            if (n_mask_global_out) *n_mask_global_out = n;
            if (n == 0) atomicOr(d_status, AGENTRL_ST_NO_TOKENS);
        }
    }
}

// zero-token batch: still define the outputs
__global__ void k_adv_empty(int32_t n_tasks, double* task_stats_out, int64_t* n_mask_global_out,
                            int64_t* meta, const double* stats, int32_t* d_status) {
    if (threadIdx.x == 0) {
        double nsum = 0.0;
        for (int32_t i = 0; i < n_tasks; ++i) {
            const double N = stats[3 * i], S = stats[3 * i + 1], Q = stats[3 * i + 2];
            const double mu = N > 0.0 ? S / N : 0.0;
            if (task_stats_out) {
                task_stats_out[3 * i] = N;
                task_stats_out[3 * i + 1] = mu;
                task_stats_out[3 * i + 2] = N > 0.0 ? sqrt(fmax(Q / N - mu * mu, 0.0)) : 0.0;
            }
            nsum += N;
        }
        meta[0] = 0;
        meta[1] = (int64_t)nsum;
        meta[2] = (int64_t)stats[3 * n_tasks];
        if (n_mask_global_out) *n_mask_global_out = (int64_t)nsum;
        if (nsum == 0.0) atomicOr(d_status, AGENTRL_ST_NO_TOKENS);
    }
}

// ---------------------------------------------------------------------------- host
AdvWs plan_adv(int64_t T, int32_t n_traj, int32_t n_groups, int32_t n_tasks, size_t base) {
    WsPlan p;
    p.off = base;
    AdvWs w;
    const int64_t n_chunks = ceil_div(T, 512);  // warp chunks (cooperative path; >= legacy)
    // the int32 scratch that must start zeroed is contiguous: n_g, grp_cnt, grp_fill
    w.n_g = p.take(sizeof(int32_t) * (size_t)(n_traj + 1));
    w.grp_cnt = p.take(sizeof(int32_t) * (size_t)(n_groups + 1));
    w.grp_fill = p.take(sizeof(int32_t) * (size_t)(n_groups + 1));
    w.grp_lo = p.take(sizeof(uint32_t) * (size_t)(n_groups + 1));  // (zeroed with the above)
    w.grp_hi = p.take(sizeof(uint32_t) * (size_t)(n_groups + 1));
    w.grp_flag = p.take(sizeof(int32_t) * 4);
    w.chunk_cnt = p.take(sizeof(int32_t) * (size_t)(n_chunks + 1));
    w.chunk_base = w.chunk_cnt;  // scanned in place
    w.grp_start = p.take(sizeof(int32_t) * (size_t)(n_groups + 1));
    w.members = p.take(sizeof(int32_t) * (size_t)(n_traj + 1));
    w.adv_hat = p.take(sizeof(double) * (size_t)(n_traj + 1));
    w.grp_task = p.take(sizeof(int32_t) * (size_t)(n_groups + 1));
    w.grp_nsq = p.take(sizeof(double) * 3 * (size_t)(n_groups + 1));
    w.chunk_first = p.take(sizeof(int32_t) * (size_t)(n_chunks + 1));
    w.wchunk_base = p.take(sizeof(int32_t) * (size_t)(n_chunks + 1));
    w.chunk_gbase = p.take(sizeof(int32_t) * (size_t)(n_chunks + 1));
    w.blk_cnt = p.take(sizeof(int32_t) * ((size_t)n_traj + 2049));
    w.lanebits = p.take(sizeof(uint16_t) * ((size_t)n_chunks * 32 + 32));
    w.blk_chunk = p.take(sizeof(int32_t) * 2048);
    w.blk_grp = p.take(sizeof(int32_t) * 2048);
    w.blk_part = p.take(sizeof(double) * 3 * 2048 * (size_t)std::max(n_tasks, 1));
    w.stats = p.take(sizeof(double) * (size_t)(3 * n_tasks + 1));
    w.meta = p.take(sizeof(int64_t) * 4);
    w.idx = p.take(sizeof(int32_t) * (size_t)(T + 1));
    w.adv_c = p.take(sizeof(float) * (size_t)(T + 1));
    w.total = p.off;
    return w;
}

int launch_adv_norm(const agentrl_batch* b, double eps_std, float* adv_tok, double* task_stats,
                    int64_t* n_mask_global, uint8_t* ws, const AdvWs& w, agentrl_comm comm,
                    int32_t* d_status, cudaStream_t stream, bool compact) {
    if (AGENTRL_ADV_COOP) {  // build switch; 0: always the 3-kernel path below
        int rc = launch_adv_norm_coop(b, eps_std, adv_tok, task_stats, n_mask_global, ws, w, comm,
                                      d_status, stream, compact);
        if (rc != AGENTRL_ERR_UNSUPPORTED) return rc;
    }
    const int64_t T = b->T;
    const int64_t n_chunks = ceil_div(T, CHUNK_TOKENS);
    int32_t* n_g = reinterpret_cast<int32_t*>(ws + w.n_g);
    int32_t* grp_cnt = reinterpret_cast<int32_t*>(ws + w.grp_cnt);
    int32_t* grp_fill = reinterpret_cast<int32_t*>(ws + w.grp_fill);
    int32_t* chunk = reinterpret_cast<int32_t*>(ws + w.chunk_cnt);
    int32_t* grp_start = reinterpret_cast<int32_t*>(ws + w.grp_start);
    int32_t* members = reinterpret_cast<int32_t*>(ws + w.members);
    double* adv_hat = reinterpret_cast<double*>(ws + w.adv_hat);
    double* stats = reinterpret_cast<double*>(ws + w.stats);
    int64_t* meta = reinterpret_cast<int64_t*>(ws + w.meta);
    int32_t* idx = reinterpret_cast<int32_t*>(ws + w.idx);
    float* adv_c = reinterpret_cast<float*>(ws + w.adv_c);

    // zero n_g, grp_cnt, grp_fill (contiguous) in one memset; stats/meta in another
    AG_CUDA(cudaMemsetAsync(ws + w.n_g, 0, w.chunk_cnt - w.n_g, stream));
    AG_CUDA(cudaMemsetAsync(ws + w.stats, 0, (w.meta + 4 * sizeof(int64_t)) - w.stats, stream));
    if (n_chunks > 0) {
        ProfScope ps(KID_COUNT, stream);
        k_count<<<(unsigned)n_chunks, CHUNK_THREADS, 0, stream>>>(
            T, b->n_traj, b->n_groups, b->n_tasks, b->traj_offsets, b->group_id, b->task_id,
            b->loss_mask, n_g, chunk, grp_cnt);
        count_launch();
    }
    {
    ProfScope ps(KID_STATS, stream);
    k_stats<<<1, STATS_THREADS, 0, stream>>>(T, b->n_traj, b->n_groups, b->n_tasks, n_chunks,
                                             b->traj_offsets, b->task_id, b->group_id, b->rewards,
                                             eps_std, n_g, chunk, grp_cnt, grp_start, grp_fill,
                                             members, adv_hat, stats, meta, d_status);
    }
    count_launch();
    AG_CUDA(cudaGetLastError());
    if (comm) {
        int rc = comm_allreduce_f64(comm, stats, (size_t)3 * b->n_tasks + 1, stream);
        if (rc != AGENTRL_OK) return rc;
    }
    ProfScope ps_apply(KID_APPLY, stream);
    if (n_chunks > 0) {
        k_apply<<<(unsigned)n_chunks, CHUNK_THREADS, 0, stream>>>(
            T, b->n_traj, b->n_tasks, b->traj_offsets, b->task_id, b->loss_mask, adv_hat, stats,
            eps_std, chunk, adv_tok, idx, adv_c, task_stats, n_mask_global, meta, d_status);
    } else {
        k_adv_empty<<<1, 32, 0, stream>>>(b->n_tasks, task_stats, n_mask_global, meta, stats,
                                          d_status);
    }
    count_launch();
    AG_CUDA(cudaGetLastError());
    return AGENTRL_OK;
}

}  // namespace agentrl
