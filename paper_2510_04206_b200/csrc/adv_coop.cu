// adv_coop.cu -- part 1 (GRPO group advantage P:1263, then task advantage normalization,
// sec 3.2 Eq.1) as ONE cooperative persistent kernel with grid-wide barriers
// between its phases (two launches around the NCCL all-reduce when a communicator is given).
//
// Token streaming (phases A and C).  Each block owns a contiguous range of 512-token warp
// chunks; warp w takes chunks w, w+8, ... of it.  The mask bytes reach shared memory through a
// per-warp ring of RING slots filled by 1-D bulk copies (cp.async.bulk, one 512 B copy per
// chunk, completion on an mbarrier), so every warp keeps RING-1 chunks in flight without
// spending registers.  Trajectory offsets are staged per block in windows of 64 chunks.
//   phase A  per-trajectory masked counts n_g: each lane counts its 16 tokens, a segmented
//            warp scan sums the lanes of one trajectory, and one lane per trajectory adds to a
//            shared counter (no same-address atomics inside a warp); per-chunk counts.
//   phase C  adv_tok[t] = mask ? A~_g(t) : 0 with the staged A~ of the window; the 16 values of
//            each lane go through a swizzled shared-memory transpose so that the stores are
//            512 B contiguous per warp instruction; optional stable compaction idx[] / adv_c[].
//
// Two drivers:
//   small  (n_traj <= 2048, n_groups <= 512; every BASELINE config): every block streams and
//          holds the whole trajectory table in smem; A + the A^ of its groups + its partial
//          moments -> ONE grid barrier -> moments (identical in every block) -> C.  Per-block
//          trajectory counts go to disjoint slots (index g + block): no zeroing pass.
//   large  three launches: (1) popcount stream (phase A: per-lane mask bits, chunk counts, K_j,
//          group bounds, the chunk -> first-trajectory table); (2) cooperative statistics:
//          chunk bases | n_g from prefix differences at the trajectory bounds | [B1 K_j scans |
//          B2 member lists: skipped when every group is one contiguous run of <= 16] | B3 group
//          advantages | B4 task moments by the last block (ticket); (3) apply (phase C) in
//          8-chunk warp units, a programmatic dependent launch of (2) without a communicator.
//          Measured and dropped: loading the first n_g bounds before the
//          grid barrier (4 us slower: the barrier waits for the slowest block's extra loads);
//          writing the all-zero sectors of adv_tok from the popcount launch (its strided
//          stores took it from 30 to 135 us, and the apply did not get faster: the L2's
//          deferred write-back of those lines lands in the apply anyway).
// Every floating-point reduction has a fixed order: results are bitwise run-to-run
// deterministic.
#include <cooperative_groups.h>
#include <algorithm>
#include <climits>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace agentrl {

constexpr int COOP_THREADS = 256;
constexpr int NWARPS = COOP_THREADS / 32;
constexpr int GMAX_BLOCKS = 2048;  // cap on the cooperative grid (per-block scratch arrays)
constexpr int WCHUNK = 512;        // tokens per warp chunk (32 lanes x 16 tokens)
#ifndef ADV_RING
#define ADV_RING 8
#endif
#ifndef ADV_LDGSTS
#define ADV_LDGSTS 1  // ring filled by per-lane cp.async (1) or one cp.async.bulk per chunk (0)
#endif
#ifndef AGENTRL_ADV_SMALL
#define AGENTRL_ADV_SMALL 1  // 0: the large driver for every batch
#endif
#ifndef ADV_LARGE_MINB
#define ADV_LARGE_MINB 2  // resident blocks per SM the large driver's register budget is cut for
#endif
constexpr int RING = ADV_RING;          // bulk-copy slots per warp
constexpr int WIN_CHUNKS = 8 * NWARPS;  // warp chunks per offset-staging window (large path)
constexpr int WIN_TRAJ = 2048;          // trajectories a block stages at once (more: windows,
                                        // then global lookups)
#ifndef ADV_KC_CAP
#define ADV_KC_CAP 2048
#endif
constexpr int KC_CAP = ADV_KC_CAP;      // chunks per staged window (chunk -> trajectory table);
                                        // a block with more chunks stages 64-chunk windows
constexpr int SMALL_TRAJ = 2048;        // small driver: all offsets staged in every block
constexpr int SMALL_GROUPS = 512;
constexpr int CT_CAP = 1024;   // small driver: chunk totals kept in smem up to this many chunks
constexpr int TASK_BATCH = 16;  // tasks reduced per barrier in the per-block partials
constexpr int REG_K = 16;       // groups up to this size are handled in registers (phase B3)

// phase timestamps of the last cooperative launch (block 0, after each grid barrier), read by
// agentrl_debug_adv_phase_ns(); 8 x %globaltimer ns
__device__ unsigned long long g_adv_phase_ns[8];
__device__ __forceinline__ void phase_mark(int i, unsigned blk = 0) {
    if (blockIdx.x == blk && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_adv_phase_ns[i] = t;
    }
}

// dynamic shared memory layout (byte offsets), identical on host and device
struct Lay {
    uint32_t ring, rwarp, bars, ostage, soff, srel, saux, skc, stask, cidx, cadv;
    uint32_t sgid, stid, srew, sah, gflag, gtask, glist, gfirst, glast, sct;  // small driver
    uint32_t total;
};
__host__ __device__ inline uint32_t lay_take(uint32_t& o, uint32_t bytes) {
    o = (o + 127u) & ~127u;
    const uint32_t r = o;
    o += bytes;
    return r;
}
__host__ __device__ inline Lay make_lay(int n_tasks, bool compact, bool small, int n_traj,
                                        int n_groups) {
    Lay L;
    uint32_t o = 0;
    L.bars = lay_take(o, NWARPS * RING * 8);
    const uint32_t stream_begin = (o + 127u) & ~127u;
    L.rwarp = RING * (uint32_t)WCHUNK;
    L.ring = lay_take(o, NWARPS * L.rwarp);
    L.ostage = lay_take(o, NWARPS * WCHUNK * 4);
    L.cidx = lay_take(o, compact ? NWARPS * WCHUNK * 4 : 0);
    L.cadv = lay_take(o, compact ? NWARPS * WCHUNK * 4 : 0);
    const uint32_t stream_end = o;
    const int nst = small ? n_traj : WIN_TRAJ;
    L.soff = lay_take(o, small ? 8u * (uint32_t)(n_traj + 1) : 0u);  // all offsets (small)
    L.srel = lay_take(o, 4u * (uint32_t)(nst + 1));
    L.saux = lay_take(o, 4u * (uint32_t)(nst + 1));
    L.skc = lay_take(o, 4u * KC_CAP);
    L.stask = lay_take(o, 16u * (uint32_t)(n_tasks > 0 ? n_tasks : 1));
    // small driver: the whole trajectory table and per-group scratch (every block streams)
    const uint32_t nt = small ? (uint32_t)n_traj : 0u, ng = small ? (uint32_t)n_groups + 1 : 0u;
    L.sgid = lay_take(o, 4u * nt);
    L.stid = lay_take(o, 4u * nt);
    L.srew = lay_take(o, 4u * nt);
    L.sah = lay_take(o, 8u * nt);
    L.gflag = lay_take(o, 4u * ng);
    L.gtask = lay_take(o, 4u * ng);
    L.glist = lay_take(o, 4u * ng);
    L.gfirst = lay_take(o, 4u * ng);  // first / last member of each group (scan bounds)
    L.glast = lay_take(o, 4u * ng);
    L.sct = lay_take(o, small ? 4u * CT_CAP : 0u);  // per-chunk masked totals of the block
    (void)stream_begin;
    (void)stream_end;
    L.total = o;
    return L;
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
    uint32_t *grp_lo, *grp_hi;  // large driver: ~(first member) and last member + 1 of each
                                // group (atomicMax from zero)
    int32_t* grp_flag;          // [0] != 0: some group is not one run of <= REG_K trajectories
    int32_t *blk_chunk, *blk_grp;  // per-block masked / member totals
    int32_t* chunk_base;           // [n_chunks] compaction base of each chunk within its block
    int32_t* chunk_gbase;          // [n_chunks] global compaction base (large driver)
    int32_t g_stats;               // grid of the statistics launch (its per-block arrays)
    int32_t* blk_cnt;              // small driver: per-block trajectory counts at [g + block]
    uint16_t* lanebits;            // large driver: the 16-token mask bits of each lane of each
                                   // chunk, [n_chunks * 32] (phase A writes them; phase C and
                                   // the trajectory-bound prefix counts read them instead of
                                   // the mask: 1 bit per token instead of 1 byte)
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
    Lay lay;
};

// ------------------------------------------------------------------ small helpers
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
// k in [lo, hi) with s[k] <= t < s[k+1] (clamped to lo / hi - 1)
__device__ __forceinline__ int32_t smem_find_in(const int64_t* s, int32_t lo, int32_t hi, int64_t t) {
    while (hi - lo > 1) {
        const int32_t mid = (lo + hi) >> 1;
        if (s[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo;
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
// the 16 mask bytes of lane `lane` of chunk c, zero past T (direct loads; tail / misaligned)
__device__ __forceinline__ uint4 mask_direct(const AdvParams& p, int64_t c, int lane) {
    const int64_t t0 = c * WCHUNK + lane * 16;
    if (t0 + 16 <= p.T && (reinterpret_cast<uintptr_t>(p.mask + t0) & 15) == 0)
        return __ldg(reinterpret_cast<const uint4*>(p.mask + t0));
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    for (int i = 0; i < 16; ++i)
        if (t0 + i < p.T) w[i >> 2] |= (uint32_t)p.mask[t0 + i] << (8 * (i & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
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
        int32_t w = lane < NWARPS ? s_w[lane] : 0;
#pragma unroll
        for (int o = 1; o < NWARPS; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NWARPS) s_w[lane] = w;
    }
    __syncthreads();
    const int32_t base = wid > 0 ? s_w[wid - 1] : 0;
    total = s_w[NWARPS - 1];
    __syncthreads();
    return base + x - v;
}
// in-place exclusive scan of a[0..n) by the block (contiguous per-thread segments); total out
__device__ int32_t coop_block_scan_array(int32_t* a, int64_t n, int32_t* s_w) {
    const int64_t per = (n + COOP_THREADS - 1) / COOP_THREADS;
    const int64_t lo = min(n, (int64_t)threadIdx.x * per), hi = min(n, lo + per);
    int32_t s = 0;
    for (int64_t i = lo; i < hi; ++i) s += a[i];
    int32_t total;
    int32_t run = coop_block_exscan(s, s_w, total);
    for (int64_t i = lo; i < hi; ++i) {
        const int32_t v = a[i];
        a[i] = run;
        run += v;
    }
    __syncthreads();
    return total;
}

// balanced contiguous partition of [0, n) over G blocks
__device__ __forceinline__ int64_t part_lo(int64_t n, int64_t b, int64_t G) { return n * b / G; }
// block owning item j under part_lo
__device__ __forceinline__ int64_t part_owner(int64_t n, int64_t j, int64_t G) {
    return ((j + 1) * G + n - 1) / n - 1;
}
// exclusive prefix over blocks of a per-block int array, computed by every block into smem
__device__ void block_prefix_smem(const int32_t* __restrict__ blk, int64_t G, int32_t* s_pre,
                                  int32_t* s_w) {
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

// ------------------------------------------------------------------ per-warp bulk-copy ring
struct WarpRing {
    uint8_t* buf;   // RING x WCHUNK bytes
    uint64_t* bar;  // RING mbarriers
    uint32_t par;   // parity of each slot's next completion
    bool on;        // mask 16 B aligned: full chunks arrive by bulk copy
};
__device__ __forceinline__ WarpRing ring_setup(const AdvParams& p, uint8_t* smem) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpRing r;
    r.buf = smem + p.lay.ring + warp * p.lay.rwarp;
    r.bar = reinterpret_cast<uint64_t*>(smem + p.lay.bars) + warp * RING;
    r.par = 0u;
    r.on = (reinterpret_cast<uintptr_t>(p.mask) & 15) == 0;
    if (lane == 0) {
        for (int s = 0; s < RING; ++s) mbar_init(&r.bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    return r;
}
__device__ __forceinline__ bool chunk_full(const AdvParams& p, int64_t c) {
    return (c + 1) * WCHUNK <= p.T;
}
// lane 0: start the copy of chunk c into `slot`
__device__ __forceinline__ void ring_issue(const AdvParams& p, WarpRing& r, int slot, int64_t c) {
    mbar_arrive_expect_tx(&r.bar[slot], WCHUNK);
    bulk_g2s(r.buf + slot * WCHUNK, p.mask + c * WCHUNK, WCHUNK, &r.bar[slot]);
}
// per-lane variant: every lane copies its own 16 bytes (cp.async, one commit group per chunk;
// a lane only ever reads its own bytes, so waiting on its own groups is enough)
__device__ __forceinline__ void lane_issue(const AdvParams& p, WarpRing& r, int slot, int64_t c,
                                           bool valid) {
    const int lane = threadIdx.x & 31;
    if (valid)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         smem_u32(r.buf + slot * WCHUNK + lane * 16)),
                     "l"(p.mask + c * WCHUNK + lane * 16)
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void lane_wait_oldest() {
    asm volatile("cp.async.wait_group %0;" ::"n"(RING - 1) : "memory");
}

// Offset staging of one window of chunks [w0, w1): trajectories [f, f + nbt) cover its
// tokens; s_rel[k] = off[f + k] - base (clamped to [0, INT_MAX]), k = 0..nbt, with base the
// window's first token, so the token loops compare 32-bit positions.  staged == false: the
// window covers more than WIN_TRAJ trajectories and uses global lookups.
struct Window {
    int32_t f, nbt;
    int64_t base;
    const int32_t* s_rel;
    bool staged;
};

// ------------------------------------------------------------------ phase C: apply
// writes the 16 values of each lane through a swizzled transpose: lane L stores its q-th
// float4 at word L*16 + 4*(q ^ ((L>>1)&3)) (conflict-free), then reads back the float4 of tokens
// i*128 + 4L (conflict-free) and stores it -- 512 contiguous bytes per warp instruction
__device__ __forceinline__ void store_transposed(const AdvParams& p, float* os, int64_t c,
                                                 const float (&v)[16], bool vec_ok) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(os + lane * 16 + 4 * (q ^ ((lane >> 1) & 3))) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    __syncwarp();
    if (vec_ok && (c + 1) * WCHUNK <= p.T) {  // a full chunk: no per-vector bounds checks
        float4* dst = reinterpret_cast<float4*>(p.adv_tok + c * WCHUNK) + lane;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int lp = (i * 128 + lane * 4) >> 4, q = lane & 3;
            dst[i * 32] = *reinterpret_cast<const float4*>(os + lp * 16 + 4 * (q ^ ((lp >> 1) & 3)));
        }
        __syncwarp();
        return;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int tok = i * 128 + lane * 4;
        const int lp = tok >> 4, q = lane & 3;
        const float4 x = *reinterpret_cast<const float4*>(os + lp * 16 + 4 * (q ^ ((lp >> 1) & 3)));
        const int64_t t = c * WCHUNK + tok;
        if (vec_ok && t + 4 <= p.T) {
            *reinterpret_cast<float4*>(p.adv_tok + t) = x;
        } else {
            if (t < p.T) p.adv_tok[t] = x.x;
            if (t + 1 < p.T) p.adv_tok[t + 1] = x.y;
            if (t + 2 < p.T) p.adv_tok[t + 2] = x.z;
            if (t + 3 < p.T) p.adv_tok[t + 3] = x.w;
        }
    }
    __syncwarp();
}

// Eq.1 from smem copies of A^ and the task ids (identical arithmetic to adv_tilde)
__device__ __forceinline__ float adv_tilde_s(const AdvParams& p, const double2* s_task,
                                             const double* ah, const int32_t* tid, int32_t g) {
    const int32_t ti = tid[g];
    return (ti >= 0 && ti < p.n_tasks) ? (float)((ah[g] - s_task[ti].x) / s_task[ti].y) : 0.f;
}
// Eq.1 for trajectory g with the block's per-task (mu, max(sigma, eps))
__device__ __forceinline__ float adv_tilde(const AdvParams& p, const double2* s_task, int32_t g) {
    const int32_t ti = p.task_id[g];
    return (ti >= 0 && ti < p.n_tasks)
               ? (float)((p.adv_hat[g] - s_task[ti].x) / s_task[ti].y)
               : 0.f;
}

// ------------------------------------------------------------------ the streaming loop
// PH 0: counting (phase A); PH 1: apply (phase C).  small: one window = the block's range,
// offsets from s_offall (all trajectories staged); else windows of WIN_CHUNKS chunks staged
// from the chunk -> first-trajectory table.
// ------------------------------------------------------------------ bit-parallel chunk code
// The 16 mask bytes of a lane -> a per-byte 0xFF/0x00 mask (4 words) and a 16-bit token mask.
struct LaneMask {
    uint32_t byte[4];  // 0xFF in every byte whose mask byte is nonzero (reading R18)
    uint32_t bits;     // bit i = token i of the lane is an assistant token
};
__device__ __forceinline__ LaneMask lane_mask(const uint4& mk) {
    const uint32_t w[4] = {mk.x, mk.y, mk.z, mk.w};
    LaneMask m;
    m.bits = 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        // high bit of each byte set iff the byte is nonzero
        const uint32_t hb = ((((w[q] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | w[q]) & 0x80808080u) >> 7;
        m.byte[q] = hb * 0xFFu;
        m.bits |= ((hb * 0x01020408u) >> 24) << (4 * q);
    }
    return m;
}

// phase A, staged window: per-trajectory masked counts of chunk c (window-relative start tc,
// first trajectory kc).  With E the exclusive prefix of the lanes' popcounts, the count below
// a boundary x is P(x) = E[x/16] + popc(bits[x/16] & low(x%16)); lane j handles the segment
// that ends at the chunk's j-th trajectory start (and adds it once: no intra-warp conflicts).
__device__ __forceinline__ int32_t count_chunk_bits(const LaneMask& m, int32_t tc, int32_t kc,
                                                    const Window& w, int32_t* s_cnt,
                                                    int32_t& chunk_total) {
    const int lane = threadIdx.x & 31;
    const int32_t pc = __popc(m.bits);
    const int32_t E = warp_incl_scan(pc) - pc;
    const int32_t total = __shfl_sync(0xffffffffu, E + pc, 31);
    int32_t prevP = 0;
    for (int32_t jb = 0;; jb += 32) {
        const int32_t kb = kc + 1 + jb + lane;  // trajectory starting at boundary jb + lane
        const int32_t b = kb < w.nbt ? w.s_rel[kb] : INT_MAX;
        const bool in = b < tc + WCHUNK;
        const int32_t nb = __popc(__ballot_sync(0xffffffffu, in));
        const int32_t x = in ? b - tc : 0;
        const int32_t o = x >> 4;
        const int32_t Eo = __shfl_sync(0xffffffffu, E, o);
        const uint32_t bo = __shfl_sync(0xffffffffu, m.bits, o);
        const int32_t P = in ? Eo + __popc(bo & ((1u << (x & 15)) - 1u)) : total;
        int32_t Pm = __shfl_up_sync(0xffffffffu, P, 1);
        if (lane == 0) Pm = prevP;
        const int32_t cnt = P - Pm;
        if (lane <= nb && cnt > 0) atomicAdd(&s_cnt[kc + jb + lane], cnt);
        if (nb < 32) break;
        prevP = __shfl_sync(0xffffffffu, P, 31);
    }
    chunk_total = total;
    return pc;
}

// phase C, staged window: the lane's 16 advantages (as bits, 0 on unmasked tokens).  Start
// from the chunk's first trajectory, then every trajectory start b inside the chunk overwrites
// the tokens at or after b (uniform loop over the chunk's few boundaries).
__device__ __forceinline__ void apply_chunk_bits(const LaneMask& m, int32_t tc, int32_t kc,
                                                 const Window& w, const int32_t* s_val,
                                                 uint32_t (&out)[16]) {
    const int lane = threadIdx.x & 31;
    const int32_t tr0 = tc + lane * 16;
    const uint32_t v0 = (uint32_t)s_val[kc];
    {  // the common case first: at most one trajectory start inside the chunk
        const int32_t kb = kc + 1 + lane;
        const int32_t b = kb < w.nbt ? w.s_rel[kb] : INT_MAX;
        const uint32_t av = kb < w.nbt ? (uint32_t)s_val[kb] : 0u;
        const uint32_t bal = __ballot_sync(0xffffffffu, b < tc + WCHUNK);
        if (bal <= 1u) {  // bal is 0 or 1: boundaries are sorted, so only lane 0 can hold one
            const int32_t rel = bal ? __shfl_sync(0xffffffffu, b, 0) - tr0 : 16;
            const uint32_t v = __shfl_sync(0xffffffffu, av, 0);
#pragma unroll
            for (int i = 0; i < 16; ++i) out[i] = (m.bits & (1u << i)) ? (i >= rel ? v : v0) : 0u;
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = v0;
    for (int32_t jb = 0;; jb += 32) {
        const int32_t kb = kc + 1 + jb + lane;
        const int32_t b = kb < w.nbt ? w.s_rel[kb] : INT_MAX;
        const uint32_t av = kb < w.nbt ? (uint32_t)s_val[kb] : 0u;
        const int32_t nb = __popc(__ballot_sync(0xffffffffu, b < tc + WCHUNK));
        for (int32_t j = 0; j < nb; ++j) {
            const int32_t rel = __shfl_sync(0xffffffffu, b, j) - tr0;
            const uint32_t v = __shfl_sync(0xffffffffu, av, j);
#pragma unroll
            for (int i = 0; i < 16; ++i) out[i] = i >= rel ? v : out[i];
        }
        if (nb < 32) break;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = (m.bits & (1u << i)) ? out[i] : 0u;
}

// resident (PH 1): the warp's chunks are still in its ring slots from phase A (same kernel,
// at most RING chunks per warp) and are not copied again.
struct NoPre {
    __device__ void operator()() const {}
};
// pre(): work run after the ring's first copies are issued (overlaps their latency)
// ah_s / tid_s (PH 1, small driver): A^ and task ids of every trajectory already in smem
template <int PH, typename Pre = NoPre>
__device__ void stream_phase(const AdvParams& p, uint8_t* smem, WarpRing& r, int64_t c_lo,
                             int64_t c_hi, bool small, const int64_t* s_offall, int32_t blk_base,
                             int32_t& warp_total, bool resident = false, Pre pre = Pre(),
                             const double* ah_s = nullptr, const int32_t* tid_s = nullptr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t B = blockIdx.x;
    int32_t* s_rel = reinterpret_cast<int32_t*>(smem + p.lay.srel);
    int32_t* s_aux = reinterpret_cast<int32_t*>(smem + p.lay.saux);
    const double2* s_task = reinterpret_cast<const double2*>(smem + p.lay.stask);
    float* os = reinterpret_cast<float*>(smem + p.lay.ostage) + warp * WCHUNK;
    int32_t* s_cidx = reinterpret_cast<int32_t*>(smem + p.lay.cidx) + warp * WCHUNK;
    float* s_cadv = reinterpret_cast<float*>(smem + p.lay.cadv) + warp * WCHUNK;
    const bool vec_ok = (reinterpret_cast<uintptr_t>(p.adv_tok) & 15) == 0;
    const bool any_traj = p.n_traj > 0;
    static_assert((RING & (RING - 1)) == 0, "RING is a power of two");
    // chunk indices fit in 32 bits (T < 2^31): keep the per-chunk bookkeeping 32-bit
    const int32_t n_full = (int32_t)(p.T / WCHUNK);  // chunks with all 512 tokens < T
    const int64_t n_mine = c_hi - c_lo > warp ? (c_hi - c_lo - warp + NWARPS - 1) / NWARPS : 0;
    const bool res = resident && n_mine <= RING;  // warp-uniform
    if (ADV_LDGSTS && r.on && !res) {
        for (int s = 0; s < RING; ++s) {
            const int32_t c = (int32_t)c_lo + warp + s * NWARPS;
            lane_issue(p, r, s, c, c < c_hi && c < n_full);
        }
    } else if (lane == 0 && r.on && !res) {
        for (int s = 0; s < RING; ++s) {
            const int64_t c = c_lo + warp + (int64_t)s * NWARPS;
            if (c < c_hi && chunk_full(p, c)) ring_issue(p, r, s, c);
        }
    }
    pre();
    // staging plan: the block's whole range if its trajectories fit, else 64-chunk windows
    int64_t wlen = max(c_hi - c_lo, (int64_t)1);
    if (wlen > KC_CAP) wlen = WIN_CHUNKS;
    if (!small && any_traj && c_lo < c_hi) {
        const int32_t f = p.chunk_first[c_lo];
        const int32_t l = c_hi < p.n_chunks ? p.chunk_first[c_hi] : p.n_traj - 1;
        if (l - f + 1 > WIN_TRAJ) wlen = WIN_CHUNKS;
    }
    int32_t* s_kc = reinterpret_cast<int32_t*>(smem + p.lay.skc);
    // small driver, phase C of the fused kernel with one window: phase A's s_rel and s_kc are
    // still in smem (the same window), only the values s_aux are restaged
    const bool reuse = PH == 1 && small && resident && wlen >= c_hi - c_lo;
    int32_t kseq = 0;
    int32_t prev_last = -1;  // last trajectory of the previous window (block-uniform)
    for (int64_t w0 = c_lo; w0 < c_hi; w0 += wlen) {
        const int64_t w1 = min(c_hi, w0 + wlen);
        // ---- stage the window's trajectories (block-wide)
        Window w{0, 0, w0 * WCHUNK, s_rel, false};
        if (any_traj) {
            int32_t f, l;
            if (small) {
                f = smem_find_in(s_offall, 0, p.n_traj, w0 * WCHUNK);
                l = smem_find_in(s_offall, 0, p.n_traj, min(w1 * WCHUNK, p.T) - 1);
            } else {
                f = p.chunk_first[w0];
                l = w1 < p.n_chunks ? p.chunk_first[w1] : p.n_traj - 1;
            }
            f = min(max(f, 0), p.n_traj - 1);
            l = min(max(l, f), p.n_traj - 1);
            w.f = f;
            w.nbt = l - f + 1;
            w.staged = small || w.nbt <= WIN_TRAJ;
            if (w.staged) {
                for (int32_t k = threadIdx.x; k <= w.nbt; k += COOP_THREADS) {
                    const int64_t o = (small ? s_offall[f + k] : p.off[f + k]) - w.base;
                    if (!reuse) s_rel[k] = (int32_t)min(max(o, (int64_t)0), (int64_t)INT_MAX);
                    if (k < w.nbt)
                        s_aux[k] = PH == 0 ? 0
                                   : (ah_s ? __float_as_int(adv_tilde_s(p, s_task, ah_s, tid_s, f + k))
                                           : __float_as_int(adv_tilde(p, s_task, f + k)));
                }
            }
        }
        __syncthreads();
        if (w.staged && !reuse) {  // chunk -> first trajectory of the window (no searches)
            const int32_t nwc = (int32_t)(w1 - w0);
            for (int32_t k = threadIdx.x; k < w.nbt; k += COOP_THREADS) {
                const int32_t lo = (w.s_rel[k] + WCHUNK - 1) / WCHUNK;
                const int32_t hi = min((int32_t)(((int64_t)w.s_rel[k + 1] + WCHUNK - 1) / WCHUNK), nwc);
                for (int32_t q = lo; q < hi; ++q) s_kc[q] = k;
            }
            __syncthreads();
        }
        // ---- this warp's chunks of the window
        for (int32_t c = (int32_t)w0 + warp; c < w1; c += NWARPS, ++kseq) {
            const int slot = kseq & (RING - 1);
            uint4 mk = make_uint4(0u, 0u, 0u, 0u);
            if (ADV_LDGSTS && r.on && !res) lane_wait_oldest();  // this chunk's group
            if (r.on && c < n_full) {
                if (!res && !ADV_LDGSTS) {
                    mbar_wait(&r.bar[slot], (r.par >> slot) & 1u);
                    r.par ^= 1u << slot;
                }
                mk = *reinterpret_cast<const uint4*>(r.buf + slot * WCHUNK + lane * 16);
            } else {
                mk = mask_direct(p, c, lane);
            }
            const int64_t t0 = (int64_t)c * WCHUNK + lane * 16;
            const int32_t tc = (int32_t)((int64_t)c * WCHUNK - w.base);  // window-relative
            const int32_t kc = (any_traj && w.staged) ? s_kc[c - (int32_t)w0] : 0;
            if (PH == 0) {  // small driver: every window is staged
                int32_t tot = 0;
                if (any_traj) (void)count_chunk_bits(lane_mask(mk), tc, kc, w, s_aux, tot);
                if (lane == 0) {
                    p.chunk[c] = tot;
                    if (c - c_lo < CT_CAP)
                        reinterpret_cast<int32_t*>(smem + p.lay.sct)[c - c_lo] = tot;
                }
                warp_total += tot;
            } else {
                const LaneMask lm = lane_mask(mk);
                const int32_t mine = any_traj ? __popc(lm.bits) : 0;
                int32_t wtotal = 0, pos = 0;
                if (p.compact) {  // positions of the lane's masked tokens in the chunk
                    const int32_t incl = warp_incl_scan(mine);
                    wtotal = __shfl_sync(0xffffffffu, incl, 31);
                    pos = incl - mine;
                }
                float outv[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) outv[i] = 0.f;
                if (any_traj && w.staged) {
                    uint32_t ob[16];
                    apply_chunk_bits(lm, tc, kc, w, s_aux, ob);
#pragma unroll
                    for (int i = 0; i < 16; ++i) outv[i] = __uint_as_float(ob[i]);
                    if (p.compact) {  // staged in smem, written coalesced below
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if ((lm.bits >> i) & 1u) {
                                s_cidx[pos] = (int32_t)(t0 + i);
                                s_cadv[pos] = outv[i];
                                ++pos;
                            }
                    }
                } else if (mine > 0 && t0 < p.T) {
                    int32_t g = coop_find_traj(p.off, p.n_traj, t0);
                    int64_t end = p.off[g + 1];
                    float at = adv_tilde(p, s_task, g);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int64_t t = t0 + i;
                        while (t >= end && g + 1 < p.n_traj) {
                            ++g;
                            end = p.off[g + 1];
                            at = adv_tilde(p, s_task, g);
                        }
                        const bool on = (lm.bits >> i) & 1u;
                        outv[i] = on ? at : 0.f;
                        if (p.compact && on) {
                            s_cidx[pos] = (int32_t)t;
                            s_cadv[pos] = at;
                            ++pos;
                        }
                    }
                }
                if (t0 - lane * 16 < p.T) store_transposed(p, os, c, outv, vec_ok);
                if (p.compact) {
                    __syncwarp();
                    const int32_t wbase =
                        small ? blk_base + p.chunk_base[c] : p.chunk_gbase[c];  // (large: global)
                    for (int32_t i = lane; i < wtotal; i += 32) {
                        p.idx[wbase + i] = s_cidx[i];
                        p.adv_c[wbase + i] = s_cadv[i];
                    }
                    __syncwarp();
                }
            }
            __syncwarp();
            if (ADV_LDGSTS && r.on && !res) {
                const int32_t c2 = c + RING * NWARPS;
                lane_issue(p, r, slot, c2, c2 < c_hi && c2 < n_full);
            } else if (lane == 0 && r.on && !res) {
                const int32_t c2 = c + RING * NWARPS;
                if (c2 < c_hi && c2 < n_full) ring_issue(p, r, slot, c2);
            }
        }
        __syncthreads();
        // ---- window epilogue (counting): per-trajectory counts out
        if (PH == 0 && w.staged) {
            for (int32_t k = threadIdx.x; k < w.nbt; k += COOP_THREADS) {
                if (small) {
                    // disjoint slot g + block; a trajectory that crosses from this block's
                    // previous window into this one adds to the count that window stored
                    // (the store is ordered before this load by the __syncthreads below)
                    if (k == 0 && w.f == prev_last) p.blk_cnt[w.f + B] += s_aux[0];
                    else p.blk_cnt[w.f + B + k] = s_aux[k];
                } else if (s_aux[k]) {
                    atomicAdd(&p.n_g[w.f + k], s_aux[k]);
                }
            }
            prev_last = w.f + w.nbt - 1;
            __syncthreads();
        }
    }
}

// per-task (mu, max(sigma, eps)) into smem from the (global) stats (readings R1, R2);
// block 0 also publishes task_stats
__device__ void task_params_smem(const AdvParams& p, double2* s_task) {
    for (int32_t i = threadIdx.x; i < p.n_tasks; i += blockDim.x) {
        const double N = p.stats[3 * i], S = p.stats[3 * i + 1], Q = p.stats[3 * i + 2];
        const double mu = N > 0.0 ? S / N : 0.0;
        const double sd = N > 0.0 ? sqrt(fmax(Q / N - mu * mu, 0.0)) : 0.0;
        s_task[i] = make_double2(mu, sd > p.eps_std ? sd : p.eps_std);
        if (blockIdx.x == 0 && p.task_stats_out) {
            p.task_stats_out[3 * i] = N;
            p.task_stats_out[3 * i + 1] = mu;
            p.task_stats_out[3 * i + 2] = sd;
        }
    }
}
// one warp (block 0): meta = (local masked rows, global N, global G), n_mask_global, status
__device__ void publish_meta(const AdvParams& p, int32_t local_rows) {
    double nsum = 0.0;
    for (int32_t i = threadIdx.x & 31; i < p.n_tasks; i += 32) nsum += p.stats[3 * i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsum += __shfl_down_sync(0xffffffffu, nsum, o);
    if ((threadIdx.x & 31) == 0) {
        const int64_t n = (int64_t)nsum;
        p.meta[0] = local_rows;  // local masked rows
        p.meta[1] = n;           // global N
        p.meta[2] = (int64_t)p.stats[3 * p.n_tasks];  // global G (groups)
        if (p.n_mask_global_out) *p.n_mask_global_out = n;
        if (n == 0) atomicOr(p.d_status, AGENTRL_ST_NO_TOKENS);
    }
}
// the above for the small driver's apply, plus every block's prefix of the stats blocks'
// masked totals (its compaction base)
__device__ void load_task_params(const AdvParams& p, uint8_t* smem, int32_t* s_pre, int32_t* s_w) {
    double2* s_task = reinterpret_cast<double2*>(smem + p.lay.stask);
    const int64_t G = p.g_stats > 0 ? p.g_stats : gridDim.x;
    task_params_smem(p, s_task);
    block_prefix_smem(p.blk_chunk, G, s_pre, s_w);  // also orders the s_task writes
    if (blockIdx.x == 0 && threadIdx.x < 32) publish_meta(p, s_pre[G]);
}

// block-local exclusive scan of the block's chunk counts -> chunk_base; block total
__device__ void chunk_bases(const AdvParams& p, int64_t c_lo, int64_t c_hi, int32_t* s_w) {
    __syncthreads();  // chunk counts of all warps written
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
    if (threadIdx.x == 0) p.blk_chunk[blockIdx.x] = total;
}

// ------------------------------------------------------------------ GRPO group advantage
// (readings R1 population std, R2 exact-equal rule and eps floor, R14 K == 1).
// mb: the K members sorted by index.  Writes adv_hat; returns (N, S, Q) of the group and
// its task; nz counts the groups with at least one member (E_{i,j} of P:1250).
template <typename GetR, typename GetT, typename GetN>
__device__ __forceinline__ void group_adv(const AdvParams& p, int32_t K, const int32_t* mb,
                                          GetR rew, GetT task, GetN ng, double& N, double& S,
                                          double& Q, int32_t& task0, int32_t& st,
                                          unsigned long long& nz) {
    N = S = Q = 0.0;
    task0 = -1;
    if (K <= 0) return;
    if (K == 1) st |= AGENTRL_ST_GROUP_TOO_SMALL;
    task0 = task(mb[0]);
    double sum = 0.0, rmax = rew(mb[0]), rmin = rmax;
    for (int a = 0; a < K; ++a) {
        const double r = rew(mb[a]);
        if (task(mb[a]) != task0) st |= AGENTRL_ST_GROUP_SPANS_TASKS;
        sum += r;
        rmax = fmax(rmax, r);
        rmin = fmin(rmin, r);
    }
    const bool flat = rmax == rmin;
    const double mean = sum / (double)K;
    double ss = 0.0;
    if (!flat)
        for (int a = 0; a < K; ++a) {
            const double dlt = (double)rew(mb[a]) - mean;
            ss += dlt * dlt;
        }
    const double sd = sqrt(ss / (double)K);
    const double den = sd > p.eps_std ? sd : p.eps_std;
    for (int a = 0; a < K; ++a) {
        const int32_t g = mb[a];
        const double ah = flat ? 0.0 : ((double)rew(g) - mean) / den;
        p.adv_hat[g] = ah;
        const int32_t nn = ng(g);
        const double n = (double)nn;
        N += n;
        S += n * ah;
        Q += n * ah * ah;
    }
    nz += 1;  // a group present in the batch (GRPO group mean)
}

// ------------------------------------------------------------------ small driver
// Every block streams a contiguous chunk range (warp w: chunks w, w+8, ...) and also owns a
// contiguous slice of the trajectories and of the groups (part_lo).  One grid barrier:
//   before it, each block
//     - loads the whole trajectory table (offsets, group / task ids, rewards) into shared
//       memory while its first mask copies are in flight;
//     - counts its chunks (phase A): c_{g,B} = masked tokens of trajectory g in block B;
//     - computes A^ of every group with a trajectory in its token range, and of the groups it
//       owns (one warp per group: ballot scans of the staged ids in index order);
//     - writes its per-task partial moments sum_g c_{g,B} (1, A^_g, A^_g^2).  Eq.1's moments
//       are linear in the counts, so the partials of the blocks sharing a trajectory add up to
//       n_g (1, A^_g, A^_g^2); N_i stays an exact integer;
//   after it, every block sums the G partials in block order (the same code and order in
//   every block, so every block holds identical mu_i, sigma_i) and applies Eq.1 to its chunks,
//   which are still resident in its ring; then it publishes n_g of the trajectories it owns.
struct SmallT {
    int32_t *gid, *tid, *gflag, *gtask, *glist, *gfirst, *glast;
    float* rew;
    double* ah;
};
__device__ __forceinline__ SmallT small_t(const AdvParams& p, uint8_t* smem) {
    SmallT a;
    a.gid = reinterpret_cast<int32_t*>(smem + p.lay.sgid);
    a.tid = reinterpret_cast<int32_t*>(smem + p.lay.stid);
    a.rew = reinterpret_cast<float*>(smem + p.lay.srew);
    a.ah = reinterpret_cast<double*>(smem + p.lay.sah);
    a.gflag = reinterpret_cast<int32_t*>(smem + p.lay.gflag);
    a.gtask = reinterpret_cast<int32_t*>(smem + p.lay.gtask);
    a.glist = reinterpret_cast<int32_t*>(smem + p.lay.glist);
    a.gfirst = reinterpret_cast<int32_t*>(smem + p.lay.gfirst);
    a.glast = reinterpret_cast<int32_t*>(smem + p.lay.glast);
    return a;
}

__device__ void stage_all_offsets(const AdvParams& p, uint8_t* smem) {
    int64_t* s_off = reinterpret_cast<int64_t*>(smem + p.lay.soff);
    for (int32_t k = threadIdx.x; k <= p.n_traj; k += COOP_THREADS) s_off[k] = p.off[k];
    __syncthreads();
}

__device__ __forceinline__ bool small_member(const AdvParams& p, int32_t j, int32_t i) {
    return j >= 0 && j < p.n_groups && i >= 0 && i < p.n_tasks;
}

// the whole trajectory table into smem: every load of a thread is issued before its first store
// (one DRAM round trip); the trajectories this block owns are validated here (ids, offsets;
// A^ = 0 outside any group)
constexpr int TBL_PER = (SMALL_TRAJ + 1 + COOP_THREADS - 1) / COOP_THREADS;
__device__ void small_load_table(const AdvParams& p, uint8_t* smem, int32_t& st) {
    const SmallT a = small_t(p, smem);
    int64_t* s_off = reinterpret_cast<int64_t*>(smem + p.lay.soff);
    const int64_t G = gridDim.x, B = blockIdx.x;
    const int64_t t_lo = part_lo(p.n_traj, B, G), t_hi = part_lo(p.n_traj, B + 1, G);
    int64_t o[TBL_PER];
    int32_t jj[TBL_PER], ii[TBL_PER];
    float rr[TBL_PER];
#pragma unroll
    for (int q = 0; q < TBL_PER; ++q) {
        const int32_t g = threadIdx.x + q * COOP_THREADS;
        o[q] = g <= p.n_traj ? p.off[g] : 0;
        const bool in = g < p.n_traj;
        jj[q] = in ? p.group_id[g] : -1;
        ii[q] = in ? p.task_id[g] : -1;
        rr[q] = in ? p.rewards[g] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < TBL_PER; ++q) {
        const int32_t g = threadIdx.x + q * COOP_THREADS;
        if (g <= p.n_traj) s_off[g] = o[q];
        if (g < p.n_traj) {
            a.gid[g] = small_member(p, jj[q], ii[q]) ? jj[q] : -1;  // -1: in no group
            a.tid[g] = ii[q];
            a.rew[g] = rr[q];
            a.ah[g] = 0.0;
            if (g >= t_lo && g < t_hi && !small_member(p, jj[q], ii[q])) {
                st |= AGENTRL_ST_GROUP_SPANS_TASKS;
                p.adv_hat[g] = 0.0;
            }
        }
    }
    for (int32_t j = threadIdx.x; j < p.n_groups; j += COOP_THREADS) {
        a.gflag[j] = 0;
        a.gfirst[j] = INT_MAX;
        a.glast[j] = -1;
    }
    __syncthreads();
    for (int64_t g = t_lo + threadIdx.x; g < t_hi; g += COOP_THREADS)
        if (s_off[g + 1] < s_off[g]) st |= AGENTRL_ST_BAD_OFFSETS;
    if (B == 0 && threadIdx.x == 0 && (s_off[0] != 0 || s_off[p.n_traj] != p.T))
        st |= AGENTRL_ST_BAD_OFFSETS;
}

// One warp, group j (readings R1 population std, R2 exact-equal rule and eps floor,
// R14 K == 1): members = trajectories with group id j and valid task id, found by ballot scans
// of the staged table in index order.  A^ of every member -> a.ah; the group's task (its
// lowest-index member's) -> a.gtask.  own: also publishes K_j, the task and A^, and the status.
// Every block that handles j runs the same code on the same smem copy: identical bits.
__device__ void small_group_warp(const AdvParams& p, const SmallT& a, int32_t j, bool own,
                                 int32_t* s_mb /* 32 ints of this warp */, int32_t& st,
                                 int32_t& nz) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    int32_t K = 0, first = -1;
    double sum = 0.0;
    float fmx = -INFINITY, fmn = INFINITY;
    // a.gid holds the group id of members and -1 otherwise (invalid group or task id)
    const int32_t lo = a.gfirst[j], hi = a.glast[j];  // (INT_MAX, -1) for an empty group
#pragma unroll 4
    for (int32_t i0 = lo & ~31; i0 <= hi; i0 += 32) {
        const int32_t i = i0 + lane;
        const bool hit = i <= hi && a.gid[i] == j;
        const uint32_t bal = __ballot_sync(0xffffffffu, hit);
        if (hit) {
            const float r = a.rew[i];
            const int32_t rk = K + __popc(bal & lt);
            if (rk < 32) s_mb[rk] = i;  // the first 32 members, in index order
            sum += (double)r;
            fmx = fmaxf(fmx, r);
            fmn = fminf(fmn, r);
        }
        if (first < 0 && bal) first = i0 + __ffs(bal) - 1;
        K += __popc(bal);
    }
    // butterfly: a + b == b + a, so every lane ends with the same bits; max / min of the f32
    // rewards through order-preserving integer keys (one redux each)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    auto okey = [](float x) {
        const uint32_t u = __float_as_uint(x);
        return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    };
    auto ounkey = [](uint32_t k) {
        return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
    };
    const double rmax = (double)ounkey(__reduce_max_sync(0xffffffffu, okey(fmx)));
    const double rmin = (double)ounkey(__reduce_min_sync(0xffffffffu, okey(fmn)));
    __syncwarp();
    if (K == 0) {
        if (lane == 0) {
            a.gtask[j] = -1;
            if (own) {
                p.grp_cnt[j] = 0;
                p.grp_task[j] = -1;
            }
        }
        return;
    }
    const int32_t task0 = a.tid[first];
    const bool flat = rmax == rmin;
    const double mean = sum / (double)K;
    const bool few = K <= 32;  // members in registers (lane L = member L)
    const int32_t m = (few && lane < K) ? s_mb[lane] : -1;
    double ss = 0.0;
    bool spans = false;
    if (few) {
        if (m >= 0) {
            spans = a.tid[m] != task0;
            const double dl = (double)a.rew[m] - mean;
            ss = flat ? 0.0 : dl * dl;
        }
    } else {
        for (int32_t i = lo + lane; i <= hi; i += 32)
            if (a.gid[i] == j) {
                spans |= a.tid[i] != task0;
                const double dl = (double)a.rew[i] - mean;
                ss += flat ? 0.0 : dl * dl;
            }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    spans = __any_sync(0xffffffffu, spans);
    const double sd = sqrt(ss / (double)K);
    const double den = sd > p.eps_std ? sd : p.eps_std;
    auto put = [&](int32_t i) {
        const double ah = flat ? 0.0 : ((double)a.rew[i] - mean) / den;
        a.ah[i] = ah;
        if (own) p.adv_hat[i] = ah;
    };
    if (few) {
        if (m >= 0) put(m);
    } else {
        for (int32_t i = lo + lane; i <= hi; i += 32)
            if (a.gid[i] == j) put(i);
    }
    if (lane == 0) {
        a.gtask[j] = task0;
        if (own) {
            p.grp_cnt[j] = K;
            p.grp_task[j] = task0;
            if (K == 1) st |= AGENTRL_ST_GROUP_TOO_SMALL;
            if (spans) st |= AGENTRL_ST_GROUP_SPANS_TASKS;
            nz += 1;  // a group present in the batch (GRPO group mean)
        }
    }
}

__device__ __forceinline__ void small_range(const AdvParams& p, int64_t& c_lo, int64_t& c_hi) {
    c_lo = part_lo(p.n_chunks, blockIdx.x, gridDim.x);
    c_hi = part_lo(p.n_chunks, (int64_t)blockIdx.x + 1, gridDim.x);
}

// the trajectories overlapping the block's token range [f, l] (stream_phase's staging rule);
// false: the block has no chunks
__device__ __forceinline__ bool small_traj_range(const AdvParams& p, const int64_t* s_off,
                                                 int64_t c_lo, int64_t c_hi, int32_t& f,
                                                 int32_t& l) {
    if (c_lo >= c_hi || p.n_traj <= 0) return false;
    f = smem_find_in(s_off, 0, p.n_traj, c_lo * WCHUNK);
    l = smem_find_in(s_off, 0, p.n_traj, min(c_hi * WCHUNK, p.T) - 1);
    f = min(max(f, 0), p.n_traj - 1);
    l = min(max(l, f), p.n_traj - 1);
    return true;
}

// the groups this block needs -- those of the trajectories overlapping its token range (bit
// 0) and those it owns (bit 1) -- one warp each; blk_grp[B] = the owned groups with members
__device__ void small_groups(const AdvParams& p, uint8_t* smem, int64_t c_lo, int64_t c_hi,
                             int32_t& st) {
    const SmallT a = small_t(p, smem);
    const int64_t G = gridDim.x, B = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t* s_off = reinterpret_cast<const int64_t*>(smem + p.lay.soff);
    int32_t f = 0, l = -1;
    const bool any = small_traj_range(p, s_off, c_lo, c_hi, f, l);
    const int64_t j_lo = part_lo(p.n_groups, B, G), j_hi = part_lo(p.n_groups, B + 1, G);
    // every group's first and last member (the bounds of its ballot scans: one or two 32-wide
    // steps when a group's members are contiguous), then the flags
    for (int32_t g = threadIdx.x; g < p.n_traj; g += COOP_THREADS) {
        const int32_t j = a.gid[g];
        if (j >= 0) {
            atomicMin(&a.gfirst[j], g);
            atomicMax(&a.glast[j], g);
        }
    }
    if (any)
        for (int32_t g = f + threadIdx.x; g <= l; g += COOP_THREADS)
            if (a.gid[g] >= 0) atomicOr(&a.gflag[a.gid[g]], 1);
    for (int64_t j = j_lo + threadIdx.x; j < j_hi; j += COOP_THREADS) atomicOr(&a.gflag[j], 2);
    __shared__ int32_t s_nl, s_nz;
    if (threadIdx.x == 0) s_nl = s_nz = 0;
    __syncthreads();
    for (int32_t j = threadIdx.x; j < p.n_groups; j += COOP_THREADS)
        if (a.gflag[j]) a.glist[atomicAdd(&s_nl, 1)] = j;
    __syncthreads();
    __shared__ int32_t s_mb[NWARPS][32];
    int32_t nz = 0;
    for (int32_t q = wid; q < s_nl; q += NWARPS) {
        const int32_t j = a.glist[q];
        small_group_warp(p, a, j, (a.gflag[j] & 2) != 0, s_mb[wid], st, nz);
    }
    if (lane == 0 && nz) atomicAdd(&s_nz, nz);
    __syncthreads();  // A^ of the block's trajectories and the groups' tasks in smem
    if (threadIdx.x == 0) p.blk_grp[B] = s_nz;
}

// block-local exclusive scan of the block's chunk totals (kept in smem by phase A up to CT_CAP
// chunks) -> chunk_base; blk_chunk[B] = the block total
__device__ void small_chunk_bases(const AdvParams& p, uint8_t* smem, int64_t c_lo, int64_t c_hi,
                                  int32_t* s_w) {
    const int64_t n = c_hi - c_lo;
    if (n > CT_CAP) {
        chunk_bases(p, c_lo, c_hi, s_w);
        return;
    }
    const int32_t* s_ct = reinterpret_cast<const int32_t*>(smem + p.lay.sct);
    __syncthreads();  // chunk totals of all warps written
    const int64_t per = (n + COOP_THREADS - 1) / COOP_THREADS;
    const int64_t lo = min(n, (int64_t)threadIdx.x * per), hi = min(n, lo + per);
    int32_t sum = 0;
    for (int64_t c = lo; c < hi; ++c) sum += s_ct[c];
    int32_t total;
    int32_t run = coop_block_exscan(sum, s_w, total);
    for (int64_t c = lo; c < hi; ++c) {
        p.chunk_base[c_lo + c] = run;
        run += s_ct[c];
    }
    if (threadIdx.x == 0) p.blk_chunk[blockIdx.x] = total;
}

// phase A (with the trajectory table and the group advantages computed while the block's first
// mask copies are in flight) + the block's partial moments: everything before the barrier
__device__ void small_pre_barrier(const AdvParams& p, uint8_t* smem, WarpRing& r, int32_t* s_w) {
    const SmallT a = small_t(p, smem);
    const int64_t B = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t* s_off = reinterpret_cast<const int64_t*>(smem + p.lay.soff);
    int32_t st = 0;
    int64_t c_lo, c_hi;
    small_range(p, c_lo, c_hi);
    int32_t warp_total = 0;
    stream_phase<0>(p, smem, r, c_lo, c_hi, true, s_off, 0, warp_total, false, [&]() {
        small_load_table(p, smem, st);
        phase_mark(1);
        small_groups(p, smem, c_lo, c_hi, st);
        phase_mark(2);
    });
    phase_mark(3);
    small_chunk_bases(p, smem, c_lo, c_hi, s_w);  // per-chunk compaction bases, blk_chunk[B]
    // ---- per-task partial (N, S, Q) = sum over the block's trajectories of c_{g,B} (1, A^,
    // A^^2), attributed to the group's task; fixed order (lanes stride the trajectories,
    // shuffle tree).  Counts: the window's s_aux (one staged window) or the block's slots.
    int32_t f = 0, l = -1;
    const bool any = small_traj_range(p, s_off, c_lo, c_hi, f, l);
    const int32_t* s_aux = reinterpret_cast<const int32_t*>(smem + p.lay.saux);
    const bool one_window = c_hi - c_lo <= KC_CAP;
    for (int32_t i = wid; i < p.n_tasks; i += NWARPS) {
        double N = 0.0, S = 0.0, Q = 0.0;
        if (any)
            for (int32_t g = f + lane; g <= l; g += 32) {
                const int32_t j = a.gid[g];
                if (!small_member(p, j, a.tid[g]) || a.gtask[j] != i) continue;
                // (an empty trajectory between two windows has no slot: count 0)
                const int32_t c = one_window ? s_aux[g - f]
                                  : s_off[g + 1] > s_off[g] ? p.blk_cnt[g + B] : 0;
                const double n = (double)c, ah = a.ah[g];
                N += n;
                S += n * ah;
                Q += n * ah * ah;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            N += __shfl_down_sync(0xffffffffu, N, o);
            S += __shfl_down_sync(0xffffffffu, S, o);
            Q += __shfl_down_sync(0xffffffffu, Q, o);
        }
        if (lane == 0) {
            double* bp = p.blk_part + 3 * (B * p.n_tasks + i);
            bp[0] = N;
            bp[1] = S;
            bp[2] = Q;
        }
    }
    phase_mark(4);
    if (st) atomicOr(p.d_status, st);
}

// after the barrier (every block, identical code and order -> identical results): the per-task
// moments = the block partials summed in block order (warp w: tasks w, w+8, ...; lanes stride
// the blocks, shuffle tree); mu_i and max(sigma_i, eps) into s_task; s_pre = exclusive prefix
// of the blocks' masked totals (compaction bases).  Block 0 publishes task_stats, N, G and the
// local masked-row count; stats_only (a communicator follows): block 0 writes the raw sums.
__device__ void small_moments(const AdvParams& p, uint8_t* smem, int32_t* s_pre, int32_t* s_w,
                              bool stats_only) {
    double2* s_task = reinterpret_cast<double2*>(smem + p.lay.stask);
    __shared__ double s_nsum[NWARPS];
    __shared__ int32_t s_ngrp;
    const int64_t G = gridDim.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool blk0 = blockIdx.x == 0;
    if (stats_only && !blk0) return;
    // one round trip: every block partial, the block totals (compaction bases) and the group
    // counts are loaded by the whole block into smem (the idle output-staging region) first
    const bool one = G <= COOP_THREADS;
    const int64_t nparts = 3 * G * (int64_t)p.n_tasks;
    double* s_bp = reinterpret_cast<double*>(smem + p.lay.ostage);
    const bool staged = nparts <= (int64_t)(NWARPS * WCHUNK * 4 / sizeof(double));
    const int32_t my_cnt = (one && !stats_only && threadIdx.x < G) ? p.blk_chunk[threadIdx.x] : 0;
    const int32_t my_grp = (one && blk0 && threadIdx.x < G) ? p.blk_grp[threadIdx.x] : 0;
    if (threadIdx.x == 0) s_ngrp = 0;
    if (staged) {
        for (int64_t k = threadIdx.x; k < nparts; k += COOP_THREADS) s_bp[k] = p.blk_part[k];
    }
    __syncthreads();
    if (one && my_grp) atomicAdd(&s_ngrp, my_grp);  // integers: exact in any order
    const double* bsrc = staged ? s_bp : p.blk_part;
    double nsum = 0.0;
    for (int32_t i = wid; i < p.n_tasks; i += NWARPS) {
        double N = 0.0, S = 0.0, Q = 0.0;
        for (int64_t b = lane; b < G; b += 32) {
            const double* bp = bsrc + 3 * (b * p.n_tasks + i);
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
            if (stats_only) {
                p.stats[3 * i] = N;
                p.stats[3 * i + 1] = S;
                p.stats[3 * i + 2] = Q;
            } else {
                const double mu = N > 0.0 ? S / N : 0.0;
                const double sd = N > 0.0 ? sqrt(fmax(Q / N - mu * mu, 0.0)) : 0.0;
                s_task[i] = make_double2(mu, sd > p.eps_std ? sd : p.eps_std);
                if (blk0 && p.task_stats_out) {
                    p.task_stats_out[3 * i] = N;
                    p.task_stats_out[3 * i + 1] = mu;
                    p.task_stats_out[3 * i + 2] = sd;
                }
            }
            nsum += N;
        }
    }
    if (blk0) {
        if (lane == 0) s_nsum[wid] = nsum;
        if (wid == 0 && !one) {
            int32_t c = 0;
            for (int64_t b = lane; b < G; b += 32) c += p.blk_grp[b];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
            if (lane == 0) s_ngrp = c;
        }
    }
    if (stats_only) {
        __syncthreads();
        if (threadIdx.x == 0) p.stats[3 * p.n_tasks] = (double)s_ngrp;  // G (local)
        return;
    }
    if (one) {  // (the scan's barriers also order s_task / s_nsum)
        int32_t total;
        const int32_t pre = coop_block_exscan(my_cnt, s_w, total);
        if (threadIdx.x < G) s_pre[threadIdx.x] = pre;
        if (threadIdx.x == 0) s_pre[G] = total;
        __syncthreads();
    } else {
        block_prefix_smem(p.blk_chunk, G, s_pre, s_w);
    }
    if (blk0 && threadIdx.x == 0) {
        double n = 0.0;
        // tasks were summed warp by warp: add the warp totals in warp order -- any fixed order
        // gives the exact integer here
        for (int w = 0; w < NWARPS; ++w) n += s_nsum[w];
        const int64_t nn = (int64_t)n;
        p.meta[0] = s_pre[G];  // local masked rows
        p.meta[1] = nn;        // global N
        p.meta[2] = s_ngrp;    // global G (groups)
        if (p.n_mask_global_out) *p.n_mask_global_out = nn;
        if (nn == 0) atomicOr(p.d_status, AGENTRL_ST_NO_TOKENS);
    }
    __syncthreads();
}

// n_g of the trajectories this block owns: the slots of the blocks whose ranges it spans,
// summed in block order (exact integers).  Loaded before phase C (the loads are in flight
// while it streams), stored after it.
constexpr int NG_PER = (SMALL_TRAJ + COOP_THREADS - 1) / COOP_THREADS;
struct NgRegs {
    int32_t n[NG_PER];
};
__device__ __forceinline__ NgRegs small_ng_load(const AdvParams& p, const int64_t* s_off) {
    const int64_t G = gridDim.x, B = blockIdx.x;
    const int64_t t_lo = part_lo(p.n_traj, B, G), t_hi = part_lo(p.n_traj, B + 1, G);
    NgRegs r;
#pragma unroll
    for (int q = 0; q < NG_PER; ++q) {
        const int64_t g = t_lo + threadIdx.x + (int64_t)q * COOP_THREADS;
        int32_t n = 0;
        if (g < t_hi) {
            const int64_t s0 = s_off[g], e = s_off[g + 1];
            if (e > s0 && s0 >= 0) {
                const int64_t b0 = part_owner(p.n_chunks, s0 / WCHUNK, G);
                const int64_t b1 = part_owner(p.n_chunks, (e - 1) / WCHUNK, G);
                for (int64_t b = max(b0, (int64_t)0); b <= min(b1, G - 1); ++b) n += p.blk_cnt[g + b];
            }
        }
        r.n[q] = n;
    }
    return r;
}
__device__ __forceinline__ void small_ng_store(const AdvParams& p, const NgRegs& r) {
    const int64_t G = gridDim.x, B = blockIdx.x;
    const int64_t t_lo = part_lo(p.n_traj, B, G), t_hi = part_lo(p.n_traj, B + 1, G);
#pragma unroll
    for (int q = 0; q < NG_PER; ++q) {
        const int64_t g = t_lo + threadIdx.x + (int64_t)q * COOP_THREADS;
        if (g < t_hi) p.n_g[g] = r.n[q];
    }
}


// masked tokens before position t (large driver, after phase A): block prefix + the chunk's
// local base + the popcount of the chunk's lane bits below t
__device__ __forceinline__ int32_t masked_before(const AdvParams& p, const int32_t* s_pre, int64_t G, int64_t t) {
    if (t <= 0) return 0;
    if (t >= p.T) return s_pre[G];
    const int64_t c = t / WCHUNK;
    const int r = (int)(t - c * WCHUNK);  // bits below r of the chunk's 512-bit mask
    int32_t P = s_pre[part_owner(p.n_chunks, c, G)] + p.chunk_base[c];
    const uint4* b4 = reinterpret_cast<const uint4*>(p.lanebits + c * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 128 bits (8 lanes) per vector
        const uint4 v = b4[q];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int b0 = (q * 4 + k) * 32;  // first token of this word
            const int keep = min(max(r - b0, 0), 32);
            const uint32_t m = keep == 32 ? 0xffffffffu : ((1u << keep) - 1u);
            P += __popc(w[k] & m);
        }
    }
    return P;
}

// ------------------------------------------------------------------ large driver
// Three launches (round 2): k_adv_large_pop streams phase A at full occupancy; the cooperative
// k_adv_large_stats runs the statistics phases B1..B4; k_adv_large_apply streams phase C with
// its own (smaller) register and shared-memory budget.  With a communicator the all-reduce of
// (N, S, Q) sits between the last two.

// phase A as an ordinary kernel: per-lane mask bits and per-chunk masked counts (4 chunks per
// warp iteration: 4 x 16 B loads in flight per lane), plus the per-trajectory work that needs
// no counts -- K_j, validation, the chunk -> first-trajectory table.  grp_cnt / grp_fill are
// zeroed by the host before the launch.
constexpr int POP_THREADS = 256;
#ifndef ADV_POP_UNROLL
#define ADV_POP_UNROLL 4
#endif
constexpr int POP_UNROLL = ADV_POP_UNROLL;
#ifndef ADV_POP_PIPE
#define ADV_POP_PIPE 1  // the next POP_UNROLL chunks' loads in flight while the current reduce
#endif
__global__ void __launch_bounds__(POP_THREADS) k_adv_large_pop(const AdvParams p) {
    phase_mark(0);
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * POP_THREADS + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * POP_THREADS) >> 5;
    const int64_t n_full = p.T / WCHUNK;
    const bool aligned = (reinterpret_cast<uintptr_t>(p.mask) & 15) == 0;
    const bool any_traj = p.n_traj > 0;
    // software-pipelined: the loads of the warp's next POP_UNROLL chunks are in flight while
    // the current ones are reduced
    auto load = [&](uint4 (&mk)[POP_UNROLL], int64_t c0) {
#pragma unroll
        for (int u = 0; u < POP_UNROLL; ++u) {
            const int64_t c = c0 + u;
            mk[u] = make_uint4(0u, 0u, 0u, 0u);
            if (c < n_full && aligned)
                mk[u] = __ldcs(reinterpret_cast<const uint4*>(p.mask + c * WCHUNK) + lane);
            else if (c < p.n_chunks)
                mk[u] = mask_direct(p, c, lane);
        }
    };
    const int64_t step = nw * POP_UNROLL;
    uint4 cur[POP_UNROLL];
#if ADV_POP_PIPE
    uint4 nxt[POP_UNROLL];
#endif
    int64_t c0 = gw * POP_UNROLL;
#if ADV_POP_PIPE
    if (c0 < p.n_chunks) load(cur, c0);
#endif
    for (; c0 < p.n_chunks; c0 += step) {
#if ADV_POP_PIPE
        if (c0 + step < p.n_chunks) load(nxt, c0 + step);
#else
        load(cur, c0);
#endif
#pragma unroll
        for (int u = 0; u < POP_UNROLL; ++u) {
            const int64_t c = c0 + u;
            if (c < p.n_chunks) {
                const uint32_t lb = any_traj ? lane_mask(cur[u]).bits : 0u;
                p.lanebits[c * 32 + lane] = (uint16_t)lb;  // 64 B per chunk
                const int32_t tot = __reduce_add_sync(0xffffffffu, __popc(lb));
                if (lane == 0) p.chunk[c] = tot;
            }
        }
#if ADV_POP_PIPE
#pragma unroll
        for (int u = 0; u < POP_UNROLL; ++u) cur[u] = nxt[u];
#endif
    }
    const int64_t gtid = (int64_t)blockIdx.x * POP_THREADS + threadIdx.x;
    const int64_t gstride = (int64_t)gridDim.x * POP_THREADS;
    int32_t st = 0;
    bool bad_member = false;
    for (int64_t g = gtid; g < p.n_traj; g += gstride) {
        const int64_t a = p.off[g], b = p.off[g + 1];
        const int32_t j = p.group_id[g], i = p.task_id[g];
        // chunks whose first token is in g
        const int64_t lo = (a + WCHUNK - 1) / WCHUNK;
        const int64_t hi = min((b + WCHUNK - 1) / WCHUNK, p.n_chunks);
        for (int64_t c = max(lo, (int64_t)0); c < hi; ++c) p.chunk_first[c] = (int32_t)g;
        if (j < 0 || j >= p.n_groups || i < 0 || i >= p.n_tasks) {
            st |= AGENTRL_ST_GROUP_SPANS_TASKS;
            bad_member = true;
            continue;
        }
        atomicAdd(&p.grp_cnt[j], 1);
        atomicMax(&p.grp_lo[j], ~(uint32_t)g);  // ~min(g)
        atomicMax(&p.grp_hi[j], (uint32_t)g + 1u);
        if (b < a) st |= AGENTRL_ST_BAD_OFFSETS;
    }
    if (bad_member) atomicOr(p.grp_flag, 1);  // a trajectory in no group: the general path
    if (gtid == 0 && (p.off[0] != 0 || p.off[p.n_traj] != p.T)) st |= AGENTRL_ST_BAD_OFFSETS;
    if (st) atomicOr(p.d_status, st);
}

// GRPO group advantage (R1, R2, R14) of a group of K <= REG_K members m[0..K), sorted
// by index: the arithmetic and order of group_adv on register copies of the members' reward,
// task and count (their loads issued together: no dependent global round trips)
__device__ __forceinline__ void group_regs(const AdvParams& p, int32_t K, const int32_t (&m)[REG_K],
                                           double& N, double& S, double& Q, int32_t& task0,
                                           int32_t& st, unsigned long long& nz) {
    float rr[REG_K];
    int32_t tt[REG_K], nn[REG_K];
#pragma unroll
    for (int a = 0; a < REG_K; ++a) {
        rr[a] = a < K ? p.rewards[m[a]] : 0.f;
        tt[a] = a < K ? p.task_id[m[a]] : 0;
        nn[a] = a < K ? p.n_g[m[a]] : 0;
    }
    // same arithmetic and order as group_adv, on the register copies
    N = S = Q = 0.0;
    task0 = -1;
    if (K > 0) {
        if (K == 1) st |= AGENTRL_ST_GROUP_TOO_SMALL;
        task0 = tt[0];
        double sum = 0.0, rmax = rr[0], rmin = rmax;
#pragma unroll
        for (int a = 0; a < REG_K; ++a)
            if (a < K) {
                const double rv = rr[a];
                if (tt[a] != task0) st |= AGENTRL_ST_GROUP_SPANS_TASKS;
                sum += rv;
                rmax = fmax(rmax, rv);
                rmin = fmin(rmin, rv);
            }
        const bool flat = rmax == rmin;
        const double mean = sum / (double)K;
        double ss = 0.0;
        if (!flat) {
#pragma unroll
            for (int a = 0; a < REG_K; ++a)
                if (a < K) {
                    const double dlt = (double)rr[a] - mean;
                    ss += dlt * dlt;
                }
        }
        const double sd = sqrt(ss / (double)K);
        const double den = sd > p.eps_std ? sd : p.eps_std;
#pragma unroll
        for (int a = 0; a < REG_K; ++a)
            if (a < K) {
                const double ah = flat ? 0.0 : ((double)rr[a] - mean) / den;
                p.adv_hat[m[a]] = ah;
                const double n = (double)nn[a];
                N += n;
                S += n * ah;
                Q += n * ah * ah;
            }
        nz += 1;  // a group present in the batch (GRPO group mean)
    }
}

__device__ void large_stats_phases(const AdvParams& p, uint8_t* smem, cg::grid_group& grid,
                                   int32_t* s_w, int32_t* s_pre) {
    const int64_t G = gridDim.x, B = blockIdx.x;
    const int64_t gtid = B * blockDim.x + threadIdx.x;
    const int64_t gstride = G * blockDim.x;
    int32_t st = 0;
    phase_mark(1);
    const int64_t c_lo = part_lo(p.n_chunks, B, G), c_hi = part_lo(p.n_chunks, B + 1, G);
    const int64_t j_lo = part_lo(p.n_groups, B, G), j_hi = part_lo(p.n_groups, B + 1, G);
    if (gtid == 0) p.meta[3] = 0;  // local count of groups with members (G)
    chunk_bases(p, c_lo, c_hi, s_w);  // block-local bases of the popcount launch's chunk counts
    // contiguous groups (the usual rollout layout: a prompt's K samples stored together): when
    // every group is one run of at most REG_K trajectories (K_j == last - first + 1) and every
    // trajectory is in a group, the members of group j are first_j .. first_j + K_j - 1 in index
    // order, so the member-list phases B1/B2 and their two grid barriers are skipped
    {
        bool bad = false;
        for (int64_t j = j_lo + threadIdx.x; j < j_hi; j += COOP_THREADS) {
            const int32_t K = p.grp_cnt[j];
            if (K > 0) bad |= K > REG_K || p.grp_hi[j] - ~p.grp_lo[j] != (uint32_t)K;
        }
        if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(p.grp_flag, 1);
    }
    grid.sync();
    phase_mark(2);
    const bool contig = __ldcg(p.grp_flag) == 0;  // grid-uniform

    block_prefix_smem(p.blk_chunk, G, s_pre, s_w);
    // global compaction base of this block's chunks (the apply launch has its own grid; only
    // the fused step compacts)
    if (p.compact)
        for (int64_t c = c_lo + threadIdx.x; c < c_hi; c += COOP_THREADS)
            p.chunk_gbase[c] = s_pre[B] + p.chunk_base[c];
    // n_g = masked tokens in [off_g, off_{g+1}) from prefix differences (exact integers), one
    // masked_before per trajectory bound: warp iteration i covers bounds 31i .. 31i + 31 (lane
    // L: bound 31i + L) and writes n_g of trajectories 31i .. 31i + 30 from the next lane's
    // bound.  NG_U iterations' loads are issued together (this phase is latency-bound).
    {
        constexpr int NG_U = 4;
        const int lane = threadIdx.x & 31;
        const int64_t wg = gtid >> 5, nwg = gstride >> 5;
        const int64_t n_it = ((int64_t)p.n_traj + 30) / 31;
        for (int64_t i0 = wg; i0 < n_it; i0 += NG_U * nwg) {
            int64_t t[NG_U];
            int32_t mb[NG_U];
#pragma unroll
            for (int u = 0; u < NG_U; ++u) {
                const int64_t i = i0 + u * nwg, k = i * 31 + lane;
                t[u] = (i < n_it && k <= p.n_traj) ? p.off[k] : -1;
            }
#pragma unroll
            for (int u = 0; u < NG_U; ++u) mb[u] = t[u] >= 0 ? masked_before(p, s_pre, G, t[u]) : 0;
#pragma unroll
            for (int u = 0; u < NG_U; ++u) {
                const int64_t i = i0 + u * nwg, g = i * 31 + lane;
                const int32_t mn = __shfl_down_sync(0xffffffffu, mb[u], 1);
                const int64_t tn = __shfl_down_sync(0xffffffffu, t[u], 1);
                if (lane < 31 && i < n_it && g < p.n_traj) p.n_g[g] = tn > t[u] ? mn - mb[u] : 0;
            }
        }
    }
    if (contig) {
        grid.sync();  // every n_g written
        phase_mark(3);
        phase_mark(4);
    } else {
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
    {
        // BATCH trajectories per thread at a time: their loads, then their slot atomics are
        // issued together (one dependent round trip per batch instead of per trajectory)
        constexpr int BATCH = 4;
        for (int64_t g0 = gtid; g0 < p.n_traj; g0 += BATCH * gstride) {
            int32_t jj[BATCH], sl[BATCH], gs[BATCH];
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int64_t g = g0 + u * gstride;
                jj[u] = -1;
                if (g < p.n_traj) {
                    const int32_t j = p.group_id[g], i = p.task_id[g];
                    if (j >= 0 && j < p.n_groups && i >= 0 && i < p.n_tasks) jj[u] = j;
                }
            }
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
                if (jj[u] >= 0) {
                    sl[u] = atomicAdd(&p.grp_fill[jj[u]], 1);
                    gs[u] = p.grp_start[jj[u]];
                }
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
                if (jj[u] >= 0) {
                    const int64_t owner = part_owner(p.n_groups, jj[u], G);
                    p.members[s_pre[owner] + gs[u] + sl[u]] = (int32_t)(g0 + u * gstride);
                }
        }
    }
    grid.sync();
    phase_mark(4);
    }  // !contig

    // phase B3: this block's groups, then the block's per-task partial (N, S, Q) in a fixed
    // order.  Groups of <= REG_K members: ids sorted by a register sorting network and their
    // reward / task / count loads issued together (no dependent global round trips).
    unsigned long long nz = 0;
    // at most one group per thread (the usual case): its (task, N, S, Q) stay in registers for
    // the per-task partials below instead of being re-read from global per task
    const bool one_per_thread = j_hi - j_lo <= COOP_THREADS;
    int32_t my_task = -1;
    double my_N = 0.0, my_S = 0.0, my_Q = 0.0;
    for (int64_t j = j_lo + threadIdx.x; j < j_hi; j += COOP_THREADS) {
        const int32_t K = p.grp_cnt[j];
        int32_t* mbg = contig ? nullptr : p.members + s_pre[B] + p.grp_start[j];
        double N, S, Q;
        int32_t task0;
        if (contig) {  // members first_j .. first_j + K - 1: already in index order
            const int32_t f = (int32_t)~p.grp_lo[j];
            int32_t m[REG_K];
#pragma unroll
            for (int a = 0; a < REG_K; ++a) m[a] = a < K ? f + a : INT_MAX;
            group_regs(p, K, m, N, S, Q, task0, st, nz);
        } else if (K <= REG_K) {
            int32_t m[REG_K];
#pragma unroll
            for (int a = 0; a < REG_K; ++a) m[a] = a < K ? mbg[a] : INT_MAX;
#pragma unroll
            for (int k2 = 2; k2 <= REG_K; k2 <<= 1)
#pragma unroll
                for (int jj = k2 >> 1; jj > 0; jj >>= 1)
#pragma unroll
                    for (int i = 0; i < REG_K; ++i) {
                        const int l = i ^ jj;
                        if (l > i) {
                            const bool up = (i & k2) == 0;
                            const int32_t a0 = m[i], b0 = m[l];
                            if ((a0 > b0) == up) {
                                m[i] = b0;
                                m[l] = a0;
                            }
                        }
                    }
            group_regs(p, K, m, N, S, Q, task0, st, nz);
        } else {
            for (int a = 1; a < K; ++a) {
                const int32_t x = mbg[a];
                int b = a - 1;
                while (b >= 0 && mbg[b] > x) {
                    mbg[b + 1] = mbg[b];
                    --b;
                }
                mbg[b + 1] = x;
            }
            group_adv(
                p, K, mbg, [&](int32_t g) { return p.rewards[g]; },
                [&](int32_t g) { return p.task_id[g]; }, [&](int32_t g) { return p.n_g[g]; }, N,
                S, Q, task0, st, nz);
        }
        p.grp_task[j] = task0;
        p.grp_nsq[3 * j + 0] = N;
        p.grp_nsq[3 * j + 1] = S;
        p.grp_nsq[3 * j + 2] = Q;
        my_task = task0;
        my_N = N;
        my_S = S;
        my_Q = Q;
    }
    {  // one atomic per block (same-address atomics from every thread serialise at L2)
        int32_t nzt = 0;
        (void)coop_block_exscan((int32_t)nz, s_w, nzt);
        if (threadIdx.x == 0 && nzt)
            atomicAdd(reinterpret_cast<unsigned long long*>(&p.meta[3]),
                      (unsigned long long)nzt);  // integer: exact
    }
    __syncthreads();
    {
        __shared__ double s_wp[NWARPS][TASK_BATCH][3];
        const int warp_b = threadIdx.x >> 5, lane_b = threadIdx.x & 31;
        for (int32_t i0 = 0; i0 < p.n_tasks; i0 += TASK_BATCH) {
            const int32_t nb = min(TASK_BATCH, p.n_tasks - i0);
            for (int32_t ii = 0; ii < nb; ++ii) {
                double N = 0.0, S = 0.0, Q = 0.0;
                if (one_per_thread) {
                    if (my_task == i0 + ii) {
                        N = my_N;
                        S = my_S;
                        Q = my_Q;
                    }
                } else {
                    for (int64_t j = j_lo + threadIdx.x; j < j_hi; j += COOP_THREADS)
                        if (p.grp_task[j] == i0 + ii) {
                            N += p.grp_nsq[3 * j];
                            S += p.grp_nsq[3 * j + 1];
                            Q += p.grp_nsq[3 * j + 2];
                        }
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

    // phase B4 by the LAST block to finish B3 (a ticket instead of a grid barrier: every block
    // fences its partials before taking its ticket, so the last one sees them all): per-task
    // moments over the token set = fixed-order sum of the block partials (warp w
    // handles tasks w, w+8, ...; lanes stride over blocks; the same bits whichever block it is).
    // The ticket grp_fill[n_groups] is zeroed with the member-list counters before the launch.
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&p.grp_fill[p.n_groups], 1) == (int)G - 1;
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (s_last) {
        phase_mark(5, (unsigned)B);
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        for (int32_t i = wid; i < p.n_tasks; i += NWARPS) {
            double N = 0.0, S = 0.0, Q = 0.0;
            for (int64_t b = lane; b < G; b += 32) {
                const double* bp = p.blk_part + 3 * (b * p.n_tasks + i);
                N += __ldcg(bp);
                S += __ldcg(bp + 1);
                Q += __ldcg(bp + 2);
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
        if (threadIdx.x == 0)  // G (local)
            p.stats[3 * p.n_tasks] = (double)__ldcg(reinterpret_cast<const long long*>(p.meta + 3));
    }
}

// phase C of the large driver (round 2, lean apply; its own launch and one-wave grid).
// A warp takes a unit of APPLY_SC consecutive 512-token chunks; units are strided over every
// warp of the grid (equal work per warp: no block-range tail).  All loads of a unit are issued
// together (one memory round trip per 4 chunks: the launch is otherwise latency-bound on these
// cold loads): the chunk -> first-trajectory table gives g0 (holding the unit's first token,
// loaded one unit ahead); lane L loads the start, A^ and task of trajectory g0 + 1 + L, and a
// ballot finds the starts inside the unit (sorted: a prefix of the lanes); each lane computes
// Eq.1 for the trajectory it loaded, and shuffles broadcast the values.  Lane L
// writes the float4s of tokens q*128 + 4L .. +3 (q = 0..3) of each chunk, so every store
// instruction writes 512 contiguous bytes with no shared-memory transpose.  The mask comes from
// phase A's stored lane bits (64 B per chunk instead of 512 mask bytes).  Compaction positions
// (fused step): the statistics launch's global chunk base + the popcount of the chunk's bits
// below the token.  A unit with 32 or more trajectory starts (trajectories shorter than ~64
// tokens) takes its chunks one at a time with global batches of starts.
constexpr int APPLY_THREADS = 256;
static_assert(APPLY_THREADS == COOP_THREADS && POP_THREADS == COOP_THREADS,
              "coop_grid sizes the one-wave grids with COOP_THREADS");
#ifndef ADV_APPLY_MINB
#define ADV_APPLY_MINB 2  // resident blocks per SM the apply launch's register budget is cut for
#endif
#ifndef ADV_APPLY_SC
#define ADV_APPLY_SC 8  // 512-token chunks per warp unit of the apply (one load round trip each)
#endif
constexpr int APPLY_SC = ADV_APPLY_SC;
#ifndef ADV_APPLY_PF
#define ADV_APPLY_PF 1  // 1: a unit's loads are issued while the previous unit is processed
#endif
#ifndef ADV_APPLY_DIAG
#define ADV_APPLY_DIAG 0  // timing experiment: stores only (wrong results; never a product build)
#endif
#ifndef ADV_APPLY_PDL
#define ADV_APPLY_PDL 1  // 1: the apply is a programmatic dependent launch of the statistics
#endif
// Eq.1 value of trajectory g as float bits (the arithmetic of adv_tilde)
__device__ __forceinline__ uint32_t adv_tilde_u(const double2* s_task, int32_t n_tasks, double ah,
                                                int32_t ti) {
    return (ti >= 0 && ti < n_tasks) ? __float_as_uint((float)((ah - s_task[ti].x) / s_task[ti].y))
                                     : 0u;
}

// the 16 values of one 512-token chunk c from its own trajectory starts, 32 starts per global
// batch (a unit with 32 or more trajectory starts: trajectories shorter than ~64 tokens)
// mask (the chunk's stored lane bits bk), store the 16 values of one chunk starting at token cbk
// and, in the fused step, its compaction (global base gbk)
__device__ __forceinline__ void apply_emit(const AdvParams& p, int64_t cbk, uint32_t (&o)[16],
                                           uint32_t bk, int32_t gbk, bool vec_ok) {
    const int lane = threadIdx.x & 31;
    // the mask bits of tokens q*128 + 4L .. +3 sit in lane (8q + L/4)'s 16 bits,
    // nibble L%4
    const int sh = (lane & 3) * 4;
    if (!p.compact && vec_ok && cbk + WCHUNK <= p.T) {  // the common case: no per-vector checks
        uint4* dst = reinterpret_cast<uint4*>(p.adv_tok + cbk) + lane;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t nib = __shfl_sync(0xffffffffu, bk, 8 * q + (lane >> 2)) >> sh;
            dst[32 * q] = make_uint4((nib & 1u) ? o[4 * q] : 0u, (nib & 2u) ? o[4 * q + 1] : 0u,
                                     (nib & 4u) ? o[4 * q + 2] : 0u, (nib & 8u) ? o[4 * q + 3] : 0u);
        }
        return;
    }
    int32_t E = 0;
    if (p.compact) {
        const int32_t pc = __popc(bk);
        E = warp_incl_scan(pc) - pc;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t word = __shfl_sync(0xffffffffu, bk, 8 * q + (lane >> 2));
        const uint32_t nib = (word >> sh) & 0xfu;
#pragma unroll
        for (int e = 0; e < 4; ++e) o[4 * q + e] = ((nib >> e) & 1u) ? o[4 * q + e] : 0u;
        const int64_t t = cbk + q * 128 + 4 * lane;
        if (vec_ok && t + 4 <= p.T) {
            *reinterpret_cast<uint4*>(p.adv_tok + t) =
                make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (t + e < p.T) p.adv_tok[t + e] = __uint_as_float(o[4 * q + e]);
        }
        if (p.compact) {
            const int32_t Eq = __shfl_sync(0xffffffffu, E, 8 * q + (lane >> 2));
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if ((nib >> e) & 1u) {
                    const int32_t pos = gbk + Eq + __popc(word & ((1u << (sh + e)) - 1u));
                    p.idx[pos] = (int32_t)(t + e);
                    p.adv_c[pos] = __uint_as_float(o[4 * q + e]);
                }
        }
    }
}

__device__ __forceinline__ void apply_chunk_global(const AdvParams& p, const double2* s_task, int64_t c,
                                                uint32_t bk, int32_t gbk, bool vec_ok) {
    uint32_t o[16];
    const int lane = threadIdx.x & 31;
    const int32_t last = p.n_traj - 1;
    const int64_t cb = c * WCHUNK;
    const int32_t g0 = min(max(p.chunk_first[c], 0), last);
    const uint32_t v0 = adv_tilde_u(s_task, p.n_tasks, p.adv_hat[g0], p.task_id[g0]);
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i] = v0;
    for (int64_t gs = (int64_t)g0 + 1 + lane;; gs += 32) {
        const bool ex = gs <= last;
        const int64_t so = ex ? p.off[gs] : LLONG_MAX;
        const bool in = so < cb + WCHUNK;
        const int32_t rel = in ? (int32_t)(so - cb) : WCHUNK;
        const uint32_t v = in ? adv_tilde_u(s_task, p.n_tasks, p.adv_hat[gs], p.task_id[gs]) : 0u;
        const int nb = __popc(__ballot_sync(0xffffffffu, in));
        for (int j = 0; j < nb; ++j) {
            const int32_t sj = __shfl_sync(0xffffffffu, rel, j);
            const uint32_t vj = __shfl_sync(0xffffffffu, v, j);
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    o[4 * q + e] = q * 128 + 4 * lane + e >= sj ? vj : o[4 * q + e];
        }
        if (nb < 32) break;
    }
    apply_emit(p, c * WCHUNK, o, bk, gbk, vec_ok);
}

__global__ void __launch_bounds__(APPLY_THREADS, ADV_APPLY_MINB) k_adv_large_apply(const AdvParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    double2* s_task = reinterpret_cast<double2*>(smem);
#if ADV_APPLY_PDL
    // launched as a programmatic dependent of the statistics launch (no communicator): wait
    // until that grid has completed and its memory is visible before reading anything it wrote
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    phase_mark(6);
    task_params_smem(p, s_task);
    if (blockIdx.x == 0 && threadIdx.x < 32) {  // local masked rows = sum of the stats blocks'
        int32_t s = 0;                          // totals (exact integers, any order)
        for (int32_t b = threadIdx.x; b < p.g_stats; b += 32) s += p.blk_chunk[b];
        s = __reduce_add_sync(0xffffffffu, s);
        publish_meta(p, s);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    constexpr int WPB = APPLY_THREADS / 32;
    constexpr int32_t USPAN = APPLY_SC * WCHUNK;  // tokens per unit
    const int64_t n_units = (p.n_chunks + APPLY_SC - 1) / APPLY_SC;
    const int64_t nw = (int64_t)gridDim.x * WPB;
    const int64_t gw = (int64_t)blockIdx.x * WPB + (threadIdx.x >> 5);
    // units strided over the warps (the grid writes one advancing front; a contiguous range
    // per warp measured 5% slower at 2^27)
    int64_t u = gw;
    const int64_t u_end = n_units, u_step = nw;
    const bool any = p.n_traj > 0;
    const bool vec_ok = (reinterpret_cast<uintptr_t>(p.adv_tok) & 15) == 0;
    const int32_t last = p.n_traj - 1;
    // a unit's loads: the lane bits of its chunks, A^ / task of g0 (uniform) and of trajectory
    // g0 + 1 + lane with its start (issued together; with ADV_APPLY_PF one unit ahead)
    struct UnitLd {
        uint32_t bits[APPLY_SC];
        double ah0, ah;
        int32_t ti0, ti;
        int64_t so;
    };
    auto load_unit = [&](int64_t uu, int32_t gf) {
        UnitLd L;
        const int64_t c0 = uu * APPLY_SC;
        const int32_t g0 = min(max(gf, 0), max(last, 0));
#pragma unroll
        for (int k = 0; k < APPLY_SC; ++k)
            L.bits[k] = (any && c0 + k < p.n_chunks) ? (uint32_t)p.lanebits[(c0 + k) * 32 + lane] : 0u;
        L.ah0 = L.ah = 0.0;
        L.ti0 = L.ti = -1;
        L.so = LLONG_MAX;
        if (any) {
            L.ah0 = p.adv_hat[g0];
            L.ti0 = p.task_id[g0];
            const int64_t gs = (int64_t)g0 + 1 + lane;
            if (gs <= last) {
                L.so = p.off[gs];
                L.ah = p.adv_hat[gs];
                L.ti = p.task_id[gs];
            }
        }
        return L;
    };
    int32_t g_next = (any && u < u_end) ? p.chunk_first[u * APPLY_SC] : 0;
#if ADV_APPLY_PF
    UnitLd nxt;
    if (u < u_end) {
        nxt = load_unit(u, g_next);
        g_next = (any && u + u_step < u_end) ? p.chunk_first[(u + u_step) * APPLY_SC] : 0;
    }
#endif
    for (; u < u_end; u += u_step) {
        const int64_t c0 = u * APPLY_SC, cb = c0 * WCHUNK;
        const int nsub = (int)min((int64_t)APPLY_SC, p.n_chunks - c0);
#if ADV_APPLY_DIAG  // timing experiment only (NOT the method): the unit's stores alone
        for (int k = 0; k < nsub; ++k)
            if (cb + (k + 1) * WCHUNK <= p.T)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    reinterpret_cast<uint4*>(p.adv_tok + cb + k * WCHUNK)[32 * q + lane] =
                        make_uint4(0u, 0u, 0u, 0u);
        continue;
#endif
#if ADV_APPLY_PF
        const UnitLd L = nxt;
        if (u + u_step < u_end) nxt = load_unit(u + u_step, g_next);
        if (any && u + 2 * u_step < u_end) g_next = p.chunk_first[(u + 2 * u_step) * APPLY_SC];
#else
        const UnitLd L = load_unit(u, g_next);
        if (any && u + u_step < u_end) g_next = p.chunk_first[(u + u_step) * APPLY_SC];  // ahead
#endif
        const uint32_t(&bits)[APPLY_SC] = L.bits;
        const uint32_t v0 = any ? adv_tilde_u(s_task, p.n_tasks, L.ah0, L.ti0) : 0u;
        const bool in = L.so < cb + USPAN;  // starts are sorted: the in-lanes are a prefix
        const int32_t rel = in ? (int32_t)(L.so - cb) : USPAN;
        const uint32_t v = in ? adv_tilde_u(s_task, p.n_tasks, L.ah, L.ti) : 0u;
        const bool many = __ballot_sync(0xffffffffu, in) == 0xffffffffu;  // >= 32 starts
#pragma unroll 1
        for (int k = 0; k < nsub; ++k) {  // not unrolled: a small loop body stays in the I-cache
            const int32_t lo = k * WCHUNK;  // the chunk's first token, unit-relative
            uint32_t bk = bits[0];
#pragma unroll
            for (int i = 1; i < APPLY_SC; ++i) bk = k == i ? bits[i] : bk;  // no local memory
            const int32_t gbk = p.compact ? p.chunk_gbase[c0 + k] : 0;  // (fused step only)
            uint32_t o[16];
            if (!any) {
#pragma unroll
                for (int i = 0; i < 16; ++i) o[i] = 0u;
            } else if (!many) {
                // value at the chunk's first token: the last start at or before it; then the
                // starts inside the chunk (lanes ka .. kb - 1) overwrite in order
                const int ka = __popc(__ballot_sync(0xffffffffu, in && rel <= lo));
                const int kb = __popc(__ballot_sync(0xffffffffu, in && rel < lo + WCHUNK));
                const uint32_t vs = ka ? __shfl_sync(0xffffffffu, v, max(ka - 1, 0)) : v0;
                // per float4 of the lane: one value unless a start falls strictly inside it
                uint32_t w[4] = {vs, vs, vs, vs};
                bool split = false;
                for (int j = ka; j < kb; ++j) {
                    // start relative to the lane's first token of float4 q = 0
                    const int32_t dj = __shfl_sync(0xffffffffu, rel, j) - lo - 4 * lane;
                    const uint32_t vj = __shfl_sync(0xffffffffu, v, j);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int32_t r = dj - q * 128;  // relative to float4 q's first token
                        w[q] = r <= 0 ? vj : w[q];
                        split |= (uint32_t)(r - 1) < 3u;  // at element 1..3 of the float4
                    }
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) o[i] = w[i >> 2];
                if (__any_sync(0xffffffffu, split)) {  // rare: element-wise over the starts
#pragma unroll
                    for (int i = 0; i < 16; ++i) o[i] = vs;
                    for (int j = ka; j < kb; ++j) {
                        const int32_t dj = __shfl_sync(0xffffffffu, rel, j) - lo - 4 * lane;
                        const uint32_t vj = __shfl_sync(0xffffffffu, v, j);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                o[4 * q + e] = q * 128 + e >= dj ? vj : o[4 * q + e];
                    }
                }
            } else {
                apply_chunk_global(p, s_task, c0 + k, bk, gbk, vec_ok);
                continue;
            }
            apply_emit(p, cb + lo, o, bk, gbk, vec_ok);
        }
    }
    phase_mark(7);
}

// static shared memory of the kernels (the rest is the dynamic Lay arena)
struct CoopStatic {
    int32_t s_w[NWARPS];
    int32_t s_pre[GMAX_BLOCKS + 1];
};

__global__ void __launch_bounds__(COOP_THREADS, ADV_LARGE_MINB) k_adv_large_stats(const AdvParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ CoopStatic ss;
    cg::grid_group grid = cg::this_grid();
    large_stats_phases(p, smem, grid, ss.s_w, ss.s_pre);
}
// phase C of the second launch (after the all-reduce): everything reloaded, mu, sigma from the
// reduced stats, A^ and task ids from global
__device__ __forceinline__ void small_apply(const AdvParams& p, uint8_t* smem, WarpRing& r,
                                            int32_t* s_pre, int32_t* s_w) {
    int64_t c_lo, c_hi;
    small_range(p, c_lo, c_hi);
    const int64_t* s_off = reinterpret_cast<const int64_t*>(smem + p.lay.soff);
    load_task_params(p, smem, s_pre, s_w);
    int32_t dummy = 0;
    stream_phase<1>(p, smem, r, c_lo, c_hi, true, s_off, s_pre[blockIdx.x], dummy, false);
}

// phase stamps (agentrl_debug_adv_phase_ns), small driver, block 0: [0] start, [1] trajectory
// table staged, [2] group advantages done, [3] counts done, [4] partial moments written, [5] after
// the grid barrier, [6] moments done, [7] apply done
__global__ void __launch_bounds__(COOP_THREADS, 1) k_adv_small_all(const AdvParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ CoopStatic ss;
    cg::grid_group grid = cg::this_grid();
    phase_mark(0);
    WarpRing r = ring_setup(p, smem);
    small_pre_barrier(p, smem, r, ss.s_w);
    grid.sync();
    phase_mark(5);
    small_moments(p, smem, ss.s_pre, ss.s_w, false);  // every block: mu_i, sigma_i, bases
    phase_mark(6);
    int64_t c_lo, c_hi;
    small_range(p, c_lo, c_hi);
    const int64_t* s_off = reinterpret_cast<const int64_t*>(smem + p.lay.soff);
    const SmallT a = small_t(p, smem);
    const NgRegs ng = small_ng_load(p, s_off);
    int32_t dummy = 0;
    // the mask is still in the ring from phase A; A^ and task ids from smem
    stream_phase<1>(p, smem, r, c_lo, c_hi, true, s_off, ss.s_pre[blockIdx.x], dummy, true,
                    NoPre(), a.ah, a.tid);
    phase_mark(7);
    small_ng_store(p, ng);
}
__global__ void __launch_bounds__(COOP_THREADS, 1) k_adv_small_stats(const AdvParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ CoopStatic ss;
    cg::grid_group grid = cg::this_grid();
    WarpRing r = ring_setup(p, smem);
    small_pre_barrier(p, smem, r, ss.s_w);
    grid.sync();
    small_moments(p, smem, ss.s_pre, ss.s_w, true);  // block 0: raw (N, S, Q) and G
    small_ng_store(p, small_ng_load(p, reinterpret_cast<const int64_t*>(smem + p.lay.soff)));
}
__global__ void __launch_bounds__(COOP_THREADS, 1) k_adv_small_apply(const AdvParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ CoopStatic ss;
    stage_all_offsets(p, smem);
    WarpRing r = ring_setup(p, smem);
    small_apply(p, smem, r, ss.s_pre, ss.s_w);  // block 0 publishes meta / task_stats
}

static int coop_grid(const void* kern, size_t smem, int64_t want) {
    // occupancy per (kernel, dynamic smem, device), cached: keeps the per-call host work small
    struct Key {
        const void* k;
        size_t smem;
        int dev;
        int per_sm;
    };
    static thread_local Key cache[16];
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
        cache[n_cache % 16] = Key{kern, smem, dev, per_sm};
        n_cache = n_cache < 16 ? n_cache + 1 : 16;
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
    p.grp_lo = reinterpret_cast<uint32_t*>(ws + w.grp_lo);
    p.grp_hi = reinterpret_cast<uint32_t*>(ws + w.grp_hi);
    p.grp_flag = reinterpret_cast<int32_t*>(ws + w.grp_flag);
    p.members = reinterpret_cast<int32_t*>(ws + w.members);
    p.grp_task = reinterpret_cast<int32_t*>(ws + w.grp_task);
    p.chunk_first = reinterpret_cast<int32_t*>(ws + w.chunk_first);
    p.blk_chunk = reinterpret_cast<int32_t*>(ws + w.blk_chunk);
    p.chunk_base = reinterpret_cast<int32_t*>(ws + w.wchunk_base);
    p.blk_grp = reinterpret_cast<int32_t*>(ws + w.blk_grp);
    p.blk_cnt = reinterpret_cast<int32_t*>(ws + w.blk_cnt);
    p.lanebits = reinterpret_cast<uint16_t*>(ws + w.lanebits);
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
    // AGENTRL_ADV_SMALL=0 (build): always the large driver (A/B and layout tests)
    const bool small = AGENTRL_ADV_SMALL && b->n_traj <= SMALL_TRAJ &&
                       b->n_groups <= SMALL_GROUPS && b->n_tasks <= 64;
    p.chunk_gbase = reinterpret_cast<int32_t*>(ws + w.chunk_gbase);
    p.g_stats = 0;
    {  // dynamic smem attribute, per device, set once for every kernel of this file
        static std::atomic<uint64_t> done[5];
        const void* ks[5] = {(const void*)k_adv_small_all, (const void*)k_adv_small_stats,
                             (const void*)k_adv_small_apply, (const void*)k_adv_large_stats,
                             (const void*)k_adv_large_apply};
        for (int i = 0; i < 5; ++i)
            if (!func_attr_once(done[i], ks[i], 200 * 1024)) return AGENTRL_ERR_UNSUPPORTED;
    }
    void* args[] = {&p};
    if (small) {
        p.lay = make_lay(b->n_tasks, compact, true, b->n_traj, b->n_groups);
        const size_t smem = p.lay.total;
        if (smem > 200 * 1024) return AGENTRL_ERR_UNSUPPORTED;
        const int64_t want = std::max<int64_t>(ceil_div(p.n_chunks, NWARPS), 1);  // a chunk per warp
        if (!comm) {
            const int grid = coop_grid((const void*)k_adv_small_all, smem, want);
            if (!grid) return AGENTRL_ERR_UNSUPPORTED;
            p.g_stats = grid;
            ProfScope ps(KID_STATS, stream);
            AG_CUDA(cudaLaunchCooperativeKernel((const void*)k_adv_small_all, grid, COOP_THREADS,
                                                args, smem, stream));
            count_launch();
            return AGENTRL_OK;
        }
        const int grid = std::min(coop_grid((const void*)k_adv_small_stats, smem, want),
                                  coop_grid((const void*)k_adv_small_apply, smem, want));
        if (!grid) return AGENTRL_ERR_UNSUPPORTED;
        p.g_stats = grid;
        {
            ProfScope ps(KID_STATS, stream);
            AG_CUDA(cudaLaunchCooperativeKernel((const void*)k_adv_small_stats, grid, COOP_THREADS,
                                                args, smem, stream));
            count_launch();
        }
        int rc = comm_allreduce_f64(comm, p.stats, (size_t)3 * b->n_tasks + 1, stream);
        if (rc != AGENTRL_OK) return rc;
        ProfScope ps(KID_APPLY, stream);
        // same grid as the stats launch: phase C reuses its contiguous chunk partition
        AG_CUDA(cudaLaunchKernel((const void*)k_adv_small_apply, grid, COOP_THREADS, args, smem,
                                 stream));
        count_launch();
        return AGENTRL_OK;
    }
    // large driver: popcount stream -> cooperative statistics -> [C1] -> apply stream
    {
        ProfScope ps(KID_STATS, stream);
        // K_j, the member-list fill counters (+ the B4 ticket), the group bounds and the
        // contiguity flag start at zero (contiguous in the workspace)
        AG_CUDA(cudaMemsetAsync(p.grp_cnt, 0,
                                (size_t)(reinterpret_cast<uint8_t*>(p.grp_flag + 4) -
                                         reinterpret_cast<uint8_t*>(p.grp_cnt)),
                                stream));
        const int64_t pop_want = std::max<int64_t>(
            ceil_div(p.n_chunks, (int64_t)POP_UNROLL * (POP_THREADS / 32)), 1);
        // one wave: a second partial wave of blocks left a tail (1,184 blocks for 888 slots)
        const int pop_grid = coop_grid((const void*)k_adv_large_pop, 0, pop_want);
        if (!pop_grid) return AGENTRL_ERR_UNSUPPORTED;
        k_adv_large_pop<<<pop_grid, POP_THREADS, 0, stream>>>(p);
        count_launch();
        AG_CUDA(cudaGetLastError());
        const int64_t want = std::max<int64_t>({ceil_div(p.n_chunks, NWARPS),
                                                ceil_div(p.n_traj, COOP_THREADS),
                                                ceil_div(p.n_groups, COOP_THREADS), 1});
        const int grid = coop_grid((const void*)k_adv_large_stats, 0, want);
        if (!grid) return AGENTRL_ERR_UNSUPPORTED;
        p.g_stats = grid;
        AG_CUDA(cudaLaunchCooperativeKernel((const void*)k_adv_large_stats, grid, COOP_THREADS,
                                            args, 0, stream));
        count_launch();
    }
    if (comm) {
        int rc = comm_allreduce_f64(comm, p.stats, (size_t)3 * b->n_tasks + 1, stream);
        if (rc != AGENTRL_OK) return rc;
    }
    ProfScope ps(KID_APPLY, stream);
    const size_t smem = (size_t)16 * std::max(b->n_tasks, 1);  // per-task (mu, sigma)
    if (smem > 200 * 1024) return AGENTRL_ERR_UNSUPPORTED;
    // one wave (every block resident), chunks strided over its warps
    const int grid_a = coop_grid((const void*)k_adv_large_apply, smem,
                                 std::max<int64_t>(ceil_div(p.n_chunks, APPLY_THREADS / 32), 1));
    if (!grid_a) return AGENTRL_ERR_UNSUPPORTED;
    if (ADV_APPLY_PDL && !comm) {  // its launch overlaps the statistics launch's tail
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid_a);
        cfg.blockDim = dim3(APPLY_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelExC(&cfg, (const void*)k_adv_large_apply, args) != cudaSuccess) {
            // (a driver without programmatic dependent launch: an ordinary launch instead; the
            // kernel's griddepcontrol.wait then returns at once)
            (void)cudaGetLastError();
            AG_CUDA(cudaLaunchKernel((const void*)k_adv_large_apply, grid_a, APPLY_THREADS,
                                     args, smem, stream));
        }
    } else {
        AG_CUDA(cudaLaunchKernel((const void*)k_adv_large_apply, grid_a, APPLY_THREADS, args,
                                 smem, stream));
    }
    count_launch();
    return AGENTRL_OK;
}

int debug_adv_phase_ns(unsigned long long* host8) {
    return cudaMemcpyFromSymbol(host8, g_adv_phase_ns, sizeof(unsigned long long) * 8) ==
                   cudaSuccess
               ? AGENTRL_OK
               : AGENTRL_ERR_CUDA;
}

}  // namespace agentrl
