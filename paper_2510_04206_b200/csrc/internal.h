// internal.h -- host-side declarations shared by the CUDA translation units of libagentrl.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <atomic>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys / ncu --nvtx, no-ops without a tool

#include "../../include/agentrl.h"

namespace agentrl {

constexpr int CHUNK_TOKENS = 4096;  // tokens per block in the token-parallel kernels
constexpr int CHUNK_THREADS = 256;  // 16 tokens per thread

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over the caller's workspace (offsets only; the plan is computed identically
// by the *_workspace_size() query and by the entry point).
struct WsPlan {
    size_t off = 0;
    size_t take(size_t bytes, size_t align = 256) {
        off = align_up(off, align);
        size_t o = off;
        off += bytes;
        return o;
    }
};

// ---- part 1 workspace (see adv_norm.cu) ----
struct AdvWs {
    size_t n_g, chunk_cnt, chunk_base, grp_cnt, grp_start, grp_fill, members;  // int32
    size_t grp_lo, grp_hi;  // uint32 [n_groups + 1]: ~(first member), last member + 1 (large
                            // coop driver: atomicMax from zero; contiguous-group check)
    size_t grp_flag;        // int32 [4]: [0] some group is not one contiguous run of <= 16
    size_t adv_hat;                                                               // double
    size_t grp_task;  // int32 [n_groups] task of each group (cooperative path)
    size_t grp_nsq;   // double [3*n_groups] per-group (N, S, Q) partials (cooperative path)
    size_t chunk_first;  // int32 [n_chunks] trajectory holding each chunk's first token
    size_t blk_chunk, blk_grp, blk_part;  // per cooperative block: int32, int32, double[3*n_tasks]
    size_t wchunk_base;                   // int32 [n_chunks] local compaction base per chunk
    size_t chunk_gbase;                   // int32 [n_chunks] global compaction base (large)
    size_t blk_cnt;  // int32 [n_traj + 2049] per-block trajectory counts (small coop driver)
    size_t lanebits;  // uint16 [n_chunks * 32] per-lane mask bits (large coop driver)
    size_t stats;     // double [3*n_tasks]: N_i, S_i, Q_i (local, then global)
    size_t meta;      // int64 [4]: n_mask_local, n_mask_global, pad
    size_t idx;       // int32 [T] compacted token positions
    size_t adv_c;     // float [T] compacted advantages
    size_t total;
};
AdvWs plan_adv(int64_t T, int32_t n_traj, int32_t n_groups, int32_t n_tasks, size_t base = 0);

// Cooperative single-kernel path (adv_coop.cu); returns AGENTRL_ERR_UNSUPPORTED if the grid
// cannot be co-resident (caller falls back to the 3-kernel path).
int launch_adv_norm_coop(const agentrl_batch* b, double eps_std, float* adv_tok,
                         double* task_stats, int64_t* n_mask_global, uint8_t* ws, const AdvWs& w,
                         agentrl_comm comm, int32_t* d_status, cudaStream_t stream,
                         bool compact);

// Enqueue part 1.  Returns AGENTRL_* code.  comm may be null.
// compact: also write the compaction (idx / adv_c) that part 2 consumes (fused step only)
int launch_adv_norm(const agentrl_batch* b, double eps_std, float* adv_tok, double* task_stats,
                    int64_t* n_mask_global, uint8_t* ws, const AdvWs& w, agentrl_comm comm,
                    int32_t* d_status, cudaStream_t stream, bool compact = true);

// ---- part 2 workspace (see lmhead.cu) ----
struct LossWs {
    size_t idx, meta;                       // int32 [T] (standalone path), int64 [4]
    size_t chunk_cnt, chunk_base;           // int32 compaction scratch (standalone path)
    size_t tgt_c, old_c;                    // compacted per-row inputs [rows_cap]
    size_t adv_c;                           // float [T] compacted advantages (standalone path)
    size_t H;                               // bf16 [rows_cap, d] gathered hidden rows
    size_t P;                               // bf16 [rows_cap, V]: P~ = exp(z - m_tile)
    size_t part;                            // float2 [rows_cap, n_tiles] (m_tile, l'_tile)
    size_t fscale;                          // float [rows_cap, n_tiles] gradient scale f
    size_t xrow;                            // int2 [rows_cap] (target column, G value bits)
    size_t zy;                              // float [rows_cap]
    size_t row_term, row_rho, row_logp;     // double/float per row
    size_t row_clip;                        // int32 per row
    size_t row_kl, w_c, ref_c;              // float per row: KL_t, weight w_t, ref log-prob
    size_t rows_eff;                        // int64 [2]: min(T_eff, rows_cap)
    size_t sched;                           // int [32] GEMM tile counters (dynamic scheduler)
    size_t prog;                            // int64 [3][PROG_UNITS] GEMM progress
    int32_t ksplit;                         // grad_hidden split-K factor (1: none)
    size_t splitk;                          // float [ksplit][rows_cap, d] partials (ksplit > 1)
    size_t vpstat;                          // vocab-parallel: float2 [world][rows_cap] (M_r, L'_r)
    size_t vp_gh;                           // vocab-parallel: float [rows_cap, d] grad_h partial
    int32_t vp_world;                       // 0 = not planned for the vocab-parallel head
    int64_t rows_cap;                       // row capacity (max_rows rounded up to 256)
    size_t total;
    int32_t n_tiles;
};
constexpr int PROG_UNITS = 256;  // >= GEMM units (SMs, or SM pairs)
int64_t loss_rows_cap(int64_t T, int64_t max_rows);
LossWs plan_loss(int64_t T, int64_t max_rows, int32_t d, int32_t V, size_t base = 0,
                 int32_t vp_world = 0);

// Enqueue part 2.  If `idx_dev` / `rows_dev` are given (fused step) the compaction is reused:
//   idx_dev  int32 [T] compacted token positions, rows_dev -> int64 number of rows (local T_eff),
//   adv_c    float [T] compacted advantages, nglob -> int64 global masked count.
// batch information the fused step hands to part 2 (GRPO group-mean weights, loss_agg == 1)
struct FusedExtras {
    const int64_t* off;   // traj_offsets [n_traj+1]
    int32_t n_traj;
    const int32_t* n_g;       // masked tokens per trajectory (part 1 workspace)
    const int32_t* group_id;  // [n_traj] (batch descriptor)
    const int32_t* grp_cnt;   // [n_groups] K_j, members per group (part 1 workspace)
    int32_t n_groups;
    const int64_t* ngrp;      // global number of groups with members, G (device)
};
int launch_policy_loss(const agentrl_loss_args* a, const agentrl_loss_out* o, uint8_t* ws,
                       const LossWs& w, const int32_t* idx_dev, const int64_t* rows_dev,
                       const float* adv_c_dev, const int64_t* nglob_dev, agentrl_comm comm,
                       int32_t* d_status, cudaStream_t stream,
                       const FusedExtras* fx = nullptr);

// ---- forward-only log-prob / entropy (lmhead.cu) ----
struct LogpWs {
    size_t idx, meta, chunk, tgt_c, H, part4, zy, sched, total;
    int64_t rows_cap;
    int32_t n_tiles;
};
LogpWs plan_logp(int64_t T, int64_t max_rows, int32_t d, int32_t V, size_t base = 0);
int launch_logprob(const agentrl_logprob_args* a, float* logp, float* entropy, uint8_t* ws,
                   const LogpWs& w, int32_t* d_status, cudaStream_t stream);

// ---- comm (comm.cpp) ----
int comm_allreduce_f64(agentrl_comm c, double* buf, size_t n, cudaStream_t s);
int comm_allreduce_f32(agentrl_comm c, float* buf, size_t n, cudaStream_t s);
int comm_allreduce_i64(agentrl_comm c, int64_t* buf, size_t n, cudaStream_t s);
int comm_reduce_scatter_f32(agentrl_comm c, float* buf, size_t n, cudaStream_t s);
int comm_world(agentrl_comm c);
int comm_rank(agentrl_comm c);

// ---- peer window (peer.cu): the grad_W reduce-scatter fused into the grad_W GEMM epilogue
struct PeerWindow {
    static constexpr int MAX_RANKS = 64;
    int world = 0, rank = 0;
    size_t bytes = 0;              // staging bytes per rank (world slots of one grad_W shard)
    float* staging = nullptr;      // this rank's window (cudaMalloc, comm-owned)
    int64_t* flags = nullptr;      // [2][world]: ready[r], consumed[o] epochs
    float** d_staging = nullptr;   // device [world]: every rank's window (IPC-mapped)
    int64_t** d_flags = nullptr;   // device [world]: every rank's flags
    int32_t* done_ctr = nullptr;   // reduce-kernel block counter
    int64_t* d_epoch = nullptr;    // device [1]: the current epoch (advanced by the guard
                                   // kernel, so a captured step replays with fresh epochs)
    void* opened[MAX_RANKS] = {};
    void* opened_flags[MAX_RANKS] = {};
};
int peer_window_create(agentrl_comm c, size_t bytes, PeerWindow** out);  // collective
void peer_window_destroy(PeerWindow* pw);
PeerWindow* comm_peer(agentrl_comm c);
bool peer_window_fits(const PeerWindow* pw, int32_t V, int32_t d);
int peer_guard(PeerWindow* pw, int32_t* d_status, cudaStream_t s);
int peer_signal_reduce(PeerWindow* pw, float* grad_W, int32_t V, int32_t d, int32_t* d_status,
                       cudaStream_t s);

// launch counter for the bench's gpu_launches claim
void count_launch(int n = 1);

// per-kernel event timing (agentrl_profile_start/stop)
enum KernelId {
    KID_COUNT = 0, KID_STATS, KID_APPLY, KID_COMPACT, KID_GATHER, KID_FWD, KID_ROWSTATS,
    KID_REDUCE, KID_GRADW, KID_GRADH, KID_LOGP_GEMM, KID_LOGP_MERGE, KID_N
};
void prof_mark(int kid, bool begin, cudaStream_t s);
struct ProfScope {  // per-kernel event timing and an NVTX range named after the kernel
    int kid;
    cudaStream_t s;
    ProfScope(int k, cudaStream_t st) : kid(k), s(st) {
        nvtxRangePushA(agentrl_kernel_name(kid));
        prof_mark(kid, true, s);
    }
    ~ProfScope() {
        prof_mark(kid, false, s);
        nvtxRangePop();
    }
};
struct NvtxRange {  // host-side range around an ABI call
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
constexpr int MAX_DEVICES = 64;  // per-device caches (device ids are taken modulo this)
int current_device();
int num_sms();  // of the current device
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (function, device): the attribute
// is per device, so a process or thread driving several GPUs sets it on each
bool func_attr_once(std::atomic<uint64_t>& done_mask, const void* func, int smem_bytes);
int debug_adv_phase_ns(unsigned long long* host8);
int debug_throttle_waits(unsigned long long* host3);
int check_device();  // AGENTRL_OK or AGENTRL_ERR_UNSUPPORTED / _CUDA

}  // namespace agentrl

#define AG_CUDA(x)                                     \
    do {                                               \
        cudaError_t e_ = (x);                          \
        if (e_ != cudaSuccess) return AGENTRL_ERR_CUDA; \
    } while (0)
