/*
 * agentrl.h -- C ABI of the B200-native (sm_100a) AgentRL hot-path library
 * (libagentrl.so).  Paper: arxiv 2510.04206 "AgentRL" (PAPER.md in the task's
 * reference; citations P:<line> below).
 *
 * Two operations and their composition:
 *   agentrl_task_adv_norm        GRPO group advantage followed by the
 *                                paper's task advantage normalization, sec 3.2
 *                                Eq.1, over the loss-masked
 *                                assistant tokens of each task in the GLOBAL
 *                                batch (all ranks).
 *   agentrl_policy_loss_fwd_bwd  token-level PPO-clip loss with
 *                                the DAPO token-level mean through
 *                                the LM head (token factorisation P:1182-1190),
 *                                and its exact gradients grad_hidden, grad_W.
 *   agentrl_grpo_step            the two above, back to back on one stream.
 *
 * Conventions (all entry points)
 *   - Every pointer is DEVICE memory unless its name starts with host_.
 *   - The caller owns all memory.  The library never allocates persistent
 *     device memory; scratch comes from a caller workspace whose size the
 *     matching agentrl_*_workspace_size() returns.  The workspace base must
 *     be 1024-byte aligned.
 *   - Entry points are stream-ordered and asynchronous: they enqueue work on
 *     `stream` and return; no host synchronisation happens inside (the only
 *     host<->device traffic is kernel arguments).  Distinct workspaces make
 *     concurrent calls safe.  Every launch configuration is independent of the
 *     data, so calls can be captured in a CUDA graph.
 *   - Return value: synchronous status for host-checkable problems (AGENTRL_*
 *     codes below).  Data-dependent problems are OR-ed into the device word
 *     *d_status (int32, caller zeroes it) as AGENTRL_ST_* bits; the call still
 *     completes and writes defined (possibly zero) outputs.
 *   - comm == NULL means single GPU.  With a communicator, the per-task
 *     statistics, the masked-token count and the loss are all-reduced (sum,
 *     fp64) and grad_W is all-reduced (sum, fp32) over NCCL; each rank must
 *     hold WHOLE groups (a group never spans ranks).
 */
#ifndef AGENTRL_H_
#define AGENTRL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- synchronous return codes ------------------------------------------ */
#define AGENTRL_OK 0
#define AGENTRL_ERR_INVALID_ARG (-1) /* null pointer, eps outside range, n_tasks<=0 ... */
#define AGENTRL_ERR_SHAPE (-2)       /* d % 64 != 0, V % 8 != 0, T < 0, misaligned pointer */
#define AGENTRL_ERR_WORKSPACE (-3)   /* workspace too small or misaligned */
#define AGENTRL_ERR_CUDA (-4)        /* a CUDA runtime / driver call failed */
#define AGENTRL_ERR_NCCL (-5)        /* an NCCL call failed (or NCCL unavailable) */
#define AGENTRL_ERR_UNSUPPORTED (-6) /* device is not sm_100 */

/* ---- device status bits (OR-ed into *d_status) -------------------------- */
#define AGENTRL_ST_BAD_TARGET 1          /* a masked token's target not in [0,V) */
#define AGENTRL_ST_NONFINITE 2           /* non-finite loss / logp / ratio ("abort") */
#define AGENTRL_ST_BAD_OFFSETS 4         /* traj_offsets not 0..T nondecreasing */
#define AGENTRL_ST_GROUP_SPANS_TASKS 8   /* a group's members have different task_id */
#define AGENTRL_ST_GROUP_TOO_SMALL 16    /* a group has one trajectory */
#define AGENTRL_ST_NO_TOKENS 32          /* global masked-token count N == 0 */
#define AGENTRL_ST_COMM_TIMEOUT 64       /* a peer never reached the fused reduce-scatter */
#define AGENTRL_ST_ROWS_OVERFLOW 128     /* more local masked tokens than the max_rows the
                                            workspace was sized for: only the first max_rows
                                            (in token order) entered part 2 */

typedef struct agentrl_comm_s* agentrl_comm;
typedef struct CUstream_st* agentrl_stream; /* == cudaStream_t */

/*
 * Batch descriptor: a packed local token stream of T tokens holding n_traj
 * trajectories, each a CSR segment of the stream.
 *   traj_offsets [n_traj+1] int64: segment g = [off[g], off[g+1]); off[0]=0,
 *                off[n_traj]=T, nondecreasing (else AGENTRL_ST_BAD_OFFSETS).
 *   task_id      [n_traj] int32 in [0, n_tasks) -- the task T_i;
 *                task ids are GLOBAL across ranks.
 *   group_id     [n_traj] int32 in [0, n_groups) -- the group G_{i,j} of
 *                K_{i,j} trajectories of one sample; rank-local
 *                dense ids.  All members of a group share one task_id.
 *   rewards      [n_traj] float -- trajectory reward R.
 *   loss_mask    [T] uint8 -- nonzero marks the tokens y_{t,k} of actions
 *                (assistant turns), i.e. the index set of A_i^tok.
 */
typedef struct {
    int64_t T;
    int32_t n_traj, n_groups, n_tasks;
    const int64_t* traj_offsets;
    const int32_t* task_id;
    const int32_t* group_id;
    const float* rewards;
    const uint8_t* loss_mask;
} agentrl_batch;

/*
 * Part 1 -- task advantage normalization (Eq.1 after GRPO P:1263).
 *   A_hat_g  = (R_g - mean_j) / max(std_j, eps_std), population std over the
 *              group; exactly 0 when every reward of the group is equal.
 *   mu_i, sigma_i = mean / population std of A_hat over every masked token of
 *              task i in the global batch (each token counts once).
 *   adv_tok[t] = mask_t ? (A_hat_g(t) - mu_i) / max(sigma_i, eps_std) : 0.
 * Outputs:
 *   adv_tok      [T] float (required)
 *   task_stats   [n_tasks*3] double: (N_i, mu_i, sigma_i), global; or NULL
 *   n_mask_global [1] int64: N = sum_i N_i (global); or NULL
 * eps_std > 0 (default 1e-6); n_tasks > 0.
 */
size_t agentrl_task_adv_norm_workspace_size(int64_t T, int32_t n_traj, int32_t n_groups,
                                            int32_t n_tasks);
int agentrl_task_adv_norm(const agentrl_batch* b, double eps_std, float* adv_tok,
                          double* task_stats, int64_t* n_mask_global, void* ws,
                          size_t ws_bytes, agentrl_comm comm, int32_t* d_status,
                          agentrl_stream stream);

/*
 * Part 2 -- PPO-clip loss, forward and backward, through the LM head.
 * Inputs (device):
 *   hidden   [T,d] bf16 row-major: final normed hidden state of each token
 *   W_head   [V,d] bf16 row-major (nn.Linear layout, no bias): logits
 *            z_{t,v} = logit_scale * <hidden_t, W_v>
 *   target   [T] int32: the sampled token y_t aligned with hidden_t (the
 *            caller shifts labels)
 *   adv_tok  [T] float: token advantages (from part 1)
 *   old_logp [T] float: behaviour log-probs log pi_old(y_t)
 *   loss_mask[T] uint8
 *   n_mask_global [1] int64 (device): N in the 1/N token-level mean
 * Per masked token t:
 *   logp_t = z_{t,y_t} - logsumexp_v z_{t,v};  rho_t = exp(logp_t - old_t)
 *   term_t = min(rho_t A_t, clip(rho_t, 1-eps_low, 1+eps_high) A_t)
 *   loss   = -(1/N) sum_t term_t        (the paper maximises J; loss = -J)
 * Gradients (exact; the clip branch has zero gradient only where it is
 * strictly active: A>0 & rho>1+eps_high or A<0 & rho<1-eps_low):
 *   G_{t,v} = c_t (softmax_v - [v=y_t]),  c_t = unclipped ? rho_t A_t / N : 0
 *   grad_hidden = logit_scale * G W        (rows of unmasked tokens are 0)
 *   grad_W      = logit_scale * G^T hidden (summed over ranks if grad_W_mode=1; the rank's
 *                 row shard summed if grad_W_mode=2)
 * Empty batch: T may be 0; the per-token pointers may then be NULL; the call still writes
 * loss = 0 and a zero grad_W and sets AGENTRL_ST_NO_TOKENS (as it does whenever N == 0).
 * Shapes: d % 64 == 0, V % 8 == 0, 1 <= V.  Arithmetic: bf16 operands on
 * tcgen05 tensor cores with fp32 accumulation; softmax statistics fp32; loss
 * and statistics reductions fp64.
 */
typedef struct {
    int64_t T;
    int32_t d, V;
    const void* hidden;   /* __nv_bfloat16 [T,d] */
    const void* W_head;   /* __nv_bfloat16 [V,d] */
    const int32_t* target;
    const float* adv_tok;
    const float* old_logp;
    const uint8_t* loss_mask;
    float clip_eps_low, clip_eps_high; /* [0,1) and >= 0; default 0.2, 0.2 */
    float logit_scale;                 /* > 0; default 1.0 */
    const int64_t* n_mask_global;      /* device [1] */
    int32_t grad_W_mode;               /* 0 = local sum only, 1 = all-reduce over comm,
                                          2 = reduce-scatter over comm (FSDP-style shard,
                                          P:1357): rows [rank*V/world, (rank+1)*V/world) of
                                          grad_W hold the global sum, the other rows are
                                          scratch; needs V % world == 0 (else
                                          AGENTRL_ERR_SHAPE).  A callback communicator
                                          without a reduce-scatter sums every row.
                                          3 = vocabulary-parallel head (SURVEY 8(f) rank 4,
                                          agentrl_policy_loss_fwd_bwd only, needs comm):
                                          W_head holds rows [rank*V, (rank+1)*V) of a head
                                          of V*world rows, every rank passes the SAME token
                                          rows with global target ids in [0, V*world).  Per
                                          row (max, sum-exp) over the shards and the owner's
                                          target logit are all-gathered between the forward
                                          GEMM and the row statistics; loss, logp and loss_stats come
                                          out identical on every rank; grad_hidden is the
                                          full gradient (fp32 partials summed over the group
                                          inside the call); grad_W is this rank's complete
                                          shard [V, d] (no collective).  Workspace:
                                          agentrl_policy_loss_workspace_size_vp(). */
    int32_t max_rows;                  /* upper bound on this rank's masked tokens T_eff that
                                          the workspace was sized for (the same value passed to
                                          the *_workspace_size() query); <= 0 means T.  The
                                          T_eff x V intermediate scales with it, not with T */
    /* ---- objective variants; all-zero = the base objective above ----
     * KL penalty (the "- beta D_KL" of P:1103 / P:1119; beta unstated in the paper, R11):
     *   loss += sum_t w_t * beta * KL_t,  KL_t = exp(ref_t - logp_t) - (ref_t - logp_t) - 1
     *   (k3 estimator, >= 0); needs ref_logp [T] when kl_beta > 0.
     * Aggregation weights w_t (loss = sum_t w_t (-term_t + beta KL_t)):
     *   tok_weight != NULL : w_t = tok_weight[t] (any caller-defined aggregation)
     *   else loss_agg == 0 : w_t = 1 / N (token-level mean; default)
     *   else loss_agg == 1 : w_t = 1 / (G * K_j * n_g(t)): the GRPO objective
     *                        E_{i,j}[ 1/K_{i,j} sum_g term_g ] of P:1247-1256 with token-level
     *                        ratios; term_g = the mean of term_t over trajectory g's n_g masked
     *                        tokens (0 if n_g = 0), K_j = every member of t's group j (members
     *                        without masked tokens included), G = groups with at least one
     *                        member, summed over ranks (R7b).
     *                        agentrl_grpo_step only (needs the batch descriptor). */
    float kl_beta;                     /* >= 0 */
    int32_t loss_agg;                  /* 0 or 1 */
    const float* ref_logp;             /* [T] or NULL */
    const float* tok_weight;           /* [T] or NULL */
} agentrl_loss_args;

/* Outputs.  loss and grad_hidden / grad_W are required; the others may be NULL.
 *   loss        [1] double: this rank's share -(1/N) sum_{local t} term_t; with a
 *               communicator it is all-reduced, i.e. the global loss
 *   logp        [T] float: logp_t on masked tokens, 0 elsewhere
 *   grad_hidden [T,d] bf16 (overwritten)
 *   grad_W      [V,d] float (overwritten)
 *   loss_stats  [5] double: clip fraction, mean rho, mean logp, masked tokens,
 *               mean KL (all local) */
typedef struct {
    double* loss;
    float* logp;
    void* grad_hidden;
    float* grad_W;
    double* loss_stats;
} agentrl_loss_out;

/* Workspace: about (2 V + 8 ceil(V/256) + 2 d + 64) bytes per row of max_rows (<= 0: T) plus
 * ~8 bytes per token of T -- the bf16 P~ = exp(z - m_tile) [max_rows, V] dominates (16.1 GB at
 * T_eff = 53K, V = 152K).  The host knows the mask, so it knows T_eff (or a bound). */
size_t agentrl_policy_loss_workspace_size(int64_t T, int64_t max_rows, int32_t d, int32_t V);
/* workspace of grad_W_mode = 3 (V = the rank's shard rows, world = the group size): the base
 * plan plus the all-gathered row statistics (8 * world * rows B) and the fp32 grad_hidden
 * partial (4 * rows * d B) */
size_t agentrl_policy_loss_workspace_size_vp(int64_t T, int64_t max_rows, int32_t d, int32_t V,
                                             int32_t world);
int agentrl_policy_loss_fwd_bwd(const agentrl_loss_args* a, const agentrl_loss_out* o, void* ws,
                                size_t ws_bytes, agentrl_comm comm, int32_t* d_status,
                                agentrl_stream stream);

/* Fused: part 1 then part 2 (a->adv_tok and a->n_mask_global are ignored; the
 * step uses its own).  adv_tok_out [T] float required; task_stats optional. */
size_t agentrl_grpo_step_workspace_size(int64_t T, int32_t n_traj, int32_t n_groups,
                                        int32_t n_tasks, int64_t max_rows, int32_t d, int32_t V);
int agentrl_grpo_step(const agentrl_batch* b, double eps_std, const agentrl_loss_args* a,
                      const agentrl_loss_out* o, float* adv_tok_out, double* task_stats,
                      void* ws, size_t ws_bytes, agentrl_comm comm, int32_t* d_status,
                      agentrl_stream stream);

/*
 * Forward-only token log-probs and entropies (no backward): the
 * trainer's recomputation of behaviour / reference log-probs pi_old and the policy
 * entropy that DAPO's clip-higher targets.  For every masked token t:
 *   logp[t]    = z_{t,y_t} - logsumexp_v z_{t,v},  z = logit_scale * <hidden_t, W_v>
 *   entropy[t] = -sum_v p_{t,v} log p_{t,v}        (optional output)
 * Unmasked tokens get 0.  Same shapes/alignment rules as part 2; status bits
 * AGENTRL_ST_BAD_TARGET / AGENTRL_ST_NONFINITE.
 */
typedef struct {
    int64_t T;
    int32_t d, V;
    const void* hidden;  /* __nv_bfloat16 [T,d] */
    const void* W_head;  /* __nv_bfloat16 [V,d] */
    const int32_t* target;
    const uint8_t* loss_mask;
    float logit_scale;
    int32_t max_rows; /* bound on the masked tokens (<= 0: T), as in agentrl_loss_args */
} agentrl_logprob_args;

size_t agentrl_logprob_workspace_size(int64_t T, int64_t max_rows, int32_t d, int32_t V);
int agentrl_logprob_fwd(const agentrl_logprob_args* a, float* logp /*[T]*/,
                        float* entropy /*[T] or NULL*/, void* ws, size_t ws_bytes,
                        int32_t* d_status, agentrl_stream stream);

/*
 * Test / debug export of part 1's integer bookkeeping (north_star: bit-exact vs the oracle).
 * Copies, stream-ordered after the last agentrl_task_adv_norm / agentrl_grpo_step call that
 * used workspace `ws` with the same (T, n_traj, n_groups, n_tasks), into caller buffers:
 *   n_g  [n_traj]   int32: masked tokens of each trajectory, the per-trajectory part of the
 *                   token set A_i^tok
 *   K    [n_groups] int32: members of each group, K_{i,j}
 *   idx  [T]        int32: stable compaction, the positions of the local masked tokens in
 *                   increasing order (written by agentrl_grpo_step only; the first *rows
 *                   entries are defined)
 *   rows [1]        int64: the local masked-token count (entries of idx)
 * Every output may be NULL.  Device-to-device copies only; no kernel. */
int agentrl_debug_bookkeeping(const void* ws, int64_t T, int32_t n_traj, int32_t n_groups,
                              int32_t n_tasks, int32_t* n_g, int32_t* K, int32_t* idx,
                              int64_t* rows, agentrl_stream stream);

/* ---- communicator (NCCL over NVLink; loaded lazily with dlopen) ----------
 * Rank 0 calls agentrl_comm_unique_id, the caller broadcasts the 128 bytes
 * (e.g. over a torch.distributed process group), then every rank calls
 * agentrl_comm_init on its own device.  Returns AGENTRL_ERR_NCCL if
 * libnccl.so.2 cannot be loaded. */
int agentrl_comm_unique_id(unsigned char host_id[128]);
int agentrl_comm_init(agentrl_comm* out, int world, int rank, const unsigned char host_id[128]);
int agentrl_comm_destroy(agentrl_comm comm);

/* Callback communicator: every all-reduce (sum, in place on the device buffer, ordered on
 * `stream`) is delegated to fn(user, dev_buf, count, dtype, stream), called on the host at
 * enqueue time in the same order on every rank; fn returns 0 on success.  For hosts without
 * NCCL between the ranks (e.g. several ranks sharing one GPU in tests, or a custom fabric).
 * dtype: AGENTRL_DTYPE_*. */
#define AGENTRL_DTYPE_F64 0
#define AGENTRL_DTYPE_F32 1
#define AGENTRL_DTYPE_I64 2
typedef int (*agentrl_allreduce_fn)(void* user, void* dev_buf, size_t count, int dtype,
                                    agentrl_stream stream);
int agentrl_comm_init_callback(agentrl_comm* out, int world, int rank, agentrl_allreduce_fn fn,
                               void* user);
/* Optional in-place reduce-scatter for a callback communicator (grad_W_mode = 2): dev_buf holds
 * world * recv_count elements; afterwards block [rank*recv_count, (rank+1)*recv_count) holds
 * the sum over ranks (other blocks unspecified), ordered on `stream`.  Without it the
 * communicator's all-reduce is used (a superset).  INVALID_ARG for an NCCL communicator. */
typedef int (*agentrl_reduce_scatter_fn)(void* user, void* dev_buf, size_t recv_count, int dtype,
                                         agentrl_stream stream);
int agentrl_comm_set_reduce_scatter(agentrl_comm comm, agentrl_reduce_scatter_fn fn);
/* Fused grad_W reduce-scatter over peer memory (grad_W_mode = 2).  Collective: every rank
 * calls it with the same bytes_per_rank.  The communicator allocates a staging window of
 * bytes_per_rank device bytes (and a few flags) on each rank and maps every other rank's window
 * with CUDA IPC (NVLink / NVSwitch peer memory across GPUs; the same device across processes).
 * The IPC handles travel through one sum all-reduce of the communicator.  From then on a call
 * with grad_W_mode = 2 and a window of at least V*d*4 bytes makes the grad_W GEMM epilogue
 * store each fp32 tile directly into the window of the rank that owns its rows (owner
 * o = rows [o*V/world, (o+1)*V/world)), so the transfer overlaps the GEMM.  After a
 * system-scope flag barrier the owner sums the world slots in rank order (deterministic) into
 * its grad_W shard; the collective path is not used.  Every wait is bounded: a peer that never
 * arrives sets AGENTRL_ST_COMM_TIMEOUT instead of hanging.  AGENTRL_C3_P2P=0 in the
 * environment selects the collective path.  Every rank must make the same sequence of
 * grad_W_mode = 2 calls on the communicator: each call is one epoch of the flag protocol, and
 * the epoch counter is kept in device memory (advanced by the call's first kernel), so the call
 * may be captured in a CUDA graph and replayed.  The window is freed by agentrl_comm_destroy (the
 * one place the library allocates persistent device memory: it must be IPC-exportable), or by
 * a call with bytes_per_rank = 0, which returns to the collective path (every rank must make it,
 * after its last grad_W_mode = 2 call has completed). */
int agentrl_comm_enable_peer_window(agentrl_comm comm, size_t bytes_per_rank);

/* ---- misc -------------------------------------------------------------- */
const char* agentrl_status_string(int code); /* text for a return code or status bit */
int agentrl_version(void);                    /* major*10000 + minor*100 + patch */
/* Number of kernel launches the last call on this thread enqueued (for the
 * bench's gpu_launches claim). */
int agentrl_last_launch_count(void);

/* ---- per-kernel timing (CUDA events on the launching stream) -------------
 * agentrl_profile_start(n) pre-creates 2n events and makes every following call
 * record an event pair around each of its kernels (on the stream it launches
 * on), up to n pairs.  agentrl_profile_stop synchronises those events and
 * writes, per kernel id, the summed milliseconds and the launch count.  Kernel
 * ids: 0 count, 1 stats, 2 apply, 3 compact, 4 gather, 5 fwd GEMM, 6 row statistics
 * (loss terms and gradient scales), 7 loss reduce, 8 grad_W GEMM, 9 grad_hidden GEMM,
 * 10 log-prob GEMM, 11 log-prob merge. */
#define AGENTRL_NUM_KERNEL_IDS 12
int agentrl_profile_start(int max_pairs);
int agentrl_profile_stop(double* host_ms_sum, int* host_counts, int n_ids);
const char* agentrl_kernel_name(int id);
/* Debug: %globaltimer stamps (ns) of the last single-GPU part-1 launch at its phase
 * boundaries: [0] start, [1] after zero/table, [2] counts, [3] group scans, [4] member lists,
 * [5] group advantages + task partials, [6] task moments, [7] apply/compaction end. */
int agentrl_debug_adv_phase_ns(unsigned long long host_ns8[8]);
/* Debug: wait episodes of the GEMM progress throttle since the library was loaded, summed over
 * calls: [0] forward, [1] grad_W, [2] grad_hidden (a pair leader more than the lead ahead of the
 * slowest active pair sleeps until it is not; one episode per wait). */
int agentrl_debug_throttle_waits(unsigned long long host3[3]);

#ifdef __cplusplus
}
#endif
#endif /* AGENTRL_H_ */
