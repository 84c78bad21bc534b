// api.cu -- the C ABI declared in include/agentrl.h: argument validation, workspace planning,
// device checks, the NCCL communicator (loaded lazily with dlopen) and status strings.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <vector>

#include <algorithm>

#include "internal.h"

namespace agentrl {

static thread_local int g_launches = 0;
void count_launch(int n) { g_launches += n; }

// ---------------------------------------------------------------------------- profiling
struct ProfRec {
    int kid;
    cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<cudaEvent_t> g_prof_pool;
static std::vector<ProfRec> g_prof_recs;
static size_t g_prof_next = 0;
static int g_prof_open[KID_N];

void prof_mark(int kid, bool begin, cudaStream_t s) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (begin) {
        if (g_prof_next + 2 > g_prof_pool.size()) {
            g_prof_open[kid] = -1;
            return;
        }
        ProfRec r{kid, g_prof_pool[g_prof_next], g_prof_pool[g_prof_next + 1]};
        g_prof_next += 2;
        cudaEventRecord(r.a, s);
        g_prof_open[kid] = (int)g_prof_recs.size();
        g_prof_recs.push_back(r);
    } else {
        const int i = g_prof_open[kid];
        if (i < 0) return;
        cudaEventRecord(g_prof_recs[i].b, s);
        g_prof_open[kid] = -1;
    }
}

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int num_sms() {
    // per device (a process or thread may drive several GPUs)
    static std::atomic<int> cache[MAX_DEVICES];
    const int dev = current_device();
    const int slot = dev & (MAX_DEVICES - 1);
    int n = cache[slot].load(std::memory_order_relaxed);
    if (n == 0) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cache[slot].store(n, std::memory_order_relaxed);
    }
    return n;
}

bool func_attr_once(std::atomic<uint64_t>& done_mask, const void* func, int smem_bytes) {
    const int dev = current_device();
    const uint64_t bit = 1ull << (dev & (MAX_DEVICES - 1));
    if (done_mask.load(std::memory_order_acquire) & bit) return true;
    if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) !=
        cudaSuccess)
        return false;
    done_mask.fetch_or(bit, std::memory_order_acq_rel);
    return true;
}

int check_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return AGENTRL_ERR_CUDA;
    static thread_local int ok_dev = -1;  // last device that passed the check
    if (dev == ok_dev) return AGENTRL_OK;
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
        return AGENTRL_ERR_CUDA;
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) return AGENTRL_ERR_UNSUPPORTED;  // built for sm_100a only
    ok_dev = dev;
    return AGENTRL_OK;
}

// ---------------------------------------------------------------------------- NCCL (dlopen)
typedef struct {
    char internal[128];
} nccl_uid_t;
typedef void* nccl_comm_t;
typedef int (*fn_getUniqueId)(nccl_uid_t*);
typedef int (*fn_commInitRank)(nccl_comm_t*, int, nccl_uid_t, int);
typedef int (*fn_commDestroy)(nccl_comm_t);
typedef int (*fn_allReduce)(const void*, void*, size_t, int /*dtype*/, int /*op*/, nccl_comm_t,
                            cudaStream_t);
typedef int (*fn_reduceScatter)(const void*, void*, size_t /*recvcount*/, int, int, nccl_comm_t,
                                cudaStream_t);
enum { NCCL_INT64 = 4, NCCL_FLOAT32 = 7, NCCL_FLOAT64 = 8, NCCL_SUM = 0 };

struct NcclApi {
    void* h = nullptr;
    fn_getUniqueId getUniqueId = nullptr;
    fn_commInitRank commInitRank = nullptr;
    fn_commDestroy commDestroy = nullptr;
    fn_allReduce allReduce = nullptr;
    fn_reduceScatter reduceScatter = nullptr;
};
static NcclApi* nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // prefer a libnccl already loaded into the process (e.g. torch's), else the system one
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.h = h;
        api.getUniqueId = (fn_getUniqueId)dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (fn_commInitRank)dlsym(h, "ncclCommInitRank");
        api.commDestroy = (fn_commDestroy)dlsym(h, "ncclCommDestroy");
        api.allReduce = (fn_allReduce)dlsym(h, "ncclAllReduce");
        api.reduceScatter = (fn_reduceScatter)dlsym(h, "ncclReduceScatter");
    });
    if (!api.getUniqueId || !api.commInitRank || !api.commDestroy || !api.allReduce)
        return nullptr;
    return &api;
}

}  // namespace agentrl

struct agentrl_comm_s {
    agentrl::nccl_comm_t comm;
    int world, rank;
    agentrl_allreduce_fn fn;  // callback backend (non-null) instead of NCCL
    void* user;
    agentrl_reduce_scatter_fn rs;  // optional callback reduce-scatter
    agentrl::PeerWindow* peer = nullptr;  // fused GEMM + reduce-scatter window (or none)
};

namespace agentrl {
static int allreduce(agentrl_comm c, void* buf, size_t n, int dtype, cudaStream_t s) {
    if (!c) return AGENTRL_ERR_NCCL;
    if (n == 0) return AGENTRL_OK;
    if (c->fn) {  // callback backend: dtype codes of include/agentrl.h
        const int code = dtype == NCCL_FLOAT64 ? AGENTRL_DTYPE_F64
                                               : (dtype == NCCL_FLOAT32 ? AGENTRL_DTYPE_F32
                                                                        : AGENTRL_DTYPE_I64);
        return c->fn(c->user, buf, n, code, reinterpret_cast<agentrl_stream>(s)) == 0
                   ? AGENTRL_OK
                   : AGENTRL_ERR_NCCL;
    }
    NcclApi* api = nccl();
    if (!api) return AGENTRL_ERR_NCCL;
    return api->allReduce(buf, buf, n, dtype, NCCL_SUM, c->comm, s) == 0 ? AGENTRL_OK
                                                                         : AGENTRL_ERR_NCCL;
}
int comm_allreduce_f64(agentrl_comm c, double* b, size_t n, cudaStream_t s) {
    return allreduce(c, b, n, NCCL_FLOAT64, s);
}
int comm_allreduce_f32(agentrl_comm c, float* b, size_t n, cudaStream_t s) {
    return allreduce(c, b, n, NCCL_FLOAT32, s);
}
int comm_allreduce_i64(agentrl_comm c, int64_t* b, size_t n, cudaStream_t s) {
    return allreduce(c, b, n, NCCL_INT64, s);
}
// in-place sum reduce-scatter of n = world * m floats: rank r's block [r m, (r+1) m) receives
// the global sum.  The callback backend has only an all-reduce, which is a superset.
int comm_reduce_scatter_f32(agentrl_comm c, float* b, size_t n, cudaStream_t s) {
    if (!c) return AGENTRL_ERR_NCCL;
    if (n == 0) return AGENTRL_OK;
    if (c->fn && c->rs) {
        if (c->world <= 0 || n % (size_t)c->world != 0) return AGENTRL_ERR_NCCL;
        return c->rs(c->user, b, n / (size_t)c->world, AGENTRL_DTYPE_F32,
                     reinterpret_cast<agentrl_stream>(s)) == 0
                   ? AGENTRL_OK
                   : AGENTRL_ERR_NCCL;
    }
    if (c->fn) return allreduce(c, b, n, NCCL_FLOAT32, s);
    NcclApi* api = nccl();
    if (!api || !api->reduceScatter || c->world <= 0 || n % (size_t)c->world != 0)
        return AGENTRL_ERR_NCCL;
    const size_t m = n / (size_t)c->world;
    return api->reduceScatter(b, b + (size_t)c->rank * m, m, NCCL_FLOAT32, NCCL_SUM, c->comm, s) == 0
               ? AGENTRL_OK
               : AGENTRL_ERR_NCCL;
}
int comm_world(agentrl_comm c) { return c ? c->world : 1; }
int comm_rank(agentrl_comm c) { return c ? c->rank : 0; }
PeerWindow* comm_peer(agentrl_comm c) { return c ? c->peer : nullptr; }

static bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

static int check_batch(const agentrl_batch* b, double eps_std) {
    if (!b || !(eps_std > 0.0) || b->n_tasks <= 0 || b->n_traj < 0 || b->n_groups < 0)
        return AGENTRL_ERR_INVALID_ARG;
    if (b->T < 0 || b->T >= (int64_t)1 << 31) return AGENTRL_ERR_SHAPE;
    if (!b->traj_offsets || (b->n_traj > 0 && (!b->task_id || !b->group_id || !b->rewards)) ||
        (b->T > 0 && !b->loss_mask))
        return AGENTRL_ERR_INVALID_ARG;
    return AGENTRL_OK;
}

static int check_loss(const agentrl_loss_args* a, const agentrl_loss_out* o, bool fused) {
    if (!a || !o || !o->loss || !o->grad_W || (a->T > 0 && !o->grad_hidden))
        return AGENTRL_ERR_INVALID_ARG;
    if (!(a->clip_eps_low >= 0.f && a->clip_eps_low < 1.f) || !(a->clip_eps_high >= 0.f) ||
        !(a->logit_scale > 0.f))
        return AGENTRL_ERR_INVALID_ARG;
    if (a->T < 0 || a->T >= (int64_t)1 << 31 || a->d <= 0 || a->d % 64 != 0 || a->V < 8 ||
        a->V % 8 != 0)
        return AGENTRL_ERR_SHAPE;
    // per-token arrays may be empty (null) when T == 0
    if (!a->W_head || (a->T > 0 && (!a->hidden || !a->target || !a->old_logp || !a->loss_mask)))
        return AGENTRL_ERR_INVALID_ARG;
    if (!fused && ((a->T > 0 && !a->adv_tok) || !a->n_mask_global)) return AGENTRL_ERR_INVALID_ARG;
    if (!aligned(a->hidden, 16) || !aligned(a->W_head, 16) || !aligned(o->grad_hidden, 16) ||
        !aligned(o->grad_W, 16))
        return AGENTRL_ERR_SHAPE;
    if (a->grad_W_mode < 0 || a->grad_W_mode > 3) return AGENTRL_ERR_INVALID_ARG;
    if (fused && a->grad_W_mode == 3) return AGENTRL_ERR_INVALID_ARG;  // standalone loss only
    // objective variants: beta >= 0 (ref log-probs needed when > 0); loss_agg 0/1, the
    // sequence mean only in the fused step (it needs the batch descriptor) unless the caller
    // supplies the weights
    if (!(a->kl_beta >= 0.f) || (a->kl_beta > 0.f && !a->ref_logp)) return AGENTRL_ERR_INVALID_ARG;
    if (a->loss_agg < 0 || a->loss_agg > 1) return AGENTRL_ERR_INVALID_ARG;
    if (!fused && a->loss_agg == 1 && !a->tok_weight) return AGENTRL_ERR_INVALID_ARG;
    return AGENTRL_OK;
}

}  // namespace agentrl

using namespace agentrl;

extern "C" {

size_t agentrl_task_adv_norm_workspace_size(int64_t T, int32_t n_traj, int32_t n_groups,
                                            int32_t n_tasks) {
    return plan_adv(T, n_traj, n_groups, n_tasks).total;
}

int agentrl_task_adv_norm(const agentrl_batch* b, double eps_std, float* adv_tok,
                          double* task_stats, int64_t* n_mask_global, void* ws, size_t ws_bytes,
                          agentrl_comm comm, int32_t* d_status, agentrl_stream stream) {
    NvtxRange nvtx("agentrl_task_adv_norm");
    g_launches = 0;
    int rc = check_batch(b, eps_std);
    if (rc) return rc;
    if ((b->T > 0 && !adv_tok) || !d_status || !ws) return AGENTRL_ERR_INVALID_ARG;
    if ((rc = check_device())) return rc;
    AdvWs w = plan_adv(b->T, b->n_traj, b->n_groups, b->n_tasks);
    if (ws_bytes < w.total || !aligned(ws, 1024)) return AGENTRL_ERR_WORKSPACE;
    return launch_adv_norm(b, eps_std, adv_tok, task_stats, n_mask_global,
                           static_cast<uint8_t*>(ws), w, comm, d_status,
                           reinterpret_cast<cudaStream_t>(stream), /*compact=*/false);
}

size_t agentrl_policy_loss_workspace_size(int64_t T, int64_t max_rows, int32_t d, int32_t V) {
    return plan_loss(T, max_rows, d, V).total;
}

size_t agentrl_policy_loss_workspace_size_vp(int64_t T, int64_t max_rows, int32_t d, int32_t V,
                                             int32_t world) {
    return plan_loss(T, max_rows, d, V, 0, std::max(world, 1)).total;
}

int agentrl_policy_loss_fwd_bwd(const agentrl_loss_args* a, const agentrl_loss_out* o, void* ws,
                                size_t ws_bytes, agentrl_comm comm, int32_t* d_status,
                                agentrl_stream stream) {
    NvtxRange nvtx("agentrl_policy_loss_fwd_bwd");
    g_launches = 0;
    int rc = check_loss(a, o, false);
    if (!rc && a->grad_W_mode == 2 && comm && a->V % comm_world(comm) != 0) rc = AGENTRL_ERR_SHAPE;
    if (!rc && a->grad_W_mode == 3 && !comm) rc = AGENTRL_ERR_INVALID_ARG;  // needs the group
    if (rc) return rc;
    if (!d_status || !ws) return AGENTRL_ERR_INVALID_ARG;
    if ((rc = check_device())) return rc;
    LossWs w = plan_loss(a->T, a->max_rows, a->d, a->V, 0,
                         a->grad_W_mode == 3 ? comm_world(comm) : 0);
    if (ws_bytes < w.total || !aligned(ws, 1024)) return AGENTRL_ERR_WORKSPACE;
    return launch_policy_loss(a, o, static_cast<uint8_t*>(ws), w, nullptr, nullptr, nullptr,
                              nullptr, comm, d_status, reinterpret_cast<cudaStream_t>(stream));
}

size_t agentrl_logprob_workspace_size(int64_t T, int64_t max_rows, int32_t d, int32_t V) {
    return plan_logp(T, max_rows, d, V).total;
}

int agentrl_logprob_fwd(const agentrl_logprob_args* a, float* logp, float* entropy, void* ws,
                        size_t ws_bytes, int32_t* d_status, agentrl_stream stream) {
    NvtxRange nvtx("agentrl_logprob_fwd");
    g_launches = 0;
    if (!a || !logp || !d_status || !ws || !a->hidden || !a->W_head || !a->target ||
        !a->loss_mask || !(a->logit_scale > 0.f))
        return AGENTRL_ERR_INVALID_ARG;
    if (a->T < 0 || a->T >= (int64_t)1 << 31 || a->d <= 0 || a->d % 64 != 0 || a->V < 8 ||
        a->V % 8 != 0 || !aligned(a->hidden, 16) || !aligned(a->W_head, 16))
        return AGENTRL_ERR_SHAPE;
    int rc = check_device();
    if (rc) return rc;
    LogpWs w = plan_logp(a->T, a->max_rows, a->d, a->V);
    if (ws_bytes < w.total || !aligned(ws, 1024)) return AGENTRL_ERR_WORKSPACE;
    return launch_logprob(a, logp, entropy, static_cast<uint8_t*>(ws), w, d_status,
                          reinterpret_cast<cudaStream_t>(stream));
}

size_t agentrl_grpo_step_workspace_size(int64_t T, int32_t n_traj, int32_t n_groups,
                                        int32_t n_tasks, int64_t max_rows, int32_t d, int32_t V) {
    AdvWs wa = plan_adv(T, n_traj, n_groups, n_tasks);
    return plan_loss(T, max_rows, d, V, align_up(wa.total, 1024)).total;
}

int agentrl_grpo_step(const agentrl_batch* b, double eps_std, const agentrl_loss_args* a,
                      const agentrl_loss_out* o, float* adv_tok_out, double* task_stats, void* ws,
                      size_t ws_bytes, agentrl_comm comm, int32_t* d_status,
                      agentrl_stream stream) {
    NvtxRange nvtx("agentrl_grpo_step");
    g_launches = 0;
    int rc = check_batch(b, eps_std);
    if (rc) return rc;
    if ((rc = check_loss(a, o, true))) return rc;
    if (a->grad_W_mode == 2 && comm && a->V % comm_world(comm) != 0) return AGENTRL_ERR_SHAPE;
    if (a->T != b->T || a->loss_mask != b->loss_mask) return AGENTRL_ERR_INVALID_ARG;
    if ((b->T > 0 && !adv_tok_out) || !d_status || !ws) return AGENTRL_ERR_INVALID_ARG;
    if ((rc = check_device())) return rc;
    AdvWs wa = plan_adv(b->T, b->n_traj, b->n_groups, b->n_tasks);
    LossWs wl = plan_loss(a->T, a->max_rows, a->d, a->V, align_up(wa.total, 1024));
    if (ws_bytes < wl.total || !aligned(ws, 1024)) return AGENTRL_ERR_WORKSPACE;
    uint8_t* w8 = static_cast<uint8_t*>(ws);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int64_t* meta = reinterpret_cast<int64_t*>(w8 + wa.meta);
    if ((rc = launch_adv_norm(b, eps_std, adv_tok_out, task_stats, nullptr, w8, wa, comm,
                              d_status, s)))
        return rc;
    const int before = g_launches;
    const FusedExtras fx{b->traj_offsets,
                         b->n_traj,
                         reinterpret_cast<const int32_t*>(w8 + wa.n_g),
                         b->group_id,
                         reinterpret_cast<const int32_t*>(w8 + wa.grp_cnt),
                         b->n_groups,
                         meta + 2 /* global G */};
    rc = launch_policy_loss(a, o, w8, wl, reinterpret_cast<const int32_t*>(w8 + wa.idx),
                            meta /* [0] local rows */,
                            reinterpret_cast<const float*>(w8 + wa.adv_c),
                            meta + 1 /* global N */, comm, d_status, s, &fx);
    (void)before;
    return rc;
}

int agentrl_comm_unique_id(unsigned char host_id[128]) {
    NcclApi* api = nccl();
    if (!api || !host_id) return AGENTRL_ERR_NCCL;
    nccl_uid_t id;
    if (api->getUniqueId(&id) != 0) return AGENTRL_ERR_NCCL;
    memcpy(host_id, id.internal, 128);
    return AGENTRL_OK;
}

int agentrl_comm_init(agentrl_comm* out, int world, int rank, const unsigned char host_id[128]) {
    NcclApi* api = nccl();
    if (!out || world <= 0 || rank < 0 || rank >= world || !host_id)
        return AGENTRL_ERR_INVALID_ARG;
    if (!api) return AGENTRL_ERR_NCCL;
    nccl_uid_t id;
    memcpy(id.internal, host_id, 128);
    agentrl_comm c = new agentrl_comm_s{nullptr, world, rank, nullptr, nullptr, nullptr};
    if (api->commInitRank(&c->comm, world, id, rank) != 0) {
        delete c;
        return AGENTRL_ERR_NCCL;
    }
    *out = c;
    return AGENTRL_OK;
}

int agentrl_comm_init_callback(agentrl_comm* out, int world, int rank, agentrl_allreduce_fn fn,
                               void* user) {
    if (!out || world <= 0 || rank < 0 || rank >= world || !fn) return AGENTRL_ERR_INVALID_ARG;
    *out = new agentrl_comm_s{nullptr, world, rank, fn, user, nullptr};
    return AGENTRL_OK;
}

int agentrl_comm_set_reduce_scatter(agentrl_comm comm, agentrl_reduce_scatter_fn fn) {
    if (!comm || !comm->fn) return AGENTRL_ERR_INVALID_ARG;
    comm->rs = fn;
    return AGENTRL_OK;
}

int agentrl_comm_enable_peer_window(agentrl_comm comm, size_t bytes_per_rank) {
    if (!comm) return AGENTRL_ERR_INVALID_ARG;
    if (comm->peer) {
        peer_window_destroy(comm->peer);
        comm->peer = nullptr;
    }
    if (bytes_per_rank == 0) return AGENTRL_OK;  // disabled: the collective C3 path
    return peer_window_create(comm, bytes_per_rank, &comm->peer);
}

int agentrl_comm_destroy(agentrl_comm comm) {
    if (!comm) return AGENTRL_OK;
    if (comm->peer) {
        peer_window_destroy(comm->peer);
        comm->peer = nullptr;
    }
    if (comm->fn) {
        delete comm;
        return AGENTRL_OK;
    }
    NcclApi* api = nccl();
    int rc = AGENTRL_OK;
    if (api && comm->comm && api->commDestroy(comm->comm) != 0) rc = AGENTRL_ERR_NCCL;
    delete comm;
    return rc;
}

const char* agentrl_status_string(int code) {
    switch (code) {
        case AGENTRL_OK: return "ok";
        case AGENTRL_ERR_INVALID_ARG: return "invalid argument";
        case AGENTRL_ERR_SHAPE: return "unsupported shape or misaligned pointer";
        case AGENTRL_ERR_WORKSPACE: return "workspace too small or misaligned";
        case AGENTRL_ERR_CUDA: return "CUDA error";
        case AGENTRL_ERR_NCCL: return "NCCL error or NCCL unavailable";
        case AGENTRL_ERR_UNSUPPORTED: return "device is not sm_100 (B200)";
        case AGENTRL_ST_BAD_TARGET: return "target token id outside [0, V)";
        case AGENTRL_ST_NONFINITE: return "non-finite loss, log-prob or ratio";
        case AGENTRL_ST_BAD_OFFSETS: return "trajectory offsets inconsistent with T";
        case AGENTRL_ST_GROUP_SPANS_TASKS: return "a group spans tasks (or ids out of range)";
        case AGENTRL_ST_GROUP_TOO_SMALL: return "a group has fewer than 2 trajectories";
        case AGENTRL_ST_NO_TOKENS: return "no loss-masked tokens in the batch";
        case AGENTRL_ST_COMM_TIMEOUT: return "a peer never reached the fused reduce-scatter";
        case AGENTRL_ST_ROWS_OVERFLOW: return "more masked tokens than the workspace's max_rows";
        default: return "unknown";
    }
}

int agentrl_version(void) { return 100; }

int agentrl_debug_bookkeeping(const void* ws, int64_t T, int32_t n_traj, int32_t n_groups,
                              int32_t n_tasks, int32_t* n_g, int32_t* K, int32_t* idx,
                              int64_t* rows, agentrl_stream stream) {
    if (!ws || T < 0 || n_traj < 0 || n_groups < 0 || n_tasks <= 0) return AGENTRL_ERR_INVALID_ARG;
    const AdvWs w = plan_adv(T, n_traj, n_groups, n_tasks);  // part 1's plan starts at offset 0
    const uint8_t* b = static_cast<const uint8_t*>(ws);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (n_g && n_traj > 0)
        AG_CUDA(cudaMemcpyAsync(n_g, b + w.n_g, sizeof(int32_t) * (size_t)n_traj,
                                cudaMemcpyDeviceToDevice, s));
    if (K && n_groups > 0)
        AG_CUDA(cudaMemcpyAsync(K, b + w.grp_cnt, sizeof(int32_t) * (size_t)n_groups,
                                cudaMemcpyDeviceToDevice, s));
    if (idx && T > 0)
        AG_CUDA(cudaMemcpyAsync(idx, b + w.idx, sizeof(int32_t) * (size_t)T,
                                cudaMemcpyDeviceToDevice, s));
    if (rows)
        AG_CUDA(cudaMemcpyAsync(rows, b + w.meta, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    return AGENTRL_OK;
}

int agentrl_debug_throttle_waits(unsigned long long host3[3]) {
    return host3 ? debug_throttle_waits(host3) : AGENTRL_ERR_INVALID_ARG;
}

int agentrl_debug_adv_phase_ns(unsigned long long* host_ns8) {
    return host_ns8 ? debug_adv_phase_ns(host_ns8) : AGENTRL_ERR_INVALID_ARG;
}

int agentrl_profile_start(int max_pairs) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (max_pairs <= 0) return AGENTRL_ERR_INVALID_ARG;
    for (auto e : g_prof_pool) cudaEventDestroy(e);
    g_prof_pool.assign(2 * (size_t)max_pairs, nullptr);
    for (auto& e : g_prof_pool)
        if (cudaEventCreate(&e) != cudaSuccess) return AGENTRL_ERR_CUDA;
    g_prof_recs.clear();
    g_prof_next = 0;
    for (int k = 0; k < KID_N; ++k) g_prof_open[k] = -1;
    g_prof_on = true;
    return AGENTRL_OK;
}

int agentrl_profile_stop(double* ms_sum, int* counts, int n_ids) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = false;
    for (int k = 0; k < n_ids; ++k) {
        if (ms_sum) ms_sum[k] = 0.0;
        if (counts) counts[k] = 0;
    }
    int rc = AGENTRL_OK;
    for (auto& r : g_prof_recs) {
        if (cudaEventSynchronize(r.b) != cudaSuccess) {
            rc = AGENTRL_ERR_CUDA;
            continue;
        }
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) {
            rc = AGENTRL_ERR_CUDA;
            continue;
        }
        if (r.kid < n_ids) {
            if (ms_sum) ms_sum[r.kid] += ms;
            if (counts) counts[r.kid] += 1;
        }
    }
    g_prof_recs.clear();
    g_prof_next = 0;
    return rc;
}

const char* agentrl_kernel_name(int id) {
    static const char* names[KID_N] = {"k_count", "k_stats", "k_apply", "k_compact",
                                       "k_gather", "gemm_fwd", "k_row_stats", "k_loss_reduce",
                                       "gemm_grad_W", "gemm_grad_hidden", "gemm_logp",
                                       "k_logp_merge"};
    return (id >= 0 && id < KID_N) ? names[id] : "unknown";
}
int agentrl_last_launch_count(void) { return g_launches; }

}  // extern "C"
