// peer.cu -- the grad_W reduce-scatter (C3, grad_W_mode 2) fused into the grad_W GEMM over peer
// memory.
//
// Every rank maps every other rank's staging window (CUDA IPC; NVLink/NVSwitch peer memory
// between GPUs, the same device between processes sharing one GPU).  Rank o owns grad_W rows
// [o V/R, (o+1) V/R).  The grad_W GEMM epilogue stores each finished fp32 tile row straight into
// its owner's window, in this rank's slot, so the transfer overlaps the math tile by tile.
// Then:
//   signal  after its GEMM, rank r publishes epoch e into every owner's ready[r] (a system-scope
//           release store, after a system-scope fence in every GEMM CTA);
//   reduce  owner o waits until ready[r] >= e for all r, sums its R slots in rank order (fixed:
//           bitwise deterministic), writes its grad_W shard, then publishes e into every
//           writer's consumed[o];
//   guard   before the next GEMM writes into owner o's window, rank r waits until consumed[o]
//           >= e - 1 (o has finished reading the previous epoch's slots).
// The epoch lives in device memory: the guard kernel advances it and the signal and reduce
// kernels read it (stream-ordered after the guard), so a captured step can be replayed.
// No cycle exists (writers never wait for anything but the previous epoch's readers), and
// every wait is bounded: on timeout the kernel sets AGENTRL_ST_COMM_TIMEOUT and returns instead
// of hanging the GPU.
#include <cuda_runtime.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "internal.h"

namespace agentrl {

// about 20 s of polling with 1 us sleeps before declaring a peer dead
constexpr long long SPIN_LIMIT = 20000000LL;

__device__ __forceinline__ long long ld_acquire_sys(const int64_t* p) {
    long long v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(int64_t* p, long long v) {
    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// wait until flags[i] >= want for i in [0, n); false on timeout
__device__ bool wait_flags(const int64_t* flags, int n, long long want) {
    for (int i = 0; i < n; ++i) {
        long long it = 0;
        while (ld_acquire_sys(flags + i) < want) {
            __nanosleep(1000);
            if (++it > SPIN_LIMIT) return false;
        }
    }
    return true;
}

// rank r -> every owner o: "my tiles of epoch e are in your window"  (flags[0][r])
__global__ void k_peer_signal(int64_t* const* peer_flags, int world, int rank,
                              const int64_t* d_epoch) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const long long epoch = *d_epoch;
        __threadfence_system();
        for (int o = 0; o < world; ++o) st_release_sys(peer_flags[o] + rank, epoch);
    }
}

// owner: wait for every writer, sum the R slots in rank order into the grad_W shard, then tell
// every writer its slot may be rewritten (flags[1][owner] on the writer)
__global__ void __launch_bounds__(256)
    k_peer_reduce(const int64_t* my_flags, int64_t* const* peer_flags, int world, int rank,
                  const int64_t* d_epoch, const float* staging, float* __restrict__ out,
                  int64_t n, int32_t* done_ctr, int32_t* d_status) {
    __shared__ int ok;
    __shared__ long long epoch;
    if (threadIdx.x == 0) {
        epoch = *d_epoch;
        ok = wait_flags(my_flags, world, epoch);
        if (!ok) atomicOr(d_status, AGENTRL_ST_COMM_TIMEOUT);
    }
    __syncthreads();
    if (ok) {
        const int64_t n4 = n / 4;
        const float4* s4 = reinterpret_cast<const float4*>(staging);
        float4* o4 = reinterpret_cast<float4*>(out);
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
             i += (int64_t)gridDim.x * blockDim.x) {
            // L2 loads (ld.global.cg): the slots are written by peers while this kernel waits,
            // so the non-coherent read-only path is not allowed here
            float4 acc = __ldcg(s4 + i);
            for (int r = 1; r < world; ++r) {
                const float4 v = __ldcg(s4 + (int64_t)r * n4 + i);
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
            o4[i] = acc;
        }
    }
    // the last block to finish releases the slots
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(done_ctr, 1) == (int)gridDim.x - 1) {
            *done_ctr = 0;
            __threadfence_system();
            for (int w = 0; w < world; ++w) st_release_sys(peer_flags[w] + world + rank, epoch);
        }
    }
}

// writer: before writing into the owners' windows for epoch e, every owner must have consumed
// epoch e - 1 (flags[1][o] on this rank)
__global__ void k_peer_guard(const int64_t* my_flags, int world, int64_t* d_epoch,
                             int32_t* d_status) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const long long prev = *d_epoch;
        *d_epoch = prev + 1;  // this call's epoch (every rank makes the same sequence of calls)
        if (prev > 0 && !wait_flags(my_flags + world, world, prev))
            atomicOr(d_status, AGENTRL_ST_COMM_TIMEOUT);
    }
}

// ------------------------------------------------------------------ host
static bool p2p_disabled() {
    const char* e = getenv("AGENTRL_C3_P2P");
    return e && e[0] == '0';
}

int peer_window_create(agentrl_comm c, size_t bytes, PeerWindow** out) {
    const int R = comm_world(c), rank = comm_rank(c);
    if (R <= 0 || R > PeerWindow::MAX_RANKS) return AGENTRL_ERR_UNSUPPORTED;
    PeerWindow* pw = new PeerWindow();
    pw->world = R;
    pw->rank = rank;
    pw->bytes = (bytes + 255) / 256 * 256;
    cudaStream_t s = nullptr;
    int64_t* xch = nullptr;
    constexpr int HWORDS = (int)(sizeof(cudaIpcMemHandle_t) / sizeof(int64_t));  // 8
    static_assert(sizeof(cudaIpcMemHandle_t) % sizeof(int64_t) == 0, "handle size");
    std::vector<int64_t> host((size_t)R * 2 * HWORDS, 0);
    int rc = AGENTRL_ERR_CUDA;
    auto fail = [&](int code) {
        if (xch) cudaFree(xch);
        if (s) cudaStreamDestroy(s);
        peer_window_destroy(pw);
        return code;
    };
    if (cudaMalloc(&pw->staging, pw->bytes) != cudaSuccess) return fail(AGENTRL_ERR_CUDA);
    if (cudaMalloc(&pw->flags, sizeof(int64_t) * 2 * R) != cudaSuccess) return fail(AGENTRL_ERR_CUDA);
    if (cudaMemset(pw->flags, 0, sizeof(int64_t) * 2 * R) != cudaSuccess) return fail(AGENTRL_ERR_CUDA);
    if (cudaMalloc(&pw->d_staging, sizeof(float*) * R) != cudaSuccess) return fail(AGENTRL_ERR_CUDA);
    if (cudaMalloc(&pw->d_flags, sizeof(int64_t*) * R) != cudaSuccess) return fail(AGENTRL_ERR_CUDA);
    // exchange the IPC handles of (staging, flags) with a sum all-reduce of slot buffers
    if (R > 1) {
        cudaIpcMemHandle_t hs, hf;
        if (cudaIpcGetMemHandle(&hs, pw->staging) != cudaSuccess ||
            cudaIpcGetMemHandle(&hf, pw->flags) != cudaSuccess)
            return fail(AGENTRL_ERR_CUDA);
        memcpy(&host[(size_t)rank * 2 * HWORDS], &hs, sizeof(hs));
        memcpy(&host[(size_t)rank * 2 * HWORDS + HWORDS], &hf, sizeof(hf));
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaMalloc(&xch, sizeof(int64_t) * host.size()) != cudaSuccess ||
            cudaMemcpy(xch, host.data(), sizeof(int64_t) * host.size(), cudaMemcpyHostToDevice) !=
                cudaSuccess)
            return fail(AGENTRL_ERR_CUDA);
        if ((rc = comm_allreduce_i64(c, xch, host.size(), s)) != AGENTRL_OK) return fail(rc);
        if (cudaStreamSynchronize(s) != cudaSuccess ||
            cudaMemcpy(host.data(), xch, sizeof(int64_t) * host.size(), cudaMemcpyDeviceToHost) !=
                cudaSuccess)
            return fail(AGENTRL_ERR_CUDA);
    }
    std::vector<float*> st(R);
    std::vector<int64_t*> fl(R);
    for (int o = 0; o < R; ++o) {
        if (o == rank) {
            st[o] = pw->staging;
            fl[o] = pw->flags;
            continue;
        }
        cudaIpcMemHandle_t hs, hf;
        memcpy(&hs, &host[(size_t)o * 2 * HWORDS], sizeof(hs));
        memcpy(&hf, &host[(size_t)o * 2 * HWORDS + HWORDS], sizeof(hf));
        void* ps = nullptr;
        void* pf = nullptr;
        if (cudaIpcOpenMemHandle(&ps, hs, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
            return fail(AGENTRL_ERR_CUDA);
        pw->opened[o] = ps;
        if (cudaIpcOpenMemHandle(&pf, hf, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
            return fail(AGENTRL_ERR_CUDA);
        pw->opened_flags[o] = pf;
        st[o] = static_cast<float*>(ps);
        fl[o] = static_cast<int64_t*>(pf);
    }
    if (cudaMemcpy(pw->d_staging, st.data(), sizeof(float*) * R, cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaMemcpy(pw->d_flags, fl.data(), sizeof(int64_t*) * R, cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaMalloc(&pw->done_ctr, sizeof(int32_t)) != cudaSuccess ||
        cudaMemset(pw->done_ctr, 0, sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&pw->d_epoch, sizeof(int64_t)) != cudaSuccess ||
        cudaMemset(pw->d_epoch, 0, sizeof(int64_t)) != cudaSuccess)
        return fail(AGENTRL_ERR_CUDA);
    if (xch) cudaFree(xch);
    if (s) cudaStreamDestroy(s);
    *out = pw;
    return AGENTRL_OK;
}

void peer_window_destroy(PeerWindow* pw) {
    if (!pw) return;
    cudaDeviceSynchronize();
    for (int o = 0; o < PeerWindow::MAX_RANKS; ++o) {
        if (pw->opened[o]) cudaIpcCloseMemHandle(pw->opened[o]);
        if (pw->opened_flags[o]) cudaIpcCloseMemHandle(pw->opened_flags[o]);
    }
    if (pw->staging) cudaFree(pw->staging);
    if (pw->flags) cudaFree(pw->flags);
    if (pw->d_staging) cudaFree(pw->d_staging);
    if (pw->d_flags) cudaFree(pw->d_flags);
    if (pw->done_ctr) cudaFree(pw->done_ctr);
    if (pw->d_epoch) cudaFree(pw->d_epoch);
    delete pw;
}

// usable for a grad_W of V x d floats?
bool peer_window_fits(const PeerWindow* pw, int32_t V, int32_t d) {
    return pw && !p2p_disabled() && pw->world > 1 && V % pw->world == 0 &&
           (size_t)V * d * sizeof(float) <= pw->bytes && d % 4 == 0;
}

int peer_guard(PeerWindow* pw, int32_t* d_status, cudaStream_t s) {
    k_peer_guard<<<1, 32, 0, s>>>(pw->flags, pw->world, pw->d_epoch, d_status);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? AGENTRL_OK : AGENTRL_ERR_CUDA;
}

int peer_signal_reduce(PeerWindow* pw, float* grad_W, int32_t V, int32_t d, int32_t* d_status,
                       cudaStream_t s) {
    const int R = pw->world;
    const int64_t rows = V / R, n = rows * (int64_t)d;
    k_peer_signal<<<1, 32, 0, s>>>(pw->d_flags, R, pw->rank, pw->d_epoch);
    count_launch();
    const int grid = std::max(1, std::min<int>(num_sms() / 4, (int)((n / 4 + 255) / 256)));
    k_peer_reduce<<<grid, 256, 0, s>>>(pw->flags, pw->d_flags, R, pw->rank, pw->d_epoch, pw->staging,
                                       grad_W + (int64_t)pw->rank * n, n, pw->done_ctr, d_status);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? AGENTRL_OK : AGENTRL_ERR_CUDA;
}

}  // namespace agentrl
