// Host-ABI step transport probe: graph replay + sync vs a persistent kernel
// polling a doorbell in mapped page-locked memory.  Each "step" reads A f64
// per env and writes D f64 + 1 f64 + 2 bytes per env through the host link
// (the C2 host-ABI traffic: 4096 envs, A = 6, D = 12), or nothing (payload 0).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a doorbell.cu -o doorbell
#include <cuda_runtime.h>
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>

struct alignas(64) Box {
    volatile uint64_t epoch;
    volatile uint64_t cmd;
    uint64_t pad[6];
    volatile uint64_t ack[1024 * 8];   // one 64-B line per block (stride 8)
};

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t ld_acq_sys(const volatile uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_sys(volatile uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void work(int e, int n, int A, int D, const double* act, double* obs,
                                     double* rew, uint8_t* done, float* state) {
    if (e >= n || A == 0) return;
    double s = 0.0;
    for (int j = 0; j < A; ++j) s += act[(size_t)e * A + j];
    float x = state[e] + (float)s;
    for (int k = 0; k < 40; ++k) x = fmaf(x, 0.999f, 0.001f);
    state[e] = x;
    for (int j = 0; j < D; ++j) obs[(size_t)e * D + j] = x + j;
    rew[e] = x;
    done[e] = x > 1e30f;
}

__global__ void k_step(int n, int A, int D, const double* act, double* obs, double* rew,
                       uint8_t* done, float* state) {
    work(blockIdx.x * blockDim.x + threadIdx.x, n, A, D, act, obs, rew, done, state);
}

__device__ volatile uint64_t g_epoch;
__device__ unsigned g_count;

// one host poller (block 0) relays the doorbell through device memory; the
// last block to finish writes a single ack to the host
__global__ void k_relay(Box* box, uint64_t want, uint64_t idle_ns, int n, int A, int D,
                        const double* act, double* obs, double* rew, uint8_t* done,
                        float* state) {
    __shared__ uint64_t s_cmd;
    for (;;) {
        if (threadIdx.x == 0) {
            const uint64_t t0 = gtimer();
            uint64_t cmd = 1;
            for (;;) {
                uint64_t ev;
                if (blockIdx.x == 0) {
                    ev = ld_acq_sys(&box->epoch);
                    if (ev == want) {
                        cmd = box->cmd;
                        g_epoch = (want << 1) | cmd;
                        break;
                    }
                } else {
                    ev = g_epoch;
                    if ((ev >> 1) == want) {
                        cmd = ev & 1;
                        break;
                    }
                }
                if (gtimer() - t0 > idle_ns) break;
            }
            s_cmd = cmd;
        }
        __syncthreads();
        if (s_cmd != 0) return;
        work(blockIdx.x * blockDim.x + threadIdx.x, n, A, D, act, obs, rew, done, state);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            if (atomicAdd(&g_count, 1u) == gridDim.x - 1) {
                g_count = 0;
                __threadfence_system();
                st_rel_sys(&box->ack[0], want);
            }
        }
        ++want;
    }
}

template <int MODE>   // 0: ld.acquire.sys poll, 1: volatile poll + fence, 2: volatile + nanosleep
__global__ void k_persist(Box* box, uint64_t want, uint64_t idle_ns, int n, int A, int D,
                          const double* act, double* obs, double* rew, uint8_t* done,
                          float* state) {
    __shared__ uint64_t s_cmd;
    for (;;) {
        if (threadIdx.x == 0) {
            const uint64_t t0 = gtimer();
            uint64_t cmd = 1;
            for (;;) {
                uint64_t ev;
                if (MODE == 0) ev = ld_acq_sys(&box->epoch);
                else ev = box->epoch;
                if (ev == want) {
                    if (MODE != 0) __threadfence_system();
                    cmd = box->cmd;
                    break;
                }
                if (MODE == 2) __nanosleep(200);
                if (gtimer() - t0 > idle_ns) break;
            }
            s_cmd = cmd;
        }
        __syncthreads();
        if (s_cmd != 0) return;
        work(blockIdx.x * blockDim.x + threadIdx.x, n, A, D, act, obs, rew, done, state);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            st_rel_sys(&box->ack[blockIdx.x * 8], want);
        }
        ++want;
    }
}

template <class F> double bench(const char* name, F f, int n = 20000) {
    for (int i = 0; i < 1000; ++i) f();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
    printf("%-52s %.3f us\n", name, us);
    return us;
}

int main() {
    const int n = 4096, A = 6, D = 12, B = 128, nb = (n + B - 1) / B;
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    double *act, *obs, *rew;
    uint8_t* done;
    float* state;
    cudaHostAlloc(&act, (size_t)n * A * 8, cudaHostAllocMapped);
    cudaHostAlloc(&obs, (size_t)n * D * 8, cudaHostAllocMapped);
    cudaHostAlloc(&rew, (size_t)n * 8, cudaHostAllocMapped);
    cudaHostAlloc(&done, (size_t)n, cudaHostAllocMapped);
    cudaMalloc(&state, (size_t)n * 4);
    cudaMemset(state, 0, (size_t)n * 4);
    memset(act, 0, (size_t)n * A * 8);
    Box* box;
    cudaHostAlloc(&box, sizeof(Box), cudaHostAllocMapped);
    memset((void*)box, 0, sizeof(Box));

    for (int payload = 0; payload < 2; ++payload) {
        const int a = payload ? A : 0, d = payload ? D : 0;
        printf("payload %s\n", payload ? "C2 (196 KB in, 430 KB out)" : "none");
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        k_step<<<nb, B, 0, s>>>(n, a, d, act, obs, rew, done, state);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        bench("graph replay + cudaStreamSynchronize", [&] {
            cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
        });
        uint64_t ep = 0;
        auto run = [&](auto kern, const char* name, int flush, int nack = -1) {
            const int na = nack < 0 ? nb : nack;
            box->epoch = ep;
            kern<<<nb, B, 0, s>>>(box, ep + 1, 2000000000ull, n, a, d, act, obs, rew, done, state);
            bench(name, [&] {
                box->cmd = 0;
                std::atomic_thread_fence(std::memory_order_release);
                box->epoch = ++ep;
                if (flush & 1) _mm_clflush((const void*)&box->epoch);
                for (int b = 0; b < na; ++b)
                    for (;;) {
                        if (flush & 2) _mm_clflush((const void*)&box->ack[b * 8]);
                        _mm_mfence();
                        if (box->ack[b * 8] == ep) break;
                    }
                std::atomic_thread_fence(std::memory_order_acquire);
            }, 5000);
            box->cmd = 1;
            std::atomic_thread_fence(std::memory_order_release);
            box->epoch = ++ep;
            _mm_clflush((const void*)&box->epoch);
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) printf("persistent exit: %s\n", cudaGetErrorString(e));
        };
        run(k_persist<0>, "persistent acq.sys poll, no flush", 0);
        run(k_persist<2>, "persistent volatile poll + nanosleep", 0);
        run(k_relay, "relay: one host poller, one ack", 0, 1);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    }
    return 0;
}
