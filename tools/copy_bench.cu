// Streaming micro-benchmarks for the Jacobi pipelines (development aid, not product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/copy_bench tools/copy_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_store_1d(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 1. plain int4 grid-stride copy, U loads in flight per thread
template <int U>
__global__ void __launch_bounds__(256) k_ldg(const int4 *__restrict__ s, int4 *__restrict__ d, int64_t n4) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
    for (; i < n4; i += stride) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++)
            if (i + u * blockDim.x < n4) v[u] = s[i + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < U; u++)
            if (i + u * blockDim.x < n4) d[i + u * blockDim.x] = v[u];
    }
}

// 2. warp-specialised TMA ring: producer warp bulk-loads tiles, consumers store
// (mode 0: STG.128 from smem, 1: STG.64 pairs, 2: consumer does 3-point avg with STG.64)
template <int MODE>
__global__ void __launch_bounds__(288) k_ring(const int *__restrict__ s, int *__restrict__ d, int64_t ntiles, int tile,
                                             int S) {
    extern __shared__ __align__(128) int smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + 8;
    int *bufs = smem + 32;
    const int nct = blockDim.x - 32;
    if (threadIdx.x == 0) {
        for (int j = 0; j < S; j++) {
            mbar_init(&full[j], 1);
            mbar_init(&empty[j], nct / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int BW = tile + 16;
    if (threadIdx.x < 32) {
        uint32_t ph = 0;
        int b = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            mbar_wait(&empty[b], ((ph >> b) & 1) ^ 1);
            ph ^= 1u << b;
            if (threadIdx.x == 0) {
                mbar_expect_tx(&full[b], tile * 4);
                tma_load_1d(bufs + b * BW, s + t * tile, tile * 4, &full[b]);
            }
            b = b + 1 == S ? 0 : b + 1;
        }
        return;
    }
    const int ct = threadIdx.x - 32;
    uint32_t ph = 0;
    int b = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&full[b], (ph >> b) & 1);
        ph ^= 1u << b;
        const int *buf = bufs + b * BW;
        int *o = d + t * tile;
        for (int q = ct; q < tile / 4; q += nct) {
            int4 v = reinterpret_cast<const int4 *>(buf)[q];
            if (MODE == 0) {
                reinterpret_cast<int4 *>(o)[q] = v;
            } else if (MODE == 1) {
                reinterpret_cast<int2 *>(o)[2 * q] = make_int2(v.x, v.y);
                reinterpret_cast<int2 *>(o)[2 * q + 1] = make_int2(v.z, v.w);
            } else {
                int l = __shfl_up_sync(0xffffffffu, v.w, 1), r = __shfl_down_sync(0xffffffffu, v.x, 1);
                reinterpret_cast<int2 *>(o)[2 * q] = make_int2((l + v.x + v.y) / 3, (v.x + v.y + v.z) / 3);
                reinterpret_cast<int2 *>(o)[2 * q + 1] = make_int2((v.y + v.z + v.w) / 3, (v.z + v.w + r) / 3);
            }
        }
        __syncwarp();
        if ((ct & 31) == 0) mbar_arrive(&empty[b]);
        b = b + 1 == S ? 0 : b + 1;
    }
}

// 3. TMA load + TMA store: consumers copy smem->smem out buffer, one thread bulk-stores
int main(int argc, char **argv) {
    const int64_t n = (int64_t)1 << 28;
    int *a, *b;
    cudaMalloc(&a, n * 4 + 64);
    cudaMalloc(&b, n * 4 + 64);
    cudaMemset(a, 1, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto fn) {
        for (int i = 0; i < 3; i++) fn();
        cudaEventRecord(e0);
        const int R = 10;
        for (int i = 0; i < R; i++) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= R;
        printf("%-40s %8.3f ms %8.1f GB/s  (%s)\n", name, ms, 8.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    int sms = 148;
    for (int g : {1, 2, 4, 8}) {
        char nm[64];
        snprintf(nm, 64, "ldg U=4 grid=%d*148", g);
        timeit(nm, [&] { k_ldg<4><<<sms * g, 256>>>((const int4 *)a, (int4 *)b, n / 4); });
        snprintf(nm, 64, "ldg U=8 grid=%d*148", g);
        timeit(nm, [&] { k_ldg<8><<<sms * g, 256>>>((const int4 *)a, (int4 *)b, n / 4); });
    }
    timeit("ldg U=1 grid=n/256", [&] { k_ldg<1><<<n / 4 / 256, 256>>>((const int4 *)a, (int4 *)b, n / 4); });
    for (int tile : {2048, 4096, 8192}) {
        for (int S : {2, 4, 6}) {
            size_t sm = 128 + (size_t)S * (tile + 16) * 4;
            for (int mode = 0; mode < 3; mode++) {
                auto k = mode == 0 ? k_ring<0> : mode == 1 ? k_ring<1> : k_ring<2>;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                int per = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 288, sm);
                char nm[80];
                snprintf(nm, 80, "ring mode=%d tile=%d S=%d per_sm=%d", mode, tile, S, per);
                timeit(nm, [&] { k<<<sms * per, 288, sm>>>(a, b, n / tile, tile, S); });
            }
        }
    }
    return 0;
}
