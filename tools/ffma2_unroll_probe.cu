// FFMA2 issue probe, part 2 (development probe): the b-pair-major 8 x 8 loop
// of the matmul leaf with the k loop unrolled U steps at a time (ptxas
// schedules within the unrolled body) and with the b loads issued before the
// a loads.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fu tools/ffma2_unroll_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ void fma2p(unsigned long long &c, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}
template <int U, bool BFIRST>
__global__ void __launch_bounds__(256, 2) k(float *out, int iters) {
    constexpr int BM = 128, BN = 128;
    extern __shared__ __align__(16) float sm[];
    float *As = sm, *Bs = sm + 32 * BM;
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    for (int i = tid; i < 32 * (BM + BN); i += 256) sm[i] = 1e-3f * (i % 7);
    __syncthreads();
    unsigned long long acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = pack2(i + tid, j);
    for (int it = 0; it < iters; it++) {
        int off = 0;
        asm volatile("" : "+r"(off));
#pragma unroll 1
        for (int k0 = 0; k0 < 32; k0 += U) {
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int kk = k0 + u;
                float4 a0, a1;
                ulonglong2 b0, b1;
                if (BFIRST) {
                    b0 = *reinterpret_cast<const ulonglong2 *>(Bs + kk * BN + tx * 4 + off);
                    b1 = *reinterpret_cast<const ulonglong2 *>(Bs + kk * BN + BN / 2 + tx * 4 + off);
                }
                a0 = *reinterpret_cast<const float4 *>(As + kk * BM + ty * 4 + off);
                a1 = *reinterpret_cast<const float4 *>(As + kk * BM + BM / 2 + ty * 4 + off);
                if (!BFIRST) {
                    b0 = *reinterpret_cast<const ulonglong2 *>(Bs + kk * BN + tx * 4 + off);
                    b1 = *reinterpret_cast<const ulonglong2 *>(Bs + kk * BN + BN / 2 + tx * 4 + off);
                }
                const float af[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const unsigned long long bp[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
                for (int jp = 0; jp < 4; jp++)
#pragma unroll
                    for (int i = 0; i < 8; i++) fma2p(acc[i][jp], pack2(af[i], af[i]), bp[jp]);
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) s += __uint_as_float((unsigned)acc[i][j]);
    out[blockIdx.x * 256 + tid] = s;
}
template <int U, bool BFIRST>
void run(int sms, float *out) {
    const int iters = 2000, blocks = sms * 2;
    const int smem = 32 * 256 * 4;
    cudaFuncSetAttribute(k<U, BFIRST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<U, BFIRST><<<blocks, 256, smem>>>(out, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 3; r++) {
        cudaEventRecord(e0);
        k<U, BFIRST><<<blocks, 256, smem>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double flop = 2.0 * blocks * 256.0 * iters * 32 * 64;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double peak = sms * 256.0 * clk * 1e3;
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k<U, BFIRST>);
    printf("unroll %2d b-first %d (%3d regs): %.2f TFLOP/s = %.3f of peak\n", U, BFIRST, fa.numRegs, flop / best / 1e9,
           flop / best * 1e3 / peak);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; cudaMalloc(&out, (1 << 20) * 4);
    run<32, false>(sms, out); run<32, true>(sms, out);
    run<1, false>(sms, out); run<2, false>(sms, out); run<4, false>(sms, out); run<8, false>(sms, out);
    run<16, false>(sms, out); run<4, true>(sms, out); run<8, true>(sms, out);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
