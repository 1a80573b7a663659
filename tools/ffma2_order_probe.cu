// FFMA2 issue-order probe: the 8x8 smem-fed inner loop in several source orders.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ void fma2p(unsigned long long &c, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}
template <int ORDER, int RM, int RN, int MINB>
__global__ void __launch_bounds__(256, MINB) k(float *out, int iters) {
    constexpr int NT = 256, TY = NT / 16, BM = TY * RM, BN = 16 * RN;
    extern __shared__ __align__(16) float sm[];
    float *As = sm, *Bs = sm + 32 * BM;
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    for (int i = tid; i < 32 * (BM + BN); i += NT) sm[i] = 1e-3f * (i % 7);
    __syncthreads();
    unsigned long long acc[RM][RN / 2];
#pragma unroll
    for (int i = 0; i < RM; i++)
#pragma unroll
        for (int j = 0; j < RN / 2; j++) acc[i][j] = pack2(i + tid, j);
    for (int it = 0; it < iters; it++) {
        int off = 0;
        asm volatile("" : "+r"(off));
#pragma unroll
        for (int kk = 0; kk < 32; kk++) {
            float af[RM];
            unsigned long long bp[RN / 2];
#pragma unroll
            for (int q = 0; q < RM / 4; q++) {
                const float4 v = *reinterpret_cast<const float4 *>(As + kk * BM + q * (BM / (RM / 4)) + ty * 4 + off);
                af[4 * q] = v.x; af[4 * q + 1] = v.y; af[4 * q + 2] = v.z; af[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int q = 0; q < RN / 4; q++) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(Bs + kk * BN + q * (BN / (RN / 4)) + tx * 4 + off);
                bp[2 * q] = v.x; bp[2 * q + 1] = v.y;
            }
            if (ORDER == 0) {
#pragma unroll
                for (int i = 0; i < RM; i++)
#pragma unroll
                    for (int jp = 0; jp < RN / 2; jp++) fma2p(acc[i][jp], pack2(af[i], af[i]), bp[jp]);
            } else if (ORDER == 1) {  // a-major snake
#pragma unroll
                for (int i = 0; i < RM; i++)
#pragma unroll
                    for (int jq = 0; jq < RN / 2; jq++) {
                        const int jp = (i & 1) ? RN / 2 - 1 - jq : jq;
                        fma2p(acc[i][jp], pack2(af[i], af[i]), bp[jp]);
                    }
            } else if (ORDER == 2) {  // b-major
#pragma unroll
                for (int jp = 0; jp < RN / 2; jp++)
#pragma unroll
                    for (int i = 0; i < RM; i++) fma2p(acc[i][jp], pack2(af[i], af[i]), bp[jp]);
            } else if (ORDER == 4) {  // mirrored: a pairs, b scalars, pair-outer
#pragma unroll
                for (int ip = 0; ip < RM / 2; ip++)
#pragma unroll
                    for (int j = 0; j < RN / 2; j++) {
                        const unsigned long long ap = pack2(af[2 * ip], af[2 * ip + 1]);
                        fma2p(acc[ip * 2][j], ap, pack2(__uint_as_float((unsigned)bp[j]), __uint_as_float((unsigned)bp[j])));
                        fma2p(acc[ip * 2 + 1][j], ap, pack2(__uint_as_float((unsigned)(bp[j] >> 32)), __uint_as_float((unsigned)(bp[j] >> 32))));
                    }
            } else {  // b-major snake
#pragma unroll
                for (int jp = 0; jp < RN / 2; jp++)
#pragma unroll
                    for (int iq = 0; iq < RM; iq++) {
                        const int i = (jp & 1) ? RM - 1 - iq : iq;
                        fma2p(acc[i][jp], pack2(af[i], af[i]), bp[jp]);
                    }
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < RM; i++)
#pragma unroll
        for (int j = 0; j < RN / 2; j++) s += __uint_as_float((unsigned)acc[i][j]);
    out[blockIdx.x * 256 + tid] = s;
}
template <int ORDER, int RM, int RN, int MINB = 2>
void run(int sms, float *out) {
    const int iters = 2000, blocks = sms * MINB, NT = 256;
    const int smem = 32 * ((NT / 16) * RM + 16 * RN) * 4;
    cudaFuncSetAttribute(k<ORDER, RM, RN, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<ORDER, RM, RN, MINB><<<blocks, 256, smem>>>(out, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 3; r++) {
        cudaEventRecord(e0);
        k<ORDER, RM, RN, MINB><<<blocks, 256, smem>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double flop = 2.0 * blocks * (double)NT * iters * 32 * RM * RN;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double peak = sms * 256.0 * clk * 1e3;
    printf("order %d %dx%d minb %d: %.2f TFLOP/s = %.3f of peak\n", ORDER, RM, RN, MINB, flop / best / 1e9, flop / best * 1e3 / peak);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out; cudaMalloc(&out, (1 << 20) * 4);
    run<0, 8, 8>(sms, out); run<1, 8, 8>(sms, out); run<2, 8, 8>(sms, out); run<3, 8, 8>(sms, out); run<4, 8, 8>(sms, out);
    run<0, 8, 16, 1>(sms, out); run<2, 8, 16, 1>(sms, out); run<4, 8, 16, 1>(sms, out);
    run<0, 16, 8, 1>(sms, out); run<2, 16, 8, 1>(sms, out); run<4, 16, 8, 1>(sms, out);
    run<2, 8, 8, 1>(sms, out); run<2, 12, 8, 1>(sms, out); run<2, 8, 12, 1>(sms, out);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
