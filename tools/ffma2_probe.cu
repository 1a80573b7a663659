// FFMA2 throughput ceiling (development probe): the matmul leaf's inner loop
// (RM x RN outputs per thread, packed column pairs, scalar a broadcast) with
// its operands from shared memory (RM/4 + RN/4 LDS.128 per k step) or from
// registers only.  No barriers, no global traffic: the number is what the FFMA
// pipe gives this instruction mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2 tools/ffma2_probe.cu && /tmp/ffma2
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ void fma2p(unsigned long long &c, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}

template <bool SMEM, int MINB, int RM, int RN, int NT = 256>
__global__ void __launch_bounds__(NT, MINB) k(float *out, int iters) {
    constexpr int TX = 16, TY = NT / 16;
    constexpr int BM = TY * RM, BN = TX * RN;
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
    float4 ra = make_float4(tid, 1, 2, 3);
    ulonglong2 rb = make_ulonglong2(tid, 5);
    for (int it = 0; it < iters; it++) {
        int off = 0;  // laundered each iteration: the shared loads are not loop-invariant
        asm volatile("" : "+r"(off));
#pragma unroll
        for (int kk = 0; kk < 32; kk++) {
            float af[RM];
            unsigned long long bp[RN / 2];
#pragma unroll
            for (int q = 0; q < RM / 4; q++) {
                const float4 v = SMEM ? *reinterpret_cast<const float4 *>(As + kk * BM + q * (BM / (RM / 4)) + ty * 4 + off) : ra;
                af[4 * q] = v.x; af[4 * q + 1] = v.y; af[4 * q + 2] = v.z; af[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int q = 0; q < RN / 4; q++) {
                const ulonglong2 v = SMEM ? *reinterpret_cast<const ulonglong2 *>(Bs + kk * BN + q * (BN / (RN / 4)) + tx * 4 + off) : rb;
                bp[2 * q] = v.x; bp[2 * q + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < RM; i++) {
                const unsigned long long ai = pack2(af[i], af[i]);
#pragma unroll
                for (int jp = 0; jp < RN / 2; jp++) fma2p(acc[i][jp], ai, bp[jp]);
            }
        }
        if (!SMEM) { ra.x += 1.0f; rb.x ^= 1; }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < RM; i++)
#pragma unroll
        for (int j = 0; j < RN / 2; j++) s += __uint_as_float((unsigned)acc[i][j]);
    out[blockIdx.x * NT + tid] = s;
}

template <bool SMEM, int MINB, int RM, int RN, int NT = 256>
void run(const char *name, int per_sm, int sms, float *out, int blocks_override = 0) {
    const int iters = 1000, blocks = blocks_override ? blocks_override : sms * per_sm;
    const int smem = 32 * ((NT / 16) * RM + 16 * RN) * 4;
    cudaFuncSetAttribute(k<SMEM, MINB, RM, RN, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<SMEM, MINB, RM, RN, NT><<<blocks, 256, smem>>>(out, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<SMEM, MINB, RM, RN, NT><<<blocks, 256, smem>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * blocks * (double)NT * iters * 32 * RM * RN;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double peak = sms * 256.0 * clk * 1e3;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<SMEM, MINB, RM, RN, NT>);
    printf("%-10s %2dx%-2d %3d thr %4d CTAs (%3d regs): %.2f TFLOP/s = %.3f of %.2f (max clock)\n", name, RM, RN, NT,
           blocks, fa.numRegs, flop / ms / 1e9, flop / ms * 1e3 / peak, peak / 1e12);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, (1 << 20) * 4);
    run<false, 2, 8, 8>("registers", 2, sms, out);
    run<true, 2, 8, 8>("smem", 2, sms, out);
    run<true, 1, 8, 8>("smem", 1, sms, out);
    run<true, 1, 8, 16>("smem", 1, sms, out);
    run<true, 1, 16, 8>("smem", 1, sms, out);
    run<true, 1, 12, 8>("smem", 1, sms, out);
    run<true, 1, 8, 12>("smem", 1, sms, out);
    // n = 1024: 2^20 outputs in all; threads = 2^20 / (RM * RN)
    printf("n = 1024 (2^20 outputs):\n");
    run<true, 1, 4, 8, 256>("smem", 0, sms, out, (1 << 20) / 32 / 256);
    run<true, 1, 4, 4, 256>("smem", 0, sms, out, (1 << 20) / 16 / 256);
    run<true, 1, 8, 4, 256>("smem", 0, sms, out, (1 << 20) / 32 / 256);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
