// k_matmul_tf32.cu -- optional 3xTF32 matmul on the 5th-generation tensor
// cores (tcgen05 + TMEM + TMA), reported beside the FFMA path, never instead
// of it (BASELINE north_star: "The FP32 path stays on FFMA ... with an
// optional 3xTF32 tcgen05 variant reported separately").
//
// Same program: c[p][q] += sum_k a[p][k] * b[k][q] over the
// covered extents.  3xTF32: x = hi(x) + lo(x) with hi = tf32(x),
// lo = tf32(x - hi); a*b ~= hi(a)hi(b) + hi(a)lo(b) + lo(a)hi(b) with fp32
// accumulation in TMEM -- fp32-level accuracy (the test checks it against the
// binary64 oracle with the matmul tolerance), but NOT the FFMA path's exact
// ascending-k rounding sequence.
//
// Structure
//  * k_split_rows: a -> (a_hi, a_lo), row-major M x K (K-major for UMMA A)
//  * k_split_cols: b -> (bt_hi, bt_lo) transposed to N x K (K-major for UMMA B)
//  * k_tf32x3: one 128 x 256 output tile per CTA (4 warps):
//      warp 0 lane 0: TMA producer, 2-stage ring of {a_hi, a_lo, bt_hi, bt_lo}
//                     128B-swizzled 32-wide K slabs (96 KB per stage)
//      warp 1 lane 0: MMA issuer, tcgen05.mma.cta_group::1.kind::tf32
//                     M=128 N=256 K=8, 3 products x 4 k-steps per slab,
//                     tcgen05.commit frees the slab / signals the epilogue
//      warps 0-3:     epilogue, tcgen05.ld 32x32b.x32 from TMEM, + c, store
#include <cuda.h>

#include <cstdlib>

#include "pk_internal.cuh"

namespace pk {
namespace {

#ifndef PK_TF32_TK
#define PK_TF32_TK 32
#endif
// K slab: 32 fp32 = one 128-byte swizzle row, 2 stages of 96 KB.  (16-wide
// slabs with 64-byte swizzle and 4 stages of 48 KB compile too,
// -DPK_TF32_TK=16: 5.38 ms at n = 8192 against 4.73 -- the ring depth is not
// what limits this kernel.)
constexpr int TM = 128, TN = 256, TK = PK_TF32_TK;
constexpr int A_BYTES = TM * TK * 4;
constexpr int B_BYTES = TN * TK * 4;
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int STAGES = TK == 32 ? 2 : 4;
constexpr int SWZ_BYTES = TK * 4;                // swizzle span = one slab row (64 or 128 B)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t TMEM_COLS = 256;

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// a (M x K row-major) -> hi, lo (same layout)
__global__ void __launch_bounds__(256) k_split_rows(const float *__restrict__ a, float *__restrict__ hi,
                                                   float *__restrict__ lo, int64_t n4) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = reinterpret_cast<const float4 *>(a)[i];
        float4 h, l;
        h.x = tf32_rna(v.x); l.x = tf32_rna(v.x - h.x);
        h.y = tf32_rna(v.y); l.y = tf32_rna(v.y - h.y);
        h.z = tf32_rna(v.z); l.z = tf32_rna(v.z - h.z);
        h.w = tf32_rna(v.w); l.w = tf32_rna(v.w - h.w);
        reinterpret_cast<float4 *>(hi)[i] = h;
        reinterpret_cast<float4 *>(lo)[i] = l;
    }
}

// b (K x N row-major, leading dimension ldb) -> bt_hi, bt_lo (N x K row-major), 32x32 tiles
__global__ void __launch_bounds__(256) k_split_cols(const float *__restrict__ b, float *__restrict__ hi,
                                                   float *__restrict__ lo, int64_t K, int64_t N, int64_t ldb) {
    __shared__ float t[32][33];
    const int64_t k0 = (int64_t)blockIdx.y * 32, n0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int r = ty; r < 32; r += 8) t[r][tx] = b[(k0 + r) * ldb + n0 + tx];
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const float v = t[tx][r];  // b[k0+tx][n0+r]
        const float h = tf32_rna(v);
        hi[(n0 + r) * K + k0 + tx] = h;
        lo[(n0 + r) * K + k0 + tx] = tf32_rna(v - h);
    }
}

// ---- tcgen05 / TMA helpers ---------------------------------------------------

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// K-major swizzled UMMA shared-memory descriptor: rows of SWZ_BYTES, 8-row
// atoms stacked contiguously (SBO = 8 rows), LBO unused; layout type 2 =
// 128-byte swizzle, 4 = 64-byte swizzle (sm_100 descriptor encoding).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void *p) {
    const uint64_t addr = smem_u32(p);
    constexpr uint64_t sbo = (8 * SWZ_BYTES) >> 4, layout = SWZ_BYTES == 128 ? 2 : 4;
    return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (sbo << 32) | (1ull << 46) | (layout << 61);
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- the GEMM ------------------------------------------------------------------

__global__ void __launch_bounds__(128, 1) k_tf32x3(const __grid_constant__ CUtensorMap map_ahi,
                                                  const __grid_constant__ CUtensorMap map_alo,
                                                  const __grid_constant__ CUtensorMap map_bhi,
                                                  const __grid_constant__ CUtensorMap map_blo, float *__restrict__ c,
                                                  int64_t ldc, int64_t row0, int ntn, int kslabs) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *done = empty + STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tm = blockIdx.x / ntn, tn = blockIdx.x % ntn;
    const int m0 = tm * TM, n0 = tn * TN;  // tile origin (rows relative to row0, the shard start)

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 1) {  // TMEM: 256 fp32 columns x 128 lanes for the accumulator
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer
        for (int kb = 0; kb < kslabs; kb++) {
            const int s = kb % STAGES;
            mbar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
            unsigned char *st = smem + s * STAGE_BYTES;
            mbar_expect_tx(&full[s], STAGE_BYTES);
            const int kc = kb * TK;
            tma_load_2d(st, &map_ahi, &full[s], kc, (int)row0 + m0);
            tma_load_2d(st + A_BYTES, &map_alo, &full[s], kc, (int)row0 + m0);
            tma_load_2d(st + 2 * A_BYTES, &map_bhi, &full[s], kc, n0);
            tma_load_2d(st + 2 * A_BYTES + B_BYTES, &map_blo, &full[s], kc, n0);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer
        constexpr uint32_t idesc = idesc_tf32(TM, TN);
        for (int kb = 0; kb < kslabs; kb++) {
            const int s = kb % STAGES;
            mbar_wait(&full[s], (kb / STAGES) & 1);
            tc_fence_after();
            unsigned char *st = smem + s * STAGE_BYTES;
            const uint64_t ahi = smem_desc_sw128(st), alo = smem_desc_sw128(st + A_BYTES);
            const uint64_t bhi = smem_desc_sw128(st + 2 * A_BYTES), blo = smem_desc_sw128(st + 2 * A_BYTES + B_BYTES);
#pragma unroll
            for (int kk = 0; kk < TK / 8; kk++) {
                const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 8 tf32 = 32 B along K inside the swizzle row
                // small terms first, then the leading product
                mma_tf32(tmem, alo + adv, bhi + adv, idesc, (kb | kk) != 0);
                mma_tf32(tmem, ahi + adv, blo + adv, idesc, 1);
                mma_tf32(tmem, ahi + adv, bhi + adv, idesc, 1);
            }
            mma_commit(&empty[s]);  // slab s free once these MMAs retire
        }
        mma_commit(done);  // accumulator complete
    }
    __syncwarp();

    // ---- epilogue: all 4 warps, warp w owns TMEM lanes / tile rows 32w .. 32w+31
    mbar_wait(done, 0);
    tc_fence_after();
    const int64_t row = row0 + m0 + warp * 32 + lane;
    float *crow = c + row * ldc + n0;
#pragma unroll 1
    for (int cc = 0; cc < TN; cc += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)cc, r);
        float4 *dst = reinterpret_cast<float4 *>(crow + cc);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            float4 v = dst[q];
            v.x += __uint_as_float(r[4 * q + 0]);
            v.y += __uint_as_float(r[4 * q + 1]);
            v.z += __uint_as_float(r[4 * q + 2]);
            v.w += __uint_as_float(r[4 * q + 3]);
            dst[q] = v;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ---- the 2-CTA form (default): a CTA pair on one TPC computes a 256 x 256
// tile with tcgen05.mma.cta_group::2 (M = 256: each CTA's 128 rows of A and
// 128 of the 256 columns of B in its own shared memory, the accumulator rows
// of each CTA in its own TMEM).  Per SM and slab the operand bytes drop from
// 96 KB to 64 KB (B is split across the pair), so the ring holds 3 stages.
// Protocol (CUTLASS's 2x1SM pipeline): both CTAs' producers load their
// halves with the 2-SM TMA, which completes on the LEADER's full barrier
// (peer bit cleared from the barrier address); the leader arms that barrier
// for both halves' bytes; the leader's single MMA thread issues the MMAs and
// commits to the empty barriers of both CTAs (multicast) -- each producer
// refills its own stage -- and finally to both CTAs' done barriers.
constexpr int P_BN = 128;                              // B columns per CTA of the pair
constexpr int P_B_BYTES = P_BN * TK * 4;
constexpr int P_STAGE_BYTES = 2 * A_BYTES + 2 * P_B_BYTES;
constexpr int P_STAGES = 3;
constexpr int P_SMEM_BYTES = P_STAGES * P_STAGE_BYTES + 1024 + 256;
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;         // shared::cluster address -> CTA 0 of the pair

__device__ __forceinline__ void tma_load_2d_2sm(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void mma_tf32_2sm(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                             uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_commit_pair(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((unsigned short)3)
        : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_tf32x3_pair(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                  const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                  float *__restrict__ c, int64_t ldc, int ntn, int kslabs) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + P_STAGES * P_STAGE_BYTES);
    uint64_t *empty = full + P_STAGES;
    uint64_t *done = empty + P_STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1;
    const int tm = pair / ntn, tn = pair % ntn;
    const int m0 = tm * 2 * TM + (int)rank * TM;  // this CTA's rows (relative to the a-split buffer)
    const int nb = tn * TN + (int)rank * P_BN;     // this CTA's half of the B columns
    const int n0 = tn * TN;                         // output columns of the pair tile

    if (threadIdx.x == 0) {
        for (int s = 0; s < P_STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();  // both CTAs' barriers initialised before any remote arrival
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer (both CTAs): this CTA's halves, completing on the leader's full barrier
        for (int kb = 0; kb < kslabs; kb++) {
            const int s = kb % P_STAGES;
            mbar_wait(&empty[s], ((kb / P_STAGES) & 1) ^ 1);
            unsigned char *st = smem + s * P_STAGE_BYTES;
            if (rank == 0) mbar_expect_tx(&full[s], 2 * P_STAGE_BYTES);
            const int kc = kb * TK;
            tma_load_2d_2sm(st, &map_ahi, &full[s], kc, m0);
            tma_load_2d_2sm(st + A_BYTES, &map_alo, &full[s], kc, m0);
            tma_load_2d_2sm(st + 2 * A_BYTES, &map_bhi, &full[s], kc, nb);
            tma_load_2d_2sm(st + 2 * A_BYTES + P_B_BYTES, &map_blo, &full[s], kc, nb);
        }
    } else if (warp == 1 && lane == 0 && rank == 0) {
        // ---- MMA issuer (leader only): M = 256 across the pair, N = 256
        constexpr uint32_t idesc = idesc_tf32(2 * TM, TN);
        for (int kb = 0; kb < kslabs; kb++) {
            const int s = kb % P_STAGES;
            mbar_wait(&full[s], (kb / P_STAGES) & 1);
            tc_fence_after();
            unsigned char *st = smem + s * P_STAGE_BYTES;
            const uint64_t ahi = smem_desc_sw128(st), alo = smem_desc_sw128(st + A_BYTES);
            const uint64_t bhi = smem_desc_sw128(st + 2 * A_BYTES), blo = smem_desc_sw128(st + 2 * A_BYTES + P_B_BYTES);
#pragma unroll
            for (int kk = 0; kk < TK / 8; kk++) {
                const uint64_t adv = (uint64_t)(kk * 32) >> 4;
                mma_tf32_2sm(tmem, alo + adv, bhi + adv, idesc, (kb | kk) != 0);
                mma_tf32_2sm(tmem, ahi + adv, blo + adv, idesc, 1);
                mma_tf32_2sm(tmem, ahi + adv, bhi + adv, idesc, 1);
            }
            mma_commit_pair(&empty[s]);  // slab s free in both CTAs once these MMAs retire
        }
        mma_commit_pair(done);  // both accumulators complete
    }
    __syncwarp();

    // ---- epilogue: each CTA's 4 warps, TMEM lanes = this CTA's 128 rows
    mbar_wait(done, 0);
    tc_fence_after();
    const int64_t row = m0 + warp * 32 + lane;
    float *crow = c + row * ldc + n0;
#pragma unroll 1
    for (int cc = 0; cc < TN; cc += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)cc, r);
        float4 *dst = reinterpret_cast<float4 *>(crow + cc);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            float4 v = dst[q];
            v.x += __uint_as_float(r[4 * q + 0]);
            v.y += __uint_as_float(r[4 * q + 1]);
            v.z += __uint_as_float(r[4 * q + 2]);
            v.w += __uint_as_float(r[4 * q + 3]);
            dst[q] = v;
        }
    }
    tc_fence_before();
    cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ---- host side -------------------------------------------------------------------

typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    // resolved once; a function-local static is initialised thread-safely
    static const EncodeTiled fn = []() -> EncodeTiled {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiled>(p);
        return nullptr;
    }();
    return fn;
}

// 2-D K-major operand map: rows x K fp32, box TK x box_rows, 128B swizzle
int make_map(CUtensorMap *m, const float *base, int64_t rows, int64_t K, int box_rows) {
    EncodeTiled enc = encode_fn();
    if (!enc) return fail(PK_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 4};
    cuuint32_t box[2] = {(cuuint32_t)TK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, SWZ_BYTES == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PK_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PK_OK;
}

}  // namespace

// c[rows rlo..rhi) += a * b over K, all n x n row-major fp32; M, N, K tile-aligned.
int launch_matmul_tf32x3(const float *a, const float *b, float *c, int64_t n, int64_t rlo, int64_t rhi,
                         int64_t Nc, int64_t K, cudaStream_t st) {
    const int64_t M = rhi - rlo;
    if (M % TM || Nc % TN || K % TK || K == 0)
        return fail(PK_E_UNSUPPORTED, "3xTF32 path needs rows %% %d, cols %% %d, K %% %d (got %lld, %lld, %lld)", TM,
                    TN, TK, (long long)M, (long long)Nc, (long long)K);
    if (n > (int64_t)1 << 30) return fail(PK_E_UNSUPPORTED, "3xTF32: matrix too large for 32-bit TMA coordinates");
    // operand splits: a rows [rlo, rhi) x K, b^T: Nc x K
    float *ws = nullptr;
    const size_t a_elems = (size_t)M * K, b_elems = (size_t)Nc * K;
    cudaError_t e = scratch_alloc((void **)&ws, (2 * a_elems + 2 * b_elems) * sizeof(float), st);
    if (e != cudaSuccess) return fail(PK_E_ALLOC, "3xTF32 workspace: %s", cudaGetErrorString(e));
    float *ahi = ws, *alo = ws + a_elems, *bhi = alo + a_elems, *blo = bhi + b_elems;
    int rc = PK_OK;
    if (n == K) {
        int64_t sblocks = ceil_div((int64_t)a_elems / 4, 256);
        if (sblocks > 148 * 32) sblocks = 148 * 32;
        k_split_rows<<<(unsigned)sblocks, 256, 0, st>>>(a + rlo * n, ahi, alo, (int64_t)a_elems / 4);
        if ((rc = after_launch("tf32_split_a"))) goto out;
    } else {
        rc = fail(PK_E_UNSUPPORTED, "3xTF32: covered K != n");
        goto out;
    }
    k_split_cols<<<dim3((unsigned)(Nc / 32), (unsigned)(K / 32)), 256, 0, st>>>(b, bhi, blo, K, Nc, n);
    if ((rc = after_launch("tf32_split_b"))) goto out;
    {
        CUtensorMap mahi, malo, mbhi, mblo;
        if ((rc = make_map(&mahi, ahi, M, K, TM)) || (rc = make_map(&malo, alo, M, K, TM)) ||
            (rc = make_map(&mbhi, bhi, Nc, K, TN)) || (rc = make_map(&mblo, blo, Nc, K, TN)))
            goto out;
        const int ntn = (int)(Nc / TN);
        // the kernels' TMA row coordinate is relative to the a-split buffer (rows 0..M);
        // c rows are offset by rlo
        if (M % (2 * TM) == 0 && getenv("PK_TF32_1SM") == nullptr) {  // CTA pairs: 256 x 256 tiles
            CUtensorMap mbhi2, mblo2;
            if ((rc = make_map(&mbhi2, bhi, Nc, K, P_BN)) || (rc = make_map(&mblo2, blo, Nc, K, P_BN))) goto out;
            rc = allow_smem((const void *)k_tf32x3_pair, P_SMEM_BYTES);
            if (rc) goto out;
            const int64_t pairs = (M / (2 * TM)) * ntn;
            k_tf32x3_pair<<<(unsigned)(2 * pairs), 128, P_SMEM_BYTES, st>>>(mahi, malo, mbhi2, mblo2, c + rlo * n, n,
                                                                          ntn, (int)(K / TK));
            rc = after_launch("matmul_tf32x3_pair");
        } else {
            rc = allow_smem((const void *)k_tf32x3, SMEM_BYTES);
            if (rc) goto out;
            const int64_t tiles = (M / TM) * ntn;
            k_tf32x3<<<(unsigned)tiles, 128, SMEM_BYTES, st>>>(mahi, malo, mbhi, mblo, c + rlo * n, n, 0, ntn,
                                                               (int)(K / TK));
            rc = after_launch("matmul_tf32x3");
        }
    }
out:
    cudaFreeAsync(ws, st);
    return rc;
}

}  // namespace pk
