// k_matmul_tma.cu -- the staged matmul leaf with its shared
// tiles fed by TMA: FP32 on the FFMA pipe, numerics identical to
// k_matmul_tiled / k_matmul_generic (every output starts from c and runs
// fma(a[p][k], b[k][q], acc) for k ascending).
//
// * a's rows of this launch are transposed once (k_transpose_rows, ~1 % of
//   the multiply at n = 8192) so both operands are plain 2-D boxes: the
//   a^T slab BK x BM and the b slab BK x BN of k-step kt are one TMA each.
//   (Loading a's rows as they lie -- a 128-byte swizzled [BM][BK] box, 8
//   scalar shared loads per k step -- saves the transpose launch and 0.5 GB
//   of DRAM traffic but measured 12 % slower: 19.3 vs 17.0 ms at n = 8192,
//   the extra loads spill at the 128-register budget.)
// * Tiles (template Tile), same thread mapping (8 x 8 outputs per thread) and
//   numerics: 128 x 64 on 128 compute threads + a producer warp, 3 CTAs per SM
//   (the tuner's pick at n = 8192 and n = 1024); 128 x 128 on 256 threads, 2
//   CTAs per SM (thread 0 issues the TMAs; the best for an 8-rank share);
//   128 x 128 at one CTA per SM with a producer warp (Big1P), which the
//   launcher takes when the 128 x 128 tiles fill one wave (n = 2048); 64 x 64
//   on 64 threads (16-deep slabs, up to 7 CTAs per SM) for small matrices.
// * Small grids.  The exact result forbids splitting a tile's reduction except
//   in k order, so a tile's KS slabs run in sequence at one CTA's speed (1/c of
//   an SM with c CTAs per SM); the order-preserving split below balances the
//   SMs only when every run is at least one tile long, i.e. with at least
//   148 c tiles.  n = 2048: 128 x 128 has 256 tiles for 296 two-per-SM slots
//   (0.865 balance at best), hence Big1P (256 tiles for 148 CTAs: runs of 1.73
//   tiles).  Measured and dropped (tools/mm_kernel_probe.py; DESIGN.md section
//   7 lists the numbers): 256 x 128 on 512 threads; 8 x 16 and 8 x 4 outputs
//   per thread; BK = 16 rings; pacing the CTAs of an SM in the split phase;
//   transposing a inside the kernel or beside it.
// * Issue order of the FFMA2s.  An FFMA2 with a scalar a, a b pair and a c pair
//   reads up to 5 registers; when neither the a nor the b operand carries over
//   from the previous instruction (operand reuse cache) one register bank is
//   read three times and the instruction takes an extra cycle.  Writing the
//   k step b-pair-major (each b pair meets the 8 a values in a row) lets ptxas
//   keep the pair in the reuse cache: the bare loop (no barriers, no global
//   traffic, operands from shared memory) runs at 0.923 of the FFMA peak
//   against 0.858 a-major (0.985 with operands in registers) --
//   tools/ffma2_order_probe.cu, tools/ffma2_probe.cu,
//   profiles/r02_ffma2_ceiling.md.  In the kernels: Mid 0.843 -> 0.873-0.886
//   at n = 8192, 0.769 -> 0.79-0.80 at n = 2048; Big unchanged (0.86-0.87,
//   124 of its 128 registers).
// * ROWA tiles (PK_MM_ROWA=1, tuning aid) read a's rows as they lie through a
//   128-byte-swizzled [BM][BK] box -- no a^T launch, 0.5 GB less DRAM traffic
//   at n = 8192 -- with 16-byte loads along k (8 per 4 k steps, the same count
//   as the a^T slab) and rows ty + TY*i so a warp's loads hit distinct bank
//   groups.  Bit-identical, but 13 % slower at every size.  Likely cause (from
//   the SASS, not measured directly): more FFMA2s without a reused operand --
//   1061 of 2048 against 810 for Mid, counting an instruction as slow when
//   one bank parity is read three times.
// * STAGES-deep ring of slabs, one full/empty mbarrier pair per stage; the
//   compute warps wait on "full", run BK x 64 FFMAs per thread from 128-bit
//   shared loads, and release the stage with one arrive per warp on "empty"
//   -- no block-wide barrier in the main loop, no register staging or shared
//   stores.  The TMAs come from a producer warp where the register budget
//   allows one (its waits, and the consumers', sleep in the barrier:
//   mbar_wait_hint), else from thread 0, one slab ahead.
// * BK = 32, 3 stages (measured on B200, n = 8192: 66.1 TFLOP/s against 65.0
//   for BK = 16 / 4 stages / 3 ahead on the 128 x 128 tile; 16-deep slabs
//   lost 4-5 % on 128 x 64 too): the wider slab halves the barrier round
//   trips per FLOP.
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "pk_internal.cuh"

namespace pk {
namespace {

template <int TY_, int TX_, int BK_, int STAGES_, int MINB_, int AHEAD_, bool ROWA_ = false, bool PWARP_ = false>
struct Tile {
    static constexpr int TY = TY_, TX = TX_;              // compute threads, 8 x 8 outputs each
    static constexpr int BM = 8 * TY, BN = 8 * TX;        // block tile
    static constexpr int BK = BK_;                        // k slab per stage
    static constexpr int STAGES = STAGES_;
    static constexpr int AHEAD = AHEAD_;                  // slabs in flight ahead of the one computed on
    static constexpr int NCOMP = TY * TX;
    // PWARP: one more warp only issues the TMAs (AHEAD = STAGES - 1 slabs in
    // flight); otherwise thread 0 also issues them, AHEAD slabs ahead
    static constexpr bool PWARP = PWARP_;
    static constexpr int NTHREADS = NCOMP + (PWARP ? 32 : 0);
    static constexpr int MINB = MINB_;                    // resident CTAs per SM
    // ROWA: a's rows as they lie ([BM rows][BK] box, 128-byte swizzle), no
    // a^T launch; a thread's rows are ty + TY*i so the 16-byte a loads of a
    // warp fall in distinct bank groups
    static constexpr bool ROWA = ROWA_;
    static constexpr int A_SLAB = BK * BM * 4, B_SLAB = BK * BN * 4;
    static constexpr int STAGE_BYTES = A_SLAB + B_SLAB;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 128;  // ring + alignment + barriers
};
// BK = 32, 3 stages, 1 slab ahead for the two-per-SM tile (measured best, see
// above); the small tile keeps 3 stages of 16-deep slabs (24 KB a CTA, 7 CTAs
// in 227 KB); Mid: 128 x 64 on 128 compute threads + a producer warp, 3 CTAs
// per SM (72 KB rings).
using Big = Tile<16, 16, 32, 3, 2, 1>;
using Small = Tile<8, 8, 16, 3, 7, 1>;
// Mid: the 128 x 64 tile, 3 CTAs of 4 compute warps + 1 producer warp per SM
// (the producer sleeps in the empty-stage barrier, mbar_wait_hint): 0.872 ->
// 0.891 of peak at n = 8192 and 0.804 -> 0.826 at n = 2048 against thread 0
// as producer (paired runs on one box; without the sleep the producer warp
// gained nothing)
using Mid = Tile<16, 8, 32, 3, 3, 2, false, true>;
using BigR = Tile<16, 16, 32, 3, 2, 1, true>;
// Big1P: 128 x 128 at one CTA per SM, 6 stages, a producer warp keeping 5
// slabs in flight.  Used when the 128 x 128 tiles fill at most one wave of the
// two-per-SM kernel (n = 2048: 256 tiles for 296 slots, no split possible):
// 0.81 of peak against 0.72 (Big) and 0.80 (Mid); at n = 4096 / 8192 0.854 /
// 0.867.  Thread 0 as producer instead (4 ahead): 0.80 / 0.847 / 0.861; a
// producer warp for Mid (3 x 160 threads): no change.
using Big1P = Tile<16, 16, 32, 6, 1, 5, false, true>;
using MidR = Tile<16, 8, 32, 3, 3, 1, true>;

// Programmatic dependent launch: the a^T transpose lets the matmul grid be
// scheduled while it runs (the matmul CTAs set up their rings beside it) and
// the matmul waits for the transpose's memory before its first TMA.  The
// transpose also zeroes the split schedule's progress words and ticket, so no
// memset sits between the two launches.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void zero_words(int *zero, int nzero) {
    if (zero && blockIdx.x == 0 && blockIdx.y == 0)
        for (int i = threadIdx.x; i < nzero; i += blockDim.x) zero[i] = 0;
}

// out[k][r] = a[r][k] for r < rows (row-major a with leading dimension lda)
__global__ void __launch_bounds__(256) k_transpose_rows(const float *__restrict__ a, float *__restrict__ out,
                                                       int64_t rows, int64_t K, int64_t lda, int *zero, int nzero) {
    pdl_launch_dependents();
    zero_words(zero, nzero);
    __shared__ float t[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, k0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = ty; r < 32; r += 8) t[r][tx] = a[(r0 + r) * lda + k0 + tx];
    __syncthreads();
    for (int r = ty; r < 32; r += 8) out[(k0 + r) * rows + r0 + tx] = t[tx][r];
}

// The same on 64 x 64 blocks with 16-byte loads and stores on both sides (rows
// and K multiples of 64, lda % 4 == 0): 2.7 -> ~6 TB/s, the a^T slab the TMA
// then reads stays in L2 (plain stores, not streaming ones).
__global__ void __launch_bounds__(256) k_transpose_rows_v4(const float *__restrict__ a, float *__restrict__ out,
                                                          int64_t rows, int64_t lda, int *zero, int nzero) {
    pdl_launch_dependents();
    zero_words(zero, nzero);
    __shared__ float t[64][65];  // t[r][k]
    const int64_t r0 = (int64_t)blockIdx.y * 64, k0 = (int64_t)blockIdx.x * 64;
    const int tid = threadIdx.x;
    float4 v[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {  // 64 rows x 16 vectors of a
        const int e = tid + q * 256, r = e >> 4, kv = e & 15;
        v[q] = *reinterpret_cast<const float4 *>(a + (r0 + r) * lda + k0 + kv * 4);
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int e = tid + q * 256, r = e >> 4, kv = e & 15;
        t[r][kv * 4] = v[q].x; t[r][kv * 4 + 1] = v[q].y; t[r][kv * 4 + 2] = v[q].z; t[r][kv * 4 + 3] = v[q].w;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; q++) {  // 64 k-rows x 16 vectors of out
        const int e = tid + q * 256, k = e >> 4, rv = e & 15;
        const float4 o = make_float4(t[rv * 4][k], t[rv * 4 + 1][k], t[rv * 4 + 2][k], t[rv * 4 + 3][k]);
        *reinterpret_cast<float4 *>(out + (k0 + k) * rows + r0 + rv * 4) = o;
    }
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// sm_100 packed fp32 FMA (fma.rn.f32x2): two IEEE fma.rn per instruction --
// the same bits as two FFMAs, half the issue slots (57.8 vs 55.7 TFLOP/s).
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
// c = {a.lo * b.lo + c.lo, a.hi * b.hi + c.hi}
__device__ __forceinline__ void fma2p(unsigned long long &c, unsigned long long a, unsigned long long b) {
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifndef PK_MM_GROUP
#define PK_MM_GROUP 8
#endif

// Tile t of the grouped raster: tiles in flight together cover a GROUP x
// (some columns) block of the tile grid walked column by column, so the a
// row panels and b column panels a wave streams through k are shared by
// GROUP (resp. P / GROUP) CTAs at once -- DRAM reads per wave ~ (GROUP +
// P / GROUP) panels in lockstep.  Measured (ncu, n = 8192): the waves drift
// out of k-lockstep, so panels live about a tile-time in L2 and the small
// group wins: DRAM reads per launch 5.07 / 5.2 / 5.5 / 6.4 GB at GROUP 8 /
// 12 / 16 / 20 with the split schedule, 3.50 / 3.43 / 3.48 / 3.82 GB without
// it; the time is the same (FFMA-bound, 4 % of DRAM bandwidth).
template <class C>
__device__ __forceinline__ void tile_origin(int t, int ntm, int ntn, int group, int &m0, int &n0) {
    const int per_group = group * ntn;
    const int g = t / per_group, first = g * group;
    const int gsize = min(ntm - first, group);
    const int local = t - g * per_group;
    m0 = (first + local % gsize) * C::BM;
    // odd groups walk the columns right to left (boustrophedon), so a window
    // straddling two groups shares the b panels at the turn
    const int col = local / gsize;
    n0 = ((g & 1) ? ntn - 1 - col : col) * C::BN;
}

// Slabs [kb, ke) of tile (m0, n0): c rows -> packed accumulators, the ring,
// accumulators -> c.  gs: this CTA's running slab count (the ring's stage and
// barrier phase continue across work items).
template <class T>
__device__ __forceinline__ void mm_item(const CUtensorMap *map_at, const CUtensorMap *map_b, float *__restrict__ C,
                                        int64_t ldc, int64_t rlo, int m0, int n0, int kb, int ke, int &gs,
                                        unsigned char *smem, uint64_t *full, uint64_t *empty) {
    constexpr int TX = T::TX, TY = T::TY, BM = T::BM, BN = T::BN, BK = T::BK, STAGES = T::STAGES, AHEAD = T::AHEAD;
    constexpr int STAGE_BYTES = T::STAGE_BYTES, A_SLAB = T::A_SLAB;
    const int tid = threadIdx.x;
    const int nk = ke - kb;
    // thread 0 doubles as the TMA producer: for slab j it refills the stage of
    // slab j + AHEAD once every warp has released that stage's previous slab
    auto produce = [&](int j) {
        const int g = gs + j, s = g % STAGES;
        if (T::PWARP)
            mbar_wait_hint(&empty[s], ((g / STAGES) & 1) ^ 1, 1000);
        else
            mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
        // the consumers read the stage through the generic proxy (LDS); order
        // those reads before the async-proxy (TMA) overwrite -- without this
        // fence n = 8192 runs lost a k-slab of one tile every few launches
        fence_proxy_async();
        unsigned char *st = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        if (T::ROWA)
            tma_load_2d(st, map_at, &full[s], (kb + j) * BK, m0);  // [BM rows][BK], 128-byte swizzle
        else
            tma_load_2d(st, map_at, &full[s], m0, (kb + j) * BK);  // a^T slab [BK][BM]
        tma_load_2d(st + A_SLAB, map_b, &full[s], n0, (kb + j) * BK);
    };
    if (T::PWARP) {
        if (tid >= T::NCOMP) {  // the producer warp: one lane streams the item's slabs through the ring
            if (tid == T::NCOMP)
                for (int j = 0; j < nk; j++) produce(j);
            gs += nk;
            return;
        }
    } else if (tid == 0) {
        for (int j = 0; j < AHEAD && j < nk; j++) produce(j);
    }

    const int tx = tid % TX, ty = tid / TX;
    // this thread's 8 rows: ty*4 + {0..3} and BM/2 + ty*4 + {0..3} (a^T slab:
    // two 16-byte loads per k step), or ty + TY*i (ROWA)
    auto row_of = [&](int i) { return T::ROWA ? ty + TY * i : (i < 4 ? ty * 4 + i : BM / 2 + ty * 4 + i - 4); };
    float *cbase = C + (rlo + m0) * ldc + n0 + tx * 4;
    // accumulators as packed column pairs: acc[i][jp] = {c[i][2jp], c[i][2jp+1]}
    // (the operand format of fma.rn.f32x2, so the loop never repacks them).
    // c through L2 (.cg): a tile's earlier slabs may have been run by another SM
    unsigned long long acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const float *cr = cbase + row_of(i) * ldc;
        const ulonglong2 l = __ldcg(reinterpret_cast<const ulonglong2 *>(cr));
        const ulonglong2 h = __ldcg(reinterpret_cast<const ulonglong2 *>(cr + BN / 2));
        acc[i][0] = l.x; acc[i][1] = l.y; acc[i][2] = h.x; acc[i][3] = h.y;
    }
    for (int j = 0; j < nk; j++) {
        const int g = gs + j, s = g % STAGES;
        if (!T::PWARP && tid == 0 && j + AHEAD < nk) produce(j + AHEAD);
        // with a producer warp, a consumer that runs ahead sleeps in the barrier
        // instead of polling (paired A/B: 128 x 64 at n = 8192 0.880 -> 0.891 at
        // 200 ns or 1 us; n = 2048 -0.6 %, where the tuner picks Big1P)
        if (T::PWARP)
            mbar_wait_hint(&full[s], (g / STAGES) & 1, 200);
        else
            mbar_wait(&full[s], (g / STAGES) & 1);
        const float *As = reinterpret_cast<const float *>(smem + s * STAGE_BYTES);  // [BK][BM] or [BM][BK]
        const float *Bs = As + BK * BM;                                               // [BK][BN]
        float4 a4[8];  // ROWA: a[row_of(i)][4q .. 4q+3]
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            float af[8];
            if (T::ROWA) {
                static_assert(!T::ROWA || (BK == 32 && TY % 8 == 0), "ROWA: 128-byte rows, rows = ty mod 8");
                if (kk % 4 == 0) {
                    // 128-byte swizzle: the 16-byte chunk q of row r sits at chunk q ^ (r % 8);
                    // r % 8 = ty % 8 for every row of this thread
                    const unsigned char *ab = reinterpret_cast<const unsigned char *>(As) + ty * 128 +
                                              (((kk / 4) ^ (ty & 7)) << 4);
#pragma unroll
                    for (int i = 0; i < 8; i++) a4[i] = *reinterpret_cast<const float4 *>(ab + i * TY * 128);
                }
#pragma unroll
                for (int i = 0; i < 8; i++)
                    af[i] = kk % 4 == 0 ? a4[i].x : kk % 4 == 1 ? a4[i].y : kk % 4 == 2 ? a4[i].z : a4[i].w;
            } else {
                const float4 a0 = *reinterpret_cast<const float4 *>(As + kk * BM + ty * 4);
                const float4 a1 = *reinterpret_cast<const float4 *>(As + kk * BM + BM / 2 + ty * 4);
                af[0] = a0.x; af[1] = a0.y; af[2] = a0.z; af[3] = a0.w;
                af[4] = a1.x; af[5] = a1.y; af[6] = a1.z; af[7] = a1.w;
            }
            const ulonglong2 b0 = *reinterpret_cast<const ulonglong2 *>(Bs + kk * BN + tx * 4);
            const ulonglong2 b1 = *reinterpret_cast<const ulonglong2 *>(Bs + kk * BN + BN / 2 + tx * 4);
            const unsigned long long bp[4] = {b0.x, b0.y, b1.x, b1.y};
            // b-pair-major: each b pair meets the 8 a values in a row, so the
            // pair operand stays in the reuse cache and an FFMA2 reads at most
            // two registers per bank (a-major issue: 0.858 of the FFMA peak
            // for the bare loop, b-major 0.923 -- tools/ffma2_order_probe.cu)
#pragma unroll
            for (int jp = 0; jp < 4; jp++)
#pragma unroll
                for (int i = 0; i < 8; i++) fma2p(acc[i][jp], pack2(af[i], af[i]), bp[jp]);
        }
        __syncwarp();
        if ((tid & 31) == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    }
    gs += nk;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        float *cr = cbase + row_of(i) * ldc;
        *reinterpret_cast<ulonglong2 *>(cr) = make_ulonglong2(acc[i][0], acc[i][1]);
        *reinterpret_cast<ulonglong2 *>(cr + BN / 2) = make_ulonglong2(acc[i][2], acc[i][3]);
    }
}

template <class T>
__device__ __forceinline__ void mm_init(unsigned char *&smem, uint64_t *&full, uint64_t *&empty,
                                        unsigned char *smem_raw) {
    constexpr int STAGES = T::STAGES;
    // align by offsetting the shared array itself (not via an integer cast), so
    // the compiler keeps the shared address space and emits LDS, not generic LD
    smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    full = reinterpret_cast<uint64_t *>(smem + STAGES * T::STAGE_BYTES);
    empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], T::NCOMP / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
}

// One 128 x 128 tile per CTA, the whole reduction.
template <class T>
__global__ void __launch_bounds__(T::NTHREADS, T::MINB) k_matmul_tma(const __grid_constant__ CUtensorMap map_at,
                                                          const __grid_constant__ CUtensorMap map_b,
                                                          float *__restrict__ C, int64_t ldc, int64_t rlo,
                                                          int ntn, int ktiles, int group) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem;
    uint64_t *full, *empty;
    mm_init<T>(smem, full, empty, smem_raw);
    pdl_wait();  // a^T (and everything before it in the stream) is in memory
    int m0, n0, gs = 0;
    tile_origin<T>(blockIdx.x, (int)(gridDim.x / ntn), ntn, group, m0, n0);
    mm_item<T>(&map_at, &map_b, C, ldc, rlo, m0, n0, 0, ktiles, gs, smem, full, empty);
}

// Persistent CTAs over an order-preserving split of the work (see
// mm_schedule).  Phase 1: whole tiles [0, base) handed out in raster order by
// a ticket counter, so the tiles in flight are always a contiguous window of
// the grouped raster (L2 reuse as in a plain grid; static assignment let fast
// CTAs drift ahead and scatter the window).  Phase 2: the CTA's own items
// {tile, first slab, end slab} [off[p], off[p+1]) -- the tail waves cut into
// equal runs; an item that continues a tile's reduction waits until the part
// before it has stored c (the tile's progress word equals its first slab),
// and every item publishes its last slab after storing.  c is the fp32
// accumulator between the parts, so the bits equal one launch.
#ifdef PK_MM_TRACE
// development trace (-DPK_MM_TRACE builds only): per CTA, globaltimer at the
// start and at the end of every work item
__device__ unsigned long long g_mm_trace[1024][32];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define MM_TRACE(slot) \
    do { \
        if (threadIdx.x == 0 && blockIdx.x < 1024 && (slot) < 32) g_mm_trace[blockIdx.x][slot] = gtime(); \
    } while (0)
#else
#define MM_TRACE(slot) \
    do { \
    } while (0)
#endif

template <class T>
__global__ void __launch_bounds__(T::NTHREADS, T::MINB) k_matmul_tma_sched(const __grid_constant__ CUtensorMap map_at,
                                                                const __grid_constant__ CUtensorMap map_b,
                                                                float *__restrict__ C, int64_t ldc, int64_t rlo,
                                                                int ntm, int ntn, int group, int base, int ktiles,
                                                                const int3 *__restrict__ items,
                                                                const int *__restrict__ off, int *progress,
                                                                int *ticket) {
    extern __shared__ unsigned char smem_raw[];
    __shared__ int next;
    unsigned char *smem;
    uint64_t *full, *empty;
    int nt = 0;
    MM_TRACE(nt++);
    mm_init<T>(smem, full, empty, smem_raw);
    pdl_wait();  // a^T, the zeroed progress words and ticket (and everything before them) are in memory
    int gs = 0;
    for (;;) {
        if (threadIdx.x == 0) next = atomicAdd(ticket, 1);
        __syncthreads();
        const int t = next;
        __syncthreads();  // every thread has read next before thread 0 overwrites it
        if (t >= base) break;
        int m0, n0;
        tile_origin<T>(t, ntm, ntn, group, m0, n0);
        mm_item<T>(&map_at, &map_b, C, ldc, rlo, m0, n0, 0, ktiles, gs, smem, full, empty);
        MM_TRACE(nt++);
    }
    // Split phase.  With a producer warp the items are known up front, so on
    // the one-CTA-per-SM tile it streams all their slabs through the ring back
    // to back (the next item's first slabs load while the compute warps finish
    // the current one and store its c); the compute warps synchronise among
    // themselves only.  n = 2048: 0.839 -> 0.843 of peak; on the 128 x 64 tile
    // (3 CTAs per SM) the same cost 1.5 % at n = 8192, so it keeps the
    // item-by-item ring.
    constexpr bool STREAM = T::PWARP && T::MINB == 1;
    if (STREAM && threadIdx.x >= T::NCOMP) {
        for (int it = off[blockIdx.x]; it < off[blockIdx.x + 1]; it++) {
            const int3 w = items[it];
            int m0, n0;
            tile_origin<T>(w.x, ntm, ntn, group, m0, n0);
            mm_item<T>(&map_at, &map_b, C, ldc, rlo, m0, n0, w.y, w.z, gs, smem, full, empty);
        }
        return;
    }
    auto compute_sync = [] {
        if (STREAM)
            asm volatile("bar.sync 1, %0;" ::"r"(T::NCOMP) : "memory");
        else
            __syncthreads();
    };
    for (int it = off[blockIdx.x]; it < off[blockIdx.x + 1]; it++) {
        const int3 w = items[it];
        int m0, n0;
        tile_origin<T>(w.x, ntm, ntn, group, m0, n0);
        if (w.y > 0) {  // the tile's slabs before w.y are another CTA's: wait for their c
            if (threadIdx.x == 0) {
                int v;
                do {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(progress + w.x) : "memory");
                } while (v != w.y);
            }
            compute_sync();
        }
        MM_TRACE(nt++);
        mm_item<T>(&map_at, &map_b, C, ldc, rlo, m0, n0, w.y, w.z, gs, smem, full, empty);
        MM_TRACE(nt++);
        compute_sync();  // every thread's c stores before the publication
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(progress + w.x), "r"(w.z) : "memory");
        }
    }
}

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

// rows x cols fp32 row-major, box box_rows x box_cols, no swizzle (plain row-major slab in smem)
int make_map(CUtensorMap *m, const float *base, int64_t rows, int64_t cols, int64_t ld, int box_cols,
             int box_rows, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
    EncodeTiled enc = encode_fn();
    if (!enc) return fail(PK_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PK_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PK_OK;
}

}  // namespace

// True when a TMA-fed kernel tiles this launch: the case's block tile is one
// of the instantiated tiles (128 x 128 or 64 x 64) and divides the extents.
bool matmul_tma_fits(int64_t BM_case, int64_t BN_case, int64_t rows, int64_t Nc, int64_t K, int64_t n) {
    auto fits = [&](int bm, int bn, int bk) {
        // (K % 32: the a^T transpose works in 32 x 32 blocks)
        return BM_case == bm && BN_case == bn && rows % bm == 0 && Nc % bn == 0 && K % bk == 0 && K % 32 == 0 &&
               K > 0;
    };
    return (fits(Big::BM, Big::BN, Big::BK) || fits(Small::BM, Small::BN, Small::BK) ||
            fits(Mid::BM, Mid::BN, Mid::BK)) && n % 4 == 0 &&
           n <= ((int64_t)1 << 30);
}

namespace {

// Order-preserving split of the work over P persistent CTAs (the tail fix).
// The last 1-2 waves of tiles x KS slabs are laid end to end and cut into P
// equal runs, so every CTA gets the same number of slabs instead of whole
// tiles (T/P waves: 13.84 at n = 8192 on one B200, 1.73 per rank at 8
// ranks -- the last wave 73 % full).  A run covers [tail of tile A] [full
// tiles] [head of tile B]; the CTA runs the head of B first, then the full
// tiles, then the tail of A, so the part of a split tile that comes first in
// k runs at the start of one CTA's split phase and the part after it at the
// end of the next CTA's (a run is at least one tile long, so the wait is
// already satisfied).  Waits only go to lower-numbered CTAs, whose head item
// is the awaited one and follows only unconditional whole tiles.
struct DevSched {
    int3 *items = nullptr;
    int *off = nullptr;
};

std::mutex g_sched_mu;
std::map<std::tuple<int, int64_t, int64_t, int>, DevSched> g_sched;  // (device, T, KS, P)

// All but the last 1-2 waves are whole tiles handed out by the kernel's
// ticket counter (tiles [0, base)); the rest are split into P equal runs of
// >= one tile (so a tile is cut at most once and its second part never waits
// in practice).
int64_t schedule_base(int64_t T, int P) { return (T / P >= 2 ? T / P - 1 : 0) * P; }

int build_schedule(int64_t T, int64_t KS, int P, std::vector<int3> &items, std::vector<int> &off) {
    const int64_t base = schedule_base(T, P), S = (T - base) * KS;
    off.assign(P + 1, 0);
    for (int p = 0; p < P; p++) {
        off[p] = (int)items.size();
        const int64_t s0 = S * p / P, s1 = S * (p + 1) / P;
        if (s1 <= s0) continue;
        const int64_t t0 = s0 / KS, t1 = (s1 - 1) / KS;
        if (t0 == t1) {  // inside one tile
            items.push_back(make_int3((int)(base + t0), (int)(s0 - t0 * KS), (int)(s1 - t0 * KS)));
            continue;
        }
        const int64_t k0 = s0 - t0 * KS, k1 = s1 - t1 * KS;  // first piece from k0, last piece up to k1
        if (k1 < KS) items.push_back(make_int3((int)(base + t1), 0, (int)k1));          // head of the next split
        for (int64_t t = k0 == 0 ? t0 : t0 + 1; t <= (k1 == KS ? t1 : t1 - 1); t++)    // whole tiles
            items.push_back(make_int3((int)(base + t), 0, (int)KS));
        if (k0 > 0) items.push_back(make_int3((int)(base + t0), (int)k0, (int)KS));     // tail of the previous
    }
    off[P] = (int)items.size();
    return PK_OK;
}

int schedule_for(int dev, int64_t T, int64_t KS, int P, DevSched *out) {
    std::lock_guard<std::mutex> lock(g_sched_mu);
    const auto key = std::make_tuple(dev, T, KS, P);
    auto it = g_sched.find(key);
    if (it != g_sched.end()) {
        *out = it->second;
        return PK_OK;
    }
    std::vector<int3> items;
    std::vector<int> off;
    build_schedule(T, KS, P, items, off);
    DevSched d;
    cudaError_t e = cudaMalloc(&d.items, items.size() * sizeof(int3));
    if (e == cudaSuccess) e = cudaMalloc(&d.off, off.size() * sizeof(int));
    if (e == cudaSuccess) e = cudaMemcpy(d.items, items.data(), items.size() * sizeof(int3), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d.off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(PK_E_ALLOC, "matmul schedule: %s", cudaGetErrorString(e));
    g_sched[key] = d;
    *out = d;
    return PK_OK;
}

}  // namespace

namespace {

template <class C>
int launch_tma_t(const float *a, const float *b, float *c, int64_t n, int64_t rlo, int64_t rhi, int64_t Nc, int64_t K,
                 cudaStream_t st) {
    const int64_t rows = rhi - rlo;
    float *at = nullptr;
    int *progress = nullptr;  // split schedule: T progress words, then the ticket counter
    int rc = PK_OK;
    CUtensorMap mat, mb;
    const int ntn = (int)(Nc / C::BN), ntm = (int)(rows / C::BM);
    const int64_t T = (int64_t)ntm * ntn, KS = K / C::BK;
    // persistent split when the tiles leave the last wave part-empty
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if ((rc = allow_smem((const void *)k_matmul_tma<C>, C::SMEM_BYTES)) != PK_OK ||
        (rc = allow_smem((const void *)k_matmul_tma_sched<C>, C::SMEM_BYTES)) != PK_OK)
        return rc;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_matmul_tma_sched<C>, C::NTHREADS, C::SMEM_BYTES);
    const int64_t P = (int64_t)sms * per_sm;
    const bool split = getenv("PK_MM_NO_SPLIT") == nullptr && P > 0 && T > P && T % P != 0 && KS >= 8 &&
                       T * KS < ((int64_t)1 << 31);
    DevSched d;
    if (split) {
        if ((rc = schedule_for(dev, T, KS, (int)P, &d)) != PK_OK) return rc;
        cudaError_t e2 = scratch_alloc((void **)&progress, (size_t)(T + 1) * sizeof(int), st);
        if (e2 != cudaSuccess) return fail(PK_E_ALLOC, "matmul progress words: %s", cudaGetErrorString(e2));
    }
    // PK_MM_PDL=0: plain launches with a memset between them (comparison aid).
    // Not for a part-filled grid of several CTAs per SM: launched beside the
    // transpose, its CTAs land on the SMs with room and stack up (n = 1024 on
    // 128 x 64 tiles: 128 CTAs on ~43 SMs, 2.3x slower); the split's
    // persistent grid fills every slot.  Measured with PDL: n = 2048 0.815 ->
    // 0.824 of peak (Big1P), 0.797 -> 0.803 (Mid); n = 8192 unchanged.
    const char *penv = getenv("PK_MM_PDL");
    const bool pdl = !C::ROWA && !(penv && penv[0] == '0') && (split || T >= P || per_sm <= 1);
    if (C::ROWA) {
        rc = make_map(&mat, a + rlo * n, rows, K, n, C::BK, C::BM, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
        cudaError_t e = scratch_alloc((void **)&at, (size_t)rows * K * sizeof(float), st);
        if (e != cudaSuccess) rc = fail(PK_E_ALLOC, "matmul a^T workspace: %s", cudaGetErrorString(e));
        int *zero = pdl ? progress : nullptr;
        const int nzero = zero ? (int)(T + 1) : 0;
        if (rc == PK_OK) {
            if (rows % 64 == 0 && K % 64 == 0)
                k_transpose_rows_v4<<<dim3((unsigned)(K / 64), (unsigned)(rows / 64)), 256, 0, st>>>(
                    a + rlo * n, at, rows, n, zero, nzero);
            else
                k_transpose_rows<<<dim3((unsigned)(K / 32), (unsigned)(rows / 32)), 256, 0, st>>>(
                    a + rlo * n, at, rows, K, n, zero, nzero);
            rc = after_launch("matmul_transpose_a");
        }
        if (rc == PK_OK) rc = make_map(&mat, at, K, rows, rows, C::BM, C::BK);
    }
    if (rc == PK_OK) rc = make_map(&mb, b, K, Nc, n, C::BN, C::BK);
    if (rc == PK_OK) {
        // rows of tiles per raster group (PK_MM_GROUP overrides: tuning aid)
        const char *genv = getenv("PK_MM_GROUP");
        const int group = genv && atoi(genv) > 0 ? atoi(genv) : PK_MM_GROUP;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.blockDim = dim3(C::NTHREADS);
        cfg.dynamicSmemBytes = C::SMEM_BYTES;
        cfg.stream = st;
        cfg.attrs = pdl ? attr : nullptr;
        cfg.numAttrs = pdl ? 1 : 0;
        cudaError_t e;
        if (split) {
            e = pdl ? cudaSuccess : cudaMemsetAsync(progress, 0, (size_t)(T + 1) * sizeof(int), st);
            cfg.gridDim = dim3((unsigned)P);
            if (e == cudaSuccess)
                e = cudaLaunchKernelEx(&cfg, k_matmul_tma_sched<C>, mat, mb, c, n, rlo, ntm, ntn, group,
                                       (int)schedule_base(T, (int)P), (int)KS, (const int3 *)d.items,
                                       (const int *)d.off, progress, progress + T);
        } else {
            cfg.gridDim = dim3((unsigned)T);
            e = cudaLaunchKernelEx(&cfg, k_matmul_tma<C>, mat, mb, c, n, rlo, ntn, (int)KS, group);
        }
        rc = e != cudaSuccess ? fail(PK_E_CUDA, "matmul launch: %s", cudaGetErrorString(e))
                              : after_launch(split ? "matmul_tma_sched" : "matmul_tma");
    }
    if (progress) cudaFreeAsync(progress, st);
    if (at) cudaFreeAsync(at, st);
    return rc;
}

}  // namespace

int launch_matmul_tma(const float *a, const float *b, float *c, int64_t n, int64_t rlo, int64_t rhi, int64_t Nc,
                      int64_t K, int bm, int bn, cudaStream_t st) {
    // PK_MM_ROWA=1 selects the row-major-a kernels (measured 13 % slower, kept
    // as a tuning aid: see the ROWA note at the top of the file)
    const char *renv = getenv("PK_MM_ROWA");
    const bool rowa = renv && renv[0] == '1';
    if (bm == Small::BM && bn == Small::BN) return launch_tma_t<Small>(a, b, c, n, rlo, rhi, Nc, K, st);
    if (bm == Mid::BM && bn == Mid::BN)
        return rowa ? launch_tma_t<MidR>(a, b, c, n, rlo, rhi, Nc, K, st) : launch_tma_t<Mid>(a, b, c, n, rlo, rhi, Nc, K, st);
    // 128 x 128: one CTA per SM when the tiles fill at most one wave of the
    // two-per-SM kernel (PK_MM_TILE=big / big1p forces either: tuning aid)
    const char *tenv = getenv("PK_MM_TILE");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = ((rhi - rlo) / Big::BM) * (Nc / Big::BN);
    const bool one_wave = tenv ? !strcmp(tenv, "big1p") : tiles <= (int64_t)Big::MINB * sms;
    if (!rowa && one_wave) return launch_tma_t<Big1P>(a, b, c, n, rlo, rhi, Nc, K, st);
    return rowa ? launch_tma_t<BigR>(a, b, c, n, rlo, rhi, Nc, K, st) : launch_tma_t<Big>(a, b, c, n, rlo, rhi, Nc, K, st);
}

}  // namespace pk

#ifdef PK_MM_TRACE
extern "C" int pk_mm_trace(unsigned long long *host) {
    return (int)cudaMemcpyFromSymbol(host, pk::g_mm_trace, sizeof(pk::g_mm_trace));
}
#endif
