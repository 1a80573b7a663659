// k_matmul.cu -- tiled matrix multiplication (paper Fig. 3; SURVEY App. A.1 matmul.mfk):
//   dim0 = n/B0, dim1 = n/(ub1*s), kdim = n/B0
//   for k < kdim: for every (p, q): for z < B0:
//       c[p][q] = c[p][q] + a[p][B0*k+z] * b[B0*k+z][q]
//   p < dim0*B0, q < dim1*ub1*s, reduction index kk = B0*k+z ascending over [0, kdim*B0).
//
// Numerics (identical in every kernel below, so the result does not depend on
// the case, the tile or the kernel): each output starts from its input value
// c[p][q] and accumulates acc = fma(a[p][kk], b[kk][q], acc) for kk = 0, 1, ...
// in order -- the reference's left-to-right sum with one rounding per step.
// float32 stays on the FFMA pipe (no tensor cores on this path).
//
// Kernels:
//  * k_matmul_generic: the program's own thread mapping -- a B0 x ub1 block,
//    thread (v, u) owns row p and columns q = j*ub1*s + w*ub1 + u (w < s).
//    STAGED keeps cache(a, b): per k step the B0 x B0 slab of a and the
//    B0 x (ub1*s) slab of b sit in shared memory (the footprint
//    B0^2 + B0*ub1*s of the case).  DIRECT (caching-off) reads global memory.
//  * k_matmul_tiled: the same block tile B0 x (ub1*s) register-blocked for
//    B200 -- every thread owns an 8 x 8 sub-tile, k slabs of 16 move through
//    a double-buffered shared ring (a transposed on the way in), so each
//    pair of 128-bit shared loads feeds 64 FFMAs.  Used for the staged leaf
//    whenever the tile is one of the instantiated shapes.
#include <type_traits>

#include "pk_internal.cuh"

namespace pk {
namespace {

__device__ __forceinline__ float mad(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ int mad(int a, int b, int c) { return a * b + c; }
// int64 wraps like C (exact modulo 2^64); binary64 rounds the product and the
// sum separately, c + a*b exactly as the interpreter evaluates Python floats
__device__ __forceinline__ long long mad(long long a, long long b, long long c) {
    return (long long)((unsigned long long)a * (unsigned long long)b + (unsigned long long)c);
}
__device__ __forceinline__ double mad(double a, double b, double c) { return __dadd_rn(c, __dmul_rn(a, b)); }

constexpr int kChunk = 8;  // accumulators per thread in the generic kernel

template <typename T, bool STAGED>
__global__ void __launch_bounds__(1024) k_matmul_generic(const T *__restrict__ a,
                                                        const T *__restrict__ b, T *__restrict__ c,
                                                        int64_t n, int64_t K, int64_t rlo,
                                                        int64_t rhi, int64_t ntn, int B0, int ub1,
                                                        int E) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *As = reinterpret_cast<T *>(smem_raw);          // [B0][B0]
    T *Bs = As + (size_t)B0 * B0;                      // [B0][ub1*kChunk]
    const int u = threadIdx.x, v = threadIdx.y;
    const int tid = v * ub1 + u, nthreads = B0 * ub1;
    const int64_t bid = blockIdx.x;
    const int64_t p0 = rlo + (bid / ntn) * B0;
    const int64_t q0 = (bid % ntn) * (int64_t)ub1 * E;
    const int64_t p = p0 + v;
    const bool prow = p < rhi;
    const int rows = (int)min((int64_t)B0, rhi - p0);
    for (int w0 = 0; w0 < E; w0 += kChunk) {
        const int wn = min(kChunk, E - w0);
        const int64_t qb = q0 + (int64_t)w0 * ub1;  // first column of this chunk
        const int cols = wn * ub1;
        T acc[kChunk];
#pragma unroll
        for (int w = 0; w < kChunk; w++)
            acc[w] = (prow && w < wn) ? c[p * n + qb + w * ub1 + u] : T(0);
        for (int64_t kb = 0; kb < K; kb += B0) {
            if (STAGED) {
                for (int e = tid; e < rows * B0; e += nthreads) {
                    const int r = e / B0, z = e % B0;
                    As[r * B0 + z] = a[(p0 + r) * n + kb + z];
                }
                for (int e = tid; e < B0 * cols; e += nthreads) {
                    const int z = e / cols, q = e % cols;
                    Bs[z * cols + q] = b[(kb + z) * n + qb + q];
                }
                __syncthreads();
                if (prow) {
                    for (int z = 0; z < B0; z++) {
                        const T av = As[v * B0 + z];
#pragma unroll
                        for (int w = 0; w < kChunk; w++)
                            if (w < wn) acc[w] = mad(av, Bs[z * cols + w * ub1 + u], acc[w]);
                    }
                }
                __syncthreads();
            } else if (prow) {
                for (int z = 0; z < B0; z++) {
                    const T av = a[p * n + kb + z];
                    const T *brow = b + (kb + z) * n + qb + u;
#pragma unroll
                    for (int w = 0; w < kChunk; w++)
                        if (w < wn) acc[w] = mad(av, brow[w * ub1], acc[w]);
                }
            }
        }
        if (prow) {
#pragma unroll
            for (int w = 0; w < kChunk; w++)
                if (w < wn) c[p * n + qb + w * ub1 + u] = acc[w];
        }
    }
}

// Register-blocked staged tile.  TY x TX threads, each owning rows
// {ty*4 + i, BM/2 + ty*4 + i} x cols {tx*4 + j, BN/2 + tx*4 + j}, i, j < 4.
template <typename T, int TY, int TX, int BK>
__global__ void __launch_bounds__(TY *TX, (TY * TX >= 256) ? 2 : ((TY * TX >= 128) ? 3 : 4))
    k_matmul_tiled(const T *__restrict__ A, const T *__restrict__ B, T *__restrict__ C, int64_t n,
                   int64_t K, int64_t rlo, int64_t ntn) {
    constexpr int BM = 8 * TY, BN = 8 * TX, NT = TY * TX;
    constexpr int APAD = 4;
    constexpr int A_LD = BM * BK / 4 / NT;  // int4 loads of A per thread per k slab
    constexpr int B_LD = BK * BN / 4 / NT;
    static_assert(A_LD * NT * 4 == BM * BK && B_LD * NT * 4 == BK * BN, "tile/threads");
    __shared__ __align__(16) T As[2][BK][BM + APAD];
    __shared__ __align__(16) T Bs[2][BK][BN];

    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    const int64_t bid = blockIdx.x;
    const int64_t m0 = rlo + (bid / ntn) * BM, n0 = (bid % ntn) * BN;

    // per-thread global pointers (64-bit math once, then pointer bumps)
    const T *gA[A_LD];
    const T *gB[B_LD];
#pragma unroll
    for (int r = 0; r < A_LD; r++) {
        const int e = tid + r * NT;
        gA[r] = A + (m0 + e / (BK / 4)) * n + 4 * (e % (BK / 4));
    }
#pragma unroll
    for (int r = 0; r < B_LD; r++) {
        const int e = tid + r * NT;
        gB[r] = B + (int64_t)(e / (BN / 4)) * n + n0 + 4 * (e % (BN / 4));
    }
    const int64_t bstep = (int64_t)BK * n;

    // accumulators start from c (the reference adds into c)
    T *crow = C + (m0 + ty * 4) * n + n0 + tx * 4;
    const int64_t chalf = (int64_t)(BM / 2) * n;
    T acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const T *cr = crow + (i < 4 ? i * n : chalf + (i - 4) * n);
        const int4 lo4 = *reinterpret_cast<const int4 *>(cr);
        const int4 hi4 = *reinterpret_cast<const int4 *>(cr + BN / 2);
        const T *l = reinterpret_cast<const T *>(&lo4);
        const T *h = reinterpret_cast<const T *>(&hi4);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            acc[i][j] = l[j];
            acc[i][4 + j] = h[j];
        }
    }

    int4 ra[A_LD], rb[B_LD];
    auto load_global = [&]() {
#pragma unroll
        for (int r = 0; r < A_LD; r++) {
            ra[r] = *reinterpret_cast<const int4 *>(gA[r]);
            gA[r] += BK;
        }
#pragma unroll
        for (int r = 0; r < B_LD; r++) {
            rb[r] = *reinterpret_cast<const int4 *>(gB[r]);
            gB[r] += bstep;
        }
    };
    auto store_shared = [&](int buf) {
#pragma unroll
        for (int r = 0; r < A_LD; r++) {
            const int e = tid + r * NT;
            const int row = e / (BK / 4), k4 = e % (BK / 4);
            const T *v = reinterpret_cast<const T *>(&ra[r]);
            As[buf][4 * k4 + 0][row] = v[0];
            As[buf][4 * k4 + 1][row] = v[1];
            As[buf][4 * k4 + 2][row] = v[2];
            As[buf][4 * k4 + 3][row] = v[3];
        }
#pragma unroll
        for (int r = 0; r < B_LD; r++) {
            const int e = tid + r * NT;
            const int krow = e / (BN / 4), n4 = e % (BN / 4);
            *reinterpret_cast<int4 *>(&Bs[buf][krow][4 * n4]) = rb[r];
        }
    };

    const int KT = (int)(K / BK);
    load_global();
    store_shared(0);
    __syncthreads();
    for (int kt = 0; kt < KT; kt++) {
        const int cur = kt & 1;
        if (kt + 1 < KT) load_global();
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            T af[8], bf[8];
            const int4 a0 = *reinterpret_cast<const int4 *>(&As[cur][kk][ty * 4]);
            const int4 a1 = *reinterpret_cast<const int4 *>(&As[cur][kk][BM / 2 + ty * 4]);
            const int4 b0 = *reinterpret_cast<const int4 *>(&Bs[cur][kk][tx * 4]);
            const int4 b1 = *reinterpret_cast<const int4 *>(&Bs[cur][kk][BN / 2 + tx * 4]);
            const T *pa0 = reinterpret_cast<const T *>(&a0), *pa1 = reinterpret_cast<const T *>(&a1);
            const T *pb0 = reinterpret_cast<const T *>(&b0), *pb1 = reinterpret_cast<const T *>(&b1);
#pragma unroll
            for (int j = 0; j < 4; j++) {
                af[j] = pa0[j];
                af[4 + j] = pa1[j];
                bf[j] = pb0[j];
                bf[4 + j] = pb1[j];
            }
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = mad(af[i], bf[j], acc[i][j]);
        }
        if (kt + 1 < KT) store_shared(cur ^ 1);
        __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < 8; i++) {
        T *cr = crow + (i < 4 ? i * n : chalf + (i - 4) * n);
        int4 lo4, hi4;
        T *l = reinterpret_cast<T *>(&lo4);
        T *h = reinterpret_cast<T *>(&hi4);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            l[j] = acc[i][j];
            h[j] = acc[i][4 + j];
        }
        *reinterpret_cast<int4 *>(cr) = lo4;
        *reinterpret_cast<int4 *>(cr + BN / 2) = hi4;
    }
}

template <typename T, int TY, int TX, int BK>
int launch_tiled(const T *a, const T *b, T *c, int64_t n, int64_t K, int64_t rlo, int64_t rhi,
                 int64_t Nc, cudaStream_t st) {
    constexpr int BM = 8 * TY, BN = 8 * TX;
    const int64_t ntm = (rhi - rlo) / BM, ntn = Nc / BN;
    const int64_t blocks = ntm * ntn;
    if (blocks <= 0) return PK_OK;
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "matmul: grid too large");
    k_matmul_tiled<T, TY, TX, BK><<<(unsigned)blocks, TY * TX, 0, st>>>(a, b, c, n, K, rlo, ntn);
    return after_launch("matmul_tiled");
}

// binary64 / int64: the same c + a*b sequence (two roundings per step for
// binary64, wrapping int64) on a 64 x 64 tile of 256 threads, each owning
// rows ty + 16i and columns tx + 16j (i, j < 4) so the a reads of a warp are
// 2-address broadcasts and the b reads 128-byte rows; 16-deep k slabs of a
// (row-major, pitch 18) and b double-buffered by cp.async.
constexpr int kXM = 64, kXN = 64, kXK = 16, kXAP = kXK + 2;

template <typename T>
__global__ void __launch_bounds__(256) k_matmul_exact_tiled(const T *__restrict__ a, const T *__restrict__ b,
                                                           T *__restrict__ c, int64_t n, int64_t K, int64_t rlo,
                                                           int64_t ntn) {
    __shared__ __align__(16) T As[2][kXM][kXAP];
    __shared__ __align__(16) T Bs[2][kXK][kXN];
    constexpr int V = 16 / sizeof(T);
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const int64_t bid = blockIdx.x;
    const int64_t m0 = rlo + (bid / ntn) * kXM, n0 = (bid % ntn) * kXN;
    auto load = [&](int64_t k0, int buf) {
        for (int e = tid; e < kXM * (kXK / V); e += 256) {
            const int r = e / (kXK / V), cv = e % (kXK / V);
            cp_async16(&As[buf][r][cv * V], a + (m0 + r) * n + k0 + cv * V, 16);
        }
        for (int e = tid; e < kXK * (kXN / V); e += 256) {
            const int r = e / (kXN / V), cv = e % (kXN / V);
            cp_async16(&Bs[buf][r][cv * V], b + (k0 + r) * n + n0 + cv * V, 16);
        }
        cp_async_commit();
    };
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = c[(m0 + ty + 16 * i) * n + n0 + tx + 16 * j];
    const int64_t nk = K / kXK;
    load(0, 0);
    for (int64_t kt = 0; kt < nk; kt++) {
        if (kt + 1 < nk) {
            load((kt + 1) * kXK, (int)((kt + 1) & 1));
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int buf = (int)(kt & 1);
#pragma unroll
        for (int kk = 0; kk < kXK; kk++) {
            T av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; i++) av[i] = As[buf][ty + 16 * i][kk];
#pragma unroll
            for (int j = 0; j < 4; j++) bv[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = mad(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) c[(m0 + ty + 16 * i) * n + n0 + tx + 16 * j] = acc[i][j];
}

template <typename T>
int launch_t(const pk_launch_t &L, void *const *p, cudaStream_t st, int64_t rlo, int64_t rhi,
             int64_t Nc, int64_t K) {
    const T *a = static_cast<const T *>(p[0]);
    const T *b = static_cast<const T *>(p[1]);
    T *c = static_cast<T *>(p[2]);
    const int64_t BM = L.B0, BN = L.ub1 * elems(L);
    const bool generic = (L.flags & PK_FLAG_GENERIC) != 0;
    if constexpr (std::is_same<T, float>::value) {
        if (L.flags & PK_FLAG_TF32X3)  // optional tensor-core variant, reported separately
            return launch_matmul_tf32x3(a, b, c, L.N, rlo, rhi, Nc, K, st);
        // 128 x 128 staged tile fed by TMA (same FFMA chain as the other kernels)
        if (L.variant == PK_VARIANT_STAGED && !generic && aligned16(a) && aligned16(b) && aligned16(c) &&
            matmul_tma_fits(L.B0, L.ub1 * elems(L), rhi - rlo, Nc, K, L.N) && rlo % 4 == 0)
            return launch_matmul_tma(a, b, c, L.N, rlo, rhi, Nc, K, (int)L.B0, (int)(L.ub1 * elems(L)), st);
    }
    if constexpr (sizeof(T) == 4) {
        if (L.variant == PK_VARIANT_STAGED && !generic && L.N % 4 == 0 && K % 16 == 0 &&
            aligned16(a) && aligned16(b) && aligned16(c) && (rhi - rlo) % BM == 0 && Nc % BN == 0 &&
            rlo % 4 == 0) {
            if (BM == 128 && BN == 128) return launch_tiled<T, 16, 16, 8>(a, b, c, L.N, K, rlo, rhi, Nc, st);
            if (BM == 64 && BN == 128) return launch_tiled<T, 8, 16, 8>(a, b, c, L.N, K, rlo, rhi, Nc, st);
            if (BM == 128 && BN == 64) return launch_tiled<T, 16, 8, 8>(a, b, c, L.N, K, rlo, rhi, Nc, st);
            if (BM == 64 && BN == 64) return launch_tiled<T, 8, 8, 16>(a, b, c, L.N, K, rlo, rhi, Nc, st);
        }
    }
    if constexpr (sizeof(T) == 8) {
        if (!generic && (rhi - rlo) % kXM == 0 && Nc % kXN == 0 && K % kXK == 0 && L.N % 2 == 0 &&
            aligned16(a) && aligned16(b) && aligned16(c)) {
            const int64_t ntn = Nc / kXN, blocks = (rhi - rlo) / kXM * ntn;
            if (blocks <= 0) return PK_OK;
            if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "matmul: grid too large");
            k_matmul_exact_tiled<T><<<(unsigned)blocks, 256, 0, st>>>(a, b, c, L.N, K, rlo, ntn);
            return after_launch("matmul_exact_tiled");
        }
    }
    if (L.B0 * L.ub1 > 1024)
        return fail(PK_E_PARAM, "matmul: thread block B0*ub1 = %lld exceeds 1024 (T_B)",
                    (long long)(L.B0 * L.ub1));
    const int E = (int)elems(L);
    const int64_t ntm = ceil_div(rhi - rlo, L.B0), ntn = Nc / (L.ub1 * E);
    const int64_t blocks = ntm * ntn;
    if (blocks <= 0) return PK_OK;
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "matmul: grid too large");
    dim3 block((unsigned)L.ub1, (unsigned)L.B0);
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = ((size_t)L.B0 * L.B0 + (size_t)L.B0 * L.ub1 * (E < kChunk ? E : kChunk)) * sizeof(T);
        int rc = allow_smem((const void *)k_matmul_generic<T, true>, smem);
        if (rc) return rc;
        k_matmul_generic<T, true><<<(unsigned)blocks, block, smem, st>>>(a, b, c, L.N, K, rlo, rhi, ntn,
                                                                         (int)L.B0, (int)L.ub1, E);
    } else {
        k_matmul_generic<T, false><<<(unsigned)blocks, block, 0, st>>>(a, b, c, L.N, K, rlo, rhi, ntn,
                                                                       (int)L.B0, (int)L.ub1, E);
    }
    return after_launch("matmul_generic");
}

}  // namespace

int launch_matmul(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    if (L.B0 == 0) return fail(PK_E_DIV0, "matmul: B0 == 0 in dim0 = n / B0");
    if (L.ub1 * L.s == 0) return fail(PK_E_DIV0, "matmul: ub1*s == 0 in dim1 = n / (ub1 * s)");
    if (L.B0 < 0 || L.ub1 < 0 || L.s < 0 || L.N <= 0) return PK_OK;
    const int64_t M = max0(L.N / L.B0) * L.B0;
    const int64_t Nc = max0(L.N / (L.ub1 * L.s)) * L.ub1 * L.s;
    const int64_t K = max0(L.N / L.B0) * L.B0;
    int64_t rlo, rhi;
    unit_range(L, 0, M, &rlo, &rhi);
    if (rhi <= rlo || Nc <= 0) return PK_OK;
    if (L.dtype == PK_DTYPE_F32) return launch_t<float>(L, p, st, rlo, rhi, Nc, K);
    if (L.dtype == PK_DTYPE_I32) return launch_t<int>(L, p, st, rlo, rhi, Nc, K);
    if (L.dtype == PK_DTYPE_F64) return launch_t<double>(L, p, st, rlo, rhi, Nc, K);
    if (L.dtype == PK_DTYPE_I64) return launch_t<long long>(L, p, st, rlo, rhi, Nc, K);
    return fail(PK_E_UNSUPPORTED, "matmul: dtype %d", L.dtype);
}

// The reduction slice k in [k0, k1) of rows [lo, hi): c += a[:, k0:k1] b[k0:k1, :]
// on the TMA-fed tile.  Slices run in ascending k on one stream give the bits
// of a single launch -- between slices the fp32 accumulator simply lives in c
// (every fma.rn rounds to fp32 either way).  pk_run_host uses it to start the
// first row chunk while b is still crossing PCIe.
bool matmul_kslice_ok(const pk_launch_t &L, int64_t slice) {
    if (L.family != PK_FAMILY_MATMUL || L.dtype != PK_DTYPE_F32 || L.variant != PK_VARIANT_STAGED) return false;
    if (L.flags & (PK_FLAG_GENERIC | PK_FLAG_TF32X3)) return false;
    if (L.B0 <= 0 || L.ub1 <= 0 || L.s <= 0 || L.N <= 0 || slice <= 0 || slice % 128) return false;
    const int64_t M = (L.N / L.B0) * L.B0, Nc = (L.N / (L.ub1 * L.s)) * L.ub1 * L.s;
    int64_t rlo, rhi;
    unit_range(L, 0, M, &rlo, &rhi);
    return rhi > rlo && rlo % 4 == 0 && matmul_tma_fits(L.B0, L.ub1 * elems(L), rhi - rlo, Nc, slice, L.N);
}

int launch_matmul_kslice(const pk_launch_t &L, void *const *p, int64_t k0, int64_t k1, cudaStream_t st) {
    if (!matmul_kslice_ok(L, k1 - k0) || k0 < 0 || k0 % 4 || k1 > (L.N / L.B0) * L.B0)
        return fail(PK_E_UNSUPPORTED, "matmul: reduction slice [%lld, %lld) not provided for this leaf",
                    (long long)k0, (long long)k1);
    const int64_t M = (L.N / L.B0) * L.B0, Nc = (L.N / (L.ub1 * L.s)) * L.ub1 * L.s;
    int64_t rlo, rhi;
    unit_range(L, 0, M, &rlo, &rhi);
    const float *a = static_cast<const float *>(p[0]), *b = static_cast<const float *>(p[1]);
    float *c = static_cast<float *>(p[2]);
    if (!aligned16(a) || !aligned16(b) || !aligned16(c)) return fail(PK_E_UNSUPPORTED, "matmul: unaligned operands");
    return launch_matmul_tma(a + k0, b + k0 * L.N, c, L.N, rlo, rhi, Nc, k1 - k0, (int)L.B0,
                             (int)(L.ub1 * elems(L)), st);
}

}  // namespace pk
