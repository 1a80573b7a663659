// k_jacobi.cu -- the double-buffered Jacobi stencils.
//
// 1-D (pkg/src/parakern/data/jacobi.mfk:9-25), a[2N]:
//   dim = (N-2)/(s*B); for t < T, for p < dim*s*B (position x = p+1):
//     t even: a[x]   = (a[N+x-1] + a[N+x] + a[N+x+1]) / 3
//     t odd:  a[N+x] = (a[x-1]   + a[x]   + a[x+1])   / 3
// 2-D (SURVEY App. A.4 jacobi2d.mfk), a[2N][N]:
//   rows i in [1, dim0*B0], cols j in [1, dim1*s*B1]
//   t even: a[N+i][j] = (a[i-1][j] + a[i+1][j] + a[i][j-1] + a[i][j+1] + a[i][j]) / 5
//   t odd:  the same with the halves swapped.
// One launch per time step (the serial t loop is the schedule's context
// loop, interp.py:148-152).  HBM-bound: 8 bytes of algorithmic traffic per
// updated point per step.
//
// Exact integer division.  The reference's ints are unbounded, so the sum
// of three (five) int32 values must not wrap before the truncating
// division.  A Jacobi average never leaves the value range of its inputs
// (each new value lies between the min and max of the old ones, and
// truncation toward zero stays inside that interval), so if every initial
// value satisfies |v| <= (2^31-1)/3 (resp. /5) all sums of every later step
// fit in int32.  A device-side pre-pass checks that bound once per run and
// sets a flag the sweep kernels read (no host round trip); otherwise they
// form 64-bit sums.  Both paths give identical results -- the 32-bit one
// needs about a third of the integer instructions, which is what keeps the
// sweeps memory-bound on B200.
//
// Tiles are aligned to even positions (columns) so every global access is
// a 64-bit vector access in both halves (N may be = 2 mod 4, which rules
// out 128-bit alignment of the upper half).
#include "pk_internal.cuh"

namespace pk {
namespace {

constexpr int kBound3 = 715827882;  // (2^31 - 1) / 3
constexpr int kBound5 = 429496729;  // (2^31 - 1) / 5

template <bool WIDE>
__device__ __forceinline__ int avg3(int a, int b, int c) {
    if (WIDE) return (int)(((long long)a + (long long)b + (long long)c) / 3);
    return (a + b + c) / 3;
}
template <bool WIDE>
__device__ __forceinline__ int avg5(int a, int b, int c, int d, int e) {
    if (WIDE) return (int)(((long long)a + (long long)b + (long long)c + (long long)d + (long long)e) / 5);
    return (a + b + c + d + e) / 5;
}

// flag = 1 if every |v| <= bound over a[0, n), else 0 (flag preset to 1).
__global__ void __launch_bounds__(256) k_range_flag(const int *__restrict__ a, int64_t n, int bound,
                                                   int *__restrict__ flag) {
    bool ok = true;
    const int64_t n4 = n / 4;
    const int4 *a4 = reinterpret_cast<const int4 *>(a);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 v = ld_stream(a4 + i);
        ok &= (v.x >= -bound && v.x <= bound) & (v.y >= -bound && v.y <= bound) &
              (v.z >= -bound && v.z <= bound) & (v.w >= -bound && v.w <= bound);
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        ok &= (a[i] >= -bound && a[i] <= bound);
    if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0);
}

__device__ __forceinline__ bool narrow_mode(int mode, const int *flag) {
    return mode == 2 ? (*flag != 0) : (mode == 1);
}

// ---------------------------------------------------------------- 1-D ------

// Staged (cache(a) kept): the block's window src[xs-2, xs+tile+2) is copied
// to shared memory with 64-bit loads, then each thread produces output pairs
// (x, x+1) from it and stores them with one 64-bit store.
template <bool WIDE>
__device__ __forceinline__ void j1_staged_body(const int *__restrict__ src, int *__restrict__ dst,
                                               int64_t lo, int64_t hi, int64_t xs, int tile,
                                               int64_t limit, bool vec, int *sh) {
    const int tid = threadIdx.x, nt = blockDim.x;
    int2 *sh2 = reinterpret_cast<int2 *>(sh);
    const int w2 = (tile + 4) >> 1;
#pragma unroll 4
    for (int q = tid; q < w2; q += nt) {
        const int64_t i = xs - 2 + 2 * (int64_t)q;
        if (vec && i >= 0 && i + 1 < limit) {
            sh2[q] = *reinterpret_cast<const int2 *>(src + i);
        } else {
            sh[2 * q] = (i >= 0 && i < limit) ? src[i] : 0;
            sh[2 * q + 1] = (i + 1 >= 0 && i + 1 < limit) ? src[i + 1] : 0;
        }
    }
    __syncthreads();
    const int pairs = tile >> 1;
#pragma unroll 4
    for (int p = tid; p < pairs; p += nt) {
        const int64_t x = xs + 2 * (int64_t)p;
        const int2 c = sh2[p + 1];  // src[x], src[x+1]
        const int l = sh[2 * p + 1], r = sh[2 * p + 4];
        const int v0 = avg3<WIDE>(l, c.x, c.y), v1 = avg3<WIDE>(c.x, c.y, r);
        if (vec && x >= lo && x + 1 < hi) {
            *reinterpret_cast<int2 *>(dst + x) = make_int2(v0, v1);
        } else {
            if (x >= lo && x < hi) dst[x] = v0;
            if (x + 1 >= lo && x + 1 < hi) dst[x + 1] = v1;
        }
    }
}

__global__ void __launch_bounds__(1024) k_jacobi1d_staged(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t lo,
                                                         int64_t hi, int64_t x0, int tile,
                                                         int64_t limit, int vec, const int *flag,
                                                         int mode) {
    extern __shared__ __align__(16) int sh[];
    const int64_t xs = x0 + (int64_t)blockIdx.x * tile;
    if (narrow_mode(mode, flag))
        j1_staged_body<false>(src, dst, lo, hi, xs, tile, limit, vec != 0, sh);
    else
        j1_staged_body<true>(src, dst, lo, hi, xs, tile, limit, vec != 0, sh);
}

// caching-off: every thread reads its neighbourhood straight from global
// memory (the overlapping reads of adjacent threads hit L1).
template <bool WIDE>
__device__ __forceinline__ void j1_direct_body(const int *__restrict__ src, int *__restrict__ dst,
                                               int64_t lo, int64_t hi, int64_t xs, int tile, bool vec) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int pairs = tile >> 1;
#pragma unroll 4
    for (int p = tid; p < pairs; p += nt) {
        const int64_t x = xs + 2 * (int64_t)p;
        if (x + 1 < lo || x >= hi) continue;
        const int2 c = vec ? *reinterpret_cast<const int2 *>(src + x) : make_int2(src[x], src[x + 1]);
        const int l = src[x - 1], r = src[x + 2];
        const int v0 = avg3<WIDE>(l, c.x, c.y), v1 = avg3<WIDE>(c.x, c.y, r);
        if (vec && x >= lo && x + 1 < hi) {
            *reinterpret_cast<int2 *>(dst + x) = make_int2(v0, v1);
        } else {
            if (x >= lo && x < hi) dst[x] = v0;
            if (x + 1 >= lo && x + 1 < hi) dst[x + 1] = v1;
        }
    }
}

__global__ void __launch_bounds__(1024) k_jacobi1d_direct(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t lo,
                                                         int64_t hi, int64_t x0, int tile, int vec,
                                                         const int *flag, int mode) {
    const int64_t xs = x0 + (int64_t)blockIdx.x * tile;
    if (narrow_mode(mode, flag))
        j1_direct_body<false>(src, dst, lo, hi, xs, tile, vec != 0);
    else
        j1_direct_body<true>(src, dst, lo, hi, xs, tile, vec != 0);
}

// ---------------------------------------------------------------- 2-D ------

// Staged: the (TI+2) x (TJ+4) window (rows r0-1..r0+TI, cols c0-2..c0+TJ+1)
// is copied to shared memory (64-bit loads when N is even); each thread then
// owns a column pair and marches down its rows keeping the up/centre/down
// values in registers, so a row costs one 64-bit and two 32-bit shared
// loads per two outputs.
template <bool WIDE>
__device__ __forceinline__ void j2_staged_body(const int *__restrict__ src, int *__restrict__ dst,
                                               int64_t N, int64_t r0, int64_t rhi, int64_t c0,
                                               int64_t J, int TI, int TJ, bool vec, int *sh) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int pitch = TJ + 4;
    const int nr = (int)min((int64_t)TI, rhi - r0);
    // ---- load window
    const int w2 = pitch >> 1;
    for (int e = tid; e < (nr + 2) * w2; e += nt) {
        const int rr = e / w2, q = e - rr * w2;
        const int64_t row = r0 - 1 + rr;
        const int64_t col = c0 - 2 + 2 * (int64_t)q;
        const int *s = src + row * N + col;
        int *d = sh + rr * pitch + 2 * q;
        if (vec && col >= 0 && col + 1 < N) {
            *reinterpret_cast<int2 *>(d) = *reinterpret_cast<const int2 *>(s);
        } else {
            d[0] = (col >= 0 && col < N) ? s[0] : 0;
            d[1] = (col + 1 >= 0 && col + 1 < N) ? s[1] : 0;
        }
    }
    __syncthreads();
    // ---- compute: thread -> (column pair, row group)
    const int ncp = TJ >> 1;
    auto march = [&](int cp, int rb, int re) {
        const int64_t j = c0 + 2 * (int64_t)cp;  // output columns j, j+1
        const bool in0 = j >= 1 && j <= J, in1 = j + 1 >= 1 && j + 1 <= J;
        if ((!in0 && !in1) || rb >= re) return;
        const int lc = 2 * cp + 2;  // window column of j
        int2 up = *reinterpret_cast<const int2 *>(sh + rb * pitch + lc);
        int2 cur = *reinterpret_cast<const int2 *>(sh + (rb + 1) * pitch + lc);
        for (int rr = rb; rr < re; rr++) {
            const int *crow = sh + (rr + 1) * pitch + lc;
            const int2 dn = *reinterpret_cast<const int2 *>(crow + pitch);
            const int l = crow[-1], r = crow[2];
            const int v0 = avg5<WIDE>(up.x, dn.x, l, cur.y, cur.x);
            const int v1 = avg5<WIDE>(up.y, dn.y, cur.x, r, cur.y);
            int *o = dst + (r0 + rr) * N + j;
            if (in0 && in1 && vec) {
                *reinterpret_cast<int2 *>(o) = make_int2(v0, v1);
            } else {
                if (in0) o[0] = v0;
                if (in1) o[1] = v1;
            }
            up = cur;
            cur = dn;
        }
    };
    if (nt >= ncp) {
        const int groups = nt / ncp, g = tid / ncp;
        const int rpg = (nr + groups - 1) / groups;
        if (g < groups) march(tid % ncp, g * rpg, min(nr, (g + 1) * rpg));
    } else {
        for (int cp = tid; cp < ncp; cp += nt) march(cp, 0, nr);
    }
}

__global__ void __launch_bounds__(1024) k_jacobi2d_staged(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t N,
                                                         int64_t rlo, int64_t rhi, int64_t J,
                                                         int TI, int TJ, int64_t ntj, int vec,
                                                         const int *flag, int mode) {
    extern __shared__ __align__(16) int sh[];
    const int64_t bid = blockIdx.x;
    const int64_t r0 = rlo + (bid / ntj) * TI, c0 = (bid % ntj) * TJ;
    if (narrow_mode(mode, flag))
        j2_staged_body<false>(src, dst, N, r0, rhi, c0, J, TI, TJ, vec != 0, sh);
    else
        j2_staged_body<true>(src, dst, N, r0, rhi, c0, J, TI, TJ, vec != 0, sh);
}

// caching-off: a thread owns a column pair of TI rows and reads the five
// neighbours from global memory (row above / below through L1/L2).
template <bool WIDE>
__device__ __forceinline__ void j2_direct_body(const int *__restrict__ src, int *__restrict__ dst,
                                               int64_t N, int64_t r0, int64_t rhi, int64_t c0,
                                               int64_t J, int TI, int TJ, bool vec) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int nr = (int)min((int64_t)TI, rhi - r0);
    const int ncp = TJ >> 1;
    for (int e = tid; e < nr * ncp; e += nt) {
        const int rr = e / ncp, cp = e - rr * ncp;
        const int64_t i = r0 + rr, j = c0 + 2 * (int64_t)cp;
        const bool in0 = j >= 1 && j <= J, in1 = j + 1 >= 1 && j + 1 <= J;
        if (!in0 && !in1) continue;
        const int *m = src + i * N + j;
        int2 c, u, d;
        if (vec) {
            c = *reinterpret_cast<const int2 *>(m);
            u = *reinterpret_cast<const int2 *>(m - N);
            d = *reinterpret_cast<const int2 *>(m + N);
        } else {
            c = make_int2(m[0], m[1]);
            u = make_int2(m[-N], m[1 - N]);
            d = make_int2(m[N], m[1 + N]);
        }
        const int l = m[-1], r = m[2];
        const int v0 = avg5<WIDE>(u.x, d.x, l, c.y, c.x), v1 = avg5<WIDE>(u.y, d.y, c.x, r, c.y);
        int *o = dst + i * N + j;
        if (in0 && in1 && vec) {
            *reinterpret_cast<int2 *>(o) = make_int2(v0, v1);
        } else {
            if (in0) o[0] = v0;
            if (in1) o[1] = v1;
        }
    }
}

__global__ void __launch_bounds__(1024) k_jacobi2d_direct(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t N,
                                                         int64_t rlo, int64_t rhi, int64_t J,
                                                         int TI, int TJ, int64_t ntj, int vec,
                                                         const int *flag, int mode) {
    const int64_t bid = blockIdx.x;
    const int64_t r0 = rlo + (bid / ntj) * TI, c0 = (bid % ntj) * TJ;
    if (narrow_mode(mode, flag))
        j2_direct_body<false>(src, dst, N, r0, rhi, c0, J, TI, TJ, vec != 0);
    else
        j2_direct_body<true>(src, dst, N, r0, rhi, c0, J, TI, TJ, vec != 0);
}

struct Extents1D {
    int64_t P;  // interior positions updated: 1..P
};

int extents1d(const pk_launch_t &L, Extents1D *e) {
    if (L.s * L.B == 0) return fail(PK_E_DIV0, "jacobi: s*B == 0 in dim = (N - 2) / (s * B)");
    e->P = 0;
    if (L.s < 0 || L.B < 0) return PK_OK;
    e->P = max0((L.N - 2) / (L.s * L.B)) * L.s * L.B;
    return PK_OK;
}

struct Extents2D {
    int64_t I, J;  // rows 1..I, cols 1..J
};

int extents2d(const pk_launch_t &L, Extents2D *e) {
    if (L.B0 == 0) return fail(PK_E_DIV0, "jacobi2d: B0 == 0 in dim0 = (N - 2) / B0");
    if (L.s * L.B1 == 0) return fail(PK_E_DIV0, "jacobi2d: s*B1 == 0 in dim1 = (N - 2) / (s * B1)");
    e->I = e->J = 0;
    if (L.B0 < 0 || L.B1 < 0 || L.s < 0) return PK_OK;
    e->I = max0((L.N - 2) / L.B0) * L.B0;
    e->J = max0((L.N - 2) / (L.s * L.B1)) * L.s * L.B1;
    return PK_OK;
}

// mode for a sweep: the caller's PK_FLAG_NARROW promise, a device flag, or wide
int sweep_mode(const pk_launch_t &L, const int *flag) {
    if (flag) return 2;
    return (L.flags & PK_FLAG_NARROW) ? 1 : 0;
}

int sweep1d_impl(const pk_launch_t &L, const int *src, int *dst, int64_t lo, int64_t hi,
                 const int *flag, cudaStream_t st) {
    Extents1D e;
    int rc = extents1d(L, &e);
    if (rc) return rc;
    if (lo < 1) lo = 1;
    if (hi > e.P + 1) hi = e.P + 1;
    if (hi <= lo) return PK_OK;
    int64_t tile64 = elems(L) * L.B;
    if (tile64 & 1) tile64 += 1;  // the pair layout needs an even tile; coverage is unchanged
    if (tile64 > (1 << 30)) return fail(PK_E_UNSUPPORTED, "jacobi: tile too large");
    const int tile = (int)tile64;
    const int nt = (int)(L.B < 1024 ? L.B : 1024);
    const int64_t x0 = lo & ~(int64_t)1;
    const int64_t blocks = ceil_div(hi - x0, tile);
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi: grid too large");
    const int vec = !((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 7u);
    const int mode = sweep_mode(L, flag);
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = ((size_t)tile + 4) * sizeof(int);
        rc = allow_smem((const void *)k_jacobi1d_staged, smem);
        if (rc) return rc;
        k_jacobi1d_staged<<<(unsigned)blocks, nt, smem, st>>>(src, dst, lo, hi, x0, tile, L.N, vec, flag, mode);
    } else {
        k_jacobi1d_direct<<<(unsigned)blocks, nt, 0, st>>>(src, dst, lo, hi, x0, tile, vec, flag, mode);
    }
    return after_launch("jacobi1d");
}

int sweep2d_impl(const pk_launch_t &L, const int *src, int *dst, int64_t lo, int64_t hi,
                 const int *flag, cudaStream_t st) {
    Extents2D e;
    int rc = extents2d(L, &e);
    if (rc) return rc;
    if (lo < 1) lo = 1;
    if (hi > e.I + 1) hi = e.I + 1;
    if (hi <= lo || e.J <= 0) return PK_OK;
    int64_t TI64 = L.B0, TJ64 = elems(L) * L.B1;
    if (TJ64 & 1) TJ64 += 1;
    if (TI64 * TJ64 > (1 << 26)) return fail(PK_E_UNSUPPORTED, "jacobi2d: tile too large");
    const int TI = (int)TI64, TJ = (int)TJ64;
    int64_t nthreads = L.B0 * L.B1;
    if (nthreads > 1024) nthreads = 1024;
    const int64_t nti = ceil_div(hi - lo, TI), ntj = ceil_div(e.J + 1, TJ);
    const int64_t blocks = nti * ntj;
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi2d: grid too large");
    const int vec = (L.N % 2 == 0) && !((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 7u);
    const int mode = sweep_mode(L, flag);
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = (size_t)(TI + 2) * (size_t)(TJ + 4) * sizeof(int);
        rc = allow_smem((const void *)k_jacobi2d_staged, smem);
        if (rc) return rc;
        k_jacobi2d_staged<<<(unsigned)blocks, (unsigned)nthreads, smem, st>>>(src, dst, L.N, lo, hi, e.J, TI, TJ,
                                                                              ntj, vec, flag, mode);
    } else {
        k_jacobi2d_direct<<<(unsigned)blocks, (unsigned)nthreads, 0, st>>>(src, dst, L.N, lo, hi, e.J, TI, TJ,
                                                                           ntj, vec, flag, mode);
    }
    return after_launch("jacobi2d");
}

// Device flag: 1 when the whole double buffer is within the narrow bound.
int range_flag(const int *a, int64_t n, int bound, int **flag, cudaStream_t st) {
    cudaError_t err = cudaMallocAsync((void **)flag, sizeof(int), st);
    if (err != cudaSuccess) return fail(PK_E_ALLOC, "cudaMallocAsync(flag): %s", cudaGetErrorString(err));
    // the flag starts non-zero (bytes 0x01); the check clears it with atomicAnd
    err = cudaMemsetAsync(*flag, 1, sizeof(int), st);
    if (err != cudaSuccess) return fail(PK_E_CUDA, "flag init: %s", cudaGetErrorString(err));
    int64_t blocks = ceil_div(n / 4 + 1, 256 * 8);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    k_range_flag<<<(unsigned)blocks, 256, 0, st>>>(a, n, bound, *flag);
    return after_launch("range_flag");
}

}  // namespace

int sweep_jacobi1d(const pk_launch_t &L, const void *src, void *dst, int64_t lo, int64_t hi,
                   cudaStream_t st) {
    return sweep1d_impl(L, static_cast<const int *>(src), static_cast<int *>(dst), lo, hi, nullptr, st);
}

int sweep_jacobi2d(const pk_launch_t &L, const void *src, void *dst, int64_t lo, int64_t hi,
                   cudaStream_t st) {
    return sweep2d_impl(L, static_cast<const int *>(src), static_cast<int *>(dst), lo, hi, nullptr, st);
}

int jacobi_narrow(const pk_launch_t &L, const void *a, int *narrow, cudaStream_t st) {
    const bool one = L.family == PK_FAMILY_JACOBI1D;
    const int64_t n = one ? 2 * L.N : 2 * L.N * L.N;
    int *flag = nullptr;
    int rc = range_flag(static_cast<const int *>(a), n, one ? kBound3 : kBound5, &flag, st);
    if (rc) return rc;
    cudaMemcpyAsync(narrow, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(flag, st);
    cudaError_t err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return fail(PK_E_CUDA, "range check: %s", cudaGetErrorString(err));
    return PK_OK;
}

int launch_jacobi1d(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    Extents1D e;
    int rc = extents1d(L, &e);
    if (rc) return rc;
    if (e.P <= 0 || L.T <= 0) return PK_OK;
    int64_t lo, hi;
    unit_range(L, 1, e.P + 1, &lo, &hi);
    int *a = static_cast<int *>(p[0]);
    int *flag = nullptr;
    if (!(L.flags & PK_FLAG_NARROW)) {
        rc = range_flag(a, 2 * L.N, kBound3, &flag, st);
        if (rc) return rc;
    }
    for (int64_t t = 0; t < L.T && rc == PK_OK; t++) {
        const bool even = (t % 2) == 0;
        int *dst = even ? a : a + L.N;
        const int *src = even ? a + L.N : a;
        rc = sweep1d_impl(L, src, dst, lo, hi, flag, st);
    }
    if (flag) cudaFreeAsync(flag, st);
    return rc;
}

int launch_jacobi2d(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    Extents2D e;
    int rc = extents2d(L, &e);
    if (rc) return rc;
    if (e.I <= 0 || e.J <= 0 || L.T <= 0) return PK_OK;
    int64_t lo, hi;
    unit_range(L, 1, e.I + 1, &lo, &hi);
    int *a = static_cast<int *>(p[0]);
    int *half1 = a + L.N * L.N;
    int *flag = nullptr;
    if (!(L.flags & PK_FLAG_NARROW)) {
        rc = range_flag(a, 2 * L.N * L.N, kBound5, &flag, st);
        if (rc) return rc;
    }
    for (int64_t t = 0; t < L.T && rc == PK_OK; t++) {
        const bool even = (t % 2) == 0;
        // t even reads half 0 and writes half 1 (a[N+i][j] = ...), t odd the reverse
        rc = sweep2d_impl(L, even ? a : half1, even ? half1 : a, lo, hi, flag, st);
    }
    if (flag) cudaFreeAsync(flag, st);
    return rc;
}

}  // namespace pk
