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
// loop, interp.py:148-152).  Sums are formed in 64-bit so the truncating
// division sees the exact integer the reference's unbounded ints would.
// HBM-bound: 8 bytes of algorithmic traffic per updated point per step.
#include "pk_internal.cuh"

namespace pk {
namespace {

// ---------------------------------------------------------------- 1-D ------

__global__ void __launch_bounds__(1024) k_jacobi1d_staged(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t xlo,
                                                         int64_t xhi, int tile) {
    extern __shared__ int sh[];
    const int64_t base = xlo + (int64_t)blockIdx.x * tile;
    const int n = (int)min((int64_t)tile, xhi - base);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int *s = src + base - 1;
#pragma unroll 4
    for (int q = tid; q < n + 2; q += nt) sh[q] = s[q];
    __syncthreads();
    int *d = dst + base;
#pragma unroll 4
    for (int q = tid; q < n; q += nt)
        d[q] = div3((long long)sh[q] + (long long)sh[q + 1] + (long long)sh[q + 2]);
}

__global__ void __launch_bounds__(1024) k_jacobi1d_direct(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t xlo,
                                                         int64_t xhi, int tile) {
    const int64_t base = xlo + (int64_t)blockIdx.x * tile;
    const int n = (int)min((int64_t)tile, xhi - base);
    const int tid = threadIdx.x, nt = blockDim.x;
#pragma unroll 4
    for (int q = tid; q < n; q += nt) {
        const int64_t x = base + q;
        dst[x] = div3((long long)src[x - 1] + (long long)src[x] + (long long)src[x + 1]);
    }
}

// ---------------------------------------------------------------- 2-D ------

__global__ void __launch_bounds__(1024) k_jacobi2d_staged(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t N,
                                                         int64_t rlo, int64_t rhi, int64_t J,
                                                         int TI, int TJ, int64_t ntj) {
    extern __shared__ int sh[];
    const int pitch = TJ + 2;
    const int64_t bid = blockIdx.x;
    const int64_t r0 = rlo + (bid / ntj) * TI, c0 = 1 + (bid % ntj) * TJ;
    const int nr = (int)min((int64_t)TI, rhi - r0), nc = (int)min((int64_t)TJ, J + 1 - c0);
    const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x, by = blockDim.y;
    for (int rr = ty; rr < nr + 2; rr += by) {
        const int *row = src + (r0 - 1 + rr) * N + c0 - 1;
        for (int cc = tx; cc < nc + 2; cc += bx) sh[rr * pitch + cc] = row[cc];
    }
    __syncthreads();
    for (int rr = ty; rr < nr; rr += by) {
        int *row = dst + (r0 + rr) * N + c0;
        const int *m = sh + (rr + 1) * pitch + 1;
        for (int cc = tx; cc < nc; cc += bx) {
            const long long sum = (long long)m[cc - pitch] + (long long)m[cc + pitch] +
                                  (long long)m[cc - 1] + (long long)m[cc + 1] + (long long)m[cc];
            row[cc] = div5(sum);
        }
    }
}

__global__ void __launch_bounds__(1024) k_jacobi2d_direct(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t N,
                                                         int64_t rlo, int64_t rhi, int64_t J,
                                                         int TI, int TJ, int64_t ntj) {
    const int64_t bid = blockIdx.x;
    const int64_t r0 = rlo + (bid / ntj) * TI, c0 = 1 + (bid % ntj) * TJ;
    const int nr = (int)min((int64_t)TI, rhi - r0), nc = (int)min((int64_t)TJ, J + 1 - c0);
    const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x, by = blockDim.y;
    for (int rr = ty; rr < nr; rr += by) {
        const int64_t i = r0 + rr;
        const int *m = src + i * N + c0;
        int *row = dst + i * N + c0;
        for (int cc = tx; cc < nc; cc += bx) {
            const long long sum = (long long)m[cc - N] + (long long)m[cc + N] + (long long)m[cc - 1] +
                                  (long long)m[cc + 1] + (long long)m[cc];
            row[cc] = div5(sum);
        }
    }
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

}  // namespace

// One 1-D sweep over positions [lo, hi) clipped to the interior 1..P.
int sweep_jacobi1d(const pk_launch_t &L, const void *srcv, void *dstv, int64_t lo, int64_t hi,
                   cudaStream_t st) {
    Extents1D e;
    int rc = extents1d(L, &e);
    if (rc) return rc;
    if (lo < 1) lo = 1;
    if (hi > e.P + 1) hi = e.P + 1;
    if (hi <= lo) return PK_OK;
    const int64_t tile64 = elems(L) * L.B;
    if (tile64 > (1 << 30)) return fail(PK_E_UNSUPPORTED, "jacobi: tile too large");
    const int tile = (int)tile64;
    const int nt = (int)(L.B < 1024 ? L.B : 1024);
    const int64_t blocks = ceil_div(hi - lo, tile);
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi: grid too large");
    const int *src = static_cast<const int *>(srcv);
    int *dst = static_cast<int *>(dstv);
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = ((size_t)tile + 2) * sizeof(int);
        rc = allow_smem((const void *)k_jacobi1d_staged, smem);
        if (rc) return rc;
        k_jacobi1d_staged<<<(unsigned)blocks, nt, smem, st>>>(src, dst, lo, hi, tile);
    } else {
        k_jacobi1d_direct<<<(unsigned)blocks, nt, 0, st>>>(src, dst, lo, hi, tile);
    }
    return after_launch("jacobi1d");
}

int launch_jacobi1d(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    Extents1D e;
    int rc = extents1d(L, &e);
    if (rc) return rc;
    if (e.P <= 0 || L.T <= 0) return PK_OK;
    int64_t lo, hi;
    unit_range(L, 1, e.P + 1, &lo, &hi);
    int *a = static_cast<int *>(p[0]);
    for (int64_t t = 0; t < L.T; t++) {
        const bool even = (t % 2) == 0;
        int *dst = even ? a : a + L.N;
        const int *src = even ? a + L.N : a;
        rc = sweep_jacobi1d(L, src, dst, lo, hi, st);
        if (rc) return rc;
    }
    return PK_OK;
}

int sweep_jacobi2d(const pk_launch_t &L, const void *srcv, void *dstv, int64_t lo, int64_t hi,
                   cudaStream_t st) {
    Extents2D e;
    int rc = extents2d(L, &e);
    if (rc) return rc;
    if (lo < 1) lo = 1;
    if (hi > e.I + 1) hi = e.I + 1;
    if (hi <= lo || e.J <= 0) return PK_OK;
    const int64_t TI64 = L.B0, TJ64 = elems(L) * L.B1;
    if (TI64 * TJ64 > (1 << 26)) return fail(PK_E_UNSUPPORTED, "jacobi2d: tile too large");
    const int TI = (int)TI64, TJ = (int)TJ64;
    int64_t nthreads = L.B0 * L.B1;
    if (nthreads > 1024) nthreads = 1024;
    dim3 block = (nthreads >= 32 && nthreads % 32 == 0) ? dim3(32, (unsigned)(nthreads / 32))
                                                         : dim3((unsigned)nthreads, 1);
    const int64_t nti = ceil_div(hi - lo, TI), ntj = ceil_div(e.J, TJ);
    const int64_t blocks = nti * ntj;
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi2d: grid too large");
    const int *src = static_cast<const int *>(srcv);
    int *dst = static_cast<int *>(dstv);
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = (size_t)(TI + 2) * (size_t)(TJ + 2) * sizeof(int);
        rc = allow_smem((const void *)k_jacobi2d_staged, smem);
        if (rc) return rc;
        k_jacobi2d_staged<<<(unsigned)blocks, block, smem, st>>>(src, dst, L.N, lo, hi, e.J, TI, TJ, ntj);
    } else {
        k_jacobi2d_direct<<<(unsigned)blocks, block, 0, st>>>(src, dst, L.N, lo, hi, e.J, TI, TJ, ntj);
    }
    return after_launch("jacobi2d");
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
    for (int64_t t = 0; t < L.T; t++) {
        const bool even = (t % 2) == 0;
        // t even reads half 0 and writes half 1 (a[N+i][j] = ...), t odd the reverse
        rc = sweep_jacobi2d(L, even ? a : half1, even ? half1 : a, lo, hi, st);
        if (rc) return rc;
    }
    return PK_OK;
}

}  // namespace pk
