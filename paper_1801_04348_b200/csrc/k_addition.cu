// k_addition.cu -- elementwise addition over flat N*N buffers
// (pkg/src/parakern/data/addition.mfk:11-23):
//   dim0 = N/B0, dim1 = N/(2*B1);  i < dim0*B0, j < dim1*B1
//   if (i < N && j < N/2) { c[iN+j] = a[iN+j] + b[iN+j];  c[iN+j+N/2] = ... (twin) }
// After granularity merged the twin stores (strategies.py:213-262) the program
// reads dim1 = N/B1 and covers j < dim1*B1 with one store; that variant is
// selected with PK_FLAG_MERGED when the caller runs the rewritten program.
// HBM-bound: 3 * sizeof(element) bytes per written element.  Element types:
// int32 / int64 wrap like C (exact whenever the sum fits; the Python shim
// picks int64 when int32 might not hold the reference's unbounded sum),
// float32 / binary64 add with one IEEE rounding -- binary64 is the
// reference's Python float addition, bit for bit.
#include "pk_internal.cuh"

namespace pk {
namespace {

// One block row-strip: rows [r0, r0+rows), columns of the covered ranges
// [0, J) and, for the twin form, [half, half+J).
__device__ __forceinline__ int add_elem(int x, int y) { return (int)((unsigned)x + (unsigned)y); }
__device__ __forceinline__ long long add_elem(long long x, long long y) {
    return (long long)((unsigned long long)x + (unsigned long long)y);
}
__device__ __forceinline__ float add_elem(float x, float y) { return __fadd_rn(x, y); }
__device__ __forceinline__ double add_elem(double x, double y) { return __dadd_rn(x, y); }

template <typename T>
__global__ void __launch_bounds__(256) k_addition(const T *__restrict__ a, const T *__restrict__ b,
                                                 T *__restrict__ c, int64_t N, int64_t rlo,
                                                 int64_t rhi, int64_t J, int64_t half, int twin,
                                                 int rows_per_block) {
    const int64_t r0 = rlo + (int64_t)blockIdx.y * rows_per_block;
    const int64_t r1 = min(r0 + rows_per_block, rhi);
    const int64_t span = twin ? 2 * J : J;
    for (int64_t r = r0; r < r1; r++) {
        const int64_t row = r * N;
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < span;
             e += (int64_t)gridDim.x * blockDim.x) {
            const int64_t j = e < J ? e : half + (e - J);
            c[row + j] = add_elem(a[row + j], b[row + j]);
        }
    }
}

// 16-byte vectors of V = 16 / sizeof(T) elements.  Vector u of the run is
// column vector w = u % per_row of row rlo + u / per_row, where a row holds
// [0, Jv) and, for the twin form, [halfv, halfv + Jv); when the covered
// columns are the whole row the rows are one contiguous run (per_row = 0
// selects that form: vector u at rlo*N/V + u).  Each thread keeps U vectors
// of a and b in flight.
template <typename T>
__device__ __forceinline__ int4 add_vec(const int4 &x, const int4 &y) {
    int4 r;
    const T *xs = reinterpret_cast<const T *>(&x), *ys = reinterpret_cast<const T *>(&y);
    T *rs = reinterpret_cast<T *>(&r);
#pragma unroll
    for (int i = 0; i < (int)(16 / sizeof(T)); i++) rs[i] = add_elem(xs[i], ys[i]);
    return r;
}

constexpr int kAddThreads = 256, kAddU = 8;

template <typename T>
__global__ void __launch_bounds__(kAddThreads) k_addition_vec(const int4 *__restrict__ a, const int4 *__restrict__ b,
                                                             int4 *__restrict__ c, int64_t Nv, int64_t rlo,
                                                             int64_t Jv, int64_t halfv, int64_t per_row,
                                                             int64_t total) {
    const int64_t stride = (int64_t)gridDim.x * kAddThreads;
    for (int64_t u0 = (int64_t)blockIdx.x * kAddThreads * kAddU + threadIdx.x; u0 < total;
         u0 += stride * kAddU) {
        int64_t off[kAddU];
        int4 x[kAddU], y[kAddU];
#pragma unroll
        for (int k = 0; k < kAddU; k++) {
            const int64_t u = u0 + (int64_t)k * kAddThreads;
            if (per_row == 0) {
                off[k] = rlo * Nv + u;
            } else {
                const int64_t r = u / per_row, w = u - r * per_row;
                off[k] = (rlo + r) * Nv + (w < Jv ? w : halfv + (w - Jv));
            }
            if (u < total) {
                x[k] = ld_stream(a + off[k]);
                y[k] = ld_stream(b + off[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < kAddU; k++)
            if (u0 + (int64_t)k * kAddThreads < total) st_stream(c + off[k], add_vec<T>(x[k], y[k]));
    }
}

template <typename T>
void launch_t(void *const *p, int64_t N, int64_t rlo, int64_t rhi, int64_t J, int64_t half, bool merged,
              int64_t span, cudaStream_t st) {
    constexpr int V = 16 / sizeof(T);
    if (N % V == 0 && J % V == 0 && half % V == 0 && aligned16(p[0]) && aligned16(p[1]) && aligned16(p[2])) {
        const int64_t Jv = J / V, halfv = half / V, Nv = N / V, rows = rhi - rlo;
        const bool whole = merged ? J == N : (J == half && 2 * half == N);
        const int64_t per_row = whole ? 0 : (merged ? Jv : 2 * Jv);
        const int64_t total = rows * (whole ? Nv : per_row);
        // one pass: every thread moves kAddU 16-byte vectors of each array, no
        // grid-stride loop (16384^2 int32: 6.42 TB/s with 4 vectors on a
        // persistent 8-blocks-per-SM grid, 6.85 / 6.96 / 7.02 with 8 vectors on
        // 16 / 32 / 64 blocks per SM, 7.12 with a block per 2048 vectors)
        const int64_t blocks = ceil_div(total, (int64_t)kAddThreads * kAddU);
        k_addition_vec<T><<<(unsigned)blocks, kAddThreads, 0, st>>>(
            static_cast<const int4 *>(p[0]), static_cast<const int4 *>(p[1]), static_cast<int4 *>(p[2]), Nv, rlo,
            Jv, halfv, per_row, total);
        return;
    }
    const int nt = 256;
    int64_t gx = ceil_div(span, nt);
    if (gx > 4096) gx = 4096;
    int rows_per_block = 8;
    if (ceil_div(rhi - rlo, rows_per_block) > 65535) rows_per_block = (int)ceil_div(rhi - rlo, 65535);  // fold rows
    const int64_t gy = ceil_div(rhi - rlo, rows_per_block);
    k_addition<T><<<dim3((unsigned)gx, (unsigned)gy), nt, 0, st>>>(
        static_cast<const T *>(p[0]), static_cast<const T *>(p[1]), static_cast<T *>(p[2]), N, rlo, rhi, J, half,
        merged ? 0 : 1, rows_per_block);
}

}  // namespace

int launch_addition(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    const bool merged = (L.flags & PK_FLAG_MERGED) != 0;
    if (L.B0 == 0) return fail(PK_E_DIV0, "addition: B0 == 0 in dim0 = N / B0");
    if ((merged ? L.B1 : 2 * L.B1) == 0) return fail(PK_E_DIV0, "addition: B1 == 0 in dim1");
    if (L.B0 < 0 || L.B1 < 0 || L.N <= 0) return PK_OK;
    const int64_t I = max0(L.N / L.B0) * L.B0;  // i < dim0*B0 <= N, so i < N always holds
    int64_t J, half = L.N / 2;
    if (merged) {
        J = max0(L.N / L.B1) * L.B1;  // j < dim1*B1 <= N
    } else {
        J = max0(L.N / (2 * L.B1)) * L.B1;  // j < dim1*B1 <= N/2
        if (J > half) J = half;
    }
    int64_t rlo, rhi;
    unit_range(L, 0, I, &rlo, &rhi);
    if (rhi <= rlo || J <= 0) return PK_OK;
    const int64_t span = merged ? J : 2 * J;
    switch (L.dtype) {
        case PK_DTYPE_I32: launch_t<int>(p, L.N, rlo, rhi, J, half, merged, span, st); break;
        case PK_DTYPE_F32: launch_t<float>(p, L.N, rlo, rhi, J, half, merged, span, st); break;
        case PK_DTYPE_I64: launch_t<long long>(p, L.N, rlo, rhi, J, half, merged, span, st); break;
        case PK_DTYPE_F64: launch_t<double>(p, L.N, rlo, rhi, J, half, merged, span, st); break;
        default: return fail(PK_E_UNSUPPORTED, "addition: dtype %d", L.dtype);
    }
    return after_launch("addition");
}

}  // namespace pk
