// k_addition.cu -- elementwise addition over flat N*N buffers
// (pkg/src/parakern/data/addition.mfk:11-23):
//   dim0 = N/B0, dim1 = N/(2*B1);  i < dim0*B0, j < dim1*B1
//   if (i < N && j < N/2) { c[iN+j] = a[iN+j] + b[iN+j];  c[iN+j+N/2] = ... (twin) }
// After granularity merged the twin stores (strategies.py:213-262) the program
// reads dim1 = N/B1 and covers j < dim1*B1 with one store; that variant is
// selected with PK_FLAG_MERGED when the caller runs the rewritten program.
// HBM-bound: 12 bytes per written element.
#include "pk_internal.cuh"

namespace pk {
namespace {

// One block row-strip: rows [r0, r0+rows), columns of the covered ranges
// [0, J) and, for the twin form, [half, half+J).  int32 wraps like C int.
__global__ void __launch_bounds__(256) k_addition(const int *__restrict__ a, const int *__restrict__ b,
                                                 int *__restrict__ c, int64_t N, int64_t rlo,
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
            c[row + j] = (int)((unsigned)a[row + j] + (unsigned)b[row + j]);
        }
    }
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
    const int nt = 256;
    int64_t gx = ceil_div(span, nt);
    if (gx > 4096) gx = 4096;
    const int rows_per_block = 8;
    const int64_t gy = ceil_div(rhi - rlo, rows_per_block);
    if (gy > 65535) {
        // fold extra rows into each block
        const int64_t rpb = ceil_div(rhi - rlo, 65535);
        k_addition<<<dim3((unsigned)gx, (unsigned)ceil_div(rhi - rlo, rpb)), nt, 0, st>>>(
            static_cast<const int *>(p[0]), static_cast<const int *>(p[1]), static_cast<int *>(p[2]),
            L.N, rlo, rhi, J, half, merged ? 0 : 1, (int)rpb);
    } else {
        k_addition<<<dim3((unsigned)gx, (unsigned)gy), nt, 0, st>>>(
            static_cast<const int *>(p[0]), static_cast<const int *>(p[1]), static_cast<int *>(p[2]),
            L.N, rlo, rhi, J, half, merged ? 0 : 1, rows_per_block);
    }
    return after_launch("addition");
}

}  // namespace pk
