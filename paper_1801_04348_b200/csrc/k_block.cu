// k_block.cu -- one thread block of a program (the reference's run_block,
// pkg/src/parakern/interp.py:228-249): the grid indices and the serial
// context loop variables fixed, the thread meta_for loops swept.  One CUDA
// block runs the program's thread loops literally (CUDA thread tid takes
// thread-loop points tid, tid + blockDim, ...; the loops of a block carry no
// dependences, interp.py:12-15), every statement of the body in the
// program's own order, on any element type:
//   int32 / int64  C integer arithmetic, truncating division
//   float32 / binary64  IEEE operations in the interpreter's order, no
//   contraction; the Jacobi "/" is the reference's c_div on Python floats
//   (interp.py:43-46: the floor division of |x| by |d| -- CPython's
//   fmod-based float floor division -- with the quotient's sign)
// Also the per-step binary64 / int64 Jacobi sweeps run_program uses for
// data the int32 register sweeps do not take.
#include "pk_internal.cuh"

namespace pk {
namespace {

template <typename T> __device__ __forceinline__ T add_(T a, T b) { return a + b; }
template <> __device__ __forceinline__ int add_(int a, int b) { return (int)((unsigned)a + (unsigned)b); }
template <> __device__ __forceinline__ long long add_(long long a, long long b) {
    return (long long)((unsigned long long)a + (unsigned long long)b);
}
template <> __device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
template <typename T> __device__ __forceinline__ T mul_(T a, T b) { return a * b; }
template <> __device__ __forceinline__ int mul_(int a, int b) { return (int)((unsigned)a * (unsigned)b); }
template <> __device__ __forceinline__ long long mul_(long long a, long long b) {
    return (long long)((unsigned long long)a * (unsigned long long)b);
}
template <> __device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }

// CPython's float floor division x // y for x >= 0, y > 0 (float_divmod):
// mod = fmod(x, y); div = (x - mod) / y; floordiv = floor(div), +1 when the
// rounding left div - floor(div) > 0.5; 0 keeps the sign of x / y.
__device__ __forceinline__ double py_floordiv(double x, double y) {
    const double mod = fmod(x, y);
    const double div = __ddiv_rn(__dsub_rn(x, mod), y);
    if (div != 0.0) {
        double fl = floor(div);
        if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
        return fl;
    }
    return copysign(0.0, __ddiv_rn(x, y));
}
// interp.py:43-46 c_div(a, b) = abs(a) // abs(b), negated when the signs differ
__device__ __forceinline__ double cdiv_(double s, int d) {
    const double q = py_floordiv(fabs(s), (double)d);
    return (s >= 0.0) ? q : -q;  // d > 0 here (3 or 5)
}
__device__ __forceinline__ float cdiv_(float s, int d) { return (float)cdiv_((double)s, d); }
// ints: the sum of 3 (5) values formed in 64 bits, C division truncates
template <typename T> struct Wide { using type = T; };
template <> struct Wide<int> { using type = long long; };
template <typename T> __device__ __forceinline__ T jdiv(typename Wide<T>::type s, int d);
template <> __device__ __forceinline__ int jdiv<int>(long long s, int d) { return (int)(s / d); }
template <> __device__ __forceinline__ long long jdiv<long long>(long long s, int d) { return s / d; }
template <> __device__ __forceinline__ float jdiv<float>(float s, int d) { return cdiv_(s, d); }
template <> __device__ __forceinline__ double jdiv<double>(double s, int d) { return cdiv_(s, d); }
template <typename T> __device__ __forceinline__ typename Wide<T>::type wadd(typename Wide<T>::type a, T b) {
    return add_<typename Wide<T>::type>(a, (typename Wide<T>::type)b);
}

// c + a*b as the family's full-program kernels evaluate it: two roundings
// for binary64 (the interpreter's Python floats), one FFMA for float32 (the
// FP32 leaves' fma chain), wrapping for the ints
template <typename T> __device__ __forceinline__ T mad_(T a, T b, T c) { return add_<T>(c, mul_<T>(a, b)); }
template <> __device__ __forceinline__ float mad_(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// one row of y += a*x: float32 sums the exact products in binary64 and
// rounds once (the leaf kernels' double-float sum is as accurate)
template <typename T>
__device__ __forceinline__ T mv_row(const T *row, const T *x, T y, int64_t N) {
    for (int64_t q = 0; q < N; q++) y = add_<T>(y, mul_<T>(row[q], x[q]));
    return y;
}
template <>
__device__ __forceinline__ float mv_row<float>(const float *row, const float *x, float y, int64_t N) {
    double acc = (double)y;
    for (int64_t q = 0; q < N; q++) acc = __dadd_rn(acc, __dmul_rn((double)row[q], (double)x[q]));
    return (float)acc;
}

struct BlockArgs {
    int64_t N, s, B, B0, B1, ub1;
    int64_t g0, g1;  // grid indices (outer, inner)
    int64_t ctx;     // context loop variable (Jacobi t, matmul k)
    int merged;      // addition: the granularity-merged program (one store, j < N)
};

template <typename T>
__global__ void k_block_reverse(const T *__restrict__ a, T *__restrict__ c, BlockArgs A) {
    for (int64_t j = threadIdx.x; j < A.B; j += blockDim.x)
        for (int64_t k = 0; k < A.s; k++) {
            const int64_t p = A.g0 * A.s * A.B + k * A.B + j;
            c[A.N - 1 - p] = a[p];
        }
}

template <typename T>
__global__ void k_block_transpose(const T *__restrict__ a, T *__restrict__ c, BlockArgs A) {
    for (int64_t t = threadIdx.x; t < A.B0 * A.B1; t += blockDim.x) {
        const int64_t u0 = t / A.B1, u1 = t % A.B1;
        for (int64_t k = 0; k < A.s; k++) {
            const int64_t i = A.g0 * A.B0 + u0, j = (A.g1 * A.s + k) * A.B1 + u1;
            c[i * A.N + j] = a[j * A.N + i];
        }
    }
}

template <typename T>
__global__ void k_block_jacobi(T *__restrict__ a, BlockArgs A) {
    using W = typename Wide<T>::type;
    const int64_t N = A.N;
    for (int64_t j = threadIdx.x; j < A.B; j += blockDim.x)
        for (int64_t k = 0; k < A.s; k++) {
            const int64_t p = A.g0 * A.s * A.B + k * A.B + j;
            if (A.ctx % 2 == 0) {
                const W s = wadd<T>(wadd<T>((W)a[N + p], a[N + p + 1]), a[N + p + 2]);
                a[p + 1] = jdiv<T>(s, 3);
            } else {
                const W s = wadd<T>(wadd<T>((W)a[p], a[p + 1]), a[p + 2]);
                a[N + p + 1] = jdiv<T>(s, 3);
            }
        }
}

template <typename T>
__device__ __forceinline__ void j2_point(T *__restrict__ a, int64_t N, int64_t i, int64_t j, int64_t t) {
    using W = typename Wide<T>::type;
    const int64_t src = t % 2 == 0 ? 0 : N, dst = t % 2 == 0 ? N : 0;
    const T *r = a + src * N;
    // ((((up + down) + left) + right) + centre), the program's left-to-right sum
    W s = wadd<T>((W)r[(i - 1) * N + j], r[(i + 1) * N + j]);
    s = wadd<T>(s, r[i * N + j - 1]);
    s = wadd<T>(s, r[i * N + j + 1]);
    s = wadd<T>(s, r[i * N + j]);
    a[(dst + i) * N + j] = jdiv<T>(s, 5);
}

template <typename T>
__global__ void k_block_jacobi2d(T *__restrict__ a, BlockArgs A) {
    for (int64_t t = threadIdx.x; t < A.B0 * A.B1; t += blockDim.x) {
        const int64_t u0 = t / A.B1, u1 = t % A.B1;
        for (int64_t k = 0; k < A.s; k++) {
            const int64_t i = A.g0 * A.B0 + u0 + 1, j = (A.g1 * A.s + k) * A.B1 + u1 + 1;
            j2_point<T>(a, A.N, i, j, A.ctx);
        }
    }
}

template <typename T>
__global__ void k_block_matvec(const T *__restrict__ a, const T *__restrict__ x, T *__restrict__ y, BlockArgs A) {
    for (int64_t j = threadIdx.x; j < A.B; j += blockDim.x)
        for (int64_t k = 0; k < A.s; k++) {
            const int64_t r = A.g0 * A.s * A.B + k * A.B + j;
            y[r] = mv_row<T>(a + r * A.N, x, y[r], A.N);
        }
}

template <typename T>
__global__ void k_block_matmul(const T *__restrict__ a, const T *__restrict__ b, T *__restrict__ c, BlockArgs A) {
    const int64_t n = A.N;
    for (int64_t t = threadIdx.x; t < A.B0 * A.ub1; t += blockDim.x) {
        const int64_t v = t / A.ub1, u = t % A.ub1;
        const int64_t p = A.g0 * A.B0 + v;
        for (int64_t w = 0; w < A.s; w++) {
            const int64_t q = A.g1 * A.ub1 * A.s + w * A.ub1 + u;
            T acc = c[p * n + q];
            for (int64_t z = 0; z < A.B0; z++) {
                const int64_t kk = A.B0 * A.ctx + z;
                acc = mad_<T>(a[p * n + kk], b[kk * n + q], acc);
            }
            c[p * n + q] = acc;
        }
    }
}

template <typename T>
__global__ void k_block_addition(const T *__restrict__ a, const T *__restrict__ b, T *__restrict__ c, BlockArgs A) {
    const int64_t N = A.N, half = N / 2;
    for (int64_t t = threadIdx.x; t < A.B0 * A.B1; t += blockDim.x) {
        const int64_t u0 = t / A.B1, u1 = t % A.B1;
        const int64_t i = A.g0 * A.B0 + u0, j = A.g1 * A.B1 + u1;
        if (A.merged) {
            if (i < N && j < N) c[i * N + j] = add_<T>(a[i * N + j], b[i * N + j]);
        } else if (i < N && j < half) {
            c[i * N + j] = add_<T>(a[i * N + j], b[i * N + j]);
            c[i * N + j + half] = add_<T>(a[i * N + j + half], b[i * N + j + half]);
        }
    }
}

template <typename T>
int launch_block_t(const pk_launch_t &L, const BlockArgs &A, void *const *p, cudaStream_t st) {
    int64_t work = 1;
    switch (L.family) {
        case PK_FAMILY_REVERSE: case PK_FAMILY_JACOBI1D: case PK_FAMILY_MATVEC: work = A.B; break;
        case PK_FAMILY_MATMUL: work = A.B0 * A.ub1; break;
        default: work = A.B0 * A.B1; break;
    }
    if (work <= 0) return PK_OK;  // an empty thread meta_for: nothing runs
    const unsigned nt = (unsigned)(work < 256 ? ((work + 31) / 32) * 32 : 256);
    switch (L.family) {
        case PK_FAMILY_REVERSE:
            k_block_reverse<T><<<1, nt, 0, st>>>(static_cast<const T *>(p[0]), static_cast<T *>(p[1]), A); break;
        case PK_FAMILY_TRANSPOSE:
            k_block_transpose<T><<<1, nt, 0, st>>>(static_cast<const T *>(p[0]), static_cast<T *>(p[1]), A); break;
        case PK_FAMILY_JACOBI1D: k_block_jacobi<T><<<1, nt, 0, st>>>(static_cast<T *>(p[0]), A); break;
        case PK_FAMILY_JACOBI2D: k_block_jacobi2d<T><<<1, nt, 0, st>>>(static_cast<T *>(p[0]), A); break;
        case PK_FAMILY_MATVEC:
            k_block_matvec<T><<<1, nt, 0, st>>>(static_cast<const T *>(p[0]), static_cast<const T *>(p[1]),
                                                 static_cast<T *>(p[2]), A);
            break;
        case PK_FAMILY_MATMUL:
            k_block_matmul<T><<<1, nt, 0, st>>>(static_cast<const T *>(p[0]), static_cast<const T *>(p[1]),
                                                 static_cast<T *>(p[2]), A);
            break;
        case PK_FAMILY_ADDITION:
            k_block_addition<T><<<1, nt, 0, st>>>(static_cast<const T *>(p[0]), static_cast<const T *>(p[1]),
                                                   static_cast<T *>(p[2]), A);
            break;
        default: return fail(PK_E_UNSUPPORTED, "run_block: family %d", L.family);
    }
    return after_launch("block");
}

// Whole-program binary64 / int64 Jacobi: one grid-stride sweep per step over
// the covered points (the reference's order inside a point; points of one
// step are independent).
template <typename T>
__global__ void k_jacobi1d_step(T *__restrict__ a, int64_t N, int64_t P, int64_t t) {
    using W = typename Wide<T>::type;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
        if (t % 2 == 0) {
            a[p + 1] = jdiv<T>(wadd<T>(wadd<T>((W)a[N + p], a[N + p + 1]), a[N + p + 2]), 3);
        } else {
            a[N + p + 1] = jdiv<T>(wadd<T>(wadd<T>((W)a[p], a[p + 1]), a[p + 2]), 3);
        }
    }
}

template <typename T>
__global__ void k_jacobi2d_step(T *__restrict__ a, int64_t N, int64_t I, int64_t J, int64_t t) {
    const int64_t total = I * J;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
        j2_point<T>(a, N, e / J + 1, e % J + 1, t);
}

template <typename T>
int jacobi_steps_t(const pk_launch_t &L, T *a, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)sms * 8;
    if (L.family == PK_FAMILY_JACOBI1D) {
        const int64_t tile = elems(L) * L.B;
        const int64_t P = max0((L.N - 2) / tile) * tile;
        if (P <= 0) return PK_OK;
        for (int64_t t = 0; t < L.T; t++) k_jacobi1d_step<T><<<grid, 256, 0, st>>>(a, L.N, P, t);
    } else {
        const int64_t I = max0((L.N - 2) / L.B0) * L.B0, J = max0((L.N - 2) / (L.s * L.B1)) * L.s * L.B1;
        if (I <= 0 || J <= 0) return PK_OK;
        for (int64_t t = 0; t < L.T; t++) k_jacobi2d_step<T><<<grid, 256, 0, st>>>(a, L.N, I, J, t);
    }
    return after_launch("jacobi_steps");
}

}  // namespace

int launch_block(const pk_launch_t &L, const int64_t *grid, int ngrid, const int64_t *ctx, int nctx, void *const *p,
                 cudaStream_t st) {
    BlockArgs A{};
    A.N = L.N;
    A.s = elems(L);
    A.B = L.B;
    A.B0 = L.B0;
    A.B1 = L.B1;
    A.ub1 = L.ub1;
    A.g0 = ngrid > 0 ? grid[0] : 0;
    A.g1 = ngrid > 1 ? grid[1] : 0;
    A.ctx = nctx > 0 ? ctx[0] : 0;
    A.merged = (L.flags & PK_FLAG_MERGED) != 0;
    switch (L.dtype) {
        case PK_DTYPE_I32: return launch_block_t<int>(L, A, p, st);
        case PK_DTYPE_I64: return launch_block_t<long long>(L, A, p, st);
        case PK_DTYPE_F32: return launch_block_t<float>(L, A, p, st);
        case PK_DTYPE_F64: return launch_block_t<double>(L, A, p, st);
        default: return fail(PK_E_UNSUPPORTED, "run_block: dtype %d", L.dtype);
    }
}

int launch_jacobi_wide(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    if (L.dtype == PK_DTYPE_F64) return jacobi_steps_t<double>(L, static_cast<double *>(p[0]), st);
    if (L.dtype == PK_DTYPE_I64) return jacobi_steps_t<long long>(L, static_cast<long long *>(p[0]), st);
    return fail(PK_E_UNSUPPORTED, "jacobi: dtype %d", L.dtype);
}

}  // namespace pk
