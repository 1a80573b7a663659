// k_matvec.cu -- matrix-vector product (SURVEY App. A.3 matvec.mfk):
//   dim = N/(s*B);  r = i*s*B + k*B + j < dim*s*B;  for q < N: y[r] = y[r] + a[r][q]*x[q]
// A block owns E*B consecutive rows (E = s, or 1 after granularity).  Rows are
// reduced by groups of lanes (a full warp when B allows): each group walks R
// rows at once with U 128-bit loads per row in flight, so a warp keeps R*U*512
// bytes of a outstanding -- the memory-level parallelism a tall mat-vec needs
// when the staged x (N words of shared memory) leaves room for only one block
// per SM.  Partial sums meet in warp shuffles.
// cache(x) kept: x is staged once per block in shared memory (the case
// requires N <= Z_B); caching-off reads x through L1/L2.
// Integers accumulate in wrapping int32 -- exact whenever the result fits, as
// two's-complement sums are exact modulo 2^32.  float32 data accumulate in a
// double-float pair (see DF), rounded once at the end.
// HBM-bound: 4*N bytes of a per row dominate (x stays on chip).
#include "pk_internal.cuh"

namespace pk {
namespace {

// float32 data: a double-float accumulator (hi + lo, both fp32).  Each
// product is split exactly (p = a*x rounded, e = fma(a, x, -p)) and added
// with TwoSum, so the running sum carries ~48 bits -- the accuracy of the
// reference's binary64 sum of Python floats -- on the FP32 pipe.  (Binary64
// accumulation measured 1.9 TB/s at N = 32768: the F2F conversions and DFMAs
// bound it; the fp32 pair keeps the kernel at HBM speed.)  Explicit _rn
// intrinsics keep nvcc from contracting the splits into FMAs.
struct DF {
    float hi, lo;
};

__device__ __forceinline__ void df_add(DF &acc, float v, float err_in) {
    const float t = __fadd_rn(acc.hi, v);
    const float bp = __fsub_rn(t, acc.hi);
    const float err = __fadd_rn(__fsub_rn(acc.hi, __fsub_rn(t, bp)), __fsub_rn(v, bp));  // TwoSum
    acc.hi = t;
    acc.lo = __fadd_rn(acc.lo, __fadd_rn(err, err_in));
}

__device__ __forceinline__ void df_add_prod(DF &acc, float a, float x) {
    const float p = __fmul_rn(a, x);
    df_add(acc, p, __fmaf_rn(a, x, -p));  // p + fma(a, x, -p) == a * x exactly
}

// The same double-float sum on packed pairs (sm_100 FADD2 / FMUL2 / FFMA2:
// two IEEE fp32 operations per instruction): lane 0 accumulates the even
// elements of a row, lane 1 the odd ones, so every 16-byte load of a is two
// exact products and two TwoSums in 11 instructions instead of 20.
struct DF2 {
    unsigned long long hi, lo;  // {even, odd} halves
};

__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// acc += v (exactly, TwoSum per half) with err_in folded into the low parts
__device__ __forceinline__ void df2_add(DF2 &acc, unsigned long long v, unsigned long long err_in) {
    const unsigned long long t = add2(acc.hi, v);
    const unsigned long long bp = sub2(t, acc.hi);
    const unsigned long long err = add2(sub2(acc.hi, sub2(t, bp)), sub2(v, bp));
    acc.hi = t;
    acc.lo = add2(acc.lo, add2(err, err_in));
}

__device__ __forceinline__ void df2_add_prod(DF2 &acc, unsigned long long a, unsigned long long x) {
    // the rounded products by two scalar mul.rn.f32: ptxas contracts a packed
    // product (mul.rn.f32x2, or fma.rn.f32x2 with -0.0) and the TwoSum's
    // add.rn.f32x2 into one FFMA2 even under --fmad=false, which would fold
    // the product's rounding into the sum; scalar .rn products it leaves alone
    const float p0 = __fmul_rn(__uint_as_float((unsigned)a), __uint_as_float((unsigned)x));
    const float p1 = __fmul_rn(__uint_as_float((unsigned)(a >> 32)), __uint_as_float((unsigned)(x >> 32)));
    const unsigned long long p = ((unsigned long long)__float_as_uint(p1) << 32) | __float_as_uint(p0);
    const unsigned long long e = fma2(a, x, sub2(0ull, p));  // a*x - p exactly (halves of +0.0 - p)
    df2_add(acc, p, e);
}

template <typename T> struct Acc;
template <> struct Acc<int> { using type = int; };
template <> struct Acc<float> { using type = DF2; };

__device__ __forceinline__ void acc_zero(int &a) { a = 0; }
__device__ __forceinline__ void acc_zero(DF &a) { a.hi = a.lo = 0.f; }
__device__ __forceinline__ void acc_zero(DF2 &a) { a.hi = a.lo = 0ull; }

__device__ __forceinline__ int group_sum(int v, int lanes) {
    for (int o = lanes >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, lanes);
    return v;
}
__device__ __forceinline__ DF group_sum(DF v, int lanes) {
    for (int o = lanes >> 1; o > 0; o >>= 1) {
        const float h = __shfl_xor_sync(0xffffffffu, v.hi, o, lanes), l = __shfl_xor_sync(0xffffffffu, v.lo, o, lanes);
        df_add(v, h, l);
    }
    return v;
}

__device__ __forceinline__ DF2 group_sum(DF2 v, int lanes) {
    for (int o = lanes >> 1; o > 0; o >>= 1) {
        const unsigned long long h = __shfl_xor_sync(0xffffffffu, v.hi, o, lanes);
        const unsigned long long l = __shfl_xor_sync(0xffffffffu, v.lo, o, lanes);
        df2_add(v, h, l);
    }
    return v;
}
__device__ __forceinline__ void dot4(DF2 &acc, const int4 &av, const float *xp) {
    const unsigned long long *x2 = reinterpret_cast<const unsigned long long *>(xp);
    df2_add_prod(acc, ((unsigned long long)(unsigned)av.y << 32) | (unsigned)av.x, x2[0]);
    df2_add_prod(acc, ((unsigned long long)(unsigned)av.w << 32) | (unsigned)av.z, x2[1]);
}
__device__ __forceinline__ void dot1(DF2 &acc, float a, float x) {  // even half only
    df2_add_prod(acc, (unsigned long long)__float_as_uint(a), (unsigned long long)__float_as_uint(x));
}
__device__ __forceinline__ float finish(float y, DF2 sum) {
    const float h0 = __uint_as_float((unsigned)sum.hi), h1 = __uint_as_float((unsigned)(sum.hi >> 32));
    const float l0 = __uint_as_float((unsigned)sum.lo), l1 = __uint_as_float((unsigned)(sum.lo >> 32));
    return (float)((((double)y + (double)h0) + (double)h1) + ((double)l0 + (double)l1));
}

__device__ __forceinline__ void dot4(int &acc, const int4 &av, const int *xp) {
    acc += av.x * xp[0] + av.y * xp[1] + av.z * xp[2] + av.w * xp[3];
}
__device__ __forceinline__ void dot4(DF &acc, const int4 &av, const float *xp) {
    df_add_prod(acc, __int_as_float(av.x), xp[0]);
    df_add_prod(acc, __int_as_float(av.y), xp[1]);
    df_add_prod(acc, __int_as_float(av.z), xp[2]);
    df_add_prod(acc, __int_as_float(av.w), xp[3]);
}
__device__ __forceinline__ void dot1(int &acc, int a, int x) { acc += a * x; }
__device__ __forceinline__ void dot1(DF &acc, float a, float x) { df_add_prod(acc, a, x); }

// y + the row's sum: ints wrap (two's complement, exact modulo 2^32); floats
// round y + hi + lo once through binary64
__device__ __forceinline__ int finish(int y, int sum) { return y + sum; }
__device__ __forceinline__ float finish(float y, DF sum) {
    return (float)(((double)y + (double)sum.hi) + (double)sum.lo);
}

#ifndef PK_MV_FUNROLL
#define PK_MV_FUNROLL 4
#endif
constexpr int kRows = 4;    // rows per lane group in flight
// 128-bit loads per row in flight: 4 for int32; 3 for float32, whose packed
// double-float accumulators (4 registers per row) would otherwise spill
template <typename T> struct Unroll { static constexpr int value = 4; };
template <> struct Unroll<float> { static constexpr int value = PK_MV_FUNROLL; };

#ifndef PK_MV_NT
#define PK_MV_NT 512
#endif
template <typename T, bool STAGED, bool VEC>
__global__ void __launch_bounds__(PK_MV_NT) k_matvec(const T *__restrict__ a, const T *__restrict__ x,
                                                T *__restrict__ y, int64_t N, int64_t rlo,
                                                int64_t rhi, int tile, int lanes) {
    using A = typename Acc<T>::type;
    constexpr int kUnroll = Unroll<T>::value;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const T *xs = x;
    if (STAGED) {
        T *sx = reinterpret_cast<T *>(smem_raw);
        if (VEC) {
            const int4 *x4 = reinterpret_cast<const int4 *>(x);
            int4 *s4 = reinterpret_cast<int4 *>(sx);
            for (int64_t q = threadIdx.x; q < N / 4; q += blockDim.x) s4[q] = x4[q];
        } else {
            for (int64_t q = threadIdx.x; q < N; q += blockDim.x) sx[q] = x[q];
        }
        __syncthreads();
        xs = sx;
    }
    const int64_t base = rlo + (int64_t)blockIdx.x * tile;
    const int64_t end = min(base + tile, rhi);
    const int lane = threadIdx.x % lanes, group = threadIdx.x / lanes;
    const int ngroups = blockDim.x / lanes;
    for (int64_t r0 = base + (int64_t)group * kRows; r0 < end; r0 += (int64_t)ngroups * kRows) {
        const int nr = (int)min((int64_t)kRows, end - r0);
        A acc[kRows];
#pragma unroll
        for (int i = 0; i < kRows; i++) acc_zero(acc[i]);
        if (VEC) {
            const int64_t n4 = N / 4;
            const int4 *rows[kRows];
#pragma unroll
            for (int i = 0; i < kRows; i++)
                rows[i] = reinterpret_cast<const int4 *>(a + (r0 + (i < nr ? i : 0)) * N);
            const int4 *xv = reinterpret_cast<const int4 *>(xs);
            for (int64_t q0 = lane; q0 < n4; q0 += (int64_t)lanes * kUnroll) {
                int4 v[kUnroll][kRows];
#pragma unroll
                for (int u = 0; u < kUnroll; u++) {
                    const int64_t q = q0 + (int64_t)u * lanes;
#pragma unroll
                    for (int i = 0; i < kRows; i++)
                        v[u][i] = (q < n4 && i < nr) ? ld_stream(rows[i] + q) : make_int4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < kUnroll; u++) {
                    const int64_t q = q0 + (int64_t)u * lanes;
                    if (q < n4) {
                        const int4 xq = xv[q];
                        const T *xp = reinterpret_cast<const T *>(&xq);
#pragma unroll
                        for (int i = 0; i < kRows; i++) dot4(acc[i], v[u][i], xp);
                    }
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < kRows; i++) {
                if (i < nr) {
                    const T *row = a + (r0 + i) * N;
                    for (int64_t q = lane; q < N; q += lanes) dot1(acc[i], row[q], xs[q]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < kRows; i++) {
            const A sum = group_sum(acc[i], lanes);
            if (lane == 0 && i < nr) y[r0 + i] = finish(y[r0 + i], sum);
        }
    }
}

template <typename T>
int launch_t(const pk_launch_t &L, void *const *p, cudaStream_t st, int64_t rlo, int64_t rhi) {
    const int64_t tile64 = elems(L) * L.B;
    if (tile64 > (1 << 30)) return fail(PK_E_UNSUPPORTED, "matvec: tile too large");
    const int tile = (int)tile64;
    // the block size is the kernel's (the groups loop over the tile, so any size
    // covers the program's B): 512 threads keep 16 warps of 16 x 16-byte loads
    // in flight beside the one staged x per SM (6.6 -> 7.1 TB/s at N = 32768)
    int nt = PK_MV_NT;
    // lanes per row: the largest power of two <= 32 dividing the block size
    int lanes = 1;
    while (lanes < 32 && nt % (lanes * 2) == 0) lanes *= 2;
    const T *a = static_cast<const T *>(p[0]);
    const T *x = static_cast<const T *>(p[1]);
    T *y = static_cast<T *>(p[2]);
    const bool vec = L.N % 4 == 0 && aligned16(a) && aligned16(x);
    const bool staged = L.variant == PK_VARIANT_STAGED;
    const size_t smem = staged ? (size_t)L.N * sizeof(T) : 0;
    const void *k = staged ? (vec ? (const void *)k_matvec<T, true, true> : (const void *)k_matvec<T, true, false>)
                           : (vec ? (const void *)k_matvec<T, false, true> : (const void *)k_matvec<T, false, false>);
    if (staged) {
        int rc = allow_smem(k, smem);
        if (rc) return rc;
    }
    // Rows per block: the case's tile, or less so that every SM gets a block --
    // the staged x (N words) allows one block per SM at N = 32768, and
    // N / (s*B) tiles would leave SMs idle (128 of 148 at the BASELINE size).
    int per_sm = 0, sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, nt, smem);
    const int64_t slots = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    const int64_t step = (int64_t)(nt / lanes) * kRows;  // rows one pass of the block's groups covers
    int64_t rows = rhi - rlo, chunk = tile;
    if (ceil_div(rows, chunk) < slots) chunk = ceil_div(ceil_div(rows, slots), step) * step;
    if (chunk < 1) chunk = 1;
    const int64_t blocks = ceil_div(rows, chunk);
    if (blocks > 0x7fffffffLL || chunk > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "matvec: grid too large");
    const int ct = (int)chunk;
    if (staged) {
        if (vec) k_matvec<T, true, true><<<(unsigned)blocks, nt, smem, st>>>(a, x, y, L.N, rlo, rhi, ct, lanes);
        else k_matvec<T, true, false><<<(unsigned)blocks, nt, smem, st>>>(a, x, y, L.N, rlo, rhi, ct, lanes);
    } else {
        if (vec) k_matvec<T, false, true><<<(unsigned)blocks, nt, 0, st>>>(a, x, y, L.N, rlo, rhi, ct, lanes);
        else k_matvec<T, false, false><<<(unsigned)blocks, nt, 0, st>>>(a, x, y, L.N, rlo, rhi, ct, lanes);
    }
    return after_launch("matvec");
}

// int64 and binary64: one thread per row in the interpreter's own order,
// acc = y[r]; acc = acc + a[r][q]*x[q] for q ascending, one rounding per
// operation (no contraction) -- bit-identical to interp.py on Python floats;
// int64 wraps like C (exact modulo 2^64, so exact whenever the result fits).
// A block owns 128 rows; 32-column tiles of a are loaded row-coalesced (each
// warp reads one 256-byte row segment per step) into a transposed shared
// tile, so every thread then walks its own row's columns.
__device__ __forceinline__ double madd(double acc, double a, double x) { return __dadd_rn(acc, __dmul_rn(a, x)); }
__device__ __forceinline__ long long madd(long long acc, long long a, long long x) {
    return (long long)((unsigned long long)acc + (unsigned long long)a * (unsigned long long)x);
}

constexpr int kExactRows = 128, kExactCols = 32;

template <typename T>
__global__ void __launch_bounds__(kExactRows) k_matvec_exact(const T *__restrict__ a, const T *__restrict__ x,
                                                            T *__restrict__ y, int64_t N, int64_t rlo, int64_t rhi) {
    __shared__ T tile[kExactCols][kExactRows + 1];
    __shared__ T xs[kExactCols];
    const int64_t r0 = rlo + (int64_t)blockIdx.x * kExactRows;
    const int t = threadIdx.x;
    const bool live = r0 + t < rhi;
    const int nrows = (int)min((int64_t)kExactRows, rhi - r0);
    T acc = live ? y[r0 + t] : T(0);
    for (int64_t q0 = 0; q0 < N; q0 += kExactCols) {
        const int nc = (int)min((int64_t)kExactCols, N - q0);
        for (int e = t; e < kExactRows * kExactCols; e += kExactRows) {
            const int rr = e / kExactCols, cc = e % kExactCols;
            tile[cc][rr] = (rr < nrows && cc < nc) ? a[(r0 + rr) * N + q0 + cc] : T(0);
        }
        if (t < kExactCols) xs[t] = t < nc ? x[q0 + t] : T(0);
        __syncthreads();
        for (int cc = 0; cc < nc; cc++) acc = madd(acc, tile[cc][t], xs[cc]);
        __syncthreads();
    }
    if (live) y[r0 + t] = acc;
}

// The same sequence fed by cp.async: a block owns groups of kXR = 16 rows
// (one computing thread per row, every thread loading), 256-column stages
// of a (32 KB) double-buffered in shared memory, the next stage in flight
// while the 16 chains run over the current one; persistent blocks stride
// over the row groups (32768 rows: 2048 groups on 3 x 148 blocks).  Needs
// N even and 16-byte aligned operands (rows then start on 16 bytes).
constexpr int kXR = 32, kXC = 128, kXT = 128, kXPitch = kXC + 2;  // pitch: 16-byte rows, 2-way banks

template <typename T>
__global__ void __launch_bounds__(kXT) k_matvec_exact_async(const T *__restrict__ a, const T *__restrict__ x,
                                                           T *__restrict__ y, int64_t N, int64_t rlo, int64_t rhi) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *tile = reinterpret_cast<T *>(smem_raw);  // [2][kXR][kXPitch]
    T *xs = tile + 2 * kXR * kXPitch;           // [2][kXC]
    const int t = threadIdx.x;
    const int64_t ngroups = ceil_div(rhi - rlo, kXR), nchunks = ceil_div(N, kXC);
    constexpr int V = 16 / sizeof(T);            // elements per 16-byte copy
    auto load = [&](int64_t r0, int64_t c, int buf) {
        const int64_t q0 = c * kXC;
        T *tb = tile + buf * kXR * kXPitch;
        for (int e = t; e < kXR * (kXC / V); e += kXT) {
            const int rr = e / (kXC / V), cv = e % (kXC / V);
            const int64_t row = r0 + rr, q = q0 + (int64_t)cv * V;
            const bool ok = row < rhi && q < N;
            cp_async16(tb + rr * kXPitch + cv * V, ok ? (const void *)(a + row * N + q) : (const void *)a,
                       ok ? 16 : 0);
        }
        for (int e = t; e < kXC / V; e += kXT) {
            const int64_t q = q0 + (int64_t)e * V;
            cp_async16(xs + buf * kXC + e * V, q < N ? (const void *)(x + q) : (const void *)x, q < N ? 16 : 0);
        }
        cp_async_commit();
    };
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int64_t r0 = rlo + g * kXR;
        const bool live = t < kXR && r0 + t < rhi;
        T acc = live ? y[r0 + t] : T(0);
        load(r0, 0, 0);
        for (int64_t c = 0; c < nchunks; c++) {
            if (c + 1 < nchunks) {
                load(r0, c + 1, (int)((c + 1) & 1));
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            if (live) {
                const T *row = tile + (c & 1) * kXR * kXPitch + t * kXPitch;
                const T *xc = xs + (c & 1) * kXC;
                const int nc = (int)min((int64_t)kXC, N - c * kXC);
                for (int cc = 0; cc < nc; cc++) acc = madd(acc, row[cc], xc[cc]);
            }
            __syncthreads();  // the buffer is refilled two stages on
        }
        if (live) y[r0 + t] = acc;
    }
}

template <typename T>
int launch_exact(void *const *p, int64_t N, int64_t rlo, int64_t rhi, cudaStream_t st) {
    if (N % 2 == 0 && aligned16(p[0]) && aligned16(p[1])) {
        const size_t smem = (size_t)(2 * kXR * kXPitch + 2 * kXC) * sizeof(T);
        int rc = allow_smem((const void *)k_matvec_exact_async<T>, smem);
        if (rc) return rc;
        int dev = 0, sms = 148, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_matvec_exact_async<T>, kXT, smem);
        int64_t blocks = ceil_div(rhi - rlo, kXR);
        const int64_t slots = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
        if (blocks > slots) blocks = slots;
        k_matvec_exact_async<T><<<(unsigned)blocks, kXT, smem, st>>>(
            static_cast<const T *>(p[0]), static_cast<const T *>(p[1]), static_cast<T *>(p[2]), N, rlo, rhi);
        return after_launch("matvec_exact_async");
    }
    const int64_t blocks = ceil_div(rhi - rlo, kExactRows);
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "matvec: grid too large");
    k_matvec_exact<T><<<(unsigned)blocks, kExactRows, 0, st>>>(static_cast<const T *>(p[0]),
                                                               static_cast<const T *>(p[1]),
                                                               static_cast<T *>(p[2]), N, rlo, rhi);
    return after_launch("matvec_exact");
}

}  // namespace

int launch_matvec(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    if (L.s * L.B == 0) return fail(PK_E_DIV0, "matvec: s*B == 0 in dim = N / (s * B)");
    if (L.s < 0 || L.B < 0 || L.N <= 0) return PK_OK;
    const int64_t R = max0(L.N / (L.s * L.B)) * L.s * L.B;
    int64_t rlo, rhi;
    unit_range(L, 0, R, &rlo, &rhi);
    if (rhi <= rlo) return PK_OK;
    if (L.dtype == PK_DTYPE_I32) return launch_t<int>(L, p, st, rlo, rhi);
    if (L.dtype == PK_DTYPE_F32) return launch_t<float>(L, p, st, rlo, rhi);
    if (L.dtype == PK_DTYPE_F64) return launch_exact<double>(p, L.N, rlo, rhi, st);
    if (L.dtype == PK_DTYPE_I64) return launch_exact<long long>(p, L.N, rlo, rhi, st);
    return fail(PK_E_UNSUPPORTED, "matvec: dtype %d", L.dtype);
}

}  // namespace pk
