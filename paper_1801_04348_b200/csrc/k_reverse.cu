// k_reverse.cu -- array reversal (SURVEY App. A.2 reverse.mfk):
//   dim = N/(s*B);  c[N-1-p] = a[p] for p < dim*s*B
// A block owns one tile of E*B consecutive input words (E = s, or 1 once
// granularity removed the s loop) and writes the mirrored output tile, which
// is also contiguous.  HBM-bound: 8 bytes of algorithmic traffic per word.
#include "pk_internal.cuh"

namespace pk {
namespace {

// cache(a) kept: the tile is staged in shared memory with 128-bit accesses on
// both sides, then written back reversed.  VEC requires 16-byte alignment of
// the tile start in a and of the mirrored tile start in c.
template <bool VEC>
__global__ void __launch_bounds__(1024) k_reverse_staged(const int *__restrict__ a,
                                                        int *__restrict__ c, int64_t N,
                                                        int64_t lo, int64_t hi, int tile) {
    extern __shared__ __align__(16) int sh[];
    const int64_t base = lo + (int64_t)blockIdx.x * tile;
    const int n = (int)min((int64_t)tile, hi - base);
    const int tid = threadIdx.x, nt = blockDim.x;
    if (VEC && n == tile) {
        const int4 *a4 = reinterpret_cast<const int4 *>(a + base);
        int4 *s4 = reinterpret_cast<int4 *>(sh);
        const int n4 = tile >> 2;
#pragma unroll 4
        for (int q = tid; q < n4; q += nt) s4[q] = ld_stream(a4 + q);
        __syncthreads();
        int4 *c4 = reinterpret_cast<int4 *>(c + (N - base - tile));
#pragma unroll 4
        for (int q = tid; q < n4; q += nt) {
            int4 v = s4[n4 - 1 - q];
            st_stream(c4 + q, make_int4(v.w, v.z, v.y, v.x));
        }
    } else {
#pragma unroll 4
        for (int q = tid; q < n; q += nt) sh[q] = a[base + q];
        __syncthreads();
        const int64_t o = N - base - n;  // c[N-1-p], p in [base, base+n)
#pragma unroll 4
        for (int q = tid; q < n; q += nt) c[o + q] = sh[n - 1 - q];
    }
}

// caching-off: every thread moves its words straight from a to c.  With VEC
// each thread reverses one int4 in registers (needs N % 4 == 0).
template <bool VEC>
__global__ void __launch_bounds__(1024) k_reverse_direct(const int *__restrict__ a,
                                                        int *__restrict__ c, int64_t N,
                                                        int64_t lo, int64_t hi, int tile) {
    const int64_t base = lo + (int64_t)blockIdx.x * tile;
    const int n = (int)min((int64_t)tile, hi - base);
    const int tid = threadIdx.x, nt = blockDim.x;
    if (VEC && n == tile) {
        const int n4 = tile >> 2;
#pragma unroll 4
        for (int q = tid; q < n4; q += nt) {
            const int64_t p = base + 4 * (int64_t)q;
            int4 v = ld_stream(reinterpret_cast<const int4 *>(a + p));
            st_stream(reinterpret_cast<int4 *>(c + (N - 4 - p)), make_int4(v.w, v.z, v.y, v.x));
        }
    } else {
#pragma unroll 4
        for (int q = tid; q < n; q += nt) c[N - 1 - (base + q)] = a[base + q];
    }
}

}  // namespace

int launch_reverse(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    if (L.s * L.B == 0) return fail(PK_E_DIV0, "reverse: s*B == 0 in dim = N / (s * B)");
    if (L.s < 0 || L.B < 0 || L.N <= 0) return PK_OK;  // empty meta_for ranges
    const int64_t dim = L.N / (L.s * L.B);
    const int64_t P = max0(dim) * L.s * L.B;
    int64_t lo, hi;
    unit_range(L, 0, P, &lo, &hi);
    if (hi <= lo) return PK_OK;
    const int64_t tile64 = elems(L) * L.B;
    if (tile64 > (1 << 30)) return fail(PK_E_UNSUPPORTED, "reverse: tile of %lld words", (long long)tile64);
    const int tile = (int)tile64;
    const int nt = (int)(L.B < 1024 ? L.B : 1024);
    const int64_t blocks = ceil_div(hi - lo, tile);
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "reverse: grid too large");
    const int *a = static_cast<const int *>(p[0]);
    int *c = static_cast<int *>(p[1]);
    const bool vec = (tile % 4 == 0) && (lo % 4 == 0) && (L.N % 4 == 0) && aligned16(a) && aligned16(c);
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = (size_t)tile * sizeof(int);
        const void *k = vec ? (const void *)k_reverse_staged<true> : (const void *)k_reverse_staged<false>;
        int rc = allow_smem(k, smem);
        if (rc) return rc;
        if (vec)
            k_reverse_staged<true><<<(unsigned)blocks, nt, smem, st>>>(a, c, L.N, lo, hi, tile);
        else
            k_reverse_staged<false><<<(unsigned)blocks, nt, smem, st>>>(a, c, L.N, lo, hi, tile);
    } else {
        if (vec)
            k_reverse_direct<true><<<(unsigned)blocks, nt, 0, st>>>(a, c, L.N, lo, hi, tile);
        else
            k_reverse_direct<false><<<(unsigned)blocks, nt, 0, st>>>(a, c, L.N, lo, hi, tile);
    }
    return after_launch("reverse");
}

}  // namespace pk
