// k_reverse.cu -- array reversal (SURVEY App. A.2 reverse.mfk):
//   dim = N/(s*B);  c[N-1-p] = a[p] for p < dim*s*B
// A block owns one tile of E*B consecutive input words (E = s, or 1 once
// granularity removed the s loop) and writes the mirrored output tile, which
// is also contiguous.  HBM-bound: 2 * sizeof(word) bytes of algorithmic
// traffic per word.  Words are moved bit-for-bit: 4-byte words for the DSL's
// int and float32, 8-byte words for int64 / binary64 (the reference's _put
// stores the fetched Python object unchanged, interp.py:134-142,189-206).
#include "pk_internal.cuh"

namespace pk {
namespace {

// Reverse the words inside one 16-byte vector: 4 x 32-bit or 2 x 64-bit.
template <typename W> __device__ __forceinline__ int4 rev_vec(const int4 &v);
template <> __device__ __forceinline__ int4 rev_vec<uint32_t>(const int4 &v) { return make_int4(v.w, v.z, v.y, v.x); }
template <> __device__ __forceinline__ int4 rev_vec<uint64_t>(const int4 &v) { return make_int4(v.z, v.w, v.x, v.y); }

// cache(a) kept: the tile is staged in shared memory with 128-bit accesses on
// both sides, then written back reversed.  VEC requires 16-byte alignment of
// the tile start in a and of the mirrored tile start in c.
template <typename W, bool VEC>
__global__ void __launch_bounds__(1024) k_reverse_staged(const W *__restrict__ a, W *__restrict__ c, int64_t N,
                                                        int64_t lo, int64_t hi, int tile) {
    extern __shared__ __align__(16) unsigned char sh_raw[];
    W *sh = reinterpret_cast<W *>(sh_raw);
    constexpr int V = 16 / sizeof(W);  // words per vector
    const int64_t base = lo + (int64_t)blockIdx.x * tile;
    const int n = (int)min((int64_t)tile, hi - base);
    const int tid = threadIdx.x, nt = blockDim.x;
    if (VEC && n == tile) {
        const int4 *a4 = reinterpret_cast<const int4 *>(a + base);
        int4 *s4 = reinterpret_cast<int4 *>(sh);
        const int n4 = tile / V;
#pragma unroll 4
        for (int q = tid; q < n4; q += nt) s4[q] = ld_stream(a4 + q);
        __syncthreads();
        int4 *c4 = reinterpret_cast<int4 *>(c + (N - base - tile));
#pragma unroll 4
        for (int q = tid; q < n4; q += nt) st_stream(c4 + q, rev_vec<W>(s4[n4 - 1 - q]));
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
// each thread reverses one 16-byte vector in registers (needs N % V == 0).
template <typename W, bool VEC>
__global__ void __launch_bounds__(1024) k_reverse_direct(const W *__restrict__ a, W *__restrict__ c, int64_t N,
                                                        int64_t lo, int64_t hi, int tile) {
    constexpr int V = 16 / sizeof(W);
    const int64_t base = lo + (int64_t)blockIdx.x * tile;
    const int n = (int)min((int64_t)tile, hi - base);
    const int tid = threadIdx.x, nt = blockDim.x;
    if (VEC && n == tile) {
        const int n4 = tile / V;
#pragma unroll 4
        for (int q = tid; q < n4; q += nt) {
            const int64_t p = base + V * (int64_t)q;
            int4 v = ld_stream(reinterpret_cast<const int4 *>(a + p));
            st_stream(reinterpret_cast<int4 *>(c + (N - V - p)), rev_vec<W>(v));
        }
    } else {
#pragma unroll 4
        for (int q = tid; q < n; q += nt) c[N - 1 - (base + q)] = a[base + q];
    }
}

template <typename W>
int launch_w(const pk_launch_t &L, void *const *p, cudaStream_t st, int64_t lo, int64_t hi, int tile) {
    constexpr int V = 16 / sizeof(W);
    const int nt = (int)(L.B < 1024 ? L.B : 1024);
    const int64_t blocks = ceil_div(hi - lo, tile);
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "reverse: grid too large");
    const W *a = static_cast<const W *>(p[0]);
    W *c = static_cast<W *>(p[1]);
    const bool vec = (tile % V == 0) && (lo % V == 0) && (L.N % V == 0) && aligned16(a) && aligned16(c);
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = (size_t)tile * sizeof(W);
        const void *k = vec ? (const void *)k_reverse_staged<W, true> : (const void *)k_reverse_staged<W, false>;
        int rc = allow_smem(k, smem);
        if (rc) return rc;
        if (vec)
            k_reverse_staged<W, true><<<(unsigned)blocks, nt, smem, st>>>(a, c, L.N, lo, hi, tile);
        else
            k_reverse_staged<W, false><<<(unsigned)blocks, nt, smem, st>>>(a, c, L.N, lo, hi, tile);
    } else {
        if (vec)
            k_reverse_direct<W, true><<<(unsigned)blocks, nt, 0, st>>>(a, c, L.N, lo, hi, tile);
        else
            k_reverse_direct<W, false><<<(unsigned)blocks, nt, 0, st>>>(a, c, L.N, lo, hi, tile);
    }
    return after_launch("reverse");
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
    if (elem_bytes(L) == 8) return launch_w<uint64_t>(L, p, st, lo, hi, (int)tile64);
    return launch_w<uint32_t>(L, p, st, lo, hi, (int)tile64);
}

}  // namespace pk
