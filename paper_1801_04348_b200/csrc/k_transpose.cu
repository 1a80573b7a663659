// k_transpose.cu -- matrix transposition (pkg/src/parakern/data/transpose.mfk:13-20):
//   dim0 = N/B0, dim1 = N/(s*B1);  c[i*N + j] = a[j][i]
//   i = v0*B0 + u0 < dim0*B0,  j = (v1*s + k)*B1 + u1 < dim1*s*B1
// A block owns the B0 x (E*B1) tile of c (E = s, or 1 after granularity).
// Words are moved bit-for-bit: 4-byte words (int, float32) or 8-byte words
// (int64, binary64 -- the reference moves Python objects unchanged,
// interp.py:134-142).  HBM-bound: 2 * sizeof(word) bytes per word.
#include "pk_internal.cuh"

namespace pk {
namespace {

// Generic staged tile (any B0, B1, s): a tile of a (TJ rows x TI cols) is read
// row-wise into shared memory, then written to c row-wise.  The shared pitch
// is odd, so column reads hit 32 distinct banks.
template <typename W>
__global__ void __launch_bounds__(1024) k_transpose_staged(const W *__restrict__ a, W *__restrict__ c, int64_t N,
                                                          int64_t ilo, int64_t ihi, int64_t J, int TI, int TJ,
                                                          int64_t ntj) {
    extern __shared__ __align__(16) unsigned char sh_raw[];
    W *sh = reinterpret_cast<W *>(sh_raw);
    const int pitch = TI | 1;
    const int64_t bid = blockIdx.x;
    const int64_t i0 = ilo + (bid / ntj) * TI, j0 = (bid % ntj) * TJ;
    const int ni = (int)min((int64_t)TI, ihi - i0), nj = (int)min((int64_t)TJ, J - j0);
    const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x, by = blockDim.y;
    for (int jj = ty; jj < nj; jj += by) {
        const W *row = a + (j0 + jj) * N + i0;
        for (int ii = tx; ii < ni; ii += bx) sh[jj * pitch + ii] = row[ii];
    }
    __syncthreads();
    for (int ii = ty; ii < ni; ii += by) {
        W *row = c + (i0 + ii) * N + j0;
        for (int jj = tx; jj < nj; jj += bx) row[jj] = sh[jj * pitch + ii];
    }
}

// Staged tile with 128-bit global accesses on both sides (TI, TJ multiples of
// 32, N % V == 0, 16-byte aligned buffers; V = words per 16-byte vector: 4
// for 4-byte words, 2 for 8-byte words).  Load: each thread reads one vector
// of a row of a and scatters it into V consecutive words of the shared row.
// Store: each thread gathers V consecutive shared rows of one column and
// writes one vector of a row of c.  The odd pitch keeps both phases free of
// bank conflicts for 4-byte words (8 threads x 16 B = 128 B per row segment).
template <typename W, int TI, int TJ, int NT>
__global__ void __launch_bounds__(NT) k_transpose_staged_v4(const W *__restrict__ a, W *__restrict__ c, int64_t N,
                                                           int64_t ilo, int64_t ntj) {
    constexpr int V = 16 / sizeof(W);
    constexpr int PITCH = TI + 1;
    __shared__ W sh[TJ * PITCH];
    const int64_t bid = blockIdx.x;
    const int64_t i0 = ilo + (bid / ntj) * TI, j0 = (bid % ntj) * TJ;
    const int tid = threadIdx.x;
    constexpr int WV = TI / V;              // vectors per row of the a tile
    constexpr int LOADS = TJ * WV / NT;     // per thread
    int4 v[LOADS];
#pragma unroll
    for (int r = 0; r < LOADS; r++) {
        const int q = tid + r * NT;
        const int jj = q / WV, iv = q % WV;
        v[r] = ld_stream(reinterpret_cast<const int4 *>(a + (j0 + jj) * N + i0) + iv);
    }
#pragma unroll
    for (int r = 0; r < LOADS; r++) {
        const int q = tid + r * NT;
        const int jj = q / WV, iv = q % WV;
        const W *w = reinterpret_cast<const W *>(&v[r]);
        W *d = sh + jj * PITCH + V * iv;
#pragma unroll
        for (int t = 0; t < V; t++) d[t] = w[t];
    }
    __syncthreads();
    constexpr int JV = TJ / V;              // vectors per row of the c tile
    constexpr int STORES = TI * JV / NT;
#pragma unroll
    for (int r = 0; r < STORES; r++) {
        const int q = tid + r * NT;
        const int ii = q / JV, jv = q % JV;
        const W *s0 = sh + (V * jv) * PITCH + ii;
        int4 o;
        W *w = reinterpret_cast<W *>(&o);
#pragma unroll
        for (int t = 0; t < V; t++) w[t] = s0[t * PITCH];
        st_stream(reinterpret_cast<int4 *>(c + (i0 + ii) * N + j0) + jv, o);
    }
}

// caching-off: threads run along j so the writes to c are coalesced; the
// reads of a walk a column (stride N) and rely on L1/L2 sector reuse.
template <typename W>
__global__ void __launch_bounds__(1024) k_transpose_direct(const W *__restrict__ a, W *__restrict__ c, int64_t N,
                                                          int64_t ilo, int64_t ihi, int64_t J,
                                                          int TI, int TJ, int64_t ntj) {
    const int64_t bid = blockIdx.x;
    const int64_t i0 = ilo + (bid / ntj) * TI, j0 = (bid % ntj) * TJ;
    const int ni = (int)min((int64_t)TI, ihi - i0), nj = (int)min((int64_t)TJ, J - j0);
    const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x, by = blockDim.y;
    for (int ii = ty; ii < ni; ii += by)
        for (int jj = tx; jj < nj; jj += bx) c[(i0 + ii) * N + j0 + jj] = a[(j0 + jj) * N + i0 + ii];
}

template <typename W, int TI, int TJ>
int launch_v4(const W *a, W *c, int64_t N, int64_t ilo, int64_t ihi, int64_t J, cudaStream_t st) {
    const int64_t nti = (ihi - ilo) / TI, ntj = J / TJ;
    const int64_t blocks = nti * ntj;
    if (blocks <= 0) return PK_OK;
    k_transpose_staged_v4<W, TI, TJ, 256><<<(unsigned)blocks, 256, 0, st>>>(a, c, N, ilo, ntj);
    return after_launch("transpose_v4");
}

template <typename W>
int launch_w(const pk_launch_t &L, void *const *p, cudaStream_t st, int64_t ilo, int64_t ihi, int64_t J, int TI,
             int TJ) {
    constexpr int V = 16 / sizeof(W);
    const W *a = static_cast<const W *>(p[0]);
    W *c = static_cast<W *>(p[1]);
    const bool vec_ok = L.N % V == 0 && aligned16(a) && aligned16(c) && (ihi - ilo) % TI == 0 &&
                        J % TJ == 0 && ilo % V == 0;
    if (L.variant == PK_VARIANT_STAGED && vec_ok) {
        if (TI == 32 && TJ == 32) return launch_v4<W, 32, 32>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 64 && TJ == 64) return launch_v4<W, 64, 64>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 32 && TJ == 64) return launch_v4<W, 32, 64>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 64 && TJ == 32) return launch_v4<W, 64, 32>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 128 && TJ == 32) return launch_v4<W, 128, 32>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 32 && TJ == 128) return launch_v4<W, 32, 128>(a, c, L.N, ilo, ihi, J, st);
    }
    // Generic geometry: the B0 x B1 block of the program, laid out 32 wide so
    // every warp touches whole 128-byte rows where the tile allows.
    int64_t nthreads = L.B0 * L.B1;
    if (nthreads > 1024) nthreads = 1024;
    dim3 block;
    if (nthreads >= 32 && nthreads % 32 == 0) block = dim3(32, (unsigned)(nthreads / 32));
    else block = dim3((unsigned)nthreads, 1);
    const int64_t nti = ceil_div(ihi - ilo, TI), ntj = ceil_div(J, TJ);
    const int64_t blocks = nti * ntj;
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "transpose: grid too large");
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = (size_t)TJ * (size_t)(TI | 1) * sizeof(W);
        int rc = allow_smem((const void *)k_transpose_staged<W>, smem);
        if (rc) return rc;
        k_transpose_staged<W><<<(unsigned)blocks, block, smem, st>>>(a, c, L.N, ilo, ihi, J, TI, TJ, ntj);
    } else {
        k_transpose_direct<W><<<(unsigned)blocks, block, 0, st>>>(a, c, L.N, ilo, ihi, J, TI, TJ, ntj);
    }
    return after_launch("transpose");
}

}  // namespace

int launch_transpose(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    if (L.B0 == 0) return fail(PK_E_DIV0, "transpose: B0 == 0 in dim0 = N / B0");
    if (L.s * L.B1 == 0) return fail(PK_E_DIV0, "transpose: s*B1 == 0 in dim1 = N / (s * B1)");
    if (L.B0 < 0 || L.B1 < 0 || L.s < 0 || L.N <= 0) return PK_OK;
    const int64_t I = max0(L.N / L.B0) * L.B0;
    const int64_t J = max0(L.N / (L.s * L.B1)) * L.s * L.B1;
    int64_t ilo, ihi;
    unit_range(L, 0, I, &ilo, &ihi);
    if (ihi <= ilo || J <= 0) return PK_OK;
    const int64_t TI64 = L.B0, TJ64 = elems(L) * L.B1;
    if (TI64 * TJ64 > (1 << 26)) return fail(PK_E_UNSUPPORTED, "transpose: tile too large");
    if (elem_bytes(L) == 8) return launch_w<uint64_t>(L, p, st, ilo, ihi, J, (int)TI64, (int)TJ64);
    return launch_w<uint32_t>(L, p, st, ilo, ihi, J, (int)TI64, (int)TJ64);
}

}  // namespace pk
