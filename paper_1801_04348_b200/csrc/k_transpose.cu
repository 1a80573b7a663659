// k_transpose.cu -- matrix transposition (pkg/src/parakern/data/transpose.mfk:13-20):
//   dim0 = N/B0, dim1 = N/(s*B1);  c[i*N + j] = a[j][i]
//   i = v0*B0 + u0 < dim0*B0,  j = (v1*s + k)*B1 + u1 < dim1*s*B1
// A block owns the B0 x (E*B1) tile of c (E = s, or 1 after granularity).
// 32-bit words are moved bit-for-bit.  HBM-bound: 8 bytes per word.
#include "pk_internal.cuh"

namespace pk {
namespace {

// Generic staged tile (any B0, B1, s): a tile of a (TJ rows x TI cols) is read
// row-wise into shared memory, then written to c row-wise.  The shared pitch
// is odd, so column reads hit 32 distinct banks.
__global__ void __launch_bounds__(1024) k_transpose_staged(const uint32_t *__restrict__ a,
                                                          uint32_t *__restrict__ c, int64_t N,
                                                          int64_t ilo, int64_t ihi, int64_t J,
                                                          int TI, int TJ, int64_t ntj) {
    extern __shared__ uint32_t sh[];
    const int pitch = TI | 1;
    const int64_t bid = blockIdx.x;
    const int64_t i0 = ilo + (bid / ntj) * TI, j0 = (bid % ntj) * TJ;
    const int ni = (int)min((int64_t)TI, ihi - i0), nj = (int)min((int64_t)TJ, J - j0);
    const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x, by = blockDim.y;
    for (int jj = ty; jj < nj; jj += by) {
        const uint32_t *row = a + (j0 + jj) * N + i0;
        for (int ii = tx; ii < ni; ii += bx) sh[jj * pitch + ii] = row[ii];
    }
    __syncthreads();
    for (int ii = ty; ii < ni; ii += by) {
        uint32_t *row = c + (i0 + ii) * N + j0;
        for (int jj = tx; jj < nj; jj += bx) row[jj] = sh[jj * pitch + ii];
    }
}

// Staged tile with 128-bit global accesses on both sides (TI, TJ multiples of
// 32, N % 4 == 0, 16-byte aligned buffers).  Load: each thread reads one int4
// of a row of a and scatters it into 4 consecutive words of the shared row.
// Store: each thread gathers 4 consecutive shared rows of one column and
// writes one int4 of a row of c.  With an odd pitch both phases are
// bank-conflict-free (8 threads x int4 = 128 B per row segment).
template <int TI, int TJ, int NT>
__global__ void __launch_bounds__(NT) k_transpose_staged_v4(const uint32_t *__restrict__ a,
                                                           uint32_t *__restrict__ c, int64_t N,
                                                           int64_t ilo, int64_t ntj) {
    constexpr int PITCH = TI + 1;
    __shared__ uint32_t sh[TJ * PITCH];
    const int64_t bid = blockIdx.x;
    const int64_t i0 = ilo + (bid / ntj) * TI, j0 = (bid % ntj) * TJ;
    const int tid = threadIdx.x;
    constexpr int W4 = TI / 4;              // int4 per row of the a tile
    constexpr int LOADS = TJ * W4 / NT;     // per thread
    int4 v[LOADS];
#pragma unroll
    for (int r = 0; r < LOADS; r++) {
        const int q = tid + r * NT;
        const int jj = q / W4, i4 = q % W4;
        v[r] = ld_stream(reinterpret_cast<const int4 *>(a + (j0 + jj) * N + i0) + i4);
    }
#pragma unroll
    for (int r = 0; r < LOADS; r++) {
        const int q = tid + r * NT;
        const int jj = q / W4, i4 = q % W4;
        uint32_t *d = sh + jj * PITCH + 4 * i4;
        d[0] = v[r].x; d[1] = v[r].y; d[2] = v[r].z; d[3] = v[r].w;
    }
    __syncthreads();
    constexpr int J4 = TJ / 4;              // int4 per row of the c tile
    constexpr int STORES = TI * J4 / NT;
#pragma unroll
    for (int r = 0; r < STORES; r++) {
        const int q = tid + r * NT;
        const int ii = q / J4, j4 = q % J4;
        const uint32_t *s0 = sh + (4 * j4) * PITCH + ii;
        int4 o = make_int4((int)s0[0], (int)s0[PITCH], (int)s0[2 * PITCH], (int)s0[3 * PITCH]);
        st_stream(reinterpret_cast<int4 *>(c + (i0 + ii) * N + j0) + j4, o);
    }
}

// caching-off: threads run along j so the writes to c are coalesced; the
// reads of a walk a column (stride N) and rely on L1/L2 sector reuse.
__global__ void __launch_bounds__(1024) k_transpose_direct(const uint32_t *__restrict__ a,
                                                          uint32_t *__restrict__ c, int64_t N,
                                                          int64_t ilo, int64_t ihi, int64_t J,
                                                          int TI, int TJ, int64_t ntj) {
    const int64_t bid = blockIdx.x;
    const int64_t i0 = ilo + (bid / ntj) * TI, j0 = (bid % ntj) * TJ;
    const int ni = (int)min((int64_t)TI, ihi - i0), nj = (int)min((int64_t)TJ, J - j0);
    const int tx = threadIdx.x, ty = threadIdx.y, bx = blockDim.x, by = blockDim.y;
    for (int ii = ty; ii < ni; ii += by)
        for (int jj = tx; jj < nj; jj += bx) c[(i0 + ii) * N + j0 + jj] = a[(j0 + jj) * N + i0 + ii];
}

template <int TI, int TJ>
int launch_v4(const uint32_t *a, uint32_t *c, int64_t N, int64_t ilo, int64_t ihi, int64_t J,
              cudaStream_t st) {
    const int64_t nti = (ihi - ilo) / TI, ntj = J / TJ;
    const int64_t blocks = nti * ntj;
    if (blocks <= 0) return PK_OK;
    k_transpose_staged_v4<TI, TJ, 256><<<(unsigned)blocks, 256, 0, st>>>(a, c, N, ilo, ntj);
    return after_launch("transpose_v4");
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
    const int TI = (int)TI64, TJ = (int)TJ64;
    const uint32_t *a = static_cast<const uint32_t *>(p[0]);
    uint32_t *c = static_cast<uint32_t *>(p[1]);
    const bool vec_ok = L.N % 4 == 0 && aligned16(a) && aligned16(c) && (ihi - ilo) % TI == 0 &&
                        J % TJ == 0 && ilo % 4 == 0;
    if (L.variant == PK_VARIANT_STAGED && vec_ok) {
        if (TI == 32 && TJ == 32) return launch_v4<32, 32>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 64 && TJ == 64) return launch_v4<64, 64>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 32 && TJ == 64) return launch_v4<32, 64>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 64 && TJ == 32) return launch_v4<64, 32>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 128 && TJ == 32) return launch_v4<128, 32>(a, c, L.N, ilo, ihi, J, st);
        if (TI == 32 && TJ == 128) return launch_v4<32, 128>(a, c, L.N, ilo, ihi, J, st);
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
        const size_t smem = (size_t)TJ * (size_t)(TI | 1) * sizeof(uint32_t);
        int rc = allow_smem((const void *)k_transpose_staged, smem);
        if (rc) return rc;
        k_transpose_staged<<<(unsigned)blocks, block, smem, st>>>(a, c, L.N, ilo, ihi, J, TI, TJ, ntj);
    } else {
        k_transpose_direct<<<(unsigned)blocks, block, 0, st>>>(a, c, L.N, ilo, ihi, J, TI, TJ, ntj);
    }
    return after_launch("transpose");
}

}  // namespace pk
