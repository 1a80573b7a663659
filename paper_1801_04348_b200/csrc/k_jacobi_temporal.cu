// k_jacobi_temporal.cu -- temporally blocked 1-D Jacobi (PK_FLAG_TEMPORAL),
// an optional variant reported beside the per-step leaf.
//
// The program (pkg/src/parakern/data/jacobi.mfk:9-25) runs T sweeps, each a
// full pass over HBM.  Here one pass advances h steps: a block loads its
// tile plus h halo points of the latest half into shared memory, iterates h
// sweeps there (the exact, shrinking-valid-region ghost-zone scheme) and
// writes only the last sweep's values.  HBM traffic per point drops from
// 8 B per step to ~8 B per h steps; the arithmetic is the per-step kernels'
// (same exact sums, same truncating division), so results are bit-identical.
//
// Which half holds what.  Step t reads half s(t) and writes half d(t)
// (t even: d = lower half).  With h odd, d(t0+h-1) != s(t0), so a pass never
// writes the half other blocks read from.  A multi-step pass leaves the
// other half stale (it would have held step t0+h-2), which no later pass
// reads; the driver therefore ends with a single ordinary sweep, after
// which both halves hold exactly the reference's final state (step T-1 in
// d(T-1), step T-2 in d(T-2)).  Positions outside 1..P (the two boundary
// points and any uncovered tail) are never written by the program; their
// value in "half d(t)" is read from that half in global memory.
#include "pk_internal.cuh"

namespace pk {
namespace {

template <bool WIDE>
__device__ __forceinline__ int avg3(int a, int b, int c) {
    if (WIDE) return (int)(((long long)a + (long long)b + (long long)c) / 3);
    return (a + b + c) / 3;
}

// One h-step pass over tiles of W outputs.  Window of a tile: positions
// [ws, ws + WN), ws = 4-aligned start at or below xs - h.
template <bool WIDE>
__device__ void tb_tile(const int *__restrict__ src, int *__restrict__ dst, const int *__restrict__ half0,
                        const int *__restrict__ half1, int64_t lo, int64_t hi, int64_t P, int64_t N, int64_t t0,
                        int h, int64_t xs, int W, int WN, int *buf0, int *buf1) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int64_t ws = (xs - h) & ~(int64_t)3;
    // ---- load the window of the latest half (src): batched 64-bit loads for
    // interior windows (ws even, halves 8-byte aligned), guarded words at the ends
    const bool interior = ws >= 0 && ws + WN <= N && ((reinterpret_cast<uintptr_t>(src) & 7u) == 0);
    if (interior) {
        const int2 *g2 = reinterpret_cast<const int2 *>(src + ws);
        int2 *b2 = reinterpret_cast<int2 *>(buf0);
        const int w2 = WN >> 1;
        for (int i = tid; i < w2; i += 4 * nt) {
            int2 v[4];
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (i + u * nt < w2) v[u] = g2[i + u * nt];
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (i + u * nt < w2) b2[i + u * nt] = v[u];
        }
    } else {
        for (int i = tid; i < WN; i += nt) {
            const int64_t x = ws + i;
            buf0[i] = (x >= 0 && x < N) ? src[x] : 0;
        }
    }
    __syncthreads();
    const int quads = WN >> 2;
    const int wlanes = min(32, nt - (tid - lane));
    const unsigned wmask = wlanes == 32 ? 0xffffffffu : ((1u << wlanes) - 1u);
    int *cur = buf0, *nxt = buf1;
    for (int k = 0; k < h; k++) {
        const int64_t t = t0 + k;
        const int *fixed_half = (t % 2 == 0) ? half0 : half1;  // d(t)
        for (int pb = tid - lane; pb < quads; pb += nt) {
            const int p = pb + lane;
            const bool act = p < quads;
            const int4 c = act ? reinterpret_cast<const int4 *>(cur)[p] : make_int4(0, 0, 0, 0);
            int l = __shfl_up_sync(wmask, c.w, 1);
            int r = __shfl_down_sync(wmask, c.x, 1);
            if (!act) continue;
            if (lane == 0) l = p > 0 ? cur[4 * p - 1] : 0;
            if (lane + 1 == wlanes || p + 1 == quads) r = p + 1 < quads ? cur[4 * p + 4] : 0;
            int4 o = make_int4(avg3<WIDE>(l, c.x, c.y), avg3<WIDE>(c.x, c.y, c.z), avg3<WIDE>(c.y, c.z, c.w),
                               avg3<WIDE>(c.z, c.w, r));
            const int64_t x = ws + 4 * (int64_t)p;
            if (x < 1 || x + 3 > P) {  // positions the program never writes keep half d(t)'s value
                int *ov = reinterpret_cast<int *>(&o);
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const int64_t xe = x + e;
                    if (xe < 1 || xe > P) ov[e] = (xe >= 0 && xe < N) ? fixed_half[xe] : 0;
                }
            }
            reinterpret_cast<int4 *>(nxt)[p] = o;
        }
        __syncthreads();
        int *tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
    // ---- write the last step's values of this tile (interior positions only)
    int64_t wlo = max(max(xs, lo), (int64_t)1);
    const int64_t whi = min(min(xs + W, hi), P + 1);
    if ((reinterpret_cast<uintptr_t>(dst) & 7u) == 0) {
        // 64-bit stores of pairs (x, x+1), x even (ws is even, so the shared side aligns too)
        if ((wlo & 1) && wlo < whi) {
            if (tid == 0) dst[wlo] = cur[wlo - ws];
            wlo++;
        }
        for (int64_t x = wlo + 2 * tid; x < whi; x += 2 * nt) {
            if (x + 1 < whi)
                *reinterpret_cast<int2 *>(dst + x) = *reinterpret_cast<const int2 *>(cur + (x - ws));
            else
                dst[x] = cur[x - ws];
        }
    } else {
        for (int64_t x = wlo + tid; x < whi; x += nt) dst[x] = cur[x - ws];
    }
}

__global__ void __launch_bounds__(256) k_jacobi1d_temporal(const int *__restrict__ src, int *__restrict__ dst,
                                                          const int *__restrict__ half0,
                                                          const int *__restrict__ half1, int64_t lo, int64_t hi,
                                                          int64_t P, int64_t N, int64_t t0, int h, int64_t x0,
                                                          int W, int WN, int64_t ntiles, const int *flag,
                                                          int mode) {
    extern __shared__ __align__(16) int sh[];
    int *buf0 = sh, *buf1 = sh + WN;
    const bool narrow = mode == 2 ? (*flag != 0) : (mode == 1);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t xs = x0 + tile * W;
        if (narrow)
            tb_tile<false>(src, dst, half0, half1, lo, hi, P, N, t0, h, xs, W, WN, buf0, buf1);
        else
            tb_tile<true>(src, dst, half0, half1, lo, hi, P, N, t0, h, xs, W, WN, buf0, buf1);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Register-resident pass (the default; the shared-memory pass above remains
// for layouts it does not take and under PK_FLAG_GENERIC).  Each warp owns a
// 512-position window [ws, ws + 512) of the latest half: lane l holds quads
// l, l+32, l+64, l+96 (coalesced 16-byte loads), and a step needs only the
// .w of the previous lane's quad and the .x of the next lane's (8 shuffles
// per 16 values; across the lane-31/lane-0 seam the neighbour quad is the
// previous / next j).  The h steps run entirely in registers: no shared
// memory, no barriers.  Values near the window ends go stale one position
// per step, so only [ws + 16, ws + 496) -- 480 outputs per warp, h <= 16 --
// is stored.  Positions the program never writes (x < 1, x > P) take half
// d(t)'s value at every step, as in tb_tile; only the one or two warps whose
// window reaches them take that path (warp-uniform branch).
#ifndef PK_RT_Q
#define PK_RT_Q 4
#endif
#ifndef PK_RT_MINB
#define PK_RT_MINB 4
#endif
constexpr int kRtQ = PK_RT_Q;             // quads per lane
constexpr int kRtSpan = 32 * 4 * kRtQ;    // 512 positions per warp window
constexpr int kRtHalo = 16;               // positions of halo on each side (h <= 16)
constexpr int kRtOut = kRtSpan - 2 * kRtHalo;  // 480 outputs per warp

template <bool WIDE, bool EDGE>
__device__ __forceinline__ void rt_warp(const int *__restrict__ src, int *__restrict__ dst,
                                        const int *__restrict__ half0, const int *__restrict__ half1, int64_t lo,
                                        int64_t hi, int64_t P, int64_t N, int64_t t0, int h, int64_t ws) {
    const int lane = threadIdx.x & 31;
    int4 q[kRtQ];
#pragma unroll
    for (int j = 0; j < kRtQ; j++) {
        const int64_t x = ws + 4 * (j * 32 + lane);
        if (!EDGE) {
            q[j] = __ldg(reinterpret_cast<const int4 *>(src + x));
        } else {
            int v[4];
#pragma unroll
            for (int e = 0; e < 4; e++) v[e] = (x + e >= 0 && x + e < N) ? __ldg(src + x + e) : 0;
            q[j] = make_int4(v[0], v[1], v[2], v[3]);
        }
    }
    for (int k = 0; k < h; k++) {
        int lw[kRtQ], rx[kRtQ];
#pragma unroll
        for (int j = 0; j < kRtQ; j++) {
            lw[j] = __shfl_sync(0xffffffffu, q[j].w, (lane + 31) & 31);
            rx[j] = __shfl_sync(0xffffffffu, q[j].x, (lane + 1) & 31);
        }
#pragma unroll
        for (int j = 0; j < kRtQ; j++) {
            // lane 0's left neighbour is lane 31's quad of the previous j, lane 31's
            // right neighbour lane 0's quad of the next j (outside the window: stale)
            const int l = lane == 0 ? (j > 0 ? lw[j - 1] : 0) : lw[j];
            const int r = lane == 31 ? (j + 1 < kRtQ ? rx[j + 1] : 0) : rx[j];
            int4 o = make_int4(avg3<WIDE>(l, q[j].x, q[j].y), avg3<WIDE>(q[j].x, q[j].y, q[j].z),
                               avg3<WIDE>(q[j].y, q[j].z, q[j].w), avg3<WIDE>(q[j].z, q[j].w, r));
            if (EDGE) {
                const int64_t x = ws + 4 * (j * 32 + lane);
                if (x < 1 || x + 3 > P) {  // positions the program never writes keep half d(t)'s value
                    const int *fh = ((t0 + k) % 2 == 0) ? half0 : half1;
                    auto fix = [&](int v, int64_t xe) {
                        return (xe >= 1 && xe <= P) ? v : (xe >= 0 && xe < N) ? fh[xe] : 0;
                    };
                    o = make_int4(fix(o.x, x), fix(o.y, x + 1), fix(o.z, x + 2), fix(o.w, x + 3));
                }
            }
            q[j] = o;
        }
    }
    // store [ws + 16, ws + 496) clipped to [lo, hi) and 1..P; dst + x is 8-byte aligned for even x - ws
    const int64_t slo = max(max(ws + kRtHalo, lo), (int64_t)1), shi = min(min(ws + kRtSpan - kRtHalo, hi), P + 1);
#pragma unroll
    for (int j = 0; j < kRtQ; j++) {
        const int64_t x = ws + 4 * (j * 32 + lane);
        if (!EDGE && x >= slo && x + 4 <= shi) {
            *reinterpret_cast<int2 *>(dst + x) = make_int2(q[j].x, q[j].y);
            *reinterpret_cast<int2 *>(dst + x + 2) = make_int2(q[j].z, q[j].w);
        } else {
            if (x >= slo && x < shi) dst[x] = q[j].x;
            if (x + 1 >= slo && x + 1 < shi) dst[x + 1] = q[j].y;
            if (x + 2 >= slo && x + 2 < shi) dst[x + 2] = q[j].z;
            if (x + 3 >= slo && x + 3 < shi) dst[x + 3] = q[j].w;
        }
    }
}

__global__ void __launch_bounds__(256, PK_RT_MINB) k_jacobi1d_rtemporal(const int *__restrict__ src, int *__restrict__ dst,
                                                           const int *__restrict__ half0,
                                                           const int *__restrict__ half1, int64_t lo, int64_t hi,
                                                           int64_t P, int64_t N, int64_t t0, int h, int64_t xs0,
                                                           int64_t nwarps, const int *flag, int mode) {
    const int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (w >= nwarps) return;  // warp-uniform
    bool narrow = mode == 1;
    if (mode == 2) {
        int v;
        asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        narrow = v != 0;
    }
    const int64_t ws = xs0 + w * kRtOut - kRtHalo;  // 16-byte aligned in src
    // interior: the whole window inside 1..P (no fixed positions, no guards)
    // and every output position stored
    const bool interior = ws >= 1 && ws + kRtSpan <= P + 1 && ws + kRtHalo >= lo && ws + kRtSpan - kRtHalo <= hi;
    if (interior) {
        if (narrow)
            rt_warp<false, false>(src, dst, half0, half1, lo, hi, P, N, t0, h, ws);
        else
            rt_warp<true, false>(src, dst, half0, half1, lo, hi, P, N, t0, h, ws);
    } else {
        if (narrow)
            rt_warp<false, true>(src, dst, half0, half1, lo, hi, P, N, t0, h, ws);
        else
            rt_warp<true, true>(src, dst, half0, half1, lo, hi, P, N, t0, h, ws);
    }
}

}  // namespace

// h-step pass starting at step t0 (h odd) over positions [lo, hi) of the
// interior 1..P, reading the half that holds step t0-1 and writing d(t0+h-1).
int jacobi1d_temporal_pass(const pk_launch_t &L, int *a, int64_t lo, int64_t hi, int64_t P, int64_t t0, int h,
                           const int *flag, int mode, cudaStream_t st) {
    if (hi <= lo) return PK_OK;
    int *half0 = a, *half1 = a + L.N;
    const int *src = (t0 % 2 == 0) ? half1 : half0;            // s(t0) = d(t0 - 1)
    int *dst = ((t0 + h - 1) % 2 == 0) ? half0 : half1;        // d(t0 + h - 1)
    // register-resident pass: needs 16-byte source quads and 8-byte output pairs
    if (!(L.flags & PK_FLAG_GENERIC) && h <= kRtHalo && (L.N % 2) == 0 && aligned16(a)) {
        const int so = (int)((reinterpret_cast<uintptr_t>(src) >> 2) & 3);
        // first window start: 16-byte aligned in src, its output region beginning at or below lo
        int64_t ws0 = lo - kRtHalo;
        ws0 -= ((ws0 + so) % 4 + 4) % 4;
        const int64_t xs0 = ws0 + kRtHalo;
        const int64_t nwarps = ceil_div(hi - xs0, kRtOut);
        const int64_t blocks = ceil_div(nwarps, 8);
        if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi: grid too large");
        k_jacobi1d_rtemporal<<<(unsigned)blocks, 256, 0, st>>>(src, dst, half0, half1, lo, hi, P, L.N, t0, h, xs0,
                                                               nwarps, flag, mode);
        return after_launch("jacobi1d_rtemporal");
    }
    const int W = 4096;
    const int64_t x0 = lo & ~(int64_t)3;  // tiles on 4-aligned positions; outputs masked to [lo, hi)
    const int64_t ntiles = ceil_div(hi - x0, W);
    // window: [ (xs-h) & ~3, xs + W + h ) rounded to quads, plus one quad of slack
    const int WN = ((W + 2 * h + 3 + 3) & ~3) + 4;
    const size_t smem = 2 * (size_t)WN * sizeof(int);
    int rc = allow_smem((const void *)k_jacobi1d_temporal, smem);
    if (rc) return rc;
    int per_sm = 0, sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi1d_temporal, 256, smem);
    int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (grid > ntiles) grid = ntiles;
    k_jacobi1d_temporal<<<(unsigned)grid, 256, smem, st>>>(src, dst, half0, half1, lo, hi, P, L.N, t0, h, x0, W, WN,
                                                           ntiles, flag, mode);
    return after_launch("jacobi1d_temporal");
}

}  // namespace pk
