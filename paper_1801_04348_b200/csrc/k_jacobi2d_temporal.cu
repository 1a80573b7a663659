// k_jacobi2d_temporal.cu -- temporally blocked 2-D Jacobi (PK_FLAG_TEMPORAL),
// an optional variant reported beside the per-step leaf.
//
// The program (jacobi2d.mfk) runs T sweeps over a[2N][N],
// each a full pass over HBM.  Here one pass advances h steps: a block loads
// a window of its tile plus h ghost rows and >= h ghost columns of the
// latest half into shared memory, iterates h sweeps there (shrinking valid
// region) and writes only the last sweep's values of the tile.  HBM traffic
// per point drops from 8 B per step to ~9 B per h steps; the arithmetic is
// the per-step kernels' (exact sums, truncating division by 5), so results
// are bit-identical.
//
// Halves.  Step t reads half s(t) and writes d(t) (t even: d = half 1,
// a[N+i][j]).  As in the 1-D variant (k_jacobi_temporal.cu): h is odd, so a
// pass never writes the half other blocks read; a pass leaves the other
// half stale, which no later pass reads, and the driver ends with an
// ordinary sweep after which both halves hold the reference's final state.
// Points the program never writes (row 0, rows > I, column 0, columns > J)
// keep, in "half d(t)", that half's own value, read from global memory.
//
// Layout.  The window is 128 columns (32 quads: one warp spans a row) by
// TI + 2h rows; the tile is the middle 128 - 2*H4 columns (H4 = h rounded
// up to 4, so window rows start on 4-column boundaries).  Each warp marches
// down a band of rows keeping up / current / down quads in registers: one
// 128-bit shared load and one 128-bit shared store per row per four points,
// left/right neighbours by warp shuffle.  Garbage entering from the window
// edges moves one point per step and never reaches the tile.
#include "pk_internal.cuh"

namespace pk {
namespace {

constexpr int kWinCols = 128;  // window width (ints): 32 quads, one per lane
constexpr int kT2Threads = 256;

template <bool WIDE>
__device__ __forceinline__ int avg5(int a, int b, int c, int d, int e) {
    if (WIDE) return (int)(((long long)a + (long long)b + (long long)c + (long long)d + (long long)e) / 5);
    return (a + b + c + d + e) / 5;
}

struct T2Geom {
    int64_t N, I, J;   // matrix order; covered rows 1..I, columns 1..J
    int64_t rlo, rhi;  // rows of this launch
    int TI, TJ, H4, h;
    int64_t ntc;       // column tiles
};

// Window geometry of one tile.
struct T2Tile {
    int64_t r0, c0;     // first output row / column
    int rows_out, WH;   // output rows, window rows
    int64_t wr0, wc0;   // window origin (global)
    bool inside;        // window inside the matrix: asynchronous 8-byte copies
};

__device__ __forceinline__ T2Tile t2_geom(const int *src, const T2Geom &G, int64_t tile) {
    T2Tile T;
    const int64_t tr = tile / G.ntc, tc = tile - tr * G.ntc;
    T.r0 = G.rlo + tr * G.TI;
    T.rows_out = (int)min((int64_t)G.TI, G.rhi - T.r0);
    T.c0 = tc * G.TJ;
    T.WH = T.rows_out + 2 * G.h;
    T.wr0 = T.r0 - G.h;
    T.wc0 = T.c0 - G.H4;
    // every window row then starts on an even column of an even-order row
    T.inside = T.wr0 >= 0 && T.wr0 + T.WH <= G.N && T.wc0 >= 0 && T.wc0 + kWinCols <= G.N && (G.N & 1) == 0 &&
               ((reinterpret_cast<uintptr_t>(src) & 7u) == 0);
    return T;
}

// Window of the latest half into buf: asynchronous 8-byte copies (the whole
// window in flight at once; the caller commits and waits), or, for windows
// reaching outside the matrix, guarded loads (0 outside).
__device__ __forceinline__ void t2_load(const int *__restrict__ src, const T2Geom &G, const T2Tile &T, int *buf,
                                        bool async) {
    const int tid = threadIdx.x;
    const int64_t N = G.N;
    if (T.inside && async) {
        // thread tid copies pair (tid & 63) of rows tid/64, tid/64 + R, ... (R = blockDim/64)
        constexpr int P2 = kWinCols / 2;
        const int R = blockDim.x / P2;
        const int64_t gstep = (int64_t)R * N;
        const int *g = src + (T.wr0 + tid / P2) * N + T.wc0 + 2 * (tid & (P2 - 1));
        uint32_t sa = smem_u32(buf) + 8u * (uint32_t)tid;
        for (int rr = tid / P2; rr < T.WH; rr += R, g += gstep, sa += 8u * blockDim.x)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
    } else if (!T.inside && !async) {
        for (int e = tid; e < T.WH * kWinCols; e += blockDim.x) {
            const int rr = e / kWinCols, cc = e - rr * kWinCols;
            const int64_t gr = T.wr0 + rr, gc = T.wc0 + cc;
            buf[e] = (gr >= 0 && gr < N && gc >= 0 && gc < N) ? src[gr * N + gc] : 0;
        }
    }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// h steps of the tile whose window is in win (scratch: tmp; h odd leaves
// the last step in tmp), then the tile's covered points to dst.
template <bool WIDE>
__device__ void t2_steps_store(int *__restrict__ dst, const int *__restrict__ half0, const int *__restrict__ half1,
                               const T2Geom &G, const T2Tile &T, int64_t t0, int *win, int *tmp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int h = G.h, WH = T.WH;
    const int64_t N = G.N, wr0 = T.wr0, wc0 = T.wc0;
    // does the window reach points the program never writes?
    const bool edge = wr0 + 1 < 1 || wr0 + WH - 1 > G.I || wc0 + 1 < 1 || wc0 + kWinCols - 1 > G.J;
    int *cur = win, *nxt = tmp;
    for (int k = 0; k < h; k++) {
        const int64_t t = t0 + k;
        const int *fixed = (t % 2 == 0) ? half1 : half0;  // d(t): t even writes a[N+i][j]
        // rows [k+1, WH-1-k) are valid after this step; split them over the warps
        const int rs = k + 1, re = WH - 1 - k, nrows = re - rs;
        const int per = (nrows + nwarps - 1) / nwarps;
        const int b0 = rs + warp * per, b1 = min(re, b0 + per);
        if (b0 < b1) {
            const int4 *c4 = reinterpret_cast<const int4 *>(cur);
            int4 up = c4[(b0 - 1) * 32 + lane], mid = c4[b0 * 32 + lane];
#pragma unroll 3
            for (int rr = b0; rr < b1; rr++) {
                const int4 dn = c4[(rr + 1) * 32 + lane];
                // lanes 0 / 31 get their own value back: garbage at the window
                // edge, which moves one column per step and never reaches the tile
                const int l = __shfl_up_sync(0xffffffffu, mid.w, 1);
                const int r = __shfl_down_sync(0xffffffffu, mid.x, 1);
                int4 o = make_int4(avg5<WIDE>(up.x, dn.x, l, mid.y, mid.x), avg5<WIDE>(up.y, dn.y, mid.x, mid.z, mid.y),
                                   avg5<WIDE>(up.z, dn.z, mid.y, mid.w, mid.z), avg5<WIDE>(up.w, dn.w, mid.z, r, mid.w));
                if (edge) {  // points the program never writes keep half d(t)'s own value
                    const int64_t gr = wr0 + rr, gc = wc0 + 4 * lane;
                    int *ov = reinterpret_cast<int *>(&o);
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const int64_t ge = gc + e;
                        if (gr < 1 || gr > G.I || ge < 1 || ge > G.J)
                            ov[e] = (gr >= 0 && gr < N && ge >= 0 && ge < N) ? fixed[gr * N + ge] : 0;
                    }
                }
                reinterpret_cast<int4 *>(nxt)[rr * 32 + lane] = o;
                up = mid;
                mid = dn;
            }
        }
        __syncthreads();
        int *sw = cur;
        cur = nxt;
        nxt = sw;
    }

    // ---- write the tile's covered points of the last step: lane = tile quad,
    // warps stride over the tile rows
    const int tq = G.TJ >> 2, hq = G.H4 >> 2;
    const int64_t rw_lo = max(T.r0, (int64_t)1), rw_hi = min(T.r0 + T.rows_out, G.I + 1);
    const bool vec = (N & 1) == 0 && ((reinterpret_cast<uintptr_t>(dst) & 7u) == 0);
    const int q = lane;
    const int64_t gc = T.c0 + 4 * q;
    for (int ro = warp; ro < T.rows_out && q < tq; ro += nwarps) {
        const int64_t gr = T.r0 + ro;
        if (gr < rw_lo || gr >= rw_hi) continue;
        const int4 v = reinterpret_cast<const int4 *>(cur)[(h + ro) * 32 + hq + q];
        int *row = dst + gr * N;
        if (vec && gc >= 1 && gc + 3 <= G.J) {
            *reinterpret_cast<int2 *>(row + gc) = make_int2(v.x, v.y);
            *reinterpret_cast<int2 *>(row + gc + 2) = make_int2(v.z, v.w);
        } else {
            const int vals[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (gc + u >= 1 && gc + u <= G.J) row[gc + u] = vals[u];
        }
    }
}

// Per block: load a window (cp.async), iterate, write, next tile.  The
// block's loads do not overlap its own arithmetic -- the other blocks on the
// SM cover them (a three-buffer prefetching ring measured no faster: the
// pass is bound by the in-shared-memory steps, and it costs occupancy).
template <bool WIDE>
__device__ void t2_run(const int *__restrict__ src, int *__restrict__ dst, const int *__restrict__ half0,
                       const int *__restrict__ half1, const T2Geom &G, int64_t t0, int64_t ntiles, int *win,
                       int *tmp) {
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const T2Tile T = t2_geom(src, G, tile);
        t2_load(src, G, T, win, true);
        cp_async_commit();
        t2_load(src, G, T, win, false);  // guarded loads when the window leaves the matrix
        cp_async_wait_all();
        __syncthreads();  // window complete and visible
        t2_steps_store<WIDE>(dst, half0, half1, G, T, t0, win, tmp);
        __syncthreads();  // results written out before the next window lands
    }
}

__global__ void __launch_bounds__(kT2Threads) k_jacobi2d_temporal(const int *__restrict__ src, int *__restrict__ dst,
                                                                  const int *__restrict__ half0,
                                                                  const int *__restrict__ half1, T2Geom G, int64_t t0,
                                                                  int64_t ntiles, const int *flag, int mode) {
    extern __shared__ __align__(16) int sh[];
    const int bw = (G.TI + 2 * G.h) * kWinCols;
    const bool narrow = mode == 2 ? (*flag != 0) : (mode == 1);
    if (narrow)
        t2_run<false>(src, dst, half0, half1, G, t0, ntiles, sh, sh + bw);
    else
        t2_run<true>(src, dst, half0, half1, G, t0, ntiles, sh, sh + bw);
}

// ---------------------------------------------------------------------------
// Register wavefront (the default; the shared-memory pass above remains for
// odd N, misaligned halves and PK_FLAG_GENERIC).  A warp owns a 128-column
// window (a column quad per lane) and walks down a band of kWfR output rows
// plus h halo rows above and below, one input row at a time.  Level k of the
// pipeline holds the last two rows it produced (A_k, B_k: 2h int4 registers
// per thread); each new level-k row n completes level k+1's row above it,
// avg5(A_k, B_k, n, left / right of B_k by shuffle), so one input row
// advances every level by one row and leaves level h (the pass's last step)
// h rows behind.  No shared memory, no barriers; every step of every point
// costs two shuffles per quad, two IADD3s and the /5.  Columns within H4
// (h rounded up to 4) of the window edges go stale and are not stored:
// windows overlap by 2 x H4 columns.  Rows of an N = 2 (mod 4) matrix
// alternate 16- / 8-byte alignment; an 8-byte row is loaded as the aligned
// quad c+2..c+5 and shifted by a shuffle (lane 0 loads its own c-2..c+1).
// Points the program never writes (row 0, rows > I, column 0, columns > J)
// take half d(t)'s value at each level, on warps whose window reaches them.
constexpr int kWfR = 128;    // output rows per band
#ifndef PK_WF_MINB
#define PK_WF_MINB 1
#endif
constexpr int kWfWarps = 4;  // warps per block

__device__ __forceinline__ int4 ldg4(const int *p) { return __ldg(reinterpret_cast<const int4 *>(p)); }

__device__ __forceinline__ int4 ldg4_guard(const int *row, int64_t c, int64_t N) {
    if (c >= 0 && c + 3 < N) return ldg4(row + c);
    int v[4];
#pragma unroll
    for (int e = 0; e < 4; e++) v[e] = (c + e >= 0 && c + e < N) ? __ldg(row + c + e) : 0;
    return make_int4(v[0], v[1], v[2], v[3]);
}

// input row r: the aligned quad (and lane 0's extra quad on an 8-byte row)
template <bool PH, bool EDGE>
__device__ __forceinline__ void wf_load(const int *src, int64_t N, int64_t r, int64_t c, int lane, int4 &raw,
                                        int4 &ext) {
    if (EDGE && (r < 0 || r >= N)) {
        raw = ext = make_int4(0, 0, 0, 0);
        return;
    }
    const int *row = src + r * N;
    if (!EDGE) {
        raw = ldg4(row + c + (PH ? 2 : 0));
        if (PH && lane == 0) ext = ldg4(row + c - 2);
    } else {
        raw = ldg4_guard(row, c + (PH ? 2 : 0), N);
        if (PH && lane == 0) ext = ldg4_guard(row, c - 2, N);
    }
}

// the row's quad at columns c .. c+3
template <bool PH>
__device__ __forceinline__ int4 wf_align(const int4 &raw, const int4 &ext, int lane) {
    if (!PH) return raw;
    int pz = __shfl_up_sync(0xffffffffu, raw.z, 1), pw = __shfl_up_sync(0xffffffffu, raw.w, 1);
    if (lane == 0) {
        pz = ext.z;
        pw = ext.w;
    }
    return make_int4(pz, pw, raw.x, raw.y);
}

struct WfGeom {
    const int *src, *half0, *half1;
    int *dst;
    int64_t N, I, J, lo, hi, t0;
    int64_t rs;       // first band's first output row (odd)
    int64_t nbands, nwin;
    int TJ;           // output columns per window
};

// One input row n (row r) through the h levels; level h's row r - h is stored.
// (Measured alternatives, h = 7, 16386^2: shuffling a row's neighbours when
// it is produced instead of when it is the centre -- 10.6 ms; one row per
// iteration with two in flight -- 14.8 ms; this pair-unrolled form -- 9.3 ms.)
template <int H, bool WIDE, bool EDGE, bool PH2>
__device__ __forceinline__ void wf_row(int4 (&A)[H], int4 (&B)[H], int4 n, int64_t r, int64_t c, int lane,
                                       int64_t slo, int64_t shi, const WfGeom &G) {
#pragma unroll
    for (int k = 0; k < H; k++) {
        // level k: A = row r-k-2, B = row r-k-1, n = row r-k -> level k+1, row i = r-k-1
        const int l = __shfl_up_sync(0xffffffffu, B[k].w, 1), rr = __shfl_down_sync(0xffffffffu, B[k].x, 1);
        int4 o = make_int4(avg5<WIDE>(A[k].x, n.x, l, B[k].y, B[k].x), avg5<WIDE>(A[k].y, n.y, B[k].x, B[k].z, B[k].y),
                           avg5<WIDE>(A[k].z, n.z, B[k].y, B[k].w, B[k].z), avg5<WIDE>(A[k].w, n.w, B[k].z, rr, B[k].w));
        if (EDGE) {
            const int64_t i = r - k - 1;
            if (i < 1 || i > G.I || c < 1 || c + 3 > G.J) {  // points the program never writes: d(t)'s value
                const int *fh = ((G.t0 + k) % 2 == 0) ? G.half1 : G.half0;  // t even writes a[N+i][j]
                const bool row_fixed = i < 1 || i > G.I;
                auto fix = [&](int v, int64_t j) {
                    if (!row_fixed && j >= 1 && j <= G.J) return v;
                    return (i >= 0 && i < G.N && j >= 0 && j < G.N) ? fh[i * G.N + j] : 0;
                };
                o = make_int4(fix(o.x, c), fix(o.y, c + 1), fix(o.z, c + 2), fix(o.w, c + 3));
            }
        }
        A[k] = B[k];
        B[k] = n;
        n = o;
    }
    constexpr int H4 = (H + 3) & ~3;
    const int64_t i = r - H;
    if (i >= slo && i < shi && lane >= H4 / 4 && lane < 32 - H4 / 4) {
        int *o = G.dst + i * G.N + c;
        const bool ph = PH2 && (i & 1);
        if (!EDGE || (c >= 1 && c + 3 <= G.J)) {
            if (!ph) {
                *reinterpret_cast<int4 *>(o) = n;
            } else {
                *reinterpret_cast<int2 *>(o) = make_int2(n.x, n.y);
                *reinterpret_cast<int2 *>(o + 2) = make_int2(n.z, n.w);
            }
        } else {
            if (c >= 1 && c <= G.J) o[0] = n.x;
            if (c + 1 >= 1 && c + 1 <= G.J) o[1] = n.y;
            if (c + 2 >= 1 && c + 2 <= G.J) o[2] = n.z;
            if (c + 3 >= 1 && c + 3 <= G.J) o[3] = n.w;
        }
    }
}

template <int H, bool WIDE, bool EDGE, bool PH2>
__device__ __forceinline__ void wf_warp(const WfGeom &G, int64_t r0, int64_t wc0) {
    const int lane = threadIdx.x & 31;
    const int64_t c = wc0 + 4 * lane;
    const int64_t slo = max(max(r0, G.lo), (int64_t)1), shi = min(min(r0 + kWfR, G.hi), G.I + 1);
    int4 A[H], B[H];
#pragma unroll
    for (int k = 0; k < H; k++) A[k] = B[k] = make_int4(0, 0, 0, 0);
    // input rows r0 - H (even) .. r0 + kWfR - 1 + H (odd), in pairs: even rows at phase 0, odd at PH2
    const int64_t rfirst = r0 - H, rlast = r0 + kWfR - 1 + H;
    int4 rawE, extE = make_int4(0, 0, 0, 0), rawO, extO = make_int4(0, 0, 0, 0);
    wf_load<false, EDGE>(G.src, G.N, rfirst, c, lane, rawE, extE);
    wf_load<PH2, EDGE>(G.src, G.N, rfirst + 1, c, lane, rawO, extO);
    for (int64_t r = rfirst; r <= rlast; r += 2) {
        const int4 cE = rawE, cO = rawO, xO = extO;
        if (r + 2 <= rlast) {  // the next pair in flight while this one runs through the levels
            wf_load<false, EDGE>(G.src, G.N, r + 2, c, lane, rawE, extE);
            wf_load<PH2, EDGE>(G.src, G.N, r + 3, c, lane, rawO, extO);
        }
        wf_row<H, WIDE, EDGE, PH2>(A, B, cE, r, c, lane, slo, shi, G);
        wf_row<H, WIDE, EDGE, PH2>(A, B, wf_align<PH2>(cO, xO, lane), r + 1, c, lane, slo, shi, G);
    }
}

// One kernel per sum width: registers are allocated for the widest path a
// kernel contains, and the 64-bit one would cost the narrow one occupancy.
// Under a device flag (mode 2) both are launched and the one that does not
// match returns at once.
template <int H, bool WIDE, bool PH2>
__global__ void __launch_bounds__(kWfWarps * 32, PK_WF_MINB) k_jacobi2d_wavefront(WfGeom G, const int *flag, int mode) {
    const int64_t w = (int64_t)blockIdx.x * kWfWarps + (threadIdx.x >> 5);
    if (w >= G.nbands * G.nwin) return;  // warp-uniform
    if (mode == 2) {
        int v;
        asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if ((v != 0) == WIDE) return;
    }
    // windows of a band side by side (consecutive warps share rows in L2)
    const int64_t band = w / G.nwin, win = w - band * G.nwin;
    constexpr int H4 = (H + 3) & ~3;
    const int64_t r0 = G.rs + band * kWfR, wc0 = win * G.TJ - H4;
    // edge: some row of the cone outside 1..I, or the window outside 1..J
    const bool edge = r0 - H - 1 < 1 || r0 + kWfR + H > G.I || wc0 < 1 || wc0 + 128 > G.J + 1;
    if (edge)
        wf_warp<H, WIDE, true, PH2>(G, r0, wc0);
    else
        wf_warp<H, WIDE, false, PH2>(G, r0, wc0);
}

template <int H, bool WIDE>
void launch_wavefront_w(const WfGeom &G, bool ph2, const int *flag, int mode, unsigned blocks, cudaStream_t st) {
    if (ph2)
        k_jacobi2d_wavefront<H, WIDE, true><<<blocks, kWfWarps * 32, 0, st>>>(G, flag, mode);
    else
        k_jacobi2d_wavefront<H, WIDE, false><<<blocks, kWfWarps * 32, 0, st>>>(G, flag, mode);
}

template <int H>
int launch_wavefront(const WfGeom &G, bool ph2, const int *flag, int mode, cudaStream_t st) {
    const int64_t warps = G.nbands * G.nwin;
    const int64_t blocks = ceil_div(warps, kWfWarps);
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi2d temporal: grid too large");
    if (mode != 0) launch_wavefront_w<H, false>(G, ph2, flag, mode, (unsigned)blocks, st);  // narrow (or flag)
    if (mode != 1) launch_wavefront_w<H, true>(G, ph2, flag, mode, (unsigned)blocks, st);   // wide (or flag)
    return after_launch("jacobi2d_wavefront");
}

}  // namespace

// h-step pass starting at step t0 (h odd, 3 <= h <= 11) over rows [lo, hi)
// of the interior 1..I, reading the half that holds step t0-1 and writing
// d(t0+h-1).
int jacobi2d_temporal_pass(const pk_launch_t &L, int *a, int64_t lo, int64_t hi, int64_t I, int64_t J, int64_t t0,
                           int h, const int *flag, int mode, cudaStream_t st) {
    if (hi <= lo || J <= 0) return PK_OK;
    if (h < 1 || h > 11 || h % 2 == 0) return fail(PK_E_PARAM, "jacobi2d temporal: h = %d (odd, <= 11)", h);
    int *half0 = a, *half1 = a + L.N * L.N;
    const int *src = (t0 % 2 == 0) ? half0 : half1;       // s(t0): t even reads half 0
    int *dst = ((t0 + h - 1) % 2 == 0) ? half1 : half0;   // d(t0 + h - 1)
    if (!(L.flags & PK_FLAG_GENERIC) && (L.N % 2) == 0 && aligned16(a)) {
        WfGeom W;
        W.src = src;
        W.dst = dst;
        W.half0 = half0;
        W.half1 = half1;
        W.N = L.N;
        W.I = I;
        W.J = J;
        W.lo = lo;
        W.hi = hi;
        W.t0 = t0;
        W.rs = (lo & 1) ? lo : lo - 1;  // bands start on odd rows (r0 - h even)
        W.nbands = ceil_div(hi - W.rs, kWfR);
        const int H4 = (h + 3) & ~3;
        W.TJ = 128 - 2 * H4;
        W.nwin = ceil_div(J + 1, W.TJ);  // output columns 0 .. J
        const bool ph2 = (L.N & 3) == 2;
        switch (h) {
            case 1: return launch_wavefront<1>(W, ph2, flag, mode, st);
            case 3: return launch_wavefront<3>(W, ph2, flag, mode, st);
            case 5: return launch_wavefront<5>(W, ph2, flag, mode, st);
            case 7: return launch_wavefront<7>(W, ph2, flag, mode, st);
            case 9: return launch_wavefront<9>(W, ph2, flag, mode, st);
            case 11: return launch_wavefront<11>(W, ph2, flag, mode, st);
            default: break;
        }
    }
    T2Geom G;
    G.N = L.N;
    G.I = I;
    G.J = J;
    G.rlo = lo;
    G.rhi = hi;
    G.h = h;
    G.H4 = (h + 3) & ~3;
    G.TJ = kWinCols - 2 * G.H4;
    G.TI = 64;
    G.ntc = ceil_div(J + 1, G.TJ);  // output columns 0..J in tiles (column 0 is never written)
    const int64_t ntiles = ceil_div(hi - lo, G.TI) * G.ntc;
    const size_t smem = 2 * (size_t)(G.TI + 2 * h) * kWinCols * sizeof(int);
    int rc = allow_smem((const void *)k_jacobi2d_temporal, smem);
    if (rc) return rc;
    int per_sm = 0, sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi2d_temporal, kT2Threads, smem);
    int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (grid > ntiles) grid = ntiles;
    k_jacobi2d_temporal<<<(unsigned)grid, kT2Threads, smem, st>>>(src, dst, half0, half1, G, t0, ntiles, flag, mode);
    return after_launch("jacobi2d_temporal");
}

}  // namespace pk
