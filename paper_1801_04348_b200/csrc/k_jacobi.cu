// k_jacobi.cu -- the double-buffered Jacobi stencils.
//
// 1-D (pkg/src/parakern/data/jacobi.mfk:9-25), a[2N]:
//   dim = (N-2)/(s*B); for t < T, for p < dim*s*B (position x = p+1):
//     t even: a[x]   = (a[N+x-1] + a[N+x] + a[N+x+1]) / 3
//     t odd:  a[N+x] = (a[x-1]   + a[x]   + a[x+1])   / 3
// 2-D (SURVEY App. A.4 jacobi2d.mfk), a[2N][N]:
//   rows i in [1, dim0*B0], cols j in [1, dim1*s*B1]
//   t even: a[N+i][j] = (a[i-1][j] + a[i+1][j] + a[i][j-1] + a[i][j+1] + a[i][j]) / 5
//   t odd:  the same with the halves swapped.
// One launch per time step (the serial t loop is the schedule's context
// loop, interp.py:148-152).  HBM-bound: 8 bytes of algorithmic traffic per
// updated point per step.
//
// Exact integer division.  The reference's ints are unbounded, so the sum
// of three (five) int32 values must not wrap before the truncating
// division.  A Jacobi average never leaves the value range of its inputs
// (each new value lies between the min and max of the old ones, and
// truncation toward zero stays inside that interval), so if every initial
// value satisfies |v| <= (2^31-1)/3 (resp. /5) all sums of every later step
// fit in int32.  A device-side pre-pass checks that bound once per run and
// sets a flag the sweep kernels read (no host round trip); otherwise they
// form 64-bit sums.  Both paths give identical results -- the 32-bit one
// needs about a third of the integer instructions.
//
// Staged tiles (cache(a) kept).  A block's window is copied to shared
// memory with unguarded, batched 64-bit loads (the interior-tile test is
// block-uniform, so only the first / last tiles take the guarded path),
// laid out so the tile's first position sits on a 16-byte boundary.  Each
// thread then computes four consecutive outputs from one 128-bit shared
// load; the left / right neighbours come from the adjacent lanes by warp
// shuffle (shared memory only at warp and row edges), and results leave as
// two 64-bit stores.  64-bit (not 128-bit) global granularity because the
// upper half starts at a + N and N = 2^28 + 2 is only 8-byte aligned.
#include "pk_internal.cuh"

namespace pk {
namespace {

constexpr int kBound3 = 715827882;  // (2^31 - 1) / 3
constexpr int kBound5 = 429496729;  // (2^31 - 1) / 5
constexpr int kBatch = 4;           // independent 64-bit loads in flight per thread

template <bool WIDE>
__device__ __forceinline__ int avg3(int a, int b, int c) {
    if (WIDE) return (int)(((long long)a + (long long)b + (long long)c) / 3);
    return (a + b + c) / 3;
}
template <bool WIDE>
__device__ __forceinline__ int avg5(int a, int b, int c, int d, int e) {
    if (WIDE) return (int)(((long long)a + (long long)b + (long long)c + (long long)d + (long long)e) / 5);
    return (a + b + c + d + e) / 5;
}

// flag = 1 if every |v| <= bound over a[0, n), else 0 (flag preset non-zero).
// a need only be 4-byte aligned: the words before its first 16-byte boundary
// are checked one by one.
__global__ void __launch_bounds__(256) k_range_flag(const int *__restrict__ a, int64_t n, int bound,
                                                   int *__restrict__ flag) {
    bool ok = true;
    int64_t head = (int64_t)(((16u - (reinterpret_cast<uintptr_t>(a) & 15u)) & 15u) >> 2);
    if (head > n) head = n;
    const int64_t n4 = (n - head) / 4;
    const int4 *a4 = reinterpret_cast<const int4 *>(a + head);
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t0; i < n4; i += stride) {
        const int4 v = ld_stream(a4 + i);
        ok &= (v.x >= -bound && v.x <= bound) & (v.y >= -bound && v.y <= bound) &
              (v.z >= -bound && v.z <= bound) & (v.w >= -bound && v.w <= bound);
    }
    if (t0 < head) ok &= (a[t0] >= -bound && a[t0] <= bound);
    for (int64_t i = head + 4 * n4 + t0; i < n; i += stride) ok &= (a[i] >= -bound && a[i] <= bound);
    if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0);
}

// the same over columns 0 and J+1 .. N-1 of rows 1 .. I of an N x N half
__global__ void __launch_bounds__(256) k_range_cols(const int *__restrict__ h, int64_t N, int64_t I, int64_t J,
                                                   int bound, int *__restrict__ flag) {
    bool ok = true;
    const int64_t w = N - J;  // column 0 plus columns J+1 .. N-1
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < I * w; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = 1 + e / w, k = e % w, j = k == 0 ? 0 : J + k;
        const int v = h[i * N + j];
        ok &= (v >= -bound && v <= bound);
    }
    if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0);
}

__device__ __forceinline__ bool narrow_mode(int mode, const int *flag) {
    return mode == 2 ? (*flag != 0) : (mode == 1);
}

__device__ __forceinline__ void store4(int *dst, int64_t x, int64_t lo, int64_t hi, bool vec, int v0,
                                       int v1, int v2, int v3) {
    if (vec && x >= lo && x + 3 < hi) {
        *reinterpret_cast<int2 *>(dst + x) = make_int2(v0, v1);
        *reinterpret_cast<int2 *>(dst + x + 2) = make_int2(v2, v3);
    } else {
        if (x >= lo && x < hi) dst[x] = v0;
        if (x + 1 >= lo && x + 1 < hi) dst[x + 1] = v1;
        if (x + 2 >= lo && x + 2 < hi) dst[x + 2] = v2;
        if (x + 3 >= lo && x + 3 < hi) dst[x + 3] = v3;
    }
}

// ---------------------------------------------------------------- 1-D ------

// Outputs x = xs + 4p .. +3 from a shared window whose index 0 holds
// position xs - 4 (sb is 16-byte aligned when al16, else 8-byte aligned).
template <bool WIDE, bool FULL = false>  // FULL: every warp of the group has 32 lanes
__device__ __forceinline__ void j1_compute(const int *sb, bool al16, int *__restrict__ dst, int64_t lo,
                                           int64_t hi, int64_t xs, int tile, bool vec, int tid, int nt) {
    const int lane = tid & 31;
    const int wlanes = min(32, nt - (tid - lane));  // lanes of this (possibly partial) warp
    const unsigned wmask = wlanes == 32 ? 0xffffffffu : ((1u << wlanes) - 1u);
    const int quads = tile >> 2;
    for (int pb = tid - lane; pb < quads; pb += nt) {  // warp-uniform trip count (shuffles)
        const int p = pb + lane;
        const bool act = p < quads;
        int4 c = make_int4(0, 0, 0, 0);  // src[x .. x+3]
        if (act) {
            const int *q = sb + 4 * p + 4;
            if (al16) {
                c = *reinterpret_cast<const int4 *>(q);
            } else {
                const int2 u = *reinterpret_cast<const int2 *>(q), w = *reinterpret_cast<const int2 *>(q + 2);
                c = make_int4(u.x, u.y, w.x, w.y);
            }
        }
        int l = __shfl_up_sync(FULL ? 0xffffffffu : wmask, c.w, 1);
        int r = __shfl_down_sync(FULL ? 0xffffffffu : wmask, c.x, 1);
        if (!act) continue;
        if (lane == 0) l = sb[4 * p + 3];
        if (lane + 1 == wlanes || p + 1 == quads) r = sb[4 * p + 8];
        const int64_t x = xs + 4 * (int64_t)p;
        if (x + 3 < lo || x >= hi) continue;
        store4(dst, x, lo, hi, vec, avg3<WIDE>(l, c.x, c.y), avg3<WIDE>(c.x, c.y, c.z),
               avg3<WIDE>(c.y, c.z, c.w), avg3<WIDE>(c.z, c.w, r));
    }
}

// Persistent, warp-specialised TMA pipeline.  Each block walks tiles
// blockIdx.x + k*gridDim.x through an S-stage ring of shared windows: warp 0
// (the producer) fills window k mod S with one cp.async.bulk (the window
// start rounded down to 16 bytes; the 8-byte remainder is the tile's shift)
// as soon as the consumers have released it, and the other warps compute.
// full[b] completes when window b has landed (TMA transaction count) or, for
// an edge window, when it is free for the consumers' own guarded fill;
// empty[b] when every consumer warp has finished reading it.  No block-wide
// barrier: each consumer warp runs ahead to the next landed window on its own.
constexpr int kTmaPad = 16;    // words of slack per buffer for the alignment shift
constexpr int kMaxStages = 8;  // ring depth limit (mbarrier header: 2 x 8 x 8 bytes)
constexpr int kRingHeader = 2 * kMaxStages * 2;  // header size in ints

__device__ __forceinline__ void j1_issue(const int *src, int64_t xs, int tile, int *buf, uint64_t *bar) {
    const uintptr_t ga = reinterpret_cast<uintptr_t>(src + xs - 4);
    const int shift = (int)((ga & 15) >> 2);
    const uint32_t bytes = (uint32_t)(((tile + 8 + shift) * 4 + 15) & ~15);
    mbar_expect_tx(bar, bytes);
    tma_load_1d(buf, reinterpret_cast<const void *>(ga & ~(uintptr_t)15), bytes, bar);
}

// Barrier among the consumer warps only (named barrier 1; the producer warp
// never joins it).
__device__ __forceinline__ void consumers_sync(int nct) {
    asm volatile("bar.sync 1, %0;" ::"r"((nct + 31) & ~31) : "memory");
}

// Producer warp.  Tiles [ta, tb) have their whole rounded window inside the
// half and go by TMA; for the one or two edge tiles outside it the producer
// only hands the (free) window to the consumers, which fill it with guarded
// loads themselves (ordered by their named barrier).
__device__ __forceinline__ void j1_produce(const int *__restrict__ src, int64_t x0, int tile, int64_t ntiles,
                                           int64_t ta, int64_t tb, int S, uint64_t *full, uint64_t *empty,
                                           int *bufs) {
    const int lane = threadIdx.x & 31;
    const int BW = tile + kTmaPad;
    uint32_t ephase = 0u;  // bit b: parity of empty[b]'s next completion
    int b = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // a fresh barrier reports the phase before its first as complete:
        // the first S waits pass at once
        mbar_wait(&empty[b], ((ephase >> b) & 1u) ^ 1u);
        ephase ^= 1u << b;
        int *buf = bufs + b * BW;
        const int64_t xs = x0 + t * tile;
        if (t >= ta && t < tb) {
            if (lane == 0) {
                fence_proxy_async();  // earlier generic accesses of buf before the async write
                j1_issue(src, xs, tile, buf, &full[b]);
            }
        } else if (lane == 0) {
            mbar_arrive(&full[b]);
        }
        b = b + 1 == S ? 0 : b + 1;
    }
}

template <bool WIDE, bool FULL>
__device__ __forceinline__ void j1_consume(const int *__restrict__ src, int *__restrict__ dst, int64_t lo,
                                           int64_t hi, int64_t x0, int tile, int64_t ntiles, int64_t ta,
                                           int64_t tb, int64_t limit, int S, uint64_t *full, uint64_t *empty,
                                           int *bufs, int ctid, int nct) {
    const int BW = tile + kTmaPad;
    uint32_t fphase = 0u;  // bit b: parity of full[b]'s next completion
    int b = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&full[b], (fphase >> b) & 1u);
        fphase ^= 1u << b;
        const int64_t xs = x0 + t * tile;
        int *buf = bufs + b * BW;
        int shift = 0;
        if (t >= ta && t < tb) {
            shift = (int)((reinterpret_cast<uintptr_t>(src + xs - 4) & 15) >> 2);
        } else {  // edge tile: guarded fill (block-uniform branch)
            for (int q = ctid; q < tile + 8; q += nct) {
                const int64_t i = xs - 4 + q;
                buf[q] = (i >= 0 && i < limit) ? src[i] : 0;
            }
            consumers_sync(nct);
        }
        j1_compute<WIDE, FULL>(buf + shift, shift == 0, dst, lo, hi, xs, tile, true, ctid, nct);
        __syncwarp();
        if ((ctid & 31) == 0) mbar_arrive(&empty[b]);
        b = b + 1 == S ? 0 : b + 1;
    }
}

// blockDim = 32 (producer) + the consumer threads
__global__ void __launch_bounds__(288) k_jacobi1d_tma(const int *__restrict__ src, int *__restrict__ dst,
                                                     int64_t lo, int64_t hi, int64_t x0, int tile,
                                                     int64_t ntiles, int64_t ta, int64_t tb, int64_t limit,
                                                     int S, const int *flag, int mode) {
    extern __shared__ __align__(128) int smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + kMaxStages;
    int *bufs = smem + kRingHeader;
    if ((int64_t)blockIdx.x >= ntiles) return;
    const int nct = blockDim.x - 32, cwarps = (nct + 31) >> 5;
    if (threadIdx.x == 0) {
        for (int j = 0; j < S; j++) {
            mbar_init(&full[j], 1);
            mbar_init(&empty[j], cwarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int ctid = threadIdx.x - 32;
    const bool narrow = narrow_mode(mode, flag), full_warps = (nct & 31) == 0;
    if (threadIdx.x < 32)
        j1_produce(src, x0, tile, ntiles, ta, tb, S, full, empty, bufs);
    else if (narrow && full_warps)
        j1_consume<false, true>(src, dst, lo, hi, x0, tile, ntiles, ta, tb, limit, S, full, empty, bufs, ctid,
                                 nct);
    else if (narrow)
        j1_consume<false, false>(src, dst, lo, hi, x0, tile, ntiles, ta, tb, limit, S, full, empty, bufs, ctid,
                                 nct);
    else if (full_warps)
        j1_consume<true, true>(src, dst, lo, hi, x0, tile, ntiles, ta, tb, limit, S, full, empty, bufs, ctid,
                                 nct);
    else
        j1_consume<true, false>(src, dst, lo, hi, x0, tile, ntiles, ta, tb, limit, S, full, empty, bufs, ctid,
                                 nct);
}

// window: positions [xs-4, xs+tile+4) at shared index pos - xs + 4 (tile % 4 == 0)
template <bool WIDE>
__device__ __forceinline__ void j1_staged_body(const int *__restrict__ src, int *__restrict__ dst,
                                               int64_t lo, int64_t hi, int64_t xs, int tile,
                                               int64_t limit, bool vec, int *sh) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int w2 = (tile + 8) >> 1;
    int2 *sh2 = reinterpret_cast<int2 *>(sh);
    const bool interior = vec && xs - 4 >= 0 && xs + tile + 4 <= limit;
    if (interior) {
        const int2 *g2 = reinterpret_cast<const int2 *>(src + xs - 4);
        for (int q = tid; q < w2; q += kBatch * nt) {
            int2 v[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; u++)
                if (q + u * nt < w2) v[u] = g2[q + u * nt];
#pragma unroll
            for (int u = 0; u < kBatch; u++)
                if (q + u * nt < w2) sh2[q + u * nt] = v[u];
        }
    } else {
        for (int q = tid; q < 2 * w2; q += nt) {
            const int64_t i = xs - 4 + q;
            sh[q] = (i >= 0 && i < limit) ? src[i] : 0;
        }
    }
    __syncthreads();
    j1_compute<WIDE>(sh, true, dst, lo, hi, xs, tile, vec, tid, nt);
}

__global__ void __launch_bounds__(1024) k_jacobi1d_staged(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t lo,
                                                         int64_t hi, int64_t x0, int tile,
                                                         int64_t limit, int vec, const int *flag,
                                                         int mode) {
    extern __shared__ __align__(16) int sh[];
    const int64_t xs = x0 + (int64_t)blockIdx.x * tile;
    if (narrow_mode(mode, flag))
        j1_staged_body<false>(src, dst, lo, hi, xs, tile, limit, vec != 0, sh);
    else
        j1_staged_body<true>(src, dst, lo, hi, xs, tile, limit, vec != 0, sh);
}

// caching-off: every thread reads its neighbourhood straight from global
// memory (the overlapping reads of adjacent threads hit L1).
template <bool WIDE>
__device__ __forceinline__ void j1_direct_body(const int *__restrict__ src, int *__restrict__ dst,
                                               int64_t lo, int64_t hi, int64_t xs, int tile, bool vec) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int quads = tile >> 2;
#pragma unroll 2
    for (int p = tid; p < quads; p += nt) {
        const int64_t x = xs + 4 * (int64_t)p;
        if (x + 3 < lo || x >= hi) continue;
        // read only what a written output needs: x-1 >= lo-1 >= 0 and x+4 <= hi <= N-1
        const int l = x >= lo ? src[x - 1] : 0;
        const int r = x + 3 < hi ? src[x + 4] : 0;
        int2 c0, c1;
        if (vec && x >= lo && x + 3 < hi) {
            c0 = *reinterpret_cast<const int2 *>(src + x);
            c1 = *reinterpret_cast<const int2 *>(src + x + 2);
        } else {
            c0 = make_int2(src[x], x + 1 <= hi ? src[x + 1] : 0);
            c1 = make_int2(x + 2 <= hi ? src[x + 2] : 0, x + 3 <= hi ? src[x + 3] : 0);
        }
        store4(dst, x, lo, hi, vec, avg3<WIDE>(l, c0.x, c0.y), avg3<WIDE>(c0.x, c0.y, c1.x),
               avg3<WIDE>(c0.y, c1.x, c1.y), avg3<WIDE>(c1.x, c1.y, r));
    }
}

__global__ void __launch_bounds__(1024) k_jacobi1d_direct(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t lo,
                                                         int64_t hi, int64_t x0, int tile, int vec,
                                                         const int *flag, int mode) {
    const int64_t xs = x0 + (int64_t)blockIdx.x * tile;
    if (narrow_mode(mode, flag))
        j1_direct_body<false>(src, dst, lo, hi, xs, tile, vec != 0);
    else
        j1_direct_body<true>(src, dst, lo, hi, xs, tile, vec != 0);
}

// ---------------------------------------------------------------- 2-D ------

// Window: rows r0-1 .. r0+nr, columns c0-4 .. c0+TJ+3 (pitch TJ+8), column j
// at shared index j - c0 + 4.  Each thread owns a column quad and marches
// down its row group keeping the rows above / at / below in registers: one
// 128-bit shared load per row per four outputs.
//
// j2_compute reads window row rr at base + rr*pitch + shift(rr), shift(rr) =
// (s0 + rr*ds) & 3 in {0, 2} words (TMA rows start on 16 bytes; rows of an
// N = 2 mod 4 matrix alternate between the two alignments).
__device__ __forceinline__ int4 lds4(const int *p, bool al16) {
    if (al16) return *reinterpret_cast<const int4 *>(p);
    const int2 u = *reinterpret_cast<const int2 *>(p), w = *reinterpret_cast<const int2 *>(p + 2);
    return make_int4(u.x, u.y, w.x, w.y);
}

// Per-thread role in a TI x TJ tile, fixed for the whole kernel: column
// quad qd of row group g (groups of nq = TJ/4 threads march rpg rows each).
struct J2Role {
    int qd, rb, rpg, passes, lc;
    bool act, lin, rin;
    unsigned wmask;
};

__device__ __forceinline__ J2Role j2_role(int TI, int TJ, int qb, int tid, int nt) {
    const int lane = tid & 31;
    const int nq = TJ >> 2;
    J2Role r;
    const int groups = nt >= nq ? nt / nq : 1;
    r.passes = nt >= nq ? 1 : (nq + nt - 1) / nt;
    r.rpg = (TI + groups - 1) / groups;
    r.qd = nt >= nq ? tid % nq : tid + qb * nt;
    const int g = nt >= nq ? tid / nq : 0;
    r.act = g < groups && r.qd < nq;
    r.rb = g * r.rpg;
    r.lc = 4 * r.qd + 4;
    const int wlanes = min(32, nt - (tid - lane));
    r.wmask = wlanes == 32 ? 0xffffffffu : ((1u << wlanes) - 1u);
    r.lin = lane > 0 && r.qd > 0;
    r.rin = lane + 1 < wlanes && r.qd + 1 < nq;
    return r;
}

// One role's column quad over its rows of the tile at (r0, c0): drow points
// at dst row r0, columns relative to c0.
template <bool WIDE, bool FULL = false>  // FULL: every warp of the group has 32 lanes
__device__ __forceinline__ void j2_march(const J2Role &R, const int *base, int pitch, int s0, int ds,
                                         int *__restrict__ drow, int64_t N, int nr, int64_t c0, int64_t J,
                                         bool vec) {
    const int64_t j = c0 + 4 * (int64_t)R.qd;  // output columns j .. j+3
    int sh = (s0 + R.rb * ds) & 3;             // alignment shift of window row rb
    const int *p = base + R.rb * pitch + sh + R.lc;
    int4 up = make_int4(0, 0, 0, 0), cur = up;
    const bool go = R.act && R.rb < nr;
    if (go) up = lds4(p, sh == 0);
    p += pitch - sh;
    sh = (sh + ds) & 3;
    p += sh;
    if (go) cur = lds4(p, sh == 0);
    int *o = drow + (int64_t)R.rb * N + 4 * R.qd;
    for (int k = 0; k < R.rpg; k++) {  // warp-uniform trip count (shuffles)
        const int *crow = p;
        const bool live = R.act && R.rb + k < nr;
        p += pitch - sh;
        sh = (sh + ds) & 3;
        p += sh;
        const int4 dn = live ? lds4(p, sh == 0) : make_int4(0, 0, 0, 0);
        int l = __shfl_up_sync(FULL ? 0xffffffffu : R.wmask, cur.w, 1);
        int r = __shfl_down_sync(FULL ? 0xffffffffu : R.wmask, cur.x, 1);
        if (live) {
            if (!R.lin) l = crow[-1];
            if (!R.rin) r = crow[4];
            const int v0 = avg5<WIDE>(up.x, dn.x, l, cur.y, cur.x);
            const int v1 = avg5<WIDE>(up.y, dn.y, cur.x, cur.z, cur.y);
            const int v2 = avg5<WIDE>(up.z, dn.z, cur.y, cur.w, cur.z);
            const int v3 = avg5<WIDE>(up.w, dn.w, cur.z, r, cur.w);
            store4(o - j, j, 1, J + 1, vec, v0, v1, v2, v3);
        }
        o += N;
        up = cur;
        cur = dn;
    }
}

template <bool WIDE, bool FULL = false>  // FULL: every warp of the group has 32 lanes
__device__ __forceinline__ void j2_compute(const int *base, int pitch, int s0, int ds, int *__restrict__ dst,
                                           int64_t N, int64_t r0, int nr, int64_t c0, int64_t J, int TI, int TJ,
                                           bool vec, int tid, int nt) {
    const int passes = j2_role(TI, TJ, 0, tid, nt).passes;
    for (int qb = 0; qb < passes; qb++)
        j2_march<WIDE, FULL>(j2_role(TI, TJ, qb, tid, nt), base, pitch, s0, ds, dst + r0 * N + c0, N, nr, c0, J, vec);
}

// Warp-specialised TMA pipeline for 2-D tiles (same ring as the 1-D one):
// the producer warp issues one bulk copy per window row (rows start on
// 16-byte boundaries; the remainder is the row's shift) into window k mod S
// once the consumer warps have released it; edge windows are filled by the
// consumers.
constexpr int kRowPad = 16;  // words of slack per window row for the alignment shift

__device__ __forceinline__ uint32_t j2_row_bytes(int TJ, int sh) {
    return (uint32_t)(((TJ + 8 + sh) * 4 + 15) & ~15);
}

// true when every rounded window row of the tile lies inside the half
// [src, src + N*N): only the first column tile of the first row band and the
// last column tile of the last band can poke out (their extra columns are
// the neighbouring rows' ends, read but never used)
__device__ __forceinline__ bool j2_window_ok(const int *src, int64_t N, int64_t r0, int nr, int64_t c0, int TJ) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(src), hi = reinterpret_cast<uintptr_t>(src + N * N);
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(src + (r0 - 1) * N + c0 - 4);
    const uintptr_t gl = reinterpret_cast<uintptr_t>(src + (r0 + nr) * N + c0 - 4);
    return (g0 & ~(uintptr_t)15) >= lo && (gl & ~(uintptr_t)15) + j2_row_bytes(TJ, (int)((gl & 15) >> 2)) <= hi;
}

__device__ __forceinline__ void j2_issue(const int *src, int64_t N, int64_t r0, int nr, int64_t c0, int TJ,
                                         int *buf, int pitch, uint64_t *bar) {
    const int lane = threadIdx.x & 31;
    const int rows = nr + 2;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src + (r0 - 1) * N + c0 - 4);
    const int s0 = (int)((a0 & 15) >> 2), ds = (int)(N & 3);
    if (lane == 0) {
        uint32_t total = 0;
        for (int rr = 0; rr < rows; rr++) total += j2_row_bytes(TJ, (s0 + rr * ds) & 3);
        mbar_expect_tx(bar, total);
    }
    __syncwarp();
    for (int rr = lane; rr < rows; rr += 32) {
        const uintptr_t ga = reinterpret_cast<uintptr_t>(src + (r0 - 1 + rr) * N + c0 - 4);
        tma_load_1d(buf + rr * pitch, reinterpret_cast<const void *>(ga & ~(uintptr_t)15),
                    j2_row_bytes(TJ, (int)((ga & 15) >> 2)), bar);
    }
}

// Tiles in row-major order (column tile fastest), blocks striding by the
// grid: at any moment the whole GPU streams a few full row bands, which
// keeps DRAM pages and the halo rows shared with the next band hot.
// (Giving each block a contiguous run down a column strip instead
// scattered the concurrent streams and measured 3x slower.)
struct J2Tile {
    int64_t r0, c0;
    int nr;
};
__device__ __forceinline__ J2Tile j2_tile(int64_t t, int64_t ntc, int64_t rlo, int64_t rhi, int TI, int TJ) {
    const uint32_t ntc32 = (uint32_t)ntc;  // tile indices < 2^31 (host check)
    const uint32_t tr = (uint32_t)t / ntc32, tc = (uint32_t)t - tr * ntc32;
    J2Tile T;
    T.r0 = rlo + (int64_t)tr * TI;
    T.c0 = (int64_t)tc * TJ;
    T.nr = (int)min((int64_t)TI, rhi - T.r0);
    return T;
}

__device__ __forceinline__ void j2_produce(const int *__restrict__ src, int64_t N, int64_t rlo, int64_t rhi,
                                           int TI, int TJ, int64_t ntc, int64_t ntiles, int S, uint64_t *full,
                                           uint64_t *empty, int *bufs) {
    const int lane = threadIdx.x & 31;
    const int pitch = TJ + kRowPad, BW = (TI + 2) * pitch;
    uint32_t ephase = 0u;  // bit b: parity of empty[b]'s next completion
    int b = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&empty[b], ((ephase >> b) & 1u) ^ 1u);  // first S waits pass at once
        ephase ^= 1u << b;
        const J2Tile T = j2_tile(t, ntc, rlo, rhi, TI, TJ);
        int *buf = bufs + b * BW;
        if (j2_window_ok(src, N, T.r0, T.nr, T.c0, TJ)) {
            fence_proxy_async();  // earlier generic accesses of buf before the async writes
            j2_issue(src, N, T.r0, T.nr, T.c0, TJ, buf, pitch, &full[b]);
        } else if (lane == 0) {
            mbar_arrive(&full[b]);  // the consumers fill this edge window themselves
        }
        b = b + 1 == S ? 0 : b + 1;
    }
}

template <bool WIDE>
__device__ __forceinline__ void j2_consume(const int *__restrict__ src, int *__restrict__ dst, int64_t N,
                                           int64_t rlo, int64_t rhi, int64_t J, int TI, int TJ, int64_t ntc,
                                           int64_t ntiles, int S, uint64_t *full, uint64_t *empty, int *bufs,
                                           int ctid, int nct) {
    const int pitch = TJ + kRowPad, BW = (TI + 2) * pitch;
    const J2Role role = j2_role(TI, TJ, 0, ctid, nct);  // fixed for every tile of this block
    uint32_t fphase = 0u;  // bit b: parity of full[b]'s next completion
    int b = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const J2Tile T = j2_tile(t, ntc, rlo, rhi, TI, TJ);
        const bool tma = j2_window_ok(src, N, T.r0, T.nr, T.c0, TJ);
        int s0 = 0, ds = 0;
        if (tma) {
            s0 = (int)((reinterpret_cast<uintptr_t>(src + (T.r0 - 1) * N + T.c0 - 4) & 15) >> 2);
            ds = (int)(N & 3);
        }
        mbar_wait(&full[b], (fphase >> b) & 1u);
        fphase ^= 1u << b;
        int *buf = bufs + b * BW;
        if (!tma) {  // edge tile: guarded fill (block-uniform branch)
            for (int e = ctid; e < (T.nr + 2) * pitch; e += nct) {
                const int rr = e / pitch, cc = e - rr * pitch;
                const int64_t col = T.c0 - 4 + cc;
                buf[e] = (cc < TJ + 8 && col >= 0 && col < N) ? src[(T.r0 - 1 + rr) * N + col] : 0;
            }
            consumers_sync(nct);
        }
        if (role.passes == 1)
            j2_march<WIDE, true>(role, buf, pitch, s0, ds, dst + T.r0 * N + T.c0, N, T.nr, T.c0, J, true);
        else
            j2_compute<WIDE, true>(buf, pitch, s0, ds, dst, N, T.r0, T.nr, T.c0, J, TI, TJ, true, ctid, nct);
        __syncwarp();
        if ((ctid & 31) == 0) mbar_arrive(&empty[b]);
        b = b + 1 == S ? 0 : b + 1;
    }
}

// blockDim = 32 (producer) + the consumer threads
__global__ void __launch_bounds__(544) k_jacobi2d_tma(const int *__restrict__ src, int *__restrict__ dst,
                                                      int64_t N, int64_t rlo, int64_t rhi, int64_t J, int TI,
                                                      int TJ, int64_t ntc, int64_t ntiles, int S, const int *flag,
                                                      int mode) {
    extern __shared__ __align__(128) int smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem), *empty = full + kMaxStages;
    int *bufs = smem + kRingHeader;
    if ((int64_t)blockIdx.x >= ntiles) return;
    const int nct = blockDim.x - 32, cwarps = (nct + 31) >> 5;
    if (threadIdx.x == 0) {
        for (int j = 0; j < S; j++) {
            mbar_init(&full[j], 1);
            mbar_init(&empty[j], cwarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x < 32)
        j2_produce(src, N, rlo, rhi, TI, TJ, ntc, ntiles, S, full, empty, bufs);
    else if (narrow_mode(mode, flag))
        j2_consume<false>(src, dst, N, rlo, rhi, J, TI, TJ, ntc, ntiles, S, full, empty, bufs, threadIdx.x - 32, nct);
    else
        j2_consume<true>(src, dst, N, rlo, rhi, J, TI, TJ, ntc, ntiles, S, full, empty, bufs, threadIdx.x - 32, nct);
}

template <bool WIDE>
__device__ __forceinline__ void j2_staged_body(const int *__restrict__ src, int *__restrict__ dst,
                                               int64_t N, int64_t r0, int64_t rhi, int64_t c0,
                                               int64_t J, int TI, int TJ, bool vec, int *sh) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    const int pitch = TJ + 8, w2 = pitch >> 1;
    const int nr = (int)min((int64_t)TI, rhi - r0);
    const int rows = nr + 2;
    const bool interior = vec && c0 - 4 >= 0 && c0 + TJ + 4 <= N;
    if (interior) {
        // batched, unguarded: element e = (row, q) advanced by nt per step
        const int drow = nt / w2, dq = nt - drow * w2;
        int row = tid / w2, q = tid - row * w2;
        const int2 *g0 = reinterpret_cast<const int2 *>(src + (r0 - 1) * N + c0 - 4);
        const int64_t rstride2 = N >> 1;  // N even on this path
        while (row < rows) {
            int2 v[kBatch];
            int rr[kBatch], qq[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; u++) {
                rr[u] = row;
                qq[u] = q;
                if (row < rows) v[u] = g0[(int64_t)row * rstride2 + q];
                row += drow;
                q += dq;
                if (q >= w2) {
                    q -= w2;
                    row++;
                }
            }
#pragma unroll
            for (int u = 0; u < kBatch; u++)
                if (rr[u] < rows) reinterpret_cast<int2 *>(sh + rr[u] * pitch)[qq[u]] = v[u];
        }
    } else {
        for (int e = tid; e < rows * pitch; e += nt) {
            const int rr = e / pitch, cc = e - rr * pitch;
            const int64_t col = c0 - 4 + cc;
            sh[e] = (col >= 0 && col < N) ? src[(r0 - 1 + rr) * N + col] : 0;
        }
    }
    __syncthreads();
    (void)lane;
    j2_compute<WIDE>(sh, pitch, 0, 0, dst, N, r0, nr, c0, J, TI, TJ, vec, threadIdx.x, blockDim.x);
}

__global__ void __launch_bounds__(1024) k_jacobi2d_staged(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t N,
                                                         int64_t rlo, int64_t rhi, int64_t J,
                                                         int TI, int TJ, int64_t tc0, int64_t ntj, int vec,
                                                         const int *flag, int mode) {
    extern __shared__ __align__(16) int sh[];
    const int64_t bid = blockIdx.x;
    const int64_t r0 = rlo + (bid / ntj) * TI, c0 = (tc0 + bid % ntj) * TJ;
    if (narrow_mode(mode, flag))
        j2_staged_body<false>(src, dst, N, r0, rhi, c0, J, TI, TJ, vec != 0, sh);
    else
        j2_staged_body<true>(src, dst, N, r0, rhi, c0, J, TI, TJ, vec != 0, sh);
}

// caching-off: a thread owns a column quad of one row and reads the five
// neighbours from global memory (rows above / below through L1/L2).
template <bool WIDE>
__device__ __forceinline__ void j2_direct_body(const int *__restrict__ src, int *__restrict__ dst,
                                               int64_t N, int64_t r0, int64_t rhi, int64_t c0,
                                               int64_t J, int TI, int TJ, bool vec) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int nr = (int)min((int64_t)TI, rhi - r0);
    const int nq = TJ >> 2;
    for (int e = tid; e < nr * nq; e += nt) {
        const int rr = e / nq, qd = e - rr * nq;
        const int64_t i = r0 + rr, j = c0 + 4 * (int64_t)qd;
        if (j + 3 < 1 || j > J) continue;
        const int *m = src + i * N;
        int v[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int64_t jj = j + k;
            if (jj >= 1 && jj <= J)
                v[k] = avg5<WIDE>(m[jj - N], m[jj + N], m[jj - 1], m[jj + 1], m[jj]);
            else
                v[k] = 0;
        }
        store4(dst + i * N, j, 1, J + 1, vec, v[0], v[1], v[2], v[3]);
    }
}

__global__ void __launch_bounds__(1024) k_jacobi2d_direct(const int *__restrict__ src,
                                                         int *__restrict__ dst, int64_t N,
                                                         int64_t rlo, int64_t rhi, int64_t J,
                                                         int TI, int TJ, int64_t ntj, int vec,
                                                         const int *flag, int mode) {
    const int64_t bid = blockIdx.x;
    const int64_t r0 = rlo + (bid / ntj) * TI, c0 = (bid % ntj) * TJ;
    if (narrow_mode(mode, flag))
        j2_direct_body<false>(src, dst, N, r0, rhi, c0, J, TI, TJ, vec != 0);
    else
        j2_direct_body<true>(src, dst, N, r0, rhi, c0, J, TI, TJ, vec != 0);
}

struct Extents1D {
    int64_t P;  // interior positions updated: 1..P
};

int extents1d(const pk_launch_t &L, Extents1D *e) {
    if (L.s * L.B == 0) return fail(PK_E_DIV0, "jacobi: s*B == 0 in dim = (N - 2) / (s * B)");
    e->P = 0;
    if (L.s < 0 || L.B < 0) return PK_OK;
    e->P = max0((L.N - 2) / (L.s * L.B)) * L.s * L.B;
    return PK_OK;
}

struct Extents2D {
    int64_t I, J;  // rows 1..I, cols 1..J
};

int extents2d(const pk_launch_t &L, Extents2D *e) {
    if (L.B0 == 0) return fail(PK_E_DIV0, "jacobi2d: B0 == 0 in dim0 = (N - 2) / B0");
    if (L.s * L.B1 == 0) return fail(PK_E_DIV0, "jacobi2d: s*B1 == 0 in dim1 = (N - 2) / (s * B1)");
    e->I = e->J = 0;
    if (L.B0 < 0 || L.B1 < 0 || L.s < 0) return PK_OK;
    e->I = max0((L.N - 2) / L.B0) * L.B0;
    e->J = max0((L.N - 2) / (L.s * L.B1)) * L.s * L.B1;
    return PK_OK;
}

// mode for a sweep: the caller's PK_FLAG_NARROW promise, a device flag, or wide
int sweep_mode(const pk_launch_t &L, const int *flag) {
    if (flag) return 2;
    return (L.flags & PK_FLAG_NARROW) ? 1 : 0;
}

inline int64_t round4(int64_t v) { return (v + 3) & ~(int64_t)3; }

// Ring depth of a TMA pipeline: enough stages that ~24 KB per block is in
// flight beyond the one being computed on, at most kMaxStages and ~160 KB of
// shared memory.  PK_TMA_STAGES overrides (tuning sweeps).
int64_t smem_optin() {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return optin;
}

int tma_stages(size_t stage_bytes) {
    int S = 1 + (int)((24 * 1024 + stage_bytes - 1) / stage_bytes);
    if (const char *e = getenv("PK_TMA_STAGES")) {
        if (atoi(e) > 0) S = atoi(e);
    }
    const int cap = (int)((160 * 1024) / stage_bytes);
    if (S > cap) S = cap;
    if (S > kMaxStages) S = kMaxStages;
    if (S < 2) S = 2;
    return S;
}

int sweep1d_impl(const pk_launch_t &L, const int *src, int *dst, int64_t lo, int64_t hi,
                 const int *flag, cudaStream_t st) {
    Extents1D e;
    int rc = extents1d(L, &e);
    if (rc) return rc;
    if (lo < 1) lo = 1;
    if (hi > e.P + 1) hi = e.P + 1;
    if (hi <= lo) return PK_OK;
    // the quad layout needs tile % 4 == 0; coverage comes from [lo, hi), not the tile
    const int64_t tile64 = round4(elems(L) * L.B);
    if (tile64 > (1 << 28)) return fail(PK_E_UNSUPPORTED, "jacobi: tile too large");
    const int tile = (int)tile64;
    const int nt = (int)(L.B < 1024 ? L.B : 1024);
    const int64_t x0 = lo & ~(int64_t)1;
    const int64_t blocks = ceil_div(hi - x0, tile);
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi: grid too large");
    const int vec = !((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 7u);
    const int mode = sweep_mode(L, flag);
    if (L.variant == PK_VARIANT_STAGED && !(L.flags & PK_FLAG_GENERIC)) {
        // the window staged in registers (k_jacobi_reg.cu) unless the layout is not its
        rc = sweep1d_reg(src, dst, lo, hi, L.N, flag, mode, st);
        if (rc != kNotTaken) return rc;
    }
    if (L.variant == PK_VARIANT_STAGED) {
        // tiles whose whole (16-byte rounded) window lies inside the half go
        // through the TMA pipeline; the one or two edge tiles through the
        // guarded kernel
        int64_t ta = 0, tb = 0;
        if (vec && tile >= 64 && tile <= 8192) {
            ta = x0 >= 8 ? 0 : ceil_div(8 - x0, tile);
            const int64_t room = L.N - 8 - tile - x0;
            tb = room >= 0 ? room / tile + 1 : 0;
            if (tb > blocks) tb = blocks;
            if (tb - ta < 2) ta = tb = 0;
        }
        const size_t smem = ((size_t)tile + 8) * sizeof(int);
        rc = allow_smem((const void *)k_jacobi1d_staged, smem);
        if (rc) return rc;
        auto generic = [&](int64_t t0, int64_t t1) -> int {
            if (t1 <= t0) return PK_OK;
            k_jacobi1d_staged<<<(unsigned)(t1 - t0), nt, smem, st>>>(src, dst, lo, hi, x0 + t0 * tile, tile,
                                                                     L.N, vec, flag, mode);
            return after_launch("jacobi1d");
        };
        if (tb > ta) {
            const size_t stage = ((size_t)tile + kTmaPad) * sizeof(int);
            const int S = tma_stages(stage);
            const size_t tsmem = kRingHeader * sizeof(int) + S * stage;
            rc = allow_smem((const void *)k_jacobi1d_tma, tsmem);
            if (rc) return rc;
            const int tnt = 32 + (nt < 256 ? nt : 256);  // producer warp + consumers
            int per_sm = 0, sms = 148, dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi1d_tma, tnt, tsmem);
            int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
            if (grid > blocks) grid = blocks;
            k_jacobi1d_tma<<<(unsigned)grid, tnt, tsmem, st>>>(src, dst, lo, hi, x0, tile, blocks, ta, tb, L.N,
                                                               S, flag, mode);
            return after_launch("jacobi1d_tma");
        }
        return generic(0, blocks);
    }
    k_jacobi1d_direct<<<(unsigned)blocks, nt, 0, st>>>(src, dst, lo, hi, x0, tile, vec, flag, mode);
    return after_launch("jacobi1d");
}

int sweep2d_impl(const pk_launch_t &L, const int *src, int *dst, int64_t lo, int64_t hi,
                 const int *flag, cudaStream_t st) {
    Extents2D e;
    int rc = extents2d(L, &e);
    if (rc) return rc;
    if (lo < 1) lo = 1;
    if (hi > e.I + 1) hi = e.I + 1;
    if (hi <= lo || e.J <= 0) return PK_OK;
    const int64_t TI64 = L.B0, TJ64 = round4(elems(L) * L.B1);
    if (TI64 * TJ64 > (1 << 26)) return fail(PK_E_UNSUPPORTED, "jacobi2d: tile too large");
    const int TI = (int)TI64, TJ = (int)TJ64;
    int64_t nthreads = L.B0 * L.B1;
    if (nthreads > 1024) nthreads = 1024;
    const int64_t nti = ceil_div(hi - lo, TI), ntj = ceil_div(e.J + 1, TJ);
    const int64_t blocks = nti * ntj;
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi2d: grid too large");
    const int vec = (L.N % 2 == 0) && !((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 7u);
    const int mode = sweep_mode(L, flag);
    if (L.variant == PK_VARIANT_STAGED && !(L.flags & PK_FLAG_GENERIC)) {
        rc = sweep2d_reg(src, dst, lo, hi, e.J, L.N, flag, mode, st);
        if (rc != kNotTaken) return rc;
    }
    if (L.variant == PK_VARIANT_STAGED) {
        const size_t smem = (size_t)(TI + 2) * (size_t)(TJ + 8) * sizeof(int);
        rc = allow_smem((const void *)k_jacobi2d_staged, smem);
        if (rc) return rc;
        auto generic = [&](int64_t tc0, int64_t ntc) -> int {
            if (ntc <= 0) return PK_OK;
            k_jacobi2d_staged<<<(unsigned)(nti * ntc), (unsigned)nthreads, smem, st>>>(
                src, dst, L.N, lo, hi, e.J, TI, TJ, tc0, ntc, vec, flag, mode);
            return after_launch("jacobi2d");
        };
        // the TMA pipeline feeds every tile whose rounded window lies inside
        // the half (the producer warp fills the rest with guarded loads)
        const size_t stage = (size_t)(TI + 2) * (size_t)(TJ + kRowPad) * sizeof(int);
        const int S = tma_stages(stage);
        const size_t tsmem = kRingHeader * sizeof(int) + S * stage;
        if (vec && nthreads % 32 == 0 && nthreads <= 512 && (int64_t)tsmem <= smem_optin()) {
            rc = allow_smem((const void *)k_jacobi2d_tma, tsmem);
            if (rc) return rc;
            const int tnt = 32 + (int)nthreads;  // producer warp + consumers
            int per_sm = 0, sms = 148, dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi2d_tma, tnt, tsmem);
            const int64_t ntiles = nti * ntj;
            int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
            if (grid > ntiles) grid = ntiles;
            k_jacobi2d_tma<<<(unsigned)grid, (unsigned)tnt, tsmem, st>>>(src, dst, L.N, lo, hi, e.J, TI, TJ, ntj,
                                                                        ntiles, S, flag, mode);
            return after_launch("jacobi2d_tma");
        }
        return generic(0, ntj);
    } else {
        k_jacobi2d_direct<<<(unsigned)blocks, (unsigned)nthreads, 0, st>>>(src, dst, L.N, lo, hi, e.J, TI, TJ,
                                                                           ntj, vec, flag, mode);
    }
    return after_launch("jacobi2d");
}

// Device flag: non-zero when the values a run can read are within the narrow
// bound.  range_flag_begin allocates and presets it; range_check clears it
// if some |v| in a[0, n) exceeds the bound.
int range_flag_begin(int **flag, cudaStream_t st) {
    cudaError_t err = scratch_alloc((void **)flag, sizeof(int), st);
    if (err != cudaSuccess) return fail(PK_E_ALLOC, "cudaMallocAsync(flag): %s", cudaGetErrorString(err));
    // the flag starts non-zero (bytes 0x01); the check clears it with atomicAnd
    err = cudaMemsetAsync(*flag, 1, sizeof(int), st);
    if (err != cudaSuccess) return fail(PK_E_CUDA, "flag init: %s", cudaGetErrorString(err));
    return PK_OK;
}

int range_check(const int *a, int64_t n, int bound, int *flag, cudaStream_t st) {
    if (n <= 0) return PK_OK;
    int64_t blocks = ceil_div(n / 4 + 1, 256 * 8);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    k_range_flag<<<(unsigned)blocks, 256, 0, st>>>(a, n, bound, flag);
    return after_launch("range_flag");
}

int range_flag(const int *a, int64_t n, int bound, int **flag, cudaStream_t st) {
    int rc = range_flag_begin(flag, st);
    return rc ? rc : range_check(a, n, bound, *flag, st);
}

// What a whole-program run can read: every value of the half step 0 reads,
// and the points of the other half the program never writes (step 0
// overwrites the rest before anything reads it).  Half the bytes of the
// whole double buffer.
int range_flag_program(const pk_launch_t &L, const int *a, int **flag, cudaStream_t st) {
    int rc = range_flag_begin(flag, st);
    if (rc) return rc;
    if (L.family == PK_FAMILY_JACOBI1D) {
        Extents1D e;
        if ((rc = extents1d(L, &e))) return rc;
        // step 0 reads the upper half and writes positions 1 .. P of the lower one
        if ((rc = range_check(a + L.N, L.N, kBound3, *flag, st))) return rc;
        if ((rc = range_check(a, 1, kBound3, *flag, st))) return rc;
        return range_check(a + e.P + 1, L.N - e.P - 1, kBound3, *flag, st);
    }
    Extents2D e;
    if ((rc = extents2d(L, &e))) return rc;
    const int64_t N = L.N;
    const int *h1 = a + N * N;  // step 0 reads half 0 and writes rows 1..I x cols 1..J of half 1
    if ((rc = range_check(a, N * N, kBound5, *flag, st))) return rc;
    if ((rc = range_check(h1, N, kBound5, *flag, st))) return rc;
    if ((rc = range_check(h1 + (e.I + 1) * N, (N - 1 - e.I) * N, kBound5, *flag, st))) return rc;
    if (e.I > 0 && N - e.J > 0) {
        int64_t blocks = ceil_div(e.I * (N - e.J), 256 * 4);
        if (blocks > 148 * 8) blocks = 148 * 8;
        k_range_cols<<<(unsigned)blocks, 256, 0, st>>>(h1, N, e.I, e.J, kBound5, *flag);
        rc = after_launch("range_cols");
    }
    return rc;
}

}  // namespace

int sweep_jacobi1d(const pk_launch_t &L, const void *src, void *dst, int64_t lo, int64_t hi,
                   cudaStream_t st) {
    return sweep1d_impl(L, static_cast<const int *>(src), static_cast<int *>(dst), lo, hi, nullptr, st);
}

int sweep_jacobi2d(const pk_launch_t &L, const void *src, void *dst, int64_t lo, int64_t hi,
                   cudaStream_t st) {
    return sweep2d_impl(L, static_cast<const int *>(src), static_cast<int *>(dst), lo, hi, nullptr, st);
}

// One step t of a Jacobi program over units [lo, hi) with the neighbours'
// ghost units written into their buffers (see PeerSweep, k_jacobi_reg.cu).
int jacobi_sweep_peer(const pk_launch_t &L, int *a, int64_t step, int64_t lo, int64_t hi, const pk_peer_t &P,
                      cudaStream_t st) {
    const bool two_d = L.family == PK_FAMILY_JACOBI2D;
    int64_t ulo = 1, uhi = 1, J = 0;
    if (two_d) {
        Extents2D e;
        int rc = extents2d(L, &e);
        if (rc) return rc;
        uhi = e.I + 1;
        J = e.J;
    } else {
        Extents1D e;
        int rc = extents1d(L, &e);
        if (rc) return rc;
        uhi = e.P + 1;
    }
    if (lo < ulo) lo = ulo;
    if (hi > uhi) hi = uhi;
    const int64_t half = two_d ? L.N * L.N : L.N;
    // 1-D: t even writes the lower half (jacobi.mfk:19-23); 2-D: t even writes the upper half
    const bool lower_dst = two_d ? (step % 2 != 0) : (step % 2 == 0);
    int *dst = lower_dst ? a : a + half;
    const int *src = lower_dst ? a + half : a;
    const int64_t off = dst - a;
    PeerHost R;
    R.left_dst = P.left_base ? static_cast<int *>(P.left_base) + off : nullptr;
    R.right_dst = P.right_base ? static_cast<int *>(P.right_base) + off : nullptr;
    R.wait_left = P.wait_left;
    R.wait_right = P.wait_right;
    R.sig_left = P.signal_left;
    R.sig_right = P.signal_right;
    R.error = P.error;
    R.step = step;
    if ((R.left_dst || R.right_dst) && !R.error) return fail(PK_E_PARAM, "pk_jacobi_sweep_peer: no error word");
    if ((R.left_dst && (!R.wait_left || !R.sig_left)) || (R.right_dst && (!R.wait_right || !R.sig_right)))
        return fail(PK_E_PARAM, "pk_jacobi_sweep_peer: a neighbour without its counters");
    const int mode = (L.flags & PK_FLAG_NARROW) ? 1 : 0;
    return sweep_reg_peer(two_d, src, dst, lo, hi, J, L.N, mode, R, st);
}

int jacobi_narrow(const pk_launch_t &L, const void *a, int *narrow, cudaStream_t st) {
    const bool one = L.family == PK_FAMILY_JACOBI1D;
    const int64_t n = one ? 2 * L.N : 2 * L.N * L.N;
    int *flag = nullptr;
    int rc = range_flag(static_cast<const int *>(a), n, one ? kBound3 : kBound5, &flag, st);
    if (rc) return rc;
    cudaMemcpyAsync(narrow, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(flag, st);
    cudaError_t err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) return fail(PK_E_CUDA, "range check: %s", cudaGetErrorString(err));
    *narrow = *narrow != 0;
    return PK_OK;
}

int launch_jacobi1d(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    Extents1D e;
    int rc = extents1d(L, &e);
    if (rc) return rc;
    if (e.P <= 0 || L.T <= 0) return PK_OK;
    int64_t lo, hi;
    unit_range(L, 1, e.P + 1, &lo, &hi);
    int *a = static_cast<int *>(p[0]);
    int *flag = nullptr;
    if (!(L.flags & PK_FLAG_NARROW)) {  // partitioned runs (L.hi > 0) check the whole double buffer
        rc = L.hi > 0 ? range_flag(a, 2 * L.N, kBound3, &flag, st) : range_flag_program(L, a, &flag, st);
        if (rc) return rc;
    }
    const bool temporal = (L.flags & PK_FLAG_TEMPORAL) && L.hi <= 0;  // whole-program runs only
    int hmax = L.tblock > 0 ? (int)L.tblock : 7;
    if (hmax > 31) hmax = 31;
    if (hmax % 2 == 0) hmax -= 1;  // odd: a pass never writes the half it reads
    for (int64_t t = 0; t < L.T && rc == PK_OK;) {
        // temporal passes leave the last step to an ordinary sweep (see k_jacobi_temporal.cu)
        int h = 1;
        if (temporal && L.T - t > 2) {
            h = (int)((L.T - t - 1) < hmax ? (L.T - t - 1) : hmax);
            if (h % 2 == 0) h -= 1;
        }
        if (h > 1) {
            rc = jacobi1d_temporal_pass(L, a, lo, hi, e.P, t, h, flag, sweep_mode(L, flag), st);
            t += h;
            continue;
        }
        const bool even = (t % 2) == 0;
        int *dst = even ? a : a + L.N;
        const int *src = even ? a + L.N : a;
        rc = sweep1d_impl(L, src, dst, lo, hi, flag, st);
        t++;
    }
    if (flag) cudaFreeAsync(flag, st);
    return rc;
}

int launch_jacobi2d(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    Extents2D e;
    int rc = extents2d(L, &e);
    if (rc) return rc;
    if (e.I <= 0 || e.J <= 0 || L.T <= 0) return PK_OK;
    int64_t lo, hi;
    unit_range(L, 1, e.I + 1, &lo, &hi);
    int *a = static_cast<int *>(p[0]);
    int *half1 = a + L.N * L.N;
    int *flag = nullptr;
    if (!(L.flags & PK_FLAG_NARROW)) {  // partitioned runs (L.hi > 0) check the whole double buffer
        rc = L.hi > 0 ? range_flag(a, 2 * L.N * L.N, kBound5, &flag, st) : range_flag_program(L, a, &flag, st);
        if (rc) return rc;
    }
    const bool temporal = (L.flags & PK_FLAG_TEMPORAL) && L.hi <= 0;  // whole-program runs only
    int hmax = L.tblock > 0 ? (int)L.tblock : 7;
    if (hmax > 11) hmax = 11;
    if (hmax % 2 == 0) hmax -= 1;  // odd: a pass never writes the half it reads
    for (int64_t t = 0; t < L.T && rc == PK_OK;) {
        // temporal passes leave the last step to an ordinary sweep (k_jacobi2d_temporal.cu)
        int h = 1;
        if (temporal && L.T - t > 2) {
            h = (int)((L.T - t - 1) < hmax ? (L.T - t - 1) : hmax);
            if (h % 2 == 0) h -= 1;
        }
        if (h > 1) {
            rc = jacobi2d_temporal_pass(L, a, lo, hi, e.I, e.J, t, h, flag, sweep_mode(L, flag), st);
            t += h;
            continue;
        }
        const bool even = (t % 2) == 0;
        // t even reads half 0 and writes half 1 (a[N+i][j] = ...), t odd the reverse
        rc = sweep2d_impl(L, even ? a : half1, even ? half1 : a, lo, hi, flag, st);
        t++;
    }
    if (flag) cudaFreeAsync(flag, st);
    return rc;
}

}  // namespace pk
