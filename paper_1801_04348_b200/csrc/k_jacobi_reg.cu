// k_jacobi_reg.cu -- the staged Jacobi leaves with the window staged in
// REGISTERS instead of shared memory (the default binding of the cache(a)
// leaf; the shared-memory TMA pipelines of k_jacobi.cu remain the binding
// for layouts these kernels do not take, and under PK_FLAG_GENERIC).
//
// The reference's staged leaf copies a window of `a` into shared memory so
// each element is read from global memory once per tile (emit.py's
// cooperative load).  On sm_100a the same reuse is cheaper
// in the register file: every thread loads the 16-byte quads it needs once,
// neighbours across lanes come by warp shuffle, and the only re-reads (the
// halo rows of a 2-D band, one quad per warp edge) are L1/L2 hits.  No
// shared memory, no barriers, no producer warp: all loads of a thread are
// issued before its first shuffle, so each thread keeps (R+2) x 16 bytes
// (2-D) or K x 16 bytes (1-D) in flight and the sweep streams at copy
// speed.  Measured on B200 (exp/ kernels, CUDA events, 2^28-point 1-D and
// 16386^2 2-D sweeps): 6.9 TB/s and 6.3 TB/s against 5.7 / 5.4 for the TMA
// pipelines.
//
// Arithmetic and coverage are those of k_jacobi.cu: outputs x in [lo, hi)
// (1-D) or rows [lo, hi) x columns [1, J] (2-D), exact int32 sums when the
// narrow flag holds, else 64-bit sums; results bit-identical to every other
// Jacobi kernel (tests/test_gpu_parity.py).
#include "pk_internal.cuh"

namespace pk {
namespace {

template <bool WIDE>
__device__ __forceinline__ int r_avg3(int a, int b, int c) {
    if (WIDE) return (int)(((long long)a + (long long)b + (long long)c) / 3);
    return (a + b + c) / 3;
}
template <bool WIDE>
__device__ __forceinline__ int r_avg5(int a, int b, int c, int d, int e) {
    if (WIDE) return (int)(((long long)a + (long long)b + (long long)c + (long long)d + (long long)e) / 5);
    return (a + b + c + d + e) / 5;
}

// Sum width of this sweep: mode 1 narrow, 0 wide, 2 the device flag set by
// the range pre-pass.  Read at kernel entry with a memory clobber so the load
// is issued ahead of the data loads (left to the compiler it was sunk below
// the shuffles, adding a dependent L2 round trip to every thread: -15 % on
// the 2-D sweep).
__device__ __forceinline__ bool r_narrow(int mode, const int *flag) {
    if (mode != 2) return mode == 1;
    int v;
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    return v != 0;
}

// Loads of the source half.  COH = false: the read-only (.nc) path -- the
// half was written by earlier kernels only.  COH = true: the edge blocks of
// a peer sweep, whose ghost rows a neighbouring GPU stores over NVLink while
// this kernel runs; they load through the coherent path (weak ld.global.cg,
// L2 -- the point of coherence for this GPU's memory), ordered after thread
// 0's ld.acquire.sys of the neighbour's counter by the block barrier, which
// the non-coherent .nc path is not.
template <bool COH = false>
__device__ __forceinline__ int4 ldq(const int *p) {
    if (!COH) return __ldg(reinterpret_cast<const int4 *>(p));
    int4 r;
    asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)
                 : "memory");
    return r;
}
template <bool COH = false>
__device__ __forceinline__ int ld1(const int *p) {
    if (!COH) return __ldg(p);
    int r;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}

// 16-byte quad at element y of a length-n array (y % 4 on a 16-byte boundary);
// elements outside [0, n) read as 0 (they only feed outputs never stored)
template <bool COH = false>
__device__ __forceinline__ int4 ldq_guard(const int *a, int64_t y, int64_t n) {
    if (y >= 0 && y + 3 < n) return ldq<COH>(a + y);
    int t[4];
#pragma unroll
    for (int e = 0; e < 4; e++) t[e] = (y + e >= 0 && y + e < n) ? ld1<COH>(a + y + e) : 0;
    return make_int4(t[0], t[1], t[2], t[3]);
}
template <bool COH = false>
__device__ __forceinline__ int ld1_guard(const int *a, int64_t y, int64_t n) {
    return (y >= 0 && y < n) ? ld1<COH>(a + y) : 0;
}
__device__ __forceinline__ int q_at(const int4 &v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// Fused halo exchange over peer memory (pk_jacobi_sweep_peer).  Every rank
// holds the whole double buffer with global indexing, so the neighbours'
// ghost point / row is written straight into their buffer (same offset,
// through the IPC mapping: NVLink stores) by the block that computes it.
// Ordering: a rank's edge blocks wait, before loading, until the neighbour's
// edge blocks of the previous step have signalled (their remote stores into
// our ghosts are done, and so are their reads of the half we are about to
// overwrite in their buffer); after storing, they signal the neighbours with
// a system-scope fence + atomic.  Interior blocks never wait.
struct PeerSweep {
    int *left_dst, *right_dst;         // neighbours' copies of this sweep's dst half (nullptr: none)
    const unsigned *wait_left, *wait_right;  // this rank's counters
    unsigned *sig_left, *sig_right;    // the neighbours' counters (mapped)
    unsigned *error;                   // set when a wait gives up (a neighbour never signalled)
    unsigned target;                   // edge blocks per step x steps already run
};

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// bounded spin (~2 s): a neighbour that never signals sets the error word
// instead of hanging the device
__device__ __forceinline__ void spin_until(const unsigned *ctr, unsigned target, unsigned *error) {
    for (unsigned k = 0; ld_acquire_sys(ctr) < target; k++) {
        if (k == (1u << 24)) {
            atomicExch(error, 1u);
            return;
        }
        __nanosleep(128);
    }
}

// thread 0 waits for the neighbours this block borders, then the block proceeds
__device__ __forceinline__ void peer_wait(const PeerSweep &P, bool left, bool right) {
    if (threadIdx.x == 0) {
        if (left) spin_until(P.wait_left, P.target, P.error);
        if (right) spin_until(P.wait_right, P.target, P.error);
    }
    __syncthreads();
}

// after every thread of the block has stored: publish to the neighbours
__device__ __forceinline__ void peer_signal(const PeerSweep &P, bool left, bool right) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (left) atomicAdd_system(P.sig_left, 1u);
        if (right) atomicAdd_system(P.sig_right, 1u);
    }
}

// ------------------------------------------------------------------ 1-D ----
//
// Output quads x = xa + 4q are 16-byte aligned in dst; the source quad a
// thread loads starts at y = x + D (16-byte aligned in src, D = phase
// difference of the halves: 2 for the BASELINE N = 2^28 + 2).  The window
// src[x-1 .. x+4] is the thread's quad plus elements of the previous lane's
// (and, for D = 0, the next lane's first); lane 0 / lane 31 load the quad
// across the warp edge themselves (an L1 hit: the neighbouring warp loads it).
constexpr int kJ1Threads = 256, kJ1K = 2;  // K quads per thread, strided by the warp

template <bool WIDE, int D, int K, bool PEER = false>
__device__ __forceinline__ void j1r_compute(const int4 (&own)[K], const int4 (&edge)[K], int *__restrict__ d,
                                            int64_t xw, int64_t lo, int64_t hi, bool interior,
                                            const PeerSweep *P = nullptr) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < K; j++) {
        const int64_t x = xw + 4 * (lane + 32 * j);
        int4 prev;  // src[x+D-4 .. x+D-1]
        prev.x = __shfl_up_sync(0xffffffffu, own[j].x, 1);
        prev.y = __shfl_up_sync(0xffffffffu, own[j].y, 1);
        prev.z = __shfl_up_sync(0xffffffffu, own[j].z, 1);
        prev.w = __shfl_up_sync(0xffffffffu, own[j].w, 1);
        int nx = __shfl_down_sync(0xffffffffu, own[j].x, 1);  // src[x+D+4] (used when D == 0)
        if (lane == 0) prev = edge[j];
        if (D == 0 && lane == 31) nx = edge[j].x;
        int w[6];  // src[x-1 .. x+4]
#pragma unroll
        for (int i = 0; i < 6; i++) {
            const int o = i - 1 - D;  // offset from the start of own
            w[i] = o < 0 ? q_at(prev, o + 4) : o < 4 ? q_at(own[j], o) : nx;
        }
        const int v0 = r_avg3<WIDE>(w[0], w[1], w[2]), v1 = r_avg3<WIDE>(w[1], w[2], w[3]);
        const int v2 = r_avg3<WIDE>(w[2], w[3], w[4]), v3 = r_avg3<WIDE>(w[3], w[4], w[5]);
        if (PEER) {  // the neighbours' ghost points: our first and last output
            const int vv[4] = {v0, v1, v2, v3};
            if (P->left_dst && lo >= x && lo < x + 4) P->left_dst[lo] = vv[lo - x];
            if (P->right_dst && hi - 1 >= x && hi - 1 < x + 4) P->right_dst[hi - 1] = vv[hi - 1 - x];
        }
        if (interior || (x >= lo && x + 4 <= hi)) {
            *reinterpret_cast<int4 *>(d + x) = make_int4(v0, v1, v2, v3);
        } else {
            if (x >= lo && x < hi) d[x] = v0;
            if (x + 1 >= lo && x + 1 < hi) d[x + 1] = v1;
            if (x + 2 >= lo && x + 2 < hi) d[x + 2] = v2;
            if (x + 3 >= lo && x + 3 < hi) d[x + 3] = v3;
        }
    }
}

template <int D, int K, bool COH>
__device__ __forceinline__ void j1r_load(const int *__restrict__ s, int64_t xw, int64_t N, bool interior,
                                         int4 (&own)[K], int4 (&edge)[K]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < K; j++) {
        const int64_t y = xw + 4 * (lane + 32 * j) + D;
        own[j] = interior ? ldq<COH>(s + y) : ldq_guard<COH>(s, y, N);
    }
    // the quads across the warp edges, loaded once the warp's own loads are in
    // flight (the neighbouring warp's loads of the same sectors are then L1 hits)
#pragma unroll
    for (int j = 0; j < K; j++) {
        const int64_t y = xw + 4 * (lane + 32 * j) + D;
        if (lane == 0) edge[j] = interior ? ldq<COH>(s + y - 4) : ldq_guard<COH>(s, y - 4, N);
        if (D == 0 && lane == 31) edge[j].x = interior ? ld1<COH>(s + y + 4) : ld1_guard<COH>(s, y + 4, N);
    }
}

// The loads do not depend on the sum width: they are issued first, the
// narrow flag (a device word set by the range pre-pass) is read beside
// them, and only the arithmetic branches on it.
template <int D, bool PEER = false>
__global__ void __launch_bounds__(kJ1Threads) k_jacobi1d_reg(const int *__restrict__ s, int *__restrict__ d,
                                                             int64_t xa, int64_t q0, int64_t lo, int64_t hi,
                                                             int64_t N, const int *flag, int mode,
                                                             PeerSweep P = PeerSweep{}) {
    constexpr int K = kJ1K;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // PEER: the last block (it holds hi - 1) runs first, then block 0 (lo), so
    // both edges are computed and signalled at the start of the sweep
    const int64_t bx = !PEER ? (int64_t)blockIdx.x
                             : (blockIdx.x == 0 ? (int64_t)gridDim.x - 1 : (int64_t)blockIdx.x - 1);
    const bool pl = PEER && bx == 0 && P.left_dst, pr = PEER && bx == (int64_t)gridDim.x - 1 && P.right_dst;
    if (PEER && (pl || pr)) peer_wait(P, pl, pr);
    const int64_t qw = q0 + (bx * (kJ1Threads / 32) + warp) * 32 * K;  // warp's first quad
    const int64_t xw = xa + 4 * qw;
    const bool narrow = r_narrow(mode, flag);
    // warp-uniform: every load inside [0, N) and every store inside [lo, hi)
    const bool interior = xw + D - 4 >= 0 && xw + 4 * 32 * K + D + 4 <= N && xw >= lo && xw + 4 * 32 * K <= hi;
    int4 own[K], edge[K];
    if (PEER && (pl || pr))
        j1r_load<D, K, true>(s, xw, N, interior, own, edge);
    else
        j1r_load<D, K, false>(s, xw, N, interior, own, edge);
    if (narrow)
        j1r_compute<false, D, K, PEER>(own, edge, d, xw, lo, hi, interior, &P);
    else
        j1r_compute<true, D, K, PEER>(own, edge, d, xw, lo, hi, interior, &P);
    if (PEER && (pl || pr)) peer_signal(P, pl, pr);
}

// ------------------------------------------------------------------ 2-D ----
//
// A warp owns 32 column quads (128 columns, c = 4k) of a band of R rows and
// loads the R + 2 rows it needs -- all of them before the first shuffle.
// Rows of an N = 2 (mod 4) matrix alternate between 16- and 8-byte
// alignment: on an 8-byte row the thread loads the aligned quad c+2..c+5 and
// takes c..c+1 (and c-1) from the previous lane.  Bands start on odd rows so
// the loaded rows' phases are the same in every band.
// Output rows per band (build option): a block loads R + 2 rows for R.
// 16386^2, T = 10: R = 4 6.45 TB/s, 6 6.27, 8 6.07, 12 5.66 (more registers,
// fewer blocks per SM) -- the halo rows come from L2 (DRAM bytes 0.98x).
#ifndef PK_J2R
#define PK_J2R 4
#endif
constexpr int kJ2Warps = 4, kJ2R = PK_J2R;

struct RowQ {
    int4 q;  // row[c .. c+3]
    int l, r;  // row[c-1], row[c+4]
};

// EDGE: the block touches a border (columns outside [0, N) or [1, J], rows
// outside [lo, hi)) and takes the guarded loads / stores; interior blocks
// (all but the first / last column block and the last band) run unguarded.
// PH2: N = 2 (mod 4), loaded row u is 8-byte aligned iff u is odd.
template <bool WIDE, bool PH2, bool EDGE>
__device__ __forceinline__ void j2r_store(int *o, int64_t c, int64_t J, bool full, bool ph, int v0, int v1,
                                          int v2, int v3) {
    if (full) {
        if (!ph) {
            *reinterpret_cast<int4 *>(o) = make_int4(v0, v1, v2, v3);
        } else {
            *reinterpret_cast<int2 *>(o) = make_int2(v0, v1);
            *reinterpret_cast<int2 *>(o + 2) = make_int2(v2, v3);
        }
    } else {
        if (c >= 1 && c <= J) o[0] = v0;
        if (c + 1 >= 1 && c + 1 <= J) o[1] = v1;
        if (c + 2 >= 1 && c + 2 <= J) o[2] = v2;
        if (c + 3 >= 1 && c + 3 <= J) o[3] = v3;
    }
}

template <bool WIDE, bool PH2, bool EDGE, bool PEER = false>
__device__ __forceinline__ void j2r_compute(const RowQ (&rows)[kJ2R + 2], int *__restrict__ d, int64_t N,
                                            int64_t i0, int64_t c, int64_t lo, int64_t hi, int64_t J,
                                            const PeerSweep *P = nullptr) {
    const bool full = !EDGE || (c >= 1 && c + 3 <= J);
#pragma unroll
    for (int u = 0; u < kJ2R; u++) {
        const int64_t i = i0 + u;
        if (EDGE && (i < lo || i >= hi)) continue;
        const bool ph = PH2 && !(u & 1);  // phase of row i (loaded row u + 1)
        const RowQ &up = rows[u], &cur = rows[u + 1], &dn = rows[u + 2];
        const int v0 = r_avg5<WIDE>(up.q.x, dn.q.x, cur.l, cur.q.y, cur.q.x);
        const int v1 = r_avg5<WIDE>(up.q.y, dn.q.y, cur.q.x, cur.q.z, cur.q.y);
        const int v2 = r_avg5<WIDE>(up.q.z, dn.q.z, cur.q.y, cur.q.w, cur.q.z);
        const int v3 = r_avg5<WIDE>(up.q.w, dn.q.w, cur.q.z, cur.r, cur.q.w);
        j2r_store<WIDE, PH2, EDGE>(d + i * N + c, c, J, full, ph, v0, v1, v2, v3);
        if (PEER) {  // the neighbours' ghost rows: our first and last output row
            if (P->left_dst && i == lo) j2r_store<WIDE, PH2, EDGE>(P->left_dst + i * N + c, c, J, full, ph, v0, v1, v2, v3);
            if (P->right_dst && i == hi - 1)
                j2r_store<WIDE, PH2, EDGE>(P->right_dst + i * N + c, c, J, full, ph, v0, v1, v2, v3);
        }
    }
}

template <bool PH2, bool EDGE, bool PEER = false, bool COH = false>
__device__ __forceinline__ void j2r_band(const int *__restrict__ s, int *__restrict__ d, int64_t N, int64_t i0,
                                         int64_t c, int64_t lo, int64_t hi, int64_t J, bool narrow,
                                         const PeerSweep *P = nullptr) {
    constexpr int R = kJ2R;
    const int lane = threadIdx.x & 31;
    const int nl = EDGE ? (int)min((int64_t)R + 2, hi + 1 - (i0 - 1)) : R + 2;  // rows i0-1 .. min(i0+R, hi)
    int4 raw[R + 2], ext[R + 2];
    const int *rp = s + (i0 - 1) * N + c;
#pragma unroll
    for (int u = 0; u < R + 2; u++) {
        const int sh = (PH2 && (u & 1)) ? 2 : 0;
        if (!EDGE)
            raw[u] = ldq<COH>(rp + sh);
        else if (u < nl)
            raw[u] = ldq_guard<COH>(rp - c, c + sh, N);
        rp += N;
    }
    // the quads across the warp edges after the warp's own loads (L1 hits then)
    rp = s + (i0 - 1) * N + c;
#pragma unroll
    for (int u = 0; u < R + 2; u++) {
        const bool ph = PH2 && (u & 1);
        const int sh = ph ? 2 : 0;
        if (!EDGE) {
            if (lane == 0) ext[u] = ldq<COH>(rp - 4 + sh);
            if (lane == 31 && !ph) ext[u].x = ld1<COH>(rp + 4);
        } else if (u < nl) {
            if (lane == 0) ext[u] = ldq_guard<COH>(rp - c, c - 4 + sh, N);
            if (lane == 31 && !ph) ext[u].x = ld1_guard<COH>(rp - c, c + 4, N);
        }
        rp += N;
    }
    RowQ rows[R + 2];
#pragma unroll
    for (int u = 0; u < R + 2; u++) {
        const bool ph = PH2 && (u & 1);
        const int4 v = raw[u];
        if (!ph) {
            rows[u].q = v;
            int l = __shfl_up_sync(0xffffffffu, v.w, 1), r = __shfl_down_sync(0xffffffffu, v.x, 1);
            if (lane == 0) l = ext[u].w;
            if (lane == 31) r = ext[u].x;
            rows[u].l = l;
            rows[u].r = r;
        } else {
            int py = __shfl_up_sync(0xffffffffu, v.y, 1), pz = __shfl_up_sync(0xffffffffu, v.z, 1),
                pw = __shfl_up_sync(0xffffffffu, v.w, 1);
            if (lane == 0) {
                py = ext[u].y;
                pz = ext[u].z;
                pw = ext[u].w;
            }
            rows[u].q = make_int4(pz, pw, v.x, v.y);
            rows[u].l = py;
            rows[u].r = v.z;
        }
    }
    if (narrow)
        j2r_compute<false, PH2, EDGE, PEER>(rows, d, N, i0, c, lo, hi, J, P);
    else
        j2r_compute<true, PH2, EDGE, PEER>(rows, d, N, i0, c, lo, hi, J, P);
}

template <bool PH2, bool PEER = false>
__global__ void __launch_bounds__(kJ2Warps * 32) k_jacobi2d_reg(const int *__restrict__ s, int *__restrict__ d,
                                                                int64_t N, int64_t rs, int64_t lo, int64_t hi,
                                                                int64_t J, int64_t ncb, const int *flag, int mode,
                                                                PeerSweep P = PeerSweep{}) {
    const bool narrow = r_narrow(mode, flag);
    const int64_t cb = blockIdx.x % ncb, rbi = blockIdx.x / ncb;
    // PEER: the last band (it holds row hi - 1) runs first, then band 0 (row lo)
    const int64_t nrb = gridDim.x / ncb;
    const int64_t rb = !PEER ? rbi : (rbi == 0 ? nrb - 1 : rbi - 1);
    const bool pl = PEER && rb == 0 && P.left_dst, pr = PEER && rb == nrb - 1 && P.right_dst;
    if (PEER && (pl || pr)) peer_wait(P, pl, pr);
    const int64_t cblk = cb * (kJ2Warps * 128);  // first column of the block
    const int64_t c = cblk + (threadIdx.x >> 5) * 128 + 4 * (threadIdx.x & 31);
    const int64_t i0 = rs + rb * kJ2R;  // odd: loaded row u has the phase of u
    const bool interior = cblk >= 4 && cblk + kJ2Warps * 128 + 8 <= N && cblk + kJ2Warps * 128 <= J + 1 &&
                          i0 >= lo && i0 + kJ2R <= hi;
    if (PEER && (pl || pr)) {  // the bands reading a ghost row a neighbour stores: coherent loads
        if (interior)
            j2r_band<PH2, false, PEER, true>(s, d, N, i0, c, lo, hi, J, narrow, &P);
        else
            j2r_band<PH2, true, PEER, true>(s, d, N, i0, c, lo, hi, J, narrow, &P);
    } else if (interior) {
        j2r_band<PH2, false, PEER>(s, d, N, i0, c, lo, hi, J, narrow, &P);
    } else {
        j2r_band<PH2, true, PEER>(s, d, N, i0, c, lo, hi, J, narrow, &P);
    }
    if (PEER && (pl || pr)) peer_signal(P, pl, pr);
}

}  // namespace

// PK_OK when the register-window sweep ran, kNotTaken when the layout is not
// one it takes (the caller then uses the shared-memory pipeline), else a
// PK_E_* code.
int sweep1d_reg(const int *src, int *dst, int64_t lo, int64_t hi, int64_t N, const int *flag, int mode,
                cudaStream_t st) {
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3u) != 0) return kNotTaken;
    if (hi <= lo) return PK_OK;
    const int so = (int)((reinterpret_cast<uintptr_t>(src) >> 2) & 3);
    const int dof = (int)((reinterpret_cast<uintptr_t>(dst) >> 2) & 3);
    const int64_t xa = (4 - dof) & 3;               // dst + xa is 16-byte aligned
    const int D = (dof - so) & 3;                   // src + x + D is 16-byte aligned
    const int64_t q0 = (lo - xa) >= 0 ? (lo - xa) / 4 : -((xa - lo + 3) / 4);  // floor
    const int64_t q1 = (hi - 1 - xa) >= 0 ? (hi - 1 - xa) / 4 : -1;
    const int64_t nq = q1 - q0 + 1;
    if (nq <= 0) return PK_OK;
    const int64_t per_block = (int64_t)kJ1Threads * kJ1K;
    const int64_t blocks = ceil_div(nq, per_block);
    if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi: grid too large");
    switch (D) {
    case 0: k_jacobi1d_reg<0><<<(unsigned)blocks, kJ1Threads, 0, st>>>(src, dst, xa, q0, lo, hi, N, flag, mode); break;
    case 1: k_jacobi1d_reg<1><<<(unsigned)blocks, kJ1Threads, 0, st>>>(src, dst, xa, q0, lo, hi, N, flag, mode); break;
    case 2: k_jacobi1d_reg<2><<<(unsigned)blocks, kJ1Threads, 0, st>>>(src, dst, xa, q0, lo, hi, N, flag, mode); break;
    default: k_jacobi1d_reg<3><<<(unsigned)blocks, kJ1Threads, 0, st>>>(src, dst, xa, q0, lo, hi, N, flag, mode); break;
    }
    return after_launch("jacobi1d_reg");
}

int sweep2d_reg(const int *src, int *dst, int64_t lo, int64_t hi, int64_t J, int64_t N, const int *flag, int mode,
                cudaStream_t st) {
    // rows must sit at phase 0 or 2: both halves 16-byte aligned and N even
    if ((N & 1) || !aligned16(src) || !aligned16(dst)) return kNotTaken;
    if (hi <= lo || J <= 0) return PK_OK;
    const int64_t rs = (lo & 1) ? lo : lo - 1;  // bands start on odd rows
    const int64_t nrb = ceil_div(hi - rs, kJ2R);
    const int64_t nq = (J + 1 + 3) / 4;  // column quads covering 0 .. J
    const int64_t ncb = ceil_div(nq, 32 * kJ2Warps);
    if (nrb * ncb > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi2d: grid too large");
    if ((N & 3) == 2)
        k_jacobi2d_reg<true><<<(unsigned)(nrb * ncb), kJ2Warps * 32, 0, st>>>(src, dst, N, rs, lo, hi, J, ncb,
                                                                             flag, mode);
    else
        k_jacobi2d_reg<false><<<(unsigned)(nrb * ncb), kJ2Warps * 32, 0, st>>>(src, dst, N, rs, lo, hi, J, ncb,
                                                                              flag, mode);
    return after_launch("jacobi2d_reg");
}

// Fused sweep + halo exchange: the register-window sweep with the edge
// blocks storing into the neighbours' buffers and ordering against them.
// R: remote dst halves already offset; counters; steps run so far.
int sweep_reg_peer(bool two_d, const int *src, int *dst, int64_t lo, int64_t hi, int64_t J, int64_t N, int mode,
                   const PeerHost &R, cudaStream_t st) {
    if (hi <= lo) return PK_OK;
    PeerSweep P;
    P.left_dst = R.left_dst;
    P.right_dst = R.right_dst;
    P.wait_left = R.wait_left;
    P.wait_right = R.wait_right;
    P.sig_left = R.sig_left;
    P.sig_right = R.sig_right;
    P.error = R.error;
    if (!two_d) {
        if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3u) != 0)
            return fail(PK_E_UNSUPPORTED, "jacobi peer sweep: halves not 4-byte aligned");
        const int so = (int)((reinterpret_cast<uintptr_t>(src) >> 2) & 3);
        const int dof = (int)((reinterpret_cast<uintptr_t>(dst) >> 2) & 3);
        const int64_t xa = (4 - dof) & 3;
        const int D = (dof - so) & 3;
        const int64_t q0 = (lo - xa) >= 0 ? (lo - xa) / 4 : -((xa - lo + 3) / 4);
        const int64_t q1 = (hi - 1 - xa) >= 0 ? (hi - 1 - xa) / 4 : -1;
        const int64_t blocks = ceil_div(q1 - q0 + 1, (int64_t)kJ1Threads * kJ1K);
        if (blocks > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi: grid too large");
        P.target = (unsigned)(1 * R.step);  // one edge block per side and step
        switch (D) {
        case 0: k_jacobi1d_reg<0, true><<<(unsigned)blocks, kJ1Threads, 0, st>>>(src, dst, xa, q0, lo, hi, N, nullptr, mode, P); break;
        case 1: k_jacobi1d_reg<1, true><<<(unsigned)blocks, kJ1Threads, 0, st>>>(src, dst, xa, q0, lo, hi, N, nullptr, mode, P); break;
        case 2: k_jacobi1d_reg<2, true><<<(unsigned)blocks, kJ1Threads, 0, st>>>(src, dst, xa, q0, lo, hi, N, nullptr, mode, P); break;
        default: k_jacobi1d_reg<3, true><<<(unsigned)blocks, kJ1Threads, 0, st>>>(src, dst, xa, q0, lo, hi, N, nullptr, mode, P); break;
        }
        return after_launch("jacobi1d_reg_peer");
    }
    if ((N & 1) || !aligned16(src) || !aligned16(dst))
        return fail(PK_E_UNSUPPORTED, "jacobi2d peer sweep: needs even N and 16-byte aligned halves");
    if (J <= 0) return PK_OK;
    const int64_t rs = (lo & 1) ? lo : lo - 1;
    const int64_t nrb = ceil_div(hi - rs, kJ2R);
    const int64_t ncb = ceil_div((J + 1 + 3) / 4, 32 * kJ2Warps);
    if (nrb * ncb > 0x7fffffffLL) return fail(PK_E_UNSUPPORTED, "jacobi2d: grid too large");
    P.target = (unsigned)(ncb * R.step);  // one band of ncb edge blocks per side and step
    if ((N & 3) == 2)
        k_jacobi2d_reg<true, true><<<(unsigned)(nrb * ncb), kJ2Warps * 32, 0, st>>>(src, dst, N, rs, lo, hi, J, ncb,
                                                                                   nullptr, mode, P);
    else
        k_jacobi2d_reg<false, true><<<(unsigned)(nrb * ncb), kJ2Warps * 32, 0, st>>>(src, dst, N, rs, lo, hi, J, ncb,
                                                                                    nullptr, mode, P);
    return after_launch("jacobi2d_reg_peer");
}

}  // namespace pk
