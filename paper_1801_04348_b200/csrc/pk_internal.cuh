// pk_internal.cuh -- shared helpers for libpk (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "pk.h"

namespace pk {

// Records the error text for pk_last_error() on this thread; returns code.
int fail(int code, const char *fmt, ...);

extern std::atomic<int64_t> g_launches;

// After a <<<>>> launch: surface configuration errors, count the launch.
inline int after_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(PK_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return PK_OK;
}

// Pageable host buffers inside pk_run_host_io (pk_staging.cu).
bool host_is_pinned(const void *p);
void parallel_copy(void *dst, const void *src, size_t bytes);  // host memcpy on the staging thread pool
class StageSession {
  public:
    explicit StageSession(int device);
    ~StageSession();
    // src (pageable) -> dst (device) through the pinned ring, DMA on st; with
    // copy_dst, the same pass also copies src there (the caller's result copy)
    int h2d(void *dst, const void *src, size_t bytes, cudaStream_t st, void *copy_dst = nullptr);
    // device src -> pinned staging at stage_off (reserve_out first) on st;
    // copied on to dst (pageable) by drain()
    int reserve_out(size_t bytes);
    int d2h(void *dst, size_t stage_off, const void *src, size_t bytes, cudaStream_t st);
    int drain();

  private:
    struct Drain {
        cudaEvent_t ev;
        const char *stage;
        char *dst;
        size_t bytes;
    };
    int device_;
    std::vector<Drain> drains_;
};

// Opt a kernel into more than 48 KB of dynamic shared memory.
int allow_smem(const void *kernel, size_t bytes);

// Stream-ordered scratch allocation from the current device's default pool,
// which is told (once per device) to keep freed memory: workspaces are
// re-used across calls instead of being unmapped at every synchronisation.
cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st);

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t max0(int64_t v) { return v > 0 ? v : 0; }

// --- device helpers ----------------------------------------------------------

// Streaming 128-bit load that does not allocate in L1 (read-once data).
__device__ __forceinline__ int4 ld_stream(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(int4 *p, const int4 &v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w));
}

// --- TMA bulk copies (cp.async.bulk) completed on an mbarrier ----------------
// Global source and shared destination 16-byte aligned, size a multiple of 16.

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make barrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order earlier generic-proxy shared accesses before later async-proxy writes
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// mbarrier wait with a suspend-time hint (ns): the thread sleeps in the
// barrier instead of re-polling.  For the producer warp's empty-stage waits
// (paired A/B on one B200: Big1P at n = 2048 0.820 -> 0.835 of peak at 1 us,
// same at 0.5 / 2 us); a thread-0 producer polls (the hint cost the 128 x 64
// tile 1.6 % at n = 8192 before it had a producer warp).
__device__ __forceinline__ void mbar_wait_hint(uint64_t *bar, uint32_t parity, uint32_t hint_ns) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
            : "memory");
}

// Asynchronous 16-byte global -> shared copy (cp.async.cg); bytes < 16
// zero-fills the rest of the destination (0: a pure zero fill).
__device__ __forceinline__ void cp_async16(void *dst_smem, const void *src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Truncating integer division of an exact (64-bit) sum, as the reference's
// c_div (interp.py:43-46): C division already truncates toward zero.
__device__ __forceinline__ int div3(long long s) { return (int)(s / 3); }
__device__ __forceinline__ int div5(long long s) { return (int)(s / 5); }

// --- per-family host launchers (one .cu each) ---------------------------------
int launch_reverse(const pk_launch_t &L, void *const *p, cudaStream_t st);
int launch_transpose(const pk_launch_t &L, void *const *p, cudaStream_t st);
int launch_jacobi1d(const pk_launch_t &L, void *const *p, cudaStream_t st);
int launch_jacobi2d(const pk_launch_t &L, void *const *p, cudaStream_t st);
int sweep_jacobi1d(const pk_launch_t &L, const void *src, void *dst, int64_t lo, int64_t hi,
                   cudaStream_t st);
int sweep_jacobi2d(const pk_launch_t &L, const void *src, void *dst, int64_t lo, int64_t hi,
                   cudaStream_t st);
int jacobi_narrow(const pk_launch_t &L, const void *a, int *narrow, cudaStream_t st);
int jacobi1d_temporal_pass(const pk_launch_t &L, int *a, int64_t lo, int64_t hi, int64_t P, int64_t t0, int h,
                           const int *flag, int mode, cudaStream_t st);
int jacobi2d_temporal_pass(const pk_launch_t &L, int *a, int64_t lo, int64_t hi, int64_t I, int64_t J, int64_t t0,
                           int h, const int *flag, int mode, cudaStream_t st);
// register-window sweeps (k_jacobi_reg.cu): kNotTaken when the layout is not theirs
constexpr int kNotTaken = -1;
int sweep1d_reg(const int *src, int *dst, int64_t lo, int64_t hi, int64_t N, const int *flag, int mode,
                cudaStream_t st);
int sweep2d_reg(const int *src, int *dst, int64_t lo, int64_t hi, int64_t J, int64_t N, const int *flag, int mode,
                cudaStream_t st);
// fused sweep + halo exchange over peer memory (k_jacobi_reg.cu)
struct PeerHost {
    int *left_dst, *right_dst;               // neighbours' dst halves, mapped (nullptr: none)
    const unsigned *wait_left, *wait_right;  // this rank's counters
    unsigned *sig_left, *sig_right;          // neighbours' counters, mapped
    unsigned *error;                         // set by a wait that gave up
    int64_t step;                            // steps run since the counters were zeroed
};
int sweep_reg_peer(bool two_d, const int *src, int *dst, int64_t lo, int64_t hi, int64_t J, int64_t N, int mode,
                   const PeerHost &R, cudaStream_t st);
int jacobi_sweep_peer(const pk_launch_t &L, int *a, int64_t step, int64_t lo, int64_t hi, const pk_peer_t &P,
                      cudaStream_t st);
int launch_matvec(const pk_launch_t &L, void *const *p, cudaStream_t st);
int launch_matmul(const pk_launch_t &L, void *const *p, cudaStream_t st);
bool matmul_tma_fits(int64_t BM_case, int64_t BN_case, int64_t rows, int64_t Nc, int64_t K, int64_t n);
int launch_matmul_tma(const float *a, const float *b, float *c, int64_t n, int64_t rlo, int64_t rhi, int64_t Nc,
                      int64_t K, int bm, int bn, cudaStream_t st);
bool matmul_kslice_ok(const pk_launch_t &L, int64_t slice);
int launch_matmul_kslice(const pk_launch_t &L, void *const *p, int64_t k0, int64_t k1, cudaStream_t st);
int launch_matmul_tf32x3(const float *a, const float *b, float *c, int64_t n, int64_t rlo, int64_t rhi,
                         int64_t Nc, int64_t K, cudaStream_t st);
int launch_addition(const pk_launch_t &L, void *const *p, cudaStream_t st);
// one thread block of the program (run_block) on any dtype (k_block.cu)
int launch_block(const pk_launch_t &L, const int64_t *grid, int ngrid, const int64_t *ctx, int nctx, void *const *p,
                 cudaStream_t st);
// the Jacobi programs on int64 / binary64 data: per-step sweeps (k_block.cu)
int launch_jacobi_wide(const pk_launch_t &L, void *const *p, cudaStream_t st);

// Shared-memory words staged per block (0 for direct variants).
int64_t footprint_words(const pk_launch_t &L);

// Bytes per array element of a launch (PK_DTYPE_*).
inline int elem_bytes(const pk_launch_t &L) {
    return (L.dtype == PK_DTYPE_I64 || L.dtype == PK_DTYPE_F64) ? 8 : 4;
}

// Elements per thread along the s axis: 1 once granularity removed the loop.
inline int64_t elems(const pk_launch_t &L) {
    return (L.flags & PK_FLAG_GRANULARITY) ? 1 : L.s;
}

// Clamp [lo, hi) of a partitioned launch to the covered units [ulo, uhi).
inline void unit_range(const pk_launch_t &L, int64_t ulo, int64_t uhi, int64_t *lo, int64_t *hi) {
    int64_t a = ulo, b = uhi;
    if (L.hi > 0) {
        a = L.lo > ulo ? L.lo : ulo;
        b = L.hi < uhi ? L.hi : uhi;
    }
    *lo = a;
    *hi = b > a ? b : a;
}

}  // namespace pk
