// pk_abi.cu -- the C ABI of libpk (include/pk.h): device-property lookup,
// validation, dispatch to the family launchers, and the host-buffer path.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "pk_internal.cuh"

namespace pk {

std::atomic<int64_t> g_launches{0};

namespace {
thread_local char t_err[1024] = "";
}

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(t_err, sizeof(t_err), fmt, ap);
    va_end(ap);
    return code;
}

int allow_smem(const void *kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return PK_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if ((long long)bytes > optin)
        return fail(PK_E_PARAM,
                    "staged tile needs %zu bytes of shared memory but the device allows %d per "
                    "block (Z_B); the case discussion selects a caching-off leaf here",
                    bytes, optin);
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return fail(PK_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return PK_OK;
}

cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t st) {
    static std::once_flag once[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64) {
        std::call_once(once[dev], [dev]() {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        });
    }
    return cudaMallocAsync(p, bytes ? bytes : 4, st);
}

int64_t footprint_words(const pk_launch_t &L) {
    if (L.variant != PK_VARIANT_STAGED) return 0;
    const int64_t E = elems(L);
    switch (L.family) {
        case PK_FAMILY_REVERSE: return E * L.B;
        case PK_FAMILY_TRANSPOSE: return E * L.B1 * (L.B0 | 1);
        case PK_FAMILY_JACOBI1D: return E * L.B + 2;
        case PK_FAMILY_JACOBI2D: return (L.B0 + 2) * (E * L.B1 + 2);
        case PK_FAMILY_MATVEC: return L.N;
        case PK_FAMILY_MATMUL: return L.B0 * L.B0 + L.B0 * L.ub1 * (E < 8 ? E : 8);
        default: return 0;
    }
}

namespace {

struct ArraySpec {
    int count;
    int64_t elems[3];
    bool written[3];
};

int array_spec(const pk_launch_t &L, ArraySpec *s) {
    const int64_t N = L.N > 0 ? L.N : 0;
    switch (L.family) {
        case PK_FAMILY_REVERSE: *s = {2, {N, N, 0}, {false, true, false}}; return PK_OK;
        case PK_FAMILY_TRANSPOSE: *s = {2, {N * N, N * N, 0}, {false, true, false}}; return PK_OK;
        case PK_FAMILY_JACOBI1D: *s = {1, {2 * N, 0, 0}, {true, false, false}}; return PK_OK;
        case PK_FAMILY_JACOBI2D: *s = {1, {2 * N * N, 0, 0}, {true, false, false}}; return PK_OK;
        case PK_FAMILY_MATVEC: *s = {3, {N * N, N, N}, {false, false, true}}; return PK_OK;
        case PK_FAMILY_MATMUL: *s = {3, {N * N, N * N, N * N}, {false, false, true}}; return PK_OK;
        case PK_FAMILY_ADDITION: *s = {3, {N * N, N * N, N * N}, {false, false, true}}; return PK_OK;
        default: return fail(PK_E_UNSUPPORTED, "unknown program family %d", L.family);
    }
}

// Element range of array i a partitioned launch (lo/hi) reads or writes, so
// pk_run_host moves only a rank's share across PCIe: rows of the row-sharded
// operands, the mirrored range for reversal, everything for the stencils.
void array_range(const pk_launch_t &L, int i, int64_t elems, int64_t *off, int64_t *cnt) {
    *off = 0;
    *cnt = elems;
    if (L.hi <= 0) return;
    const int64_t N = L.N > 0 ? L.N : 0, lo = L.lo > 0 ? L.lo : 0, hi = L.hi;
    int64_t a = 0, b = elems;
    switch (L.family) {
        case PK_FAMILY_REVERSE:
            if (i == 0) { a = lo; b = hi; } else { a = N - hi; b = N - lo; }
            break;
        case PK_FAMILY_TRANSPOSE:
            if (i == 1) { a = lo * N; b = hi * N; }
            break;
        case PK_FAMILY_MATVEC:
            if (i == 0) { a = lo * N; b = hi * N; } else if (i == 2) { a = lo; b = hi; }
            break;
        case PK_FAMILY_MATMUL:
            if (i != 1) { a = lo * N; b = hi * N; }
            break;
        case PK_FAMILY_ADDITION:
            a = lo * N;
            b = hi * N;
            break;
        default:
            break;
    }
    if (a < 0) a = 0;
    if (b > elems) b = elems;
    *off = a;
    *cnt = b > a ? b - a : 0;
}

// Elements of each array a launch touches: 1 + the largest flat index it
// reads or writes over its covered index sets (the reference raises
// IndexError for any access past the end, interp.py:209-212), 0 for an
// array it never touches.  The stencils count their whole double buffer
// (their value-range pre-pass reads it).
int required_elems(const pk_launch_t &L, int64_t need[3]) {
    need[0] = need[1] = need[2] = 0;
    const int64_t N = L.N;
    if (N <= 0) return PK_OK;
    int64_t lo, hi;
    switch (L.family) {
        case PK_FAMILY_REVERSE: {
            if (L.s * L.B == 0) return fail(PK_E_DIV0, "reverse: s*B == 0 in dim = N / (s * B)");
            if (L.s < 0 || L.B < 0) return PK_OK;
            unit_range(L, 0, max0(N / (L.s * L.B)) * L.s * L.B, &lo, &hi);
            if (hi > lo) need[0] = hi, need[1] = N - lo;
            return PK_OK;
        }
        case PK_FAMILY_TRANSPOSE: {
            if (L.B0 == 0 || L.s * L.B1 == 0) return fail(PK_E_DIV0, "transpose: zero divisor in dim0 / dim1");
            if (L.B0 < 0 || L.B1 < 0 || L.s < 0) return PK_OK;
            const int64_t J = max0(N / (L.s * L.B1)) * L.s * L.B1;
            unit_range(L, 0, max0(N / L.B0) * L.B0, &lo, &hi);
            if (hi > lo && J > 0) need[0] = (J - 1) * N + hi, need[1] = (hi - 1) * N + J;
            return PK_OK;
        }
        case PK_FAMILY_JACOBI1D:
        case PK_FAMILY_JACOBI2D: {
            const bool two = L.family == PK_FAMILY_JACOBI2D;
            const int64_t tile = two ? L.B0 : L.s * L.B;
            if (tile == 0 || (two && L.s * L.B1 == 0)) return fail(PK_E_DIV0, "jacobi: zero divisor in dim");
            if (L.T <= 0 || L.s < 0 || L.B < 0 || L.B0 < 0 || L.B1 < 0) return PK_OK;
            const int64_t P = max0((N - 2) / tile) * tile;
            const int64_t J = two ? max0((N - 2) / (L.s * L.B1)) * L.s * L.B1 : 1;
            if (P > 0 && J > 0) need[0] = two ? 2 * N * N : 2 * N;
            return PK_OK;
        }
        case PK_FAMILY_MATVEC: {
            if (L.s * L.B == 0) return fail(PK_E_DIV0, "matvec: s*B == 0 in dim = N / (s * B)");
            if (L.s < 0 || L.B < 0) return PK_OK;
            unit_range(L, 0, max0(N / (L.s * L.B)) * L.s * L.B, &lo, &hi);
            if (hi > lo) need[0] = hi * N, need[1] = N, need[2] = hi;
            return PK_OK;
        }
        case PK_FAMILY_MATMUL: {
            if (L.B0 == 0 || L.ub1 * L.s == 0) return fail(PK_E_DIV0, "matmul: zero divisor in dim0 / dim1");
            if (L.B0 < 0 || L.ub1 < 0 || L.s < 0) return PK_OK;
            const int64_t K = max0(N / L.B0) * L.B0, Nc = max0(N / (L.ub1 * L.s)) * L.ub1 * L.s;
            unit_range(L, 0, K, &lo, &hi);  // rows p < dim0*B0 == kdim*B0
            if (hi > lo && Nc > 0 && K > 0)
                need[0] = (hi - 1) * N + K, need[1] = (K - 1) * N + Nc, need[2] = (hi - 1) * N + Nc;
            return PK_OK;
        }
        case PK_FAMILY_ADDITION: {
            const bool merged = (L.flags & PK_FLAG_MERGED) != 0;
            if (L.B0 == 0 || L.B1 == 0) return fail(PK_E_DIV0, "addition: zero divisor in dim0 / dim1");
            if (L.B0 < 0 || L.B1 < 0) return PK_OK;
            int64_t J = merged ? max0(N / L.B1) * L.B1 : max0(N / (2 * L.B1)) * L.B1;
            if (!merged && J > N / 2) J = N / 2;
            unit_range(L, 0, max0(N / L.B0) * L.B0, &lo, &hi);
            if (hi > lo && J > 0) need[0] = need[1] = need[2] = (hi - 1) * N + (merged ? J : N / 2 + J);
            return PK_OK;
        }
        default: return fail(PK_E_UNSUPPORTED, "unknown program family %d", L.family);
    }
}

int dispatch(const pk_launch_t &L, void *const *p, cudaStream_t st) {
    switch (L.family) {
        case PK_FAMILY_REVERSE: return launch_reverse(L, p, st);
        case PK_FAMILY_TRANSPOSE: return launch_transpose(L, p, st);
        case PK_FAMILY_JACOBI1D: return L.dtype == PK_DTYPE_I32 ? launch_jacobi1d(L, p, st) : launch_jacobi_wide(L, p, st);
        case PK_FAMILY_JACOBI2D: return L.dtype == PK_DTYPE_I32 ? launch_jacobi2d(L, p, st) : launch_jacobi_wide(L, p, st);
        case PK_FAMILY_MATVEC: return launch_matvec(L, p, st);
        case PK_FAMILY_MATMUL: return launch_matmul(L, p, st);
        case PK_FAMILY_ADDITION: return launch_addition(L, p, st);
        default: return fail(PK_E_UNSUPPORTED, "unknown program family %d", L.family);
    }
}

int validate(const pk_launch_t *L, int nptrs) {
    if (!L) return fail(PK_E_PARAM, "null launch descriptor");
    ArraySpec s;
    int rc = array_spec(*L, &s);
    if (rc) return rc;
    if (nptrs != s.count)
        return fail(PK_E_PARAM, "family %d takes %d arrays, got %d", L->family, s.count, nptrs);
    if (L->variant != PK_VARIANT_STAGED && L->variant != PK_VARIANT_DIRECT)
        return fail(PK_E_UNSUPPORTED, "unknown variant %d", L->variant);
    const bool stencil = L->family == PK_FAMILY_JACOBI1D || L->family == PK_FAMILY_JACOBI2D;
    if (L->dtype < PK_DTYPE_I32 || L->dtype > PK_DTYPE_F64 || (stencil && L->dtype == PK_DTYPE_F32))
        return fail(PK_E_UNSUPPORTED, "dtype %d not provided for family %d", L->dtype, L->family);
    if ((L->flags & PK_FLAG_TF32X3) && !(L->family == PK_FAMILY_MATMUL && L->dtype == PK_DTYPE_F32))
        return fail(PK_E_UNSUPPORTED, "3xTF32 applies to float32 matmul only");
    if ((L->flags & PK_FLAG_TEMPORAL) && !(stencil && L->dtype == PK_DTYPE_I32))
        return fail(PK_E_UNSUPPORTED, "temporal blocking is provided for the int32 Jacobi programs only");
    return PK_OK;
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_version(void) { return (1 << 16) | 2; }  // 1.2: 8-byte dtypes, pk_launch_checked, pk_required_elems

const char *pk_last_error(void) { return t_err; }

int64_t pk_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int64_t pk_footprint_words(const pk_launch_t *L) { return L ? footprint_words(*L) : 0; }

int pk_query_machine(int device, pk_machine_t *out) {
    if (!out) return fail(PK_E_PARAM, "null pk_machine_t");
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return fail(PK_E_CUDA, "cudaGetDeviceProperties(%d): %s", device, cudaGetErrorString(e));
    memset(out, 0, sizeof(*out));
    out->device = device;
    out->cc_major = prop.major;
    out->cc_minor = prop.minor;
    out->sm_count = prop.multiProcessorCount;
    out->warp_size = prop.warpSize;
    out->max_threads_per_block = prop.maxThreadsPerBlock;
    out->max_threads_per_sm = prop.maxThreadsPerMultiProcessor;
    out->regs_per_thread = 255;  // architectural per-thread limit (not in cudaDeviceProp)
    out->regs_per_block = prop.regsPerBlock;
    out->regs_per_sm = prop.regsPerMultiprocessor;
    out->smem_per_block = (int64_t)prop.sharedMemPerBlock;
    out->smem_per_block_optin = (int64_t)prop.sharedMemPerBlockOptin;
    out->smem_per_sm = (int64_t)prop.sharedMemPerMultiprocessor;
    out->l2_bytes = prop.l2CacheSize;
    out->global_mem_bytes = (int64_t)prop.totalGlobalMem;
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, device);
    out->clock_khz = v;
    cudaDeviceGetAttribute(&v, cudaDevAttrMemoryClockRate, device);
    out->mem_clock_khz = v;
    cudaDeviceGetAttribute(&v, cudaDevAttrGlobalMemoryBusWidth, device);
    out->mem_bus_width_bits = v;
    strncpy(out->name, prop.name, sizeof(out->name) - 1);
    return PK_OK;
}

int pk_launch(const pk_launch_t *L, void *const *dev_ptrs, int nptrs, void *stream) {
    int rc = validate(L, nptrs);
    if (rc) return rc;
    for (int i = 0; i < nptrs; i++)
        if (!dev_ptrs || !dev_ptrs[i]) return fail(PK_E_PARAM, "array %d is a null pointer", i);
    return dispatch(*L, dev_ptrs, static_cast<cudaStream_t>(stream));
}

int pk_required_elems(const pk_launch_t *L, int64_t *need, int nneed) {
    if (!L || !need) return fail(PK_E_PARAM, "null argument");
    ArraySpec s;
    int rc = array_spec(*L, &s);
    if (rc) return rc;
    if (nneed < s.count) return fail(PK_E_PARAM, "family %d has %d arrays, room for %d", L->family, s.count, nneed);
    int64_t n[3];
    rc = required_elems(*L, n);
    if (rc) return rc;
    for (int i = 0; i < s.count; i++) need[i] = n[i];
    return PK_OK;
}

int pk_launch_checked(const pk_launch_t *L, void *const *dev_ptrs, const int64_t *elems, int nptrs, void *stream) {
    int rc = validate(L, nptrs);
    if (rc) return rc;
    if (!elems) return fail(PK_E_PARAM, "null element counts");
    int64_t need[3];
    rc = required_elems(*L, need);
    if (rc) return rc;
    static const char *names[7][3] = {{"a", "c", ""}, {"a", "c", ""}, {"a", "", ""}, {"a", "", ""},
                                      {"a", "x", "y"}, {"a", "b", "c"}, {"a", "b", "c"}};
    for (int i = 0; i < nptrs; i++)
        if (elems[i] < need[i])
            return fail(PK_E_BOUNDS, "access %s[%lld] out of bounds (size %lld)", names[L->family - 1][i],
                        (long long)(need[i] - 1), (long long)elems[i]);
    return pk_launch(L, dev_ptrs, nptrs, stream);
}

int pk_launch_block(const pk_launch_t *L, const int64_t *grid, int ngrid, const int64_t *ctx, int nctx,
                    void *const *dev_ptrs, int nptrs, void *stream) {
    int rc = validate(L, nptrs);
    if (rc) return rc;
    if (ngrid < 0 || ngrid > 2 || nctx < 0 || nctx > 1 || (ngrid && !grid) || (nctx && !ctx))
        return fail(PK_E_PARAM, "pk_launch_block: %d grid / %d context values", ngrid, nctx);
    for (int i = 0; i < nptrs; i++)
        if (!dev_ptrs || !dev_ptrs[i]) return fail(PK_E_PARAM, "array %d is a null pointer", i);
    return launch_block(*L, grid, ngrid, ctx, nctx, dev_ptrs, static_cast<cudaStream_t>(stream));
}

int pk_jacobi_sweep(const pk_launch_t *L, const void *src, void *dst, int64_t lo, int64_t hi,
                    void *stream) {
    if (!L || !src || !dst) return fail(PK_E_PARAM, "null argument");
    if (L->dtype != PK_DTYPE_I32) return fail(PK_E_UNSUPPORTED, "pk_jacobi_sweep: int32 only");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (L->family == PK_FAMILY_JACOBI1D) return sweep_jacobi1d(*L, src, dst, lo, hi, st);
    if (L->family == PK_FAMILY_JACOBI2D) return sweep_jacobi2d(*L, src, dst, lo, hi, st);
    return fail(PK_E_PARAM, "pk_jacobi_sweep: family %d is not a Jacobi stencil", L->family);
}

int pk_jacobi_sweep_peer(const pk_launch_t *L, void *a, int64_t step, int64_t lo, int64_t hi, const pk_peer_t *peer,
                         void *stream) {
    if (!L || !a || !peer) return fail(PK_E_PARAM, "null argument");
    if (L->family != PK_FAMILY_JACOBI1D && L->family != PK_FAMILY_JACOBI2D)
        return fail(PK_E_PARAM, "pk_jacobi_sweep_peer: family %d is not a Jacobi stencil", L->family);
    if (L->dtype != PK_DTYPE_I32) return fail(PK_E_UNSUPPORTED, "pk_jacobi_sweep_peer: int32 only");
    if (step < 0 || step >= ((int64_t)1 << 31)) return fail(PK_E_PARAM, "pk_jacobi_sweep_peer: step out of range");
    return jacobi_sweep_peer(*L, static_cast<int *>(a), step, lo, hi, *peer, static_cast<cudaStream_t>(stream));
}

namespace {
typedef int (*AddressRangeFn)(unsigned long long *, size_t *, unsigned long long);
}

int pk_ipc_export(const void *ptr, void *handle64, int64_t *offset) {
    if (!ptr || !handle64 || !offset) return fail(PK_E_PARAM, "null argument");
    // the allocation base (cudaIpcGetMemHandle takes a base pointer; torch's
    // caching allocator hands out addresses inside larger blocks)
    static const AddressRangeFn range = []() -> AddressRangeFn {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<AddressRangeFn>(p);
        return nullptr;
    }();
    if (!range) return fail(PK_E_CUDA, "cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)reinterpret_cast<uintptr_t>(ptr)) != 0)
        return fail(PK_E_PARAM, "pk_ipc_export: not a device allocation");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
    if (e != cudaSuccess) return fail(PK_E_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(handle64, &h, sizeof(h));
    *offset = (int64_t)(reinterpret_cast<uintptr_t>(ptr) - base);
    return PK_OK;
}

int pk_ipc_open(const void *handle64, int64_t offset, void **ptr) {
    if (!handle64 || !ptr || offset < 0) return fail(PK_E_PARAM, "bad argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    void *base = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(PK_E_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    *ptr = static_cast<char *>(base) + offset;
    return PK_OK;
}

int pk_ipc_close(void *ptr, int64_t offset) {
    if (!ptr || offset < 0) return fail(PK_E_PARAM, "bad argument");
    cudaError_t e = cudaIpcCloseMemHandle(static_cast<char *>(ptr) - offset);
    if (e != cudaSuccess) return fail(PK_E_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return PK_OK;
}

int pk_jacobi_narrow(const pk_launch_t *L, const void *a, int32_t *narrow, void *stream) {
    if (!L || !a || !narrow) return fail(PK_E_PARAM, "null argument");
    if (L->family != PK_FAMILY_JACOBI1D && L->family != PK_FAMILY_JACOBI2D)
        return fail(PK_E_PARAM, "pk_jacobi_narrow: family %d is not a Jacobi stencil", L->family);
    return jacobi_narrow(*L, a, narrow, static_cast<cudaStream_t>(stream));
}

namespace {

// Pipeline cut of pk_run_host (build options).  n = 8192 FP32 matmul e2e
// with the 128 x 64 producer-warp leaf: 8 x 4 22.1 ms, 12 x 4 21.1, 16 x 4
// 21.4, 12 x 6 20.85, 14 x 6 20.83, 16 x 6 20.93, 12 x 8 22.8 (chunks are
// whole 128-row multiples: 12 requested = 11 of 768 rows).  Finer uploads
// give the first chunks work sooner (tools/e2e_pipeline_model.py).
#ifndef PK_RH_CHUNKS
#define PK_RH_CHUNKS 12
#endif
#ifndef PK_RH_SLICES
#define PK_RH_SLICES 6
#endif
constexpr int kMaxChunks = PK_RH_CHUNKS;                  // pipeline depth limit of pk_run_host
constexpr int kMaxDevices = 64;                // pk_launch_multi
constexpr int64_t kChunkBytes = 48ll << 20;    // PCIe bytes per chunk (~1 ms of transfer)

// Units (rows, or elements for reversal) a host-buffer run may be cut into:
// families whose unit ranges touch disjoint slices of the streamed arrays.
// The stencils are not chunked (every step needs the whole array).
bool chunkable(const pk_launch_t &L) {
    switch (L.family) {
        case PK_FAMILY_REVERSE:
        case PK_FAMILY_TRANSPOSE:
        case PK_FAMILY_MATVEC:
        case PK_FAMILY_MATMUL:
        case PK_FAMILY_ADDITION: return true;
        default: return false;
    }
}

constexpr int kSlices = PK_RH_SLICES;  // reduction slices of matmul's first row chunk

struct HostRun {
    cudaStream_t h2d = nullptr, d2h = nullptr, cs[kMaxChunks] = {};
    cudaEvent_t ev[2 * kMaxChunks + kSlices] = {};
    void *dev[3] = {nullptr, nullptr, nullptr};
    int device = -1;
    bool timing = false;
};

// Streams and events of pk_run_host, kept per device and reused (creating
// and destroying a dozen streams and twenty events per call cost ~1 ms of a
// 23 ms n = 8192 run).  A run takes a set from the pool and returns it; a
// concurrent caller on another thread simply gets another set.
std::mutex g_run_mu;
std::vector<HostRun> g_run_pool;

cudaError_t host_run_acquire(int device, bool timing, HostRun *R) {
    {
        std::lock_guard<std::mutex> lock(g_run_mu);
        for (size_t i = 0; i < g_run_pool.size(); i++) {
            if (g_run_pool[i].device == device && g_run_pool[i].timing == timing) {
                *R = g_run_pool[i];
                g_run_pool.erase(g_run_pool.begin() + (long)i);
                return cudaSuccess;
            }
        }
    }
    R->device = device;
    R->timing = timing;
    cudaError_t e = cudaStreamCreateWithFlags(&R->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&R->d2h, cudaStreamNonBlocking);
    for (int k = 0; k < kMaxChunks && e == cudaSuccess; k++) e = cudaStreamCreateWithFlags(&R->cs[k], cudaStreamNonBlocking);
    for (int k = 0; k < 2 * kMaxChunks + kSlices && e == cudaSuccess; k++)
        e = cudaEventCreateWithFlags(&R->ev[k], timing ? cudaEventDefault : cudaEventDisableTiming);
    return e;
}

void host_run_release(HostRun &R, bool healthy) {
    for (void *&d : R.dev) d = nullptr;
    if (healthy) {
        std::lock_guard<std::mutex> lock(g_run_mu);
        if (g_run_pool.size() < 16) {
            g_run_pool.push_back(R);
            return;
        }
    }
    for (cudaEvent_t ev : R.ev)
        if (ev) cudaEventDestroy(ev);
    for (cudaStream_t s : R.cs)
        if (s) cudaStreamDestroy(s);
    for (cudaStream_t s : {R.h2d, R.d2h})
        if (s) cudaStreamDestroy(s);
}

}  // namespace

namespace {
int run_host_io(const pk_launch_t *L, const void *const *in_ptrs, void *const *out_ptrs, int nptrs, int device);
}

int pk_run_host_io(const pk_launch_t *L, const void *const *in_ptrs, void *const *out_ptrs, const int64_t *elems,
                   int nptrs, int device) {
    int rc = validate(L, nptrs);
    if (rc) return rc;
    if (!elems) return fail(PK_E_PARAM, "null element counts");
    int64_t need[3];
    rc = required_elems(*L, need);
    if (rc) return rc;
    ArraySpec spec;
    array_spec(*L, &spec);
    for (int i = 0; i < nptrs; i++) {
        // the run moves the declared extent of every array it is given
        const bool given = (in_ptrs && in_ptrs[i]) || (out_ptrs && out_ptrs[i]);
        const int64_t want = given ? spec.elems[i] : 0;
        if (elems[i] < need[i] || elems[i] < want)
            return fail(PK_E_BOUNDS, "array %d: %lld elements, the run touches %lld and copies %lld", i,
                        (long long)elems[i], (long long)need[i], (long long)want);
    }
    return run_host_io(L, in_ptrs, out_ptrs, nptrs, device);
}

int pk_run_host_checked(const pk_launch_t *L, void *const *host_ptrs, const int64_t *elems, int nptrs, int device) {
    return pk_run_host_io(L, reinterpret_cast<const void *const *>(host_ptrs), host_ptrs, elems, nptrs, device);
}

int pk_run_host(const pk_launch_t *L, void *const *host_ptrs, int nptrs, int device) {
    int rc = validate(L, nptrs);
    if (rc) return rc;
    return run_host_io(L, reinterpret_cast<const void *const *>(host_ptrs), host_ptrs, nptrs, device);
}

namespace {

int run_host_io(const pk_launch_t *L, const void *const *in_ptrs, void *const *out_ptrs, int nptrs, int device) {
    int rc = PK_OK;
    ArraySpec spec;
    array_spec(*L, &spec);
    const void *in[3] = {nullptr, nullptr, nullptr};
    void *out[3] = {nullptr, nullptr, nullptr};
    for (int i = 0; i < nptrs && i < 3; i++) {
        in[i] = in_ptrs ? in_ptrs[i] : nullptr;
        out[i] = out_ptrs ? out_ptrs[i] : nullptr;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(PK_E_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));

    // Cut the unit range into chunks so PCIe runs under the kernels: chunk k's
    // operands go up on the h2d stream while chunk k-1 computes (two compute
    // streams, so a chunk's kernel fills the previous one's tail) and chunk
    // k-2's results come down on the d2h stream.  Operands every chunk needs
    // whole (matmul's b, mat-vec's x, transpose's a) go up once, first.
    const int64_t N = L->N > 0 ? L->N : 0;
    const int64_t u0 = L->hi > 0 ? (L->lo > 0 ? L->lo : 0) : 0, u1 = L->hi > 0 ? L->hi : N;
    const int64_t eb = elem_bytes(*L);  // bytes per element
    int64_t unit_bytes = 0;  // streamed bytes per unit
    for (int i = 0; i < spec.count; i++) unit_bytes += (spec.written[i] ? 2 : 1) * (spec.elems[i] / (N > 0 ? N : 1)) * eb;
    int nchunks = 1;
    if (chunkable(*L) && u1 > u0 && unit_bytes > 0) {
        const int64_t total = (u1 - u0) * unit_bytes;
        nchunks = (int)(total / kChunkBytes);
        if (nchunks > kMaxChunks) nchunks = kMaxChunks;
        if (nchunks < 1) nchunks = 1;
    }
    int64_t step = (u1 - u0 + nchunks - 1) / nchunks;
    const int64_t align = L->family == PK_FAMILY_REVERSE ? 4096 : 128;  // whole tiles per chunk
    step = (step + align - 1) / align * align;
    if (step < 1) step = 1;
    nchunks = (int)((u1 - u0 + step - 1) / step);
    if (nchunks < 1) nchunks = 1;

    HostRun R;
    rc = PK_OK;
    const bool trace = getenv("PK_RUN_HOST_TRACE") != nullptr;
    e = host_run_acquire(device, trace, &R);
    cudaEvent_t t0ev = nullptr;
    if (trace && e == cudaSuccess) {  // PK_RUN_HOST_TRACE=1: print each event's time (development aid)
        cudaEventCreate(&t0ev);
        cudaEventRecord(t0ev, R.h2d);
    }
    if (e != cudaSuccess) rc = fail(PK_E_CUDA, "stream/event setup: %s", cudaGetErrorString(e));

    auto chunk = [&](int k) {
        pk_launch_t C = *L;
        if (nchunks > 1 || L->hi > 0) {
            C.lo = u0 + k * step;
            C.hi = u0 + (k + 1) * step < u1 ? u0 + (k + 1) * step : u1;
        }
        return C;
    };
    bool whole[3] = {false, false, false};  // needed whole by every chunk: moved once
    for (int i = 0; i < spec.count && rc == PK_OK; i++) {
        const size_t bytes = (size_t)spec.elems[i] * eb;
        e = scratch_alloc(&R.dev[i], bytes, R.h2d);
        if (e != cudaSuccess) {
            rc = fail(PK_E_ALLOC, "cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
            break;
        }
        int64_t off, cnt;
        array_range(chunk(0), i, spec.elems[i], &off, &cnt);
        whole[i] = nchunks == 1 || (off == 0 && cnt == spec.elems[i]);
    }
    // Matmul: the first row chunk runs reduction slice by reduction slice as
    // b's rows arrive (launch_matmul_kslice -- the bits of one launch), so the
    // kernels start before the 256 MiB of b have crossed PCIe.
    int64_t slice = 0, Kred = 0;
    if (rc == PK_OK && nchunks > 1 && L->family == PK_FAMILY_MATMUL && L->B0 > 0) {
        Kred = (N / L->B0) * L->B0;
        slice = Kred / kSlices / 128 * 128;
        // every chunk that runs slice by slice must take the sliced leaf
        for (int r = 0; r < nchunks && r < kSlices - 1 && slice > 0; r++)
            if (!matmul_kslice_ok(chunk(r), slice) || !matmul_kslice_ok(chunk(r), Kred - (kSlices - 1) * slice))
                slice = 0;
        if (slice < 0) slice = 0;
    }
    // Pageable buffers are staged inside the pipeline (pk_staging.cu): their
    // host copies overlap the DMA and the kernels instead of preceding them
    bool in_pg[3] = {false, false, false}, out_pg[3] = {false, false, false};
    size_t out_off[3] = {0, 0, 0}, out_total = 0;
    for (int i = 0; i < spec.count; i++) {
        in_pg[i] = in[i] && !host_is_pinned(in[i]);
        out_pg[i] = spec.written[i] && out[i] && !host_is_pinned(out[i]);
        if (out_pg[i]) {
            out_off[i] = out_total;
            out_total += (size_t)spec.elems[i] * eb;
        }
    }
    StageSession *stage = nullptr;
    alignas(StageSession) unsigned char stage_mem[sizeof(StageSession)];
    if (rc == PK_OK && (in_pg[0] || in_pg[1] || in_pg[2] || out_total)) {
        stage = new (stage_mem) StageSession(device);
        if (out_total) rc = stage->reserve_out(out_total);
    }
    // an array the program never writes, given an output buffer, ends there as
    // a copy of its input (the reference's deep copy, interp.py:183-186): made
    // in the same pass that stages the input, or right after its DMA is issued
    auto copy_out = [&](int i, int64_t off) -> char * {
        return (!spec.written[i] && out[i] && out[i] != in[i]) ? static_cast<char *>(out[i]) + off * eb : nullptr;
    };
    auto up_range = [&](int i, int64_t off, int64_t cnt) -> int {
        char *d = static_cast<char *>(R.dev[i]) + off * eb;
        char *keep = copy_out(i, off);
        if (cnt && in[i] && in_pg[i]) {
            return stage->h2d(d, static_cast<const char *>(in[i]) + off * eb, (size_t)cnt * eb, R.h2d, keep);
        } else if (cnt && in[i]) {
            cudaError_t x = cudaMemcpyAsync(d, static_cast<const char *>(in[i]) + off * eb, (size_t)cnt * eb,
                                            cudaMemcpyHostToDevice, R.h2d);
            if (x != cudaSuccess) return fail(PK_E_CUDA, "H2D copy: %s", cudaGetErrorString(x));
            if (keep) parallel_copy(keep, static_cast<const char *>(in[i]) + off * eb, (size_t)cnt * eb);
        } else if (cnt) {
            cudaMemsetAsync(d, 0, (size_t)cnt * eb, R.h2d);  // missing arrays are zero-filled (interp.py:79-81)
            if (keep) memset(keep, 0, (size_t)cnt * eb);
        }
        return PK_OK;
    };
    auto up = [&](const pk_launch_t &C, int i) -> int {
        int64_t off, cnt;
        array_range(C, i, spec.elems[i], &off, &cnt);
        return up_range(i, off, cnt);
    };
    auto down = [&](const pk_launch_t &C, int i) -> int {
        int64_t off, cnt;
        array_range(C, i, spec.elems[i], &off, &cnt);
        if (!spec.written[i] || !cnt || !out[i]) return PK_OK;
        if (out_pg[i])
            return stage->d2h(static_cast<char *>(out[i]) + off * eb, out_off[i] + (size_t)off * eb,
                              static_cast<char *>(R.dev[i]) + off * eb, (size_t)cnt * eb, R.d2h);
        cudaError_t x = cudaMemcpyAsync(static_cast<char *>(out[i]) + off * eb,
                                        static_cast<char *>(R.dev[i]) + off * eb, (size_t)cnt * eb,
                                        cudaMemcpyDeviceToHost, R.d2h);
        return x == cudaSuccess ? PK_OK : fail(PK_E_CUDA, "D2H copy: %s", cudaGetErrorString(x));
    };
    if (slice && rc == PK_OK) {
        // Matmul: uploads interleaved so the kernels start after 2 x 64 MB and
        // never idle while PCIe is the bottleneck.  h2d order: b_0, ac_0, b_1,
        // ac_1, ..., b_{S-1}, ac_{S-1}, ac_S, ... (b_j: rows of b for reduction
        // slice j; ac_r: row chunk r of a and c).  Block (r, j) runs on chunk
        // r's own stream (slices of a chunk stay in k order: c is the fp32
        // accumulator between them, so the bits equal one launch) as soon as
        // b_j and ac_r are both up; chunks whose upload follows every b slice
        // run as one full-reduction launch.  Chunk r's rows of c come down on
        // the d2h stream after its last block.
        auto slice_end = [&](int j) { return j + 1 < kSlices ? (int64_t)(j + 1) * slice : Kred; };
        auto launch_block = [&](int r, int j) -> int {
            return launch_matmul_kslice(chunk(r), R.dev, (int64_t)j * slice, slice_end(j), R.cs[r]);
        };
        auto finish_chunk = [&](int r) -> int {
            cudaEventRecord(R.ev[kSlices + nchunks + r], R.cs[r]);
            cudaStreamWaitEvent(R.d2h, R.ev[kSlices + nchunks + r], 0);
            return down(chunk(r), 2);
        };
        // the transfer list: (b_j, ac_j) pairs, then the remaining chunks
        int order[kSlices + kMaxChunks][2], nt = 0;  // {0: b_j | 1: ac_r, index}
        for (int j = 0; j < kSlices; j++) {
            order[nt][0] = 0, order[nt][1] = j, nt++;
            if (j < nchunks) order[nt][0] = 1, order[nt][1] = j, nt++;
        }
        for (int r = kSlices; r < nchunks; r++) order[nt][0] = 1, order[nt][1] = r, nt++;
        for (int t = 0; t < nt && rc == PK_OK; t++) {
            if (order[t][0] == 0) {
                const int j = order[t][1];
                const int64_t r1 = j + 1 < kSlices ? (int64_t)(j + 1) * slice : N;  // b's rows of slice j
                rc = up_range(1, (int64_t)j * slice * N, (r1 - (int64_t)j * slice) * N);
                cudaEventRecord(R.ev[t], R.h2d);
                const int up_chunks = j < nchunks ? j : nchunks;  // ac_q precedes b_j for q < j
                for (int q = 0; q < up_chunks && rc == PK_OK; q++) {
                    cudaStreamWaitEvent(R.cs[q], R.ev[t], 0);
                    rc = launch_block(q, j);
                    if (rc == PK_OK && j == kSlices - 1) rc = finish_chunk(q);
                }
            } else {
                const int r = order[t][1];
                const pk_launch_t C = chunk(r);
                rc = up(C, 0);
                if (rc == PK_OK) rc = up(C, 2);
                cudaEventRecord(R.ev[t], R.h2d);
                cudaStreamWaitEvent(R.cs[r], R.ev[t], 0);
                if (r >= kSlices - 1) {  // every slice of b is up: one launch
                    if (rc == PK_OK) rc = dispatch(C, R.dev, R.cs[r]);
                    if (rc == PK_OK) rc = finish_chunk(r);
                } else {
                    for (int q = 0; q <= r && rc == PK_OK; q++) rc = launch_block(r, q);
                }
            }
        }
    }
    for (int i = 0; i < spec.count && rc == PK_OK && !slice; i++)
        if (whole[i]) rc = up(nchunks == 1 ? *L : chunk(0), i);
    for (int k = 0; k < nchunks && rc == PK_OK && !slice; k++) {
        const pk_launch_t C = chunk(k);
        for (int i = 0; i < spec.count && rc == PK_OK; i++)
            if (!whole[i]) rc = up(C, i);
        if (rc) break;
        cudaEventRecord(R.ev[2 * k], R.h2d);
        cudaStream_t cs = R.cs[k & 1];
        cudaStreamWaitEvent(cs, R.ev[2 * k], 0);
        rc = dispatch(C, R.dev, cs);
        if (rc) break;
        cudaEventRecord(R.ev[2 * k + 1], cs);
        cudaStreamWaitEvent(R.d2h, R.ev[2 * k + 1], 0);
        for (int i = 0; i < spec.count && rc == PK_OK; i++)
            if (!whole[i] || nchunks == 1) rc = down(C, i);
    }
    // written operands moved whole come down after the last chunk (none of
    // the chunked families writes one; kept for completeness)
    for (int i = 0; i < spec.count && rc == PK_OK; i++)
        if (whole[i] && nchunks > 1) rc = down(*L, i);
    if (stage) {  // copy the staged downloads out as their pieces land, then release the staging
        const int drc = stage->drain();
        if (rc == PK_OK) rc = drc;
    }
    cudaError_t se = cudaSuccess;
    for (cudaStream_t s : R.cs) {
        if (!s) continue;
        cudaError_t x = cudaStreamSynchronize(s);
        if (se == cudaSuccess) se = x;
    }
    for (cudaStream_t s : {R.h2d, R.d2h}) {
        if (!s) continue;
        cudaError_t x = cudaStreamSynchronize(s);
        if (se == cudaSuccess) se = x;
    }
    if (se != cudaSuccess && rc == PK_OK) rc = fail(PK_E_CUDA, "kernel execution: %s", cudaGetErrorString(se));
    if (t0ev) {
        for (int k = 0; k < 2 * kMaxChunks + kSlices; k++) {
            float ms = -1.f;
            if (R.ev[k] && cudaEventElapsedTime(&ms, t0ev, R.ev[k]) == cudaSuccess)
                fprintf(stderr, "pk_run_host trace: event %2d at %8.3f ms\n", k, ms);
        }
        cudaEventDestroy(t0ev);
    }
    for (int i = 0; i < spec.count; i++)
        if (R.dev[i]) cudaFreeAsync(R.dev[i], R.d2h);
    cudaError_t fe = R.d2h ? cudaStreamSynchronize(R.d2h) : cudaSuccess;
    host_run_release(R, se == cudaSuccess && fe == cudaSuccess && e == cudaSuccess);
    if (stage) stage->~StageSession();
    return rc;
}

}  // namespace


// ---------------------------------------------------------------------------
// Single-process multi-GPU.

namespace {

// Covered units of a launch and the partitioner's alignment (one leaf tile),
// as the family launchers compute them; false when there is nothing to split.
bool covered_units(const pk_launch_t &L, int64_t *u0, int64_t *u1, int64_t *align) {
    const int64_t N = L.N, E = elems(L);
    auto cover = [](int64_t n, int64_t t) { return t > 0 && n > 0 ? (n / t) * t : (int64_t)0; };
    *u0 = 0;
    switch (L.family) {
        case PK_FAMILY_REVERSE: *u1 = cover(N, L.s * L.B); *align = 4 * L.s * L.B; break;
        case PK_FAMILY_TRANSPOSE: *u1 = cover(N, L.B0); *align = L.B0 > 4 ? L.B0 : 4; break;
        case PK_FAMILY_MATVEC: *u1 = cover(N, L.s * L.B); *align = L.s * L.B; break;
        case PK_FAMILY_MATMUL: *u1 = cover(N, L.B0); *align = L.B0 > 4 ? L.B0 : 4; break;
        case PK_FAMILY_ADDITION: *u1 = cover(N, L.B0); *align = L.B0; break;
        case PK_FAMILY_JACOBI1D: *u0 = 1; *u1 = 1 + cover(N - 2, L.s * L.B); *align = L.s * L.B; break;
        case PK_FAMILY_JACOBI2D: *u0 = 1; *u1 = 1 + cover(N - 2, L.B0); *align = L.B0; break;
        default: return false;
    }
    (void)E;
    return L.s >= 0 && L.B >= 0 && L.B0 >= 0 && L.B1 >= 0 && L.ub1 >= 0 && *align > 0 && *u1 > *u0;
}

// Device k's share: whole tiles where there are enough (partition.split).
void share(int64_t u0, int64_t u1, int64_t align, int k, int n, int64_t *lo, int64_t *hi) {
    const int64_t total = u1 - u0, blocks = total / align;
    if (n <= 1) {
        *lo = u0;
        *hi = u1;
    } else if (blocks >= n) {
        *lo = u0 + blocks * k / n * align;
        *hi = k == n - 1 ? u1 : u0 + blocks * (k + 1) / n * align;
    } else {
        *lo = u0 + total * k / n;
        *hi = u0 + total * (k + 1) / n;
    }
}

struct Multi {
    int n = 0;
    const int *dev = nullptr;
    cudaStream_t st[kMaxDevices] = {};
    cudaEvent_t done[kMaxDevices] = {}, copied[kMaxDevices] = {};
    ~Multi() {
        for (int k = 0; k < n; k++) {
            cudaSetDevice(dev[k]);
            if (st[k]) cudaStreamDestroy(st[k]);
            if (done[k]) cudaEventDestroy(done[k]);
            if (copied[k]) cudaEventDestroy(copied[k]);
        }
    }
};

// Direct peer access between every pair of distinct devices that support it
// (NVLink DMA for the peer copies), enabled once per pair for the process.
void enable_peers(int ndev, const int *devices) {
    static std::mutex mu;
    static std::vector<std::pair<int, int>> done;
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < ndev; i++)
        for (int j = 0; j < ndev; j++) {
            const int a = devices[i], b = devices[j];
            if (a == b) continue;
            bool seen = false;
            for (const auto &p : done) seen |= p.first == a && p.second == b;
            if (seen) continue;
            done.emplace_back(a, b);
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
                cudaSetDevice(a);
                if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled
            }
        }
}

int peer_copy(void *dst, int ddev, const void *src, int sdev, size_t bytes, cudaStream_t st) {
    if (!bytes) return PK_OK;
    cudaError_t e = cudaMemcpyPeerAsync(dst, ddev, src, sdev, bytes, st);
    return e == cudaSuccess ? PK_OK : fail(PK_E_CUDA, "peer copy %d -> %d: %s", sdev, ddev, cudaGetErrorString(e));
}

}  // namespace

int pk_launch_multi(const pk_launch_t *L, int ndev, const int *devices, void *const *dev_ptrs, int nptrs,
                    int64_t halo, int gather) {
    int rc = validate(L, nptrs);
    if (rc) return rc;
    if (ndev < 1 || ndev > kMaxDevices || !devices || !dev_ptrs)
        return fail(PK_E_PARAM, "pk_launch_multi: %d devices (1..%d) with their arrays", ndev, kMaxDevices);
    if (L->hi > 0) return fail(PK_E_PARAM, "pk_launch_multi splits the units itself: leave lo/hi at 0");
    for (int i = 0; i < ndev * nptrs; i++)
        if (!dev_ptrs[i]) return fail(PK_E_PARAM, "array %d of device %d is a null pointer", i % nptrs, i / nptrs);
    auto ptrs = [&](int k) { return dev_ptrs + (size_t)k * nptrs; };

    enable_peers(ndev, devices);
    Multi M;
    M.n = ndev;
    M.dev = devices;
    for (int k = 0; k < ndev; k++) {
        cudaError_t e = cudaSetDevice(devices[k]);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&M.st[k], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&M.done[k], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&M.copied[k], cudaEventDisableTiming);
        if (e != cudaSuccess) return fail(PK_E_CUDA, "device %d setup: %s", devices[k], cudaGetErrorString(e));
    }
    auto finish = [&](int code) {
        for (int k = 0; k < ndev; k++) {
            cudaSetDevice(devices[k]);
            cudaError_t e = cudaStreamSynchronize(M.st[k]);
            if (e != cudaSuccess && code == PK_OK) code = fail(PK_E_CUDA, "device %d: %s", devices[k], cudaGetErrorString(e));
        }
        return code;
    };

    int64_t u0, u1, align;
    const bool stencil = L->family == PK_FAMILY_JACOBI1D || L->family == PK_FAMILY_JACOBI2D;
    // nothing to split (or stencil data the int32 sweeps do not take): device 0 runs it
    if (ndev == 1 || !covered_units(*L, &u0, &u1, &align) || (stencil && L->dtype != PK_DTYPE_I32)) {
        cudaSetDevice(devices[0]);
        return finish(dispatch(*L, ptrs(0), M.st[0]));
    }

    if (!stencil) {
        // row / element shares, no exchange; then the written shares to device 0
        pk_launch_t Ls[kMaxDevices];
        for (int k = 0; k < ndev && rc == PK_OK; k++) {
            Ls[k] = *L;
            share(u0, u1, align, k, ndev, &Ls[k].lo, &Ls[k].hi);
            if (Ls[k].hi <= Ls[k].lo) continue;
            cudaSetDevice(devices[k]);
            rc = dispatch(Ls[k], ptrs(k), M.st[k]);
            cudaEventRecord(M.done[k], M.st[k]);
        }
        if (rc || !gather) return finish(rc);
        ArraySpec spec;
        array_spec(*L, &spec);
        const int64_t eb = elem_bytes(*L);
        cudaSetDevice(devices[0]);
        for (int k = 1; k < ndev && rc == PK_OK; k++) {
            if (Ls[k].hi <= Ls[k].lo) continue;
            cudaStreamWaitEvent(M.st[0], M.done[k], 0);
            for (int i = 0; i < spec.count && rc == PK_OK; i++) {
                if (!spec.written[i]) continue;
                int64_t off, cnt;
                array_range(Ls[k], i, spec.elems[i], &off, &cnt);
                rc = peer_copy(static_cast<char *>(ptrs(0)[i]) + off * eb, devices[0],
                               static_cast<const char *>(ptrs(k)[i]) + off * eb, devices[k], (size_t)cnt * eb, M.st[0]);
            }
        }
        return finish(rc);
    }

    // ---- stencils: slabs with ghost zones of width h refreshed every h steps
    pk_launch_t Ln = *L;
    if (!(Ln.flags & PK_FLAG_NARROW)) {  // the range check once (inputs are replicated)
        int narrow = 0;
        cudaSetDevice(devices[0]);
        rc = jacobi_narrow(Ln, ptrs(0)[0], &narrow, M.st[0]);
        if (rc) return finish(rc);
        if (narrow) Ln.flags |= PK_FLAG_NARROW;
    }
    const bool one = L->family == PK_FAMILY_JACOBI1D;
    const int64_t N = L->N, row = one ? 1 : N, half = one ? N : N * N;
    int64_t lo[kMaxDevices], hi[kMaxDevices], min_slab = u1 - u0;
    for (int k = 0; k < ndev; k++) {
        share(u0, u1, align, k, ndev, &lo[k], &hi[k]);
        if (hi[k] - lo[k] < min_slab) min_slab = hi[k] - lo[k];
    }
    // Default (halo <= 0): the halo exchange fused into the sweep -- every
    // device's edge blocks store their rows straight into the neighbours'
    // buffers (peer pointers, NVLink) and order themselves with device
    // counters (pk_jacobi_sweep_peer), ghost width 1, no copies or events per
    // step.  An explicit halo width keeps the ghost zones refreshed by peer
    // copies every h steps (below); so do layouts the register sweeps do not
    // take and devices without peer access.
    bool fused = halo <= 0 && min_slab > 0 && getenv("PK_MULTI_COPY") == nullptr;
    for (int k = 0; k < ndev && fused; k++) {
        const uintptr_t base = reinterpret_cast<uintptr_t>(ptrs(k)[0]);
        fused = one ? (base & 3u) == 0 : ((N & 1) == 0 && (base & 15u) == 0);
        for (int j = k - 1; j <= k + 1 && fused; j += 2) {
            if (j < 0 || j >= ndev || devices[j] == devices[k]) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, devices[k], devices[j]);
            fused = can != 0;
        }
    }
    if (fused) {
        unsigned *ctr[kMaxDevices] = {};
        for (int k = 0; k < ndev && rc == PK_OK; k++) {  // [from_left, from_right, error] per device
            cudaSetDevice(devices[k]);
            // cudaMalloc, not the stream-ordered pool: the neighbours' kernels
            // bump these counters with system-scope atomics over NVLink, and
            // peer access (cudaDeviceEnablePeerAccess) covers cudaMalloc
            // memory but not a memory pool without cudaMemPoolSetAccess
            cudaError_t e = cudaMalloc((void **)&ctr[k], 4 * sizeof(unsigned));
            if (e == cudaSuccess) e = cudaMemsetAsync(ctr[k], 0, 4 * sizeof(unsigned), M.st[k]);
            if (e == cudaSuccess) e = cudaEventRecord(M.done[k], M.st[k]);
            if (e != cudaSuccess) rc = fail(PK_E_CUDA, "peer counters on device %d: %s", devices[k], cudaGetErrorString(e));
        }
        for (int k = 0; k < ndev && rc == PK_OK; k++) {  // no signal before a neighbour's counters are zero
            cudaSetDevice(devices[k]);
            if (k > 0) cudaStreamWaitEvent(M.st[k], M.done[k - 1], 0);
            if (k + 1 < ndev) cudaStreamWaitEvent(M.st[k], M.done[k + 1], 0);
        }
        for (int64_t t = 0; t < L->T && rc == PK_OK; t++) {
            for (int k = 0; k < ndev && rc == PK_OK; k++) {
                cudaSetDevice(devices[k]);
                pk_peer_t P = {};
                P.left_base = k > 0 ? ptrs(k - 1)[0] : nullptr;
                P.right_base = k + 1 < ndev ? ptrs(k + 1)[0] : nullptr;
                P.wait_left = ctr[k];
                P.wait_right = ctr[k] + 1;
                P.signal_left = k > 0 ? ctr[k - 1] + 1 : nullptr;   // the left neighbour's from_right
                P.signal_right = k + 1 < ndev ? ctr[k + 1] : nullptr;  // the right neighbour's from_left
                P.error = ctr[k] + 2;
                rc = jacobi_sweep_peer(Ln, static_cast<int *>(ptrs(k)[0]), t, lo[k], hi[k], P, M.st[k]);
            }
        }
        unsigned err = 0;
        for (int k = 0; k < ndev; k++) {
            if (!ctr[k]) continue;
            cudaSetDevice(devices[k]);
            unsigned v = 0;
            if (cudaMemcpyAsync(&v, ctr[k] + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, M.st[k]) == cudaSuccess &&
                cudaStreamSynchronize(M.st[k]) == cudaSuccess)
                err |= v;
        }
        for (int k = 0; k < ndev; k++) {  // every device done before any counter goes away
            if (!ctr[k]) continue;
            cudaSetDevice(devices[k]);
            cudaStreamSynchronize(M.st[k]);
        }
        for (int k = 0; k < ndev; k++) {
            if (!ctr[k]) continue;
            cudaSetDevice(devices[k]);
            cudaFree(ctr[k]);
        }
        if (rc == PK_OK && err) rc = fail(PK_E_CUDA, "pk_launch_multi: a peer wait timed out");
    }
    int64_t h = halo > 0 ? halo : 16;
    if (h > min_slab) h = min_slab;
    if (h > L->T) h = L->T;
    if (h < 1) h = 1;
    // step t reads s(t), writes d(t): 1-D t even reads the upper half, 2-D the lower
    auto src_half = [&](int k, int64_t t) -> int * {
        int *a = static_cast<int *>(ptrs(k)[0]);
        const bool upper = one ? (t % 2 == 0) : (t % 2 == 1);
        return upper ? a + half : a;
    };
    for (int64_t t = fused ? L->T : 0; t < L->T && rc == PK_OK;) {
        const int64_t hb = (L->T - t) < h ? (L->T - t) : h;
        // exchange: the ghost rows of s(t) on both sides of every boundary; the
        // source device waits before overwriting them (step t+1 writes s(t))
        if (min_slab > 0) {
            for (int k = 0; k < ndev; k++) {
                cudaSetDevice(devices[k]);
                cudaEventRecord(M.done[k], M.st[k]);
            }
            for (int k = 0; k < ndev && rc == PK_OK; k++) {
                cudaSetDevice(devices[k]);
                if (k > 0) {  // rows [lo_k - hb, lo_k) from device k-1
                    cudaStreamWaitEvent(M.st[k], M.done[k - 1], 0);
                    rc = peer_copy(src_half(k, t) + (lo[k] - hb) * row, devices[k],
                                   src_half(k - 1, t) + (lo[k] - hb) * row, devices[k - 1],
                                   (size_t)(hb * row) * 4, M.st[k]);
                }
                if (rc == PK_OK && k + 1 < ndev) {  // rows [hi_k, hi_k + hb) from device k+1
                    cudaStreamWaitEvent(M.st[k], M.done[k + 1], 0);
                    rc = peer_copy(src_half(k, t) + hi[k] * row, devices[k], src_half(k + 1, t) + hi[k] * row,
                                   devices[k + 1], (size_t)(hb * row) * 4, M.st[k]);
                }
                cudaEventRecord(M.copied[k], M.st[k]);
            }
            for (int k = 0; k < ndev; k++) {
                cudaSetDevice(devices[k]);
                if (k > 0) cudaStreamWaitEvent(M.st[k], M.copied[k - 1], 0);
                if (k + 1 < ndev) cudaStreamWaitEvent(M.st[k], M.copied[k + 1], 0);
            }
        }
        for (int k = 0; k < ndev && rc == PK_OK; k++) {
            cudaSetDevice(devices[k]);
            for (int64_t j = 0; j < hb && rc == PK_OK; j++) {
                const int64_t ext = hb - 1 - j;  // overlap still valid after this step
                const int64_t a = lo[k] - ext > u0 ? lo[k] - ext : u0;
                const int64_t b = hi[k] + ext < u1 ? hi[k] + ext : u1;
                int *src = src_half(k, t + j);
                int *base = static_cast<int *>(ptrs(k)[0]);
                int *dst = src == base ? base + half : base;
                rc = one ? sweep_jacobi1d(Ln, src, dst, a, b, M.st[k]) : sweep_jacobi2d(Ln, src, dst, a, b, M.st[k]);
            }
        }
        t += hb;
    }
    if (rc == PK_OK && gather) {  // both halves of every slab to device 0
        for (int k = 0; k < ndev; k++) {
            cudaSetDevice(devices[k]);
            cudaEventRecord(M.done[k], M.st[k]);
        }
        cudaSetDevice(devices[0]);
        for (int k = 1; k < ndev && rc == PK_OK; k++) {
            cudaStreamWaitEvent(M.st[0], M.done[k], 0);
            for (int hsel = 0; hsel < 2 && rc == PK_OK; hsel++) {
                const int64_t off = hsel * half + lo[k] * row;
                rc = peer_copy(static_cast<int *>(ptrs(0)[0]) + off, devices[0],
                               static_cast<const int *>(ptrs(k)[0]) + off, devices[k],
                               (size_t)((hi[k] - lo[k]) * row) * 4, M.st[0]);
            }
        }
    }
    return finish(rc);
}

}  // extern "C"
