/*
 * pk.h -- C ABI of libpk, the B200 (sm_100a) executor for the parametric
 * kernels of arXiv 1801.04348.
 *
 * The reference has no FFI: its executor is the Python function
 *   parakern.interp.run_program(program, params, arrays=None, tracer=None)
 *   (/root/reference/pkg/src/parakern/interp.py:215-225)
 * which runs one program sequentially on the host.  This library replaces
 * that call for the program families below; the Python shim
 * (paper_1801_04348_b200/interp.py) keeps run_program's signature and binds
 * these entry points with ctypes.  Plain C types only: device pointers are
 * void*, streams are cudaStream_t passed as void*.
 *
 * Every entry point is re-entrant: no mutable globals except the device
 * property cache (guarded by std::once_flag per device), the thread-local
 * error text and an atomic launch counter.
 */
#ifndef PK_H
#define PK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (the shim maps them to the reference's exceptions) ---- */
#define PK_OK 0
#define PK_E_PARAM 1       /* KeyError / ValueError: missing or invalid parameter (interp.py:75) */
#define PK_E_BOUNDS 2      /* IndexError: an access would leave its array (interp.py:209-212)   */
#define PK_E_DIV0 3        /* ZeroDivisionError while evaluating a binding (interp.py:43-46)    */
#define PK_E_UNSUPPORTED 4 /* NotImplementedError: variant/dtype this library does not provide  */
#define PK_E_CUDA 5        /* CUDA runtime failure (text in pk_last_error)                      */
#define PK_E_ALLOC 6       /* device or pinned allocation failed                                */

/* ---- program families (one per .mfk program shape) ---------------------- */
#define PK_FAMILY_REVERSE 1   /* SURVEY App. A.2 reverse.mfk:   c[N-1-p] = a[p]                  */
#define PK_FAMILY_TRANSPOSE 2 /* data/transpose.mfk:             c[i*N+j] = a[j][i]              */
#define PK_FAMILY_JACOBI1D 3  /* data/jacobi.mfk:                3-point, /3, double-buffered   */
#define PK_FAMILY_JACOBI2D 4  /* SURVEY App. A.4 jacobi2d.mfk:   5-point, /5, double-buffered   */
#define PK_FAMILY_MATVEC 5    /* SURVEY App. A.3 matvec.mfk:     y[r] += a[r][q]*x[q]           */
#define PK_FAMILY_MATMUL 6    /* SURVEY App. A.1 matmul.mfk:     c[p][q] += a[p][kk]*b[kk][q]   */
#define PK_FAMILY_ADDITION 7  /* data/addition.mfk:              c = a + b (twin stores)        */

/* ---- leaf variants: what the selected case's applied strategies mean ---- */
#define PK_VARIANT_STAGED 0 /* cache(...) kept: tiles staged in shared memory            */
#define PK_VARIANT_DIRECT 1 /* caching-off applied (strategies.py:430-440): no staging   */

/* ---- flags --------------------------------------------------------------- */
#define PK_FLAG_GRANULARITY 0x1 /* granularity applied (strategies.py:302-422): the s loop is
                                   gone, one element per thread; tile = B (not s*B)           */
#define PK_FLAG_TEMPORAL 0x2    /* Jacobi only: temporally blocked sweeps (reported apart)   */
#define PK_FLAG_MERGED 0x4      /* addition only: twin stores merged by granularity          */
#define PK_FLAG_GENERIC 0x8     /* force the generic (one thread per paper thread) kernel    */
#define PK_FLAG_TF32X3 0x10     /* matmul f32 only: 3xTF32 on tcgen05 (reported apart)       */
#define PK_FLAG_NARROW 0x20     /* Jacobi only: caller guarantees |v| <= (2^31-1)/3 (1-D) or
                                   /5 (2-D) for every value, so int32 sums are exact
                                   (pk_jacobi_narrow checks it); without it pk_launch checks
                                   on the device and pk_jacobi_sweep forms 64-bit sums     */

/* ---- element types ------------------------------------------------------- */
#define PK_DTYPE_I32 0 /* the DSL's int: C int32 arithmetic, truncating / and %; 4-byte words     */
#define PK_DTYPE_F32 1 /* float32 storage: FFMA matmul, double-float mat-vec, IEEE add; 4-byte words */
#define PK_DTYPE_I64 2 /* int64: reverse/transpose move 8-byte words; addition/matvec/matmul compute
                          in wrapping int64 (exact whenever the result fits, like the reference's
                          unbounded ints)                                                          */
#define PK_DTYPE_F64 3 /* binary64, the reference's Python float: reverse/transpose move 8-byte
                          words; addition/matvec/matmul evaluate c + a*b with one rounding per
                          operation in the interpreter's order (no contraction): bit-identical
                          to interp.py on Python floats                                              */
/* dtypes per family: reverse/transpose/addition/matvec/matmul take all four;
   the Jacobi stencils take I32 (the register sweeps), I64 and F64 (per-step
   sweeps; "/" is the reference's c_div on Python floats).  Buffers hold
   elements of the dtype's size. */

/*
 * One program invocation.  Parameters carry the names of the ORIGINAL
 * program (the one the user passed to run_program); the covered index
 * sets are derived from them with the program's own bindings (C division),
 * so every variant writes exactly the elements the reference would.
 * Fields a family does not use are ignored.
 */
typedef struct pk_launch {
    int32_t family;  /* PK_FAMILY_*                                          */
    int32_t variant; /* PK_VARIANT_*                                         */
    int32_t dtype;   /* PK_DTYPE_*                                           */
    int32_t flags;   /* PK_FLAG_*                                            */
    int64_t N;       /* N (matmul: n)                                        */
    int64_t T;       /* Jacobi time steps                                    */
    int64_t s;       /* granularity                                          */
    int64_t B;       /* 1-D thread block                                     */
    int64_t B0;      /* 2-D thread block rows / matmul B0                    */
    int64_t B1;      /* 2-D thread block cols                                */
    int64_t ub1;     /* matmul thread columns                                */
    int64_t lo, hi;  /* unit sub-range for partitioned launches (hi == 0: all
                        units).  Units: reverse = input elements p, transpose /
                        matvec / matmul / addition = output rows, Jacobi =
                        interior positions (1-D) / rows (2-D).              */
    int64_t tblock;  /* PK_FLAG_TEMPORAL: steps fused per sweep (0 = auto)   */
} pk_launch_t;

/* Live device properties, the values substituted for the machine
 * parameters of the case discussion (replaces the constants of
 * pkg/src/parakern/data/fermi.machine:12-18 and machine.py:80-88). */
typedef struct pk_machine {
    int32_t device;
    int32_t cc_major, cc_minor;
    int32_t sm_count;
    int32_t warp_size;                /* not a reference parameter; executor-side filter */
    int32_t max_threads_per_block;    /* T_B */
    int32_t max_threads_per_sm;
    int32_t regs_per_thread;          /* R_B: 255 on sm_100 (architectural) */
    int32_t regs_per_block;
    int32_t regs_per_sm;
    int64_t smem_per_block;           /* Z_B (static) = /4 words */
    int64_t smem_per_block_optin;     /* Z_B (opt-in carve-out) = /4 words */
    int64_t smem_per_sm;
    int64_t l2_bytes;
    int64_t global_mem_bytes;
    int32_t clock_khz;                /* SM clock (max) */
    int32_t mem_clock_khz;
    int32_t mem_bus_width_bits;
    char name[256];
} pk_machine_t;

/* Fill *out for device `device`.  Replaces the reference's machine constants. */
int pk_query_machine(int device, pk_machine_t *out);

/* Run one program on device buffers (the pointers live on the current
 * device).  dev_ptrs follow the program's array declaration order:
 *   reverse (a, c) | transpose (a, c) | jacobi1d (a) | jacobi2d (a)
 *   matvec (a, x, y) | matmul (a, b, c) | addition (a, b, c)
 * Work is enqueued on `stream` (NULL = legacy default stream); the call
 * returns after enqueueing.  Replaces interp.run_program (interp.py:215). */
int pk_launch(const pk_launch_t *L, void *const *dev_ptrs, int nptrs, void *stream);

/* pk_launch with the element count of every buffer: PK_E_BOUNDS (the
 * reference's IndexError, interp.py:209-212) when an access of the launch
 * would leave a buffer, before anything is enqueued. */
int pk_launch_checked(const pk_launch_t *L, void *const *dev_ptrs, const int64_t *elems, int nptrs, void *stream);

/* need[i] = 1 + the largest flat index the launch reads or writes in array i
 * (0 if it never touches it); the stencils count their whole double buffer. */
int pk_required_elems(const pk_launch_t *L, int64_t *need, int nneed);

/* End-to-end call with HOST buffers (pass pinned memory for full PCIe
 * speed): copies the inputs in, runs pk_launch, copies the written arrays
 * back into the host buffers and synchronises.  With a unit sub-range
 * (L->hi > 0) only the rank's share crosses PCIe: the rows of row-sharded
 * operands (matmul a/c, mat-vec a/y, transpose c, addition), the mirrored
 * range for reversal; replicated operands (b, x, transpose's a) and the
 * stencil buffers are copied whole.  Large runs of the row-sharded families
 * are cut into up to 8 unit chunks (~48 MB of PCIe traffic each) pipelined
 * over an H2D stream, two compute streams and a D2H stream, so the copies
 * overlap the kernels; results are identical to one pk_launch. */
int pk_run_host(const pk_launch_t *L, void *const *host_ptrs, int nptrs, int device);

/* pk_run_host with element counts: PK_E_BOUNDS when a buffer is shorter than
 * what the run touches or copies (the declared extent of each array). */
int pk_run_host_checked(const pk_launch_t *L, void *const *host_ptrs, const int64_t *elems, int nptrs, int device);

/* The host-buffer run with separate inputs and outputs: array i is read from
 * in_ptrs[i] (NULL: zeros) and its final contents are written to
 * out_ptrs[i] (NULL: not copied back; may equal in_ptrs[i]) -- the result
 * for an array the program writes, a copy of the input for one it does not
 * (the reference's deep copy, made in the same pass that stages the input)
 * -- so a caller's buffers need not be copied to keep them unmutated.  Pinned buffers
 * move by DMA directly; pageable ones are staged inside the pipeline through
 * a pinned ring (host copies by a thread pool, overlapped with the DMA and
 * the kernels).  elems[i] counts both buffers of array i (PK_E_BOUNDS). */
int pk_run_host_io(const pk_launch_t *L, const void *const *in_ptrs, void *const *out_ptrs, const int64_t *elems,
                   int nptrs, int device);

/* One thread block of the program (the reference's run_block,
 * interp.py:228-249): grid[0..ngrid) the grid meta_for indices (outer
 * first: reverse / jacobi / matvec i; transpose / jacobi2d / addition
 * v0, v1; matmul i, j), ctx[0..nctx) the serial context loop variable
 * (jacobi / jacobi2d t, matmul k); the thread loops are swept by one CUDA
 * block in the program's own statement order, on any PK_DTYPE_*.  The
 * caller checks the block's accesses against its arrays. */
int pk_launch_block(const pk_launch_t *L, const int64_t *grid, int ngrid, const int64_t *ctx, int nctx,
                    void *const *dev_ptrs, int nptrs, void *stream);

/* One Jacobi sweep over an explicit position range, used by the slab
 * partitioner (one process per GPU).  src/dst point at the two halves (1-D:
 * a and a+N; 2-D: row 0 of each half, row pitch N).  Positions (1-D) or
 * rows (2-D) in [lo, hi) that are interior (1..P) are updated; columns of
 * 2-D are the program's covered columns.  Uses the tile geometry of L. */
int pk_jacobi_sweep(const pk_launch_t *L, const void *src, void *dst, int64_t lo, int64_t hi,
                    void *stream);

/* One program over several GPUs of this process (single-process multi-GPU,
 * the partitioner of SURVEY 8(e) in native code).  Device k
 * (devices[k], which may repeat) holds full-size arrays with the program's
 * global indexing -- dev_ptrs[k * nptrs + i] is array i on device k -- with
 * the inputs present on every device, and computes its aligned share of the
 * units (rows; elements for reversal; interior positions / rows for the
 * stencils).  The row families need no exchange.  The stencils (halo <= 0)
 * run the sweep with the halo exchange fused in (pk_jacobi_sweep_peer with
 * direct peer pointers: edge blocks store into the neighbours' buffers over
 * NVLink, device counters order the devices); with halo > 0 -- or layouts /
 * devices the fused sweep does not take -- they refresh ghost zones of width
 * `halo` (capped by the smallest slab and T) every `halo` steps with peer
 * copies (cudaMemcpyPeerAsync), recomputing the overlap in between.  With gather != 0 every
 * device's written share (both Jacobi halves) is copied into devices[0]'s
 * arrays, which then hold the whole result, bit-identical to pk_launch.
 * L->lo / L->hi must be 0.  Synchronises every device. */
int pk_launch_multi(const pk_launch_t *L, int ndev, const int *devices, void *const *dev_ptrs, int nptrs,
                    int64_t halo, int gather);

/* ---- fused halo exchange over peer memory (one process per GPU) ----------
 * Every rank holds the whole Jacobi double buffer `a` with the program's
 * global indexing and owns units [lo, hi) (positions / rows).  One call runs
 * step `step` (the half parity of jacobi.mfk / jacobi2d.mfk) of the
 * register-window sweep over [lo, hi); the blocks computing unit lo and unit
 * hi - 1 also store those values into the left / right neighbour's buffer
 * (the same offset through an IPC mapping: NVLink stores on an 8 x B200 box),
 * and order themselves against the neighbours with the counters below: they
 * wait, before loading, for the neighbour's edge blocks of step - 1, and
 * signal after storing (system-scope fence + atomic).  Interior blocks never
 * wait.  Counters start at 0 for step 0 (zero them, then barrier, before a
 * run).  Replaces the NCCL ghost-zone exchange of the partitioner for the
 * stencils (partition.PeerStencil).  Requires even N and 16-byte aligned
 * halves for 2-D. */
typedef struct pk_peer {
    void *left_base, *right_base;           /* neighbours' double buffers, mapped (NULL: no neighbour) */
    uint32_t *wait_left, *wait_right;       /* this rank's counters, bumped by the neighbours          */
    uint32_t *signal_left, *signal_right;   /* left neighbour's wait_right / right neighbour's wait_left */
    uint32_t *error;                        /* set to 1 when a wait gave up after ~2 s (a neighbour that
                                               never signalled): the sweep then proceeds, results are
                                               invalid, the caller must check it                        */
} pk_peer_t;
int pk_jacobi_sweep_peer(const pk_launch_t *L, void *a, int64_t step, int64_t lo, int64_t hi, const pk_peer_t *peer,
                         void *stream);

/* CUDA IPC for pk_peer_t: export a device pointer (any address inside an
 * allocation) as a 64-byte handle plus its offset from the allocation base;
 * open a handle exported by another process (returns base + offset); close
 * what pk_ipc_open returned. */
int pk_ipc_export(const void *ptr, void *handle64, int64_t *offset);
int pk_ipc_open(const void *handle64, int64_t offset, void **ptr);
int pk_ipc_close(void *ptr, int64_t offset);

/* Value-range check for the Jacobi fast path: *narrow = 1 when every value
 * of the double buffer `a` is within the PK_FLAG_NARROW bound (a Jacobi
 * average never leaves the range of its inputs, so the bound then holds for
 * every later step too).  Synchronises `stream`. */
int pk_jacobi_narrow(const pk_launch_t *L, const void *a, int32_t *narrow, void *stream);

/* Load-time compilation for programs outside the seven families: CUDA text
 * (the reference's emitted leaf, pkg/src/parakern/emit.py:268-594) compiled
 * for sm_100a with NVRTC, then launched with explicit geometry.  kinds[i]:
 * 0 = int32 scalar, 1 = device pointer; args[i] holds the value. */
int pk_jit_compile(const char *source, const char *kernel_name, const char *const *options, int nopts,
                   void **handle);
int pk_jit_launch(void *handle, const uint32_t *grid, const uint32_t *block, uint32_t smem_bytes,
                  const uint64_t *args, const int32_t *kinds, int nargs, void *stream);
int pk_jit_release(void *handle);

/* Shared-memory words the leaf kernel stages per block (the footprint the
 * case constrains against Z_B; reference counters.py:416-464). */
int64_t pk_footprint_words(const pk_launch_t *L);

/* Number of kernels libpk has launched since load (atomic). */
int64_t pk_launch_count(void);

/* Text of the last error raised on the calling thread. */
const char *pk_last_error(void);

/* ABI version: (major << 16) | minor. */
int pk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PK_H */
