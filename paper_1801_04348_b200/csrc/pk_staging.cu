// pk_staging.cu -- pageable host memory for pk_run_host_io: the copies a
// caller's ordinary (pageable) buffers need, done inside the pipeline instead
// of before and after it.
//
// * H2D: the source is copied piece by piece (8 MB) into a ring of pinned
//   slots by a pool of host threads, and each slot goes up with
//   cudaMemcpyAsync on the caller's upload stream; a slot is reused once the
//   DMA that read it has completed (its event).  The host copy of piece k+1
//   runs while piece k crosses PCIe, and the kernels already enqueued run
//   under both.
// * D2H: results land in a pinned staging buffer (stream-ordered, as for a
//   pinned destination) and are copied out to the caller's buffer piece by
//   piece as each piece's event completes, after the whole schedule has been
//   enqueued -- the copy-out of chunk k overlaps the download and compute of
//   the chunks after it.
// The staging resources are per device and reused across calls; a mutex per
// device serialises calls that stage (pinned-only calls never take it).
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "pk_internal.cuh"

namespace pk {
namespace {

// ---- a small persistent pool for parallel memcpy --------------------------
class CopyPool {
  public:
    static CopyPool &get() {
        // never destroyed: the detached workers wait on its condition variable
        // for the life of the process (a static destructor would pull it out
        // from under them and hang the exit)
        static CopyPool *pool = new CopyPool();
        return *pool;
    }
    // dst (and dst2 when given) <- src, split over the workers and the calling
    // thread; returns when done.  Two destinations read the source once.
    void copy(void *dst, const void *src, size_t bytes, void *dst2 = nullptr) {
        const size_t parts = bytes < (size_t(1) << 20) ? 1 : workers_.size() + 1;
        if (parts == 1) {
            memcpy(dst, src, bytes);
            if (dst2) memcpy(dst2, dst, bytes);
            return;
        }
        const size_t step = (bytes / parts + 4095) & ~size_t(4095);
        std::unique_lock<std::mutex> job_lock(job_mu_);  // one parallel copy at a time
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char *>(dst);
            dst2_ = static_cast<char *>(dst2);
            src_ = static_cast<const char *>(src);
            bytes_ = bytes;
            step_ = step;
            pending_ = workers_.size();
            ++gen_;
        }
        cv_.notify_all();
        const size_t own = workers_.size() * step;  // the caller copies the last part
        if (own < bytes) {
            memcpy(static_cast<char *>(dst) + own, static_cast<const char *>(src) + own, bytes - own);
            if (dst2) memcpy(static_cast<char *>(dst2) + own, static_cast<char *>(dst) + own, bytes - own);
        }
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }

  private:
    CopyPool() {
        unsigned n = std::thread::hardware_concurrency();
        if (n == 0) n = 4;
        if (n > 16) n = 16;
        for (unsigned i = 0; i + 1 < n; i++) workers_.emplace_back([this, i] { run(i); });
        for (auto &w : workers_) w.detach();  // lives for the process
    }
    void run(size_t idx) {
        unsigned long long seen = 0;
        for (;;) {
            char *d, *d2;
            const char *s;
            size_t b, st;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                d = dst_, d2 = dst2_, s = src_, b = bytes_, st = step_;
            }
            const size_t off = idx * st;
            if (off < b) {
                const size_t n = off + st < b ? st : b - off;
                memcpy(d + off, s + off, n);
                if (d2) memcpy(d2 + off, d + off, n);  // from the (cache-warm) first copy
            }
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_, done_cv_;
    char *dst_ = nullptr, *dst2_ = nullptr;
    const char *src_ = nullptr;
    size_t bytes_ = 0, step_ = 0, pending_ = 0;
    unsigned long long gen_ = 0;
};

constexpr size_t kPiece = size_t(8) << 20;  // bytes per staged piece
constexpr int kSlots = 8;                    // H2D ring depth (64 MB pinned)

struct DeviceStage {
    std::mutex mu;
    char *ring[kSlots] = {};
    cudaEvent_t ring_ev[kSlots] = {};
    bool ring_used[kSlots] = {};
    int next = 0;
    char *out = nullptr;  // D2H staging, grown on demand
    size_t out_bytes = 0;
    std::vector<cudaEvent_t> out_ev;
};

DeviceStage g_stage[64];

}  // namespace

bool host_is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Locks the device's staging resources for one pk_run_host_io call.
StageSession::StageSession(int device) : device_(device) {
    DeviceStage &S = g_stage[device & 63];
    S.mu.lock();
}

StageSession::~StageSession() {
    DeviceStage &S = g_stage[device_ & 63];
    S.mu.unlock();
}

void parallel_copy(void *dst, const void *src, size_t bytes) { CopyPool::get().copy(dst, src, bytes); }

int StageSession::h2d(void *dst, const void *src, size_t bytes, cudaStream_t st, void *copy_dst) {
    DeviceStage &S = g_stage[device_ & 63];
    for (size_t off = 0; off < bytes; off += kPiece) {
        const size_t n = bytes - off < kPiece ? bytes - off : kPiece;
        const int k = S.next;
        S.next = (S.next + 1) % kSlots;
        if (!S.ring[k]) {
            cudaError_t e = cudaHostAlloc((void **)&S.ring[k], kPiece, cudaHostAllocPortable);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&S.ring_ev[k], cudaEventDisableTiming);
            if (e != cudaSuccess) return fail(PK_E_ALLOC, "pinned staging ring: %s", cudaGetErrorString(e));
        } else if (S.ring_used[k]) {
            cudaError_t e = cudaEventSynchronize(S.ring_ev[k]);  // the DMA that last read the slot
            if (e != cudaSuccess) return fail(PK_E_CUDA, "staging slot: %s", cudaGetErrorString(e));
        }
        CopyPool::get().copy(S.ring[k], static_cast<const char *>(src) + off, n,
                             copy_dst ? static_cast<char *>(copy_dst) + off : nullptr);
        cudaError_t e = cudaMemcpyAsync(static_cast<char *>(dst) + off, S.ring[k], n, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(S.ring_ev[k], st);
        if (e != cudaSuccess) return fail(PK_E_CUDA, "staged H2D: %s", cudaGetErrorString(e));
        S.ring_used[k] = true;
    }
    return PK_OK;
}

int StageSession::reserve_out(size_t bytes) {
    DeviceStage &S = g_stage[device_ & 63];
    if (S.out_bytes >= bytes) return PK_OK;
    if (S.out) cudaFreeHost(S.out);
    S.out = nullptr;
    S.out_bytes = 0;
    size_t cap = size_t(64) << 20;
    while (cap < bytes) cap <<= 1;
    cudaError_t e = cudaHostAlloc((void **)&S.out, cap, cudaHostAllocPortable);
    if (e != cudaSuccess) return fail(PK_E_ALLOC, "pinned download staging (%zu bytes): %s", cap, cudaGetErrorString(e));
    S.out_bytes = cap;
    return PK_OK;
}

int StageSession::d2h(void *dst, size_t stage_off, const void *src, size_t bytes, cudaStream_t st) {
    DeviceStage &S = g_stage[device_ & 63];
    for (size_t off = 0; off < bytes; off += kPiece) {
        const size_t n = bytes - off < kPiece ? bytes - off : kPiece;
        cudaEvent_t ev = nullptr;
        if (drains_.size() < S.out_ev.size()) {
            ev = S.out_ev[drains_.size()];
        } else {
            cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (e != cudaSuccess) return fail(PK_E_CUDA, "staging event: %s", cudaGetErrorString(e));
            S.out_ev.push_back(ev);
        }
        char *stage = S.out + stage_off + off;
        cudaError_t e = cudaMemcpyAsync(stage, static_cast<const char *>(src) + off, n, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev, st);
        if (e != cudaSuccess) return fail(PK_E_CUDA, "staged D2H: %s", cudaGetErrorString(e));
        drains_.push_back({ev, stage, static_cast<char *>(dst) + off, n});
    }
    return PK_OK;
}

int StageSession::drain() {
    for (const Drain &d : drains_) {
        cudaError_t e = cudaEventSynchronize(d.ev);
        if (e != cudaSuccess) return fail(PK_E_CUDA, "download: %s", cudaGetErrorString(e));
        CopyPool::get().copy(d.dst, d.stage, d.bytes);
    }
    drains_.clear();
    return PK_OK;
}

}  // namespace pk
