// pk_jit.cu -- load-time compilation of CUDA text for sm_100a (NVRTC) and
// launch through the driver API.  Used for programs outside the seven
// hand-written families: the reference's own emitter renders the selected
// leaf as CUDA-C (pkg/src/parakern/emit.py:268-594); the Python side
// (paper_1801_04348_b200/jit.py) compiles that text here and launches it with
// the emitter's launch geometry.  Also the "naive emitted kernel" baseline
// the hand-written kernels are compared against.
//
// NVRTC is opened at run time (dlopen) so libpk has no link-time dependency
// on it; the CUDA driver entry points come from cudaGetDriverEntryPoint.
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "pk_internal.cuh"

namespace pk {
namespace {

struct Nvrtc {
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
    bool ok = false;
};

struct Driver {
    CUresult (*load)(CUmodule *, const void *) = nullptr;
    CUresult (*get_fn)(CUfunction *, CUmodule, const char *) = nullptr;
    CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                       void **, void **) = nullptr;
    CUresult (*unload)(CUmodule) = nullptr;
    bool ok = false;
};

Nvrtc &nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, []() {
        const char *names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
        void *h = nullptr;
        for (const char *nm : names)
            if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
        if (!h) return;
        n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
        n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
        n.log_size = reinterpret_cast<decltype(n.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
        n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
        n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
        n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
        n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy;
    });
    return n;
}

Driver &driver() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, []() {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        auto get = [&](const char *sym) -> void * {
            p = nullptr;
            if (cudaGetDriverEntryPoint(sym, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
                return nullptr;
            return p;
        };
        d.load = reinterpret_cast<decltype(d.load)>(get("cuModuleLoadData"));
        d.get_fn = reinterpret_cast<decltype(d.get_fn)>(get("cuModuleGetFunction"));
        d.launch = reinterpret_cast<decltype(d.launch)>(get("cuLaunchKernel"));
        d.unload = reinterpret_cast<decltype(d.unload)>(get("cuModuleUnload"));
        d.ok = d.load && d.get_fn && d.launch && d.unload;
    });
    return d;
}

struct JitKernel {
    CUmodule mod;
    CUfunction fn;
};

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_jit_compile(const char *source, const char *kernel_name, const char *const *options, int nopts,
                   void **handle) {
    if (!source || !kernel_name || !handle) return fail(PK_E_PARAM, "pk_jit_compile: null argument");
    Nvrtc &n = nvrtc();
    if (!n.ok) return fail(PK_E_UNSUPPORTED, "NVRTC (libnvrtc.so.12) is not available");
    Driver &d = driver();
    if (!d.ok) return fail(PK_E_CUDA, "CUDA driver entry points unavailable");
    cudaFree(nullptr);  // make the runtime's primary context current
    nvrtcProgram prog;
    if (n.create(&prog, source, "pk_emitted.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
        return fail(PK_E_CUDA, "nvrtcCreateProgram failed");
    std::vector<const char *> opts = {"--gpu-architecture=sm_100a", "-default-device"};
    for (int i = 0; i < nopts; i++) opts.push_back(options[i]);
    const nvrtcResult cr = n.compile(prog, (int)opts.size(), opts.data());
    if (cr != NVRTC_SUCCESS) {
        size_t ls = 0;
        n.log_size(prog, &ls);
        std::string log(ls, '\0');
        if (ls) n.log(prog, &log[0]);
        n.destroy(&prog);
        return fail(PK_E_PARAM, "NVRTC compile of %s failed: %.900s", kernel_name, log.c_str());
    }
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    std::vector<char> cubin(cs);
    n.cubin(prog, cubin.data());
    n.destroy(&prog);
    auto *k = new JitKernel();
    CUresult r = d.load(&k->mod, cubin.data());
    if (r != CUDA_SUCCESS) {
        delete k;
        return fail(PK_E_CUDA, "cuModuleLoadData failed (%d)", (int)r);
    }
    r = d.get_fn(&k->fn, k->mod, kernel_name);
    if (r != CUDA_SUCCESS) {
        d.unload(k->mod);
        delete k;
        return fail(PK_E_PARAM, "kernel %s not found in the compiled module (%d)", kernel_name, (int)r);
    }
    *handle = k;
    return PK_OK;
}

int pk_jit_launch(void *handle, const uint32_t *grid, const uint32_t *block, uint32_t smem, const uint64_t *args,
                  const int32_t *kinds, int nargs, void *stream) {
    if (!handle || !grid || !block || (nargs && (!args || !kinds)))
        return fail(PK_E_PARAM, "pk_jit_launch: null argument");
    Driver &d = driver();
    auto *k = static_cast<JitKernel *>(handle);
    // kinds: 0 = int32 scalar, 1 = device pointer
    std::vector<int32_t> ints(nargs);
    std::vector<void *> ptrs(nargs);
    std::vector<void *> params(nargs);
    for (int i = 0; i < nargs; i++) {
        if (kinds[i] == 1) {
            ptrs[i] = reinterpret_cast<void *>(args[i]);
            params[i] = &ptrs[i];
        } else {
            ints[i] = (int32_t)(int64_t)args[i];
            params[i] = &ints[i];
        }
    }
    CUresult r = d.launch(k->fn, grid[0], grid[1], grid[2], block[0], block[1], block[2], smem,
                          static_cast<CUstream>(stream), params.data(), nullptr);
    if (r != CUDA_SUCCESS) return fail(PK_E_CUDA, "cuLaunchKernel failed (%d)", (int)r);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return PK_OK;
}

int pk_jit_release(void *handle) {
    if (!handle) return PK_OK;
    auto *k = static_cast<JitKernel *>(handle);
    driver().unload(k->mod);
    delete k;
    return PK_OK;
}

}  // extern "C"
