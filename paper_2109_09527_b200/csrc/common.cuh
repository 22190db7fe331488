// common.cuh -- internal helpers of libprgpu (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <chrono>

#include "../../include/prgpu.h"

namespace prgpu {

void set_error(const char* fmt, ...);
extern double g_alloc_ms;  // host time spent in cudaMallocAsync (PRGPU_PROFILE diagnostics)

// Return PR_ECUDA from the enclosing int function on a CUDA error.
#define PR_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t _e = (call);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ::prgpu::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,          \
                               cudaGetErrorString(_e));                            \
            return _e == cudaErrorMemoryAllocation ? PR_ENOMEM : PR_ECUDA;         \
        }                                                                          \
    } while (0)

#define PR_TRY(expr)                 \
    do {                             \
        int _s = (expr);             \
        if (_s != PR_OK) return _s;  \
    } while (0)

// Every kernel launch goes through this so the library can count launches.
#define PR_LAUNCH(ctx, kernel, grid, block, smem, ...)                                  \
    do {                                                                                \
        kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);                 \
        (ctx).launches += 1;                                                            \
        cudaError_t _le = cudaGetLastError();                                           \
        if (_le != cudaSuccess) {                                                       \
            ::prgpu::set_error("launch %s: %s", #kernel, cudaGetErrorString(_le));      \
            return PR_ECUDA;                                                            \
        }                                                                               \
    } while (0)

// Programmatic dependent launch for the kernels of the sweep loop: the next
// kernel's CTAs are dispatched while the previous kernel drains, and wait in
// pdl_wait() (griddepcontrol.wait: full completion and visibility of the
// previous grid) before touching anything it wrote.  A kernel launched this
// way MUST call pdl_wait() before its first dependent access.
bool pdl_enabled();
#define PR_LAUNCH_PDL(ctx, kernel, grid, block, smem, ...)                                   \
    do {                                                                                     \
        cudaLaunchConfig_t _cfg = {};                                                        \
        _cfg.gridDim = dim3((unsigned)(grid));                                               \
        _cfg.blockDim = dim3((unsigned)(block));                                             \
        _cfg.dynamicSmemBytes = (size_t)(smem);                                              \
        _cfg.stream = (ctx).stream;                                                          \
        cudaLaunchAttribute _at[1];                                                          \
        _at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                      \
        _at[0].val.programmaticStreamSerializationAllowed = 1;                               \
        _cfg.attrs = _at;                                                                    \
        _cfg.numAttrs = ::prgpu::pdl_enabled() ? 1 : 0;                                      \
        cudaError_t _le = cudaLaunchKernelEx(&_cfg, kernel, __VA_ARGS__);                    \
        (ctx).launches += 1;                                                                 \
        if (_le != cudaSuccess) {                                                            \
            ::prgpu::set_error("launch %s: %s", #kernel, cudaGetErrorString(_le));           \
            return PR_ECUDA;                                                                 \
        }                                                                                    \
    } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct Ctx {
    cudaStream_t stream;
    int num_sms;
    int64_t launches;
};

// The library's own stream-ordered memory pool on the current device (api.cu):
// freed blocks stay in it for later graphs (no re-mapping in the middle of a
// call) without touching the process's default pool; pr_release_memory()
// returns them to the device.
cudaMemPool_t lib_pool();

// Stream-ordered allocation; all library memory comes from here.
template <class T>
int dalloc(T** p, size_t count, cudaStream_t s) {
    *p = nullptr;
    size_t bytes = count * sizeof(T) + 64;  // +64: vector tails may read past the end
    const auto t0 = std::chrono::steady_clock::now();
    cudaMemPool_t pool = lib_pool();
    cudaError_t e = pool ? cudaMallocFromPoolAsync((void**)p, bytes, pool, s) : cudaMallocAsync((void**)p, bytes, s);
    g_alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (e != cudaSuccess) {
        set_error("cudaMallocAsync(%zu bytes): %s", bytes, cudaGetErrorString(e));
        *p = nullptr;
        return PR_ENOMEM;
    }
    return PR_OK;
}
template <class T>
void dfree(T*& p, cudaStream_t s) {
    if (p) cudaFreeAsync((void*)p, s);
    p = nullptr;
}

// (track() keeps the ADDRESS of the pointer variable: declare the variable in
// the guard's own scope, never in an inner block that ends before the guard.)
// Frees the device temporaries registered with track() when the scope ends,
// early error returns included; a pointer already released with dfree (and so
// set to nullptr) is skipped.  Graph-owned buffers are never tracked: on error
// pr_destroy releases those.
struct TmpGuard {
    cudaStream_t s;
    void** slot[48];
    int k = 0;
    explicit TmpGuard(cudaStream_t st) : s(st) {}
    TmpGuard(const TmpGuard&) = delete;
    TmpGuard& operator=(const TmpGuard&) = delete;
    template <class T>
    void track(T*& p) {
        if (k < 48) slot[k++] = reinterpret_cast<void**>(&p);
    }
    ~TmpGuard() {
        for (int i = k - 1; i >= 0; --i)
            if (*slot[i]) {
                cudaFreeAsync(*slot[i], s);
                *slot[i] = nullptr;
            }
    }
};

constexpr int WARP = 32;

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// ---- cache-hinted memory operations (sm_100a PTX) -------------------------
// Streamed-once data (col_idx): no L1 allocation, L2 evict-first.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Read-only gathers of the contrib vector within one synchronous sweep.
__device__ __forceinline__ double ld_gather_f64(const double* ptr, uint64_t pol) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ int32_t ld_hint_s32(const int32_t* ptr, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}

// Two-tier gather: hot contribs (small index = high out-degree) stay in L1
// (evict_last), cold ones bypass it (no_allocate) so they cannot evict the
// hot lines.  One predicated load each, branch-free.
__device__ __forceinline__ double ld_gather_tiered_f64(const double* ptr, int hot, uint64_t pol) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %3, 0;\n\t"
        "@p ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;\n\t"
        "@!p ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n\t}"
        : "=d"(r)
        : "l"(ptr), "l"(pol), "r"(hot));
    return r;
}

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) + mbarrier --------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Order earlier generic-proxy accesses of shared memory before later async-proxy writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// One elected lane: arm the barrier with `bytes` and start a global->shared
// bulk copy (16-byte aligned addresses, size a multiple of 16).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// Async (No-Sync) mode: the contrib vector is read and written in the same
// launch, so loads/stores are relaxed gpu-scope atomics (never .nc).
__device__ __forceinline__ double ld_relaxed_f64(const double* ptr) {
    double r;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(r) : "l"(ptr));
    return r;
}
__device__ __forceinline__ void st_relaxed_f64(double* ptr, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(ptr), "d"(v) : "memory");
}

}  // namespace prgpu
