// cpasync_ceiling.cu -- microbenchmark (tool, not product): does the random fp64
// contrib gather run faster when the cold gathers are issued as 16-byte
// cp.async.cg (LDGSTS with L1 bypass: global -> shared memory, no L1 line held
// while the miss is in flight) instead of LDG?  Flat pass acc += y[col[e]] as
// in gather_ceiling.cu: 1024-thread CTAs, one per SM, a lane owns 8 consecutive
// edges of a 256-edge step; contribs [0, hot_n) come from a shared-memory copy.
//   ASYNC = false: cold gathers by ld.global.nc.L1::no_allocate (the control);
//   ASYNC = true : each cold gather copies the aligned 16-byte pair holding the
//                  contrib into the lane's staging slot (slot-major layout, no
//                  bank conflicts), one commit group per step, then reads it back.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double ldg_na(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ int4 ldg_stream(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <bool ASYNC>
__global__ void __launch_bounds__(1024, 1) k_flat8(const int32_t* __restrict__ col, int64_t E, const double* __restrict__ y,
                                                   int hot_n, double* out) {
    extern __shared__ __align__(16) double sm[];
    double* hot = sm;
    double2* stage = reinterpret_cast<double2*>(sm + ((hot_n + 1) & ~1));  // [8][1024]
    for (int i = threadIdx.x; i < hot_n; i += blockDim.x) hot[i] = y[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t nch = E / 256;
    const int64_t per = (nch + nwarps - 1) / nwarps;
    const int64_t cb = warp * per, ce = min(nch, cb + per);
    const uint32_t st0 = (uint32_t)__cvta_generic_to_shared(stage + threadIdx.x);
    double acc = 0.0;
    for (int64_t c = cb; c < ce; ++c) {
        const int4* p = reinterpret_cast<const int4*>(col + c * 256) + lane * 2;
        const int4 a = ldg_stream(p), b = ldg_stream(p + 1);
        const int q[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        if (ASYNC) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (q[j] >= hot_n)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st0 + (uint32_t)j * 1024u * 16u),
                                 "l"(y + (q[j] & ~1))
                                 : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (q[j] < hot_n) acc += hot[q[j]];
            asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (q[j] >= hot_n) acc += reinterpret_cast<const double*>(stage + j * 1024 + threadIdx.x)[q[j] & 1];
        } else {
            double v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = q[j] < hot_n ? hot[q[j]] : ldg_na(y + q[j]);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc += v[j];
        }
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int cpasync_run(const int32_t* col, int64_t E, const double* y, int hot_n, int async, int reps, double* out,
                           float* ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = (size_t)((hot_n + 1) & ~1) * 8 + (async ? (size_t)8 * 1024 * 16 : 0);
    auto launch = [&]() {
        if (async) {
            cudaFuncSetAttribute(k_flat8<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_flat8<true><<<sms, 1024, smem>>>(col, E, y, hot_n, out);
        } else {
            cudaFuncSetAttribute(k_flat8<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_flat8<false><<<sms, 1024, smem>>>(col, E, y, hot_n, out);
        }
    };
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    if (cudaDeviceSynchronize() != cudaSuccess) return (int)cudaGetLastError();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms / reps;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return (int)cudaGetLastError();
}
