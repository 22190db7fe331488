// hub_ceiling.cu -- microbenchmark (tool) for a slice-blocked gather of the
// hub rows' edges: the edges of high-in-degree rows are grouped by the 16K-slot
// slice of their contrib slot; a CTA loads a slice into shared memory and
// gathers its edges from there (LDS instead of one L2 request per gather).
// Measures the gather ceiling of that part (sum only, no row segmentation).
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int SL = 16384;  // slots per slice (128 KB of fp64)

// Units: unit u covers steps [u*U, (u+1)*U) of 256 edges each of the padded
// slice-major edge array; unit_slice[u] = its slice.  CTA c processes the
// contiguous unit range [c*per, (c+1)*per), reloading the slice on a change.
__global__ void __launch_bounds__(1024, 1) k_hub(const uint16_t* __restrict__ lslot, const int32_t* __restrict__ unit_slice,
                                                 int64_t nunits, int64_t per, int U, const double* __restrict__ y,
                                                 int64_t nslots, double* out) {
    extern __shared__ double sl[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t u0 = (int64_t)blockIdx.x * per, u1 = min(nunits, u0 + per);
    double acc = 0.0;
    int64_t u = u0;
    while (u < u1) {
        const int q = unit_slice[u];
        int64_t ue = u + 1;  // the run of units in the same slice
        while (ue < u1 && unit_slice[ue] == q) ++ue;
        __syncthreads();
        const int64_t base = (int64_t)q * SL;
        const int cnt = (int)min((int64_t)SL, nslots - base);
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) sl[i] = __ldcg(y + base + i);
        if (threadIdx.x == 0) sl[SL] = 0.0;
        __syncthreads();
        // warp w: steps u*U + w, + 32, ... of the run, next step's indices prefetched
        const int64_t s0 = u * U + warp, s1 = ue * U;
        uint4 nxt = make_uint4(0, 0, 0, 0);
        if (s0 < s1) nxt = __ldcs(reinterpret_cast<const uint4*>(lslot + s0 * 256 + lane * 8));
        for (int64_t st = s0; st < s1; st += 32) {
            const uint4 raw = nxt;
            if (st + 32 < s1) nxt = __ldcs(reinterpret_cast<const uint4*>(lslot + (st + 32) * 256 + lane * 8));
            const uint16_t* sv = reinterpret_cast<const uint16_t*>(&raw);
            double v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = sl[sv[j]];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc += v[j];
        }
        u = ue;
    }
    out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

extern "C" int hub_run(const uint16_t* lslot, const int32_t* unit_slice, int64_t nunits, int U, const double* y,
                       int64_t nslots, double* out, int reps, float* ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms;
    const int64_t per = (nunits + grid - 1) / grid;
    const size_t smem = (SL + 1) * sizeof(double);
    cudaFuncSetAttribute(k_hub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_hub<<<grid, 1024, smem>>>(lslot, unit_slice, nunits, per, U, y, nslots, out);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) k_hub<<<grid, 1024, smem>>>(lslot, unit_slice, nunits, per, U, y, nslots, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms / reps;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return (int)cudaGetLastError();
}
