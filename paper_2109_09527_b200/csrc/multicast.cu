// multicast.cu -- NVLS multicast buffers for the row-sharded iteration
// ("fuse the collective into K-GATHER's epilogue with NVLS
// multimem.st stores to a multicast-mapped y buffer (cuMulticastCreate), so the
// switch replicates each contrib store to all peers").
//
// Every rank's two contrib ping-pong buffers (and the device barrier's arrival
// flags) live in ONE physical allocation of 2 * seg bytes, bound at offset 0 of
// a multicast object whose team is the world's GPUs.  The rank maps its own
// allocation (unicast VA: every load of the sweep, sy[0] / sy[1]) and the
// multicast object (multicast VA: mcy[0] / mcy[1]); a multimem.st to the
// multicast VA lands in the same slot of every rank's allocation, so each new
// contrib is ONE store instead of world - 1 peer stores.
//
// The team is assembled in three collective steps (the caller orders them
// across ranks, e.g. with torch.distributed barriers):
//   create  (rank 0)  cuMulticastCreate + export of a 64-byte fabric handle
//   attach  (all)     import of the handle + cuMulticastAddDevice(own device)
//   bind    (all, after every rank attached)  cuMemCreate + cuMulticastBindMem
//                     + the unicast and multicast mappings
// Driver entry points come from cudaGetDriverEntryPoint (no libcuda link).
#include <cuda.h>
#include <string.h>

#include "internal.h"

namespace prgpu {

#define DRV(name) static decltype(&name) p_##name = nullptr
DRV(cuMulticastCreate);
DRV(cuMulticastAddDevice);
DRV(cuMulticastBindMem);
DRV(cuMulticastUnbind);
DRV(cuMulticastGetGranularity);
DRV(cuMemCreate);
DRV(cuMemRelease);
DRV(cuMemAddressReserve);
DRV(cuMemAddressFree);
DRV(cuMemMap);
DRV(cuMemUnmap);
DRV(cuMemSetAccess);
DRV(cuMemExportToShareableHandle);
DRV(cuMemImportFromShareableHandle);
DRV(cuMemGetAllocationGranularity);
DRV(cuDeviceGet);
#undef DRV

static int load_driver() {
    static int state = 0;  // 0 untried, 1 ok, -1 failed
    if (state) return state > 0 ? PR_OK : PR_ECUDA;
#define GET(name)                                                                                     \
    do {                                                                                              \
        cudaDriverEntryPointQueryResult q;                                                            \
        if (cudaGetDriverEntryPoint(#name, (void**)&p_##name, cudaEnableDefault, &q) != cudaSuccess || \
            q != cudaDriverEntryPointSuccess || !p_##name) {                                          \
            cudaGetLastError();                                                                       \
            set_error("multicast: driver entry point %s unavailable", #name);                        \
            state = -1;                                                                               \
            return PR_ECUDA;                                                                          \
        }                                                                                             \
    } while (0)
    GET(cuMulticastCreate);
    GET(cuMulticastAddDevice);
    GET(cuMulticastBindMem);
    GET(cuMulticastUnbind);
    GET(cuMulticastGetGranularity);
    GET(cuMemCreate);
    GET(cuMemRelease);
    GET(cuMemAddressReserve);
    GET(cuMemAddressFree);
    GET(cuMemMap);
    GET(cuMemUnmap);
    GET(cuMemSetAccess);
    GET(cuMemExportToShareableHandle);
    GET(cuMemImportFromShareableHandle);
    GET(cuMemGetAllocationGranularity);
    GET(cuDeviceGet);
#undef GET
    state = 1;
    return PR_OK;
}

#define CU_TRY(call)                                                                       \
    do {                                                                                   \
        CUresult _r = (call);                                                              \
        if (_r != CUDA_SUCCESS) {                                                          \
            set_error("multicast: %s failed (CUresult %d)", #call, (int)_r);               \
            return PR_ECUDA;                                                               \
        }                                                                                  \
    } while (0)

// bytes of one parity segment: ny doubles + world flags, rounded to the granularity
static size_t mc_segment(const pr_graph* g, size_t gran) {
    const int64_t ny = g->shard_hot + (int64_t)g->shard_world * g->shard_chunk + 1;
    const size_t bytes = sizeof(double) * (size_t)(ny + g->shard_world);
    return (bytes + gran - 1) / gran * gran;
}

static int granularity(const pr_graph* g, size_t* gran) {
    CUmulticastObjectProp mp = {};
    mp.numDevices = (unsigned)g->shard_world;
    mp.size = 1;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    size_t gm = 0;
    CU_TRY(p_cuMulticastGetGranularity(&gm, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = g->device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    size_t ga = 0;
    CU_TRY(p_cuMemGetAllocationGranularity(&ga, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    *gran = gm > ga ? gm : ga;
    if (*gran % ga) *gran = (*gran / ga + 1) * ga;
    return PR_OK;
}

void clear_multicast(pr_graph* g) {
    if (!g->mc) return;
    McState& m = *g->mc;
    if (m.bound) {
        cudaDeviceSynchronize();
        if (m.uva) {
            p_cuMemUnmap((CUdeviceptr)m.uva, m.size);
            p_cuMemAddressFree((CUdeviceptr)m.uva, m.size);
        }
        if (m.mva) {
            p_cuMemUnmap((CUdeviceptr)m.mva, m.size);
            p_cuMemAddressFree((CUdeviceptr)m.mva, m.size);
        }
        CUdevice dev;
        if (p_cuDeviceGet(&dev, g->device) == CUDA_SUCCESS) p_cuMulticastUnbind(m.mc, dev, 0, m.size);
        p_cuMemRelease(m.mem);
        g->sy[0] = g->sy[1] = nullptr;  // they pointed into the unicast mapping
    }
    if (m.have_mc) p_cuMemRelease(m.mc);
    delete g->mc;
    g->mc = nullptr;
}

int mc_create(pr_graph* g, void* handle_out) {
    PR_TRY(load_driver());
    if (g->speer_dev) {
        set_error("multicast: the IPC peer buffers are set (exclusive with multicast)");
        return PR_ESTATE;
    }
    clear_multicast(g);
    size_t gran = 0;
    PR_TRY(granularity(g, &gran));
    g->mc = new (std::nothrow) McState();
    if (!g->mc) {
        set_error("multicast: host allocation failed");
        return PR_ENOMEM;
    }
    McState& m = *g->mc;
    m.seg = mc_segment(g, gran);
    m.size = 2 * m.seg;
    CUmulticastObjectProp mp = {};
    mp.numDevices = (unsigned)g->shard_world;
    mp.size = m.size;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    CU_TRY(p_cuMulticastCreate(&m.mc, &mp));
    m.have_mc = true;
    if (handle_out) {
        CUmemFabricHandle fh;
        CU_TRY(p_cuMemExportToShareableHandle(&fh, m.mc, CU_MEM_HANDLE_TYPE_FABRIC, 0));
        memcpy(handle_out, &fh, sizeof(fh));
    }
    return PR_OK;
}

int mc_attach(pr_graph* g, const void* handle) {
    PR_TRY(load_driver());
    if (!g->mc) {  // not the creator: import the team's object
        if (!handle) {
            set_error("multicast: attach without a handle on a rank that did not create the object");
            return PR_EINVAL;
        }
        size_t gran = 0;
        PR_TRY(granularity(g, &gran));
        g->mc = new (std::nothrow) McState();
        if (!g->mc) {
            set_error("multicast: host allocation failed");
            return PR_ENOMEM;
        }
        g->mc->seg = mc_segment(g, gran);
        g->mc->size = 2 * g->mc->seg;
        CUmemFabricHandle fh;
        memcpy(&fh, handle, sizeof(fh));
        CU_TRY(p_cuMemImportFromShareableHandle(&g->mc->mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC));
        g->mc->have_mc = true;
    }
    CUdevice dev;
    CU_TRY(p_cuDeviceGet(&dev, g->device));
    CU_TRY(p_cuMulticastAddDevice(g->mc->mc, dev));
    return PR_OK;
}

int mc_bind(pr_graph* g, Ctx& ctx) {
    PR_TRY(load_driver());
    if (!g->mc || g->mc->bound) {
        set_error("multicast: bind needs an attached, unbound team");
        return PR_ESTATE;
    }
    McState& m = *g->mc;
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = g->device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    CU_TRY(p_cuMemCreate(&m.mem, m.size, &ap, 0));
    CU_TRY(p_cuMulticastBindMem(m.mc, 0, m.mem, 0, m.size, 0));
    CUdeviceptr u = 0, v = 0;
    CU_TRY(p_cuMemAddressReserve(&u, m.size, 0, 0, 0));
    CU_TRY(p_cuMemMap(u, m.size, 0, m.mem, 0));
    CU_TRY(p_cuMemAddressReserve(&v, m.size, 0, 0, 0));
    CU_TRY(p_cuMemMap(v, m.size, 0, m.mc, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = g->device;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU_TRY(p_cuMemSetAccess(u, m.size, &ad, 1));
    CU_TRY(p_cuMemSetAccess(v, m.size, &ad, 1));
    m.uva = (void*)u;
    m.mva = (void*)v;
    m.bound = true;
    // the sharded contrib buffers move into the unicast mapping
    for (int b = 0; b < 2; ++b)
        if (g->sy[b]) {
            cudaStreamSynchronize(ctx.stream);
            cudaFree(g->sy[b]);
        }
    PR_CUDA(cudaMemsetAsync(m.uva, 0, m.size, ctx.stream));
    PR_CUDA(cudaStreamSynchronize(ctx.stream));
    g->sy[0] = reinterpret_cast<double*>(m.uva);
    g->sy[1] = reinterpret_cast<double*>(reinterpret_cast<char*>(m.uva) + m.seg);
    m.y[0] = reinterpret_cast<double*>(m.mva);
    m.y[1] = reinterpret_cast<double*>(reinterpret_cast<char*>(m.mva) + m.seg);
    g->bar_epoch = 0;
    return PR_OK;
}

}  // namespace prgpu
