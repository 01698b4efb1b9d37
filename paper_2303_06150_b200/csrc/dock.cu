// dock.cu -- host-side dispatch of the dock kernels per atom class,
// shared-memory grid strides, occupancy queries, the score_points test hook.
// The kernels themselves are in dock_impl.cuh.
#include "dock_impl.cuh"

#include <cstdlib>
#include <cstring>

namespace vsd {

using dk::DockFn;

namespace {

DockFn pick(int AC, int NW, int PPW, int gm, int K, bool ms = false) {
    switch (AC) {
        case 32: return dk::dock_pick_32(gm, NW, PPW, K, ms);
        case 64: return dk::dock_pick_64(gm, NW, PPW, K, ms);
        case 96: return dk::dock_pick_96(gm, NW, PPW, K, ms);
        case 128: return dk::dock_pick_128(gm, NW, PPW, K, ms);
        case 160: return dk::dock_pick_160(gm, NW, PPW, K, ms);
        case 192: return dk::dock_pick_192(gm, NW, PPW, K, ms);
        case 224: return dk::dock_pick_224(gm, NW, PPW, K, ms);
        case 256: return dk::dock_pick_256(gm, NW, PPW, K, ms);
        default: return nullptr;
    }
}

}  // namespace

// Padded shared-memory strides (tools/bank_sim3.py, the lane map of 4 poses x 8 angles:
// 3.06-way bank conflicts on the sweep's corner gathers instead of 3.21 at (33, 1063) and
// 7.5 unpadded; uniform random gathers give 3.5).  Grids of at most 32^3 nodes (FIX) and the
// 32^3 window of large grids (WIN) use the fixed layout (34, 1097) with compile-time strides;
// RT grids use (nx + 1, (nx + 1) * ny + 7).  RT is chosen while its region (plus a zero plane)
// stays within the FIX budget of shared memory, so the pose buffers keep their room.
// QUAD (internal.h) whenever its window of kQuadWC cells per axis holds the whole grid or at
// least +-9 A around the docking centre (a drug-like ligand's atoms lie within ~9 A of its
// centroid: 99.96 % of the C4 library's atoms), so cells outside the window -- read
// from global memory -- stay rare.  VSDOCK_GRID_MODE=scalar selects the scalar layouts below
// (FIX / RT / WIN) for comparison.
int grid_mode(int nx, int ny, int nz, float spacing) {
    static const bool scalar = [] {
        const char* e = getenv("VSDOCK_GRID_MODE");
        return e && strcmp(e, "scalar") == 0;
    }();
    const bool fits = nx - 1 <= kQuadWC && ny - 1 <= kQuadWC && nz - 1 <= kQuadWC;
    if (!scalar && (fits || (double)spacing * (kQuadWC / 2) >= 9.0)) return kGridQuad;
    if (nx <= kWin && ny <= kWin && nz <= kWin) return kGridFix;
    const size_t rt = (size_t)(nz + 1) * ((size_t)(nx + 1) * ny + 7) + (nx + 1) + 2;
    return rt <= (size_t)kWin * dk::kFixPS + 2048 ? kGridRT : kGridWin;
}

// TYPED (Q24): the largest window edge W <= kQuadWC whose nch channel windows fit kTypedBudget
// (W = 18, 15, 13, 12, 11, 10, 10, 9 for 1..8 channels)
// VSDOCK_TYPED_BUDGET (measurement override): the channel windows' budget in quads (16 bytes)
static long typed_budget() {
    const char* e = getenv("VSDOCK_TYPED_BUDGET");
    return e ? atol(e) : (long)kTypedBudget;
}

int typed_window(int nch) {
    int W = kQuadWC;
    const long budget = typed_budget();
    while (W > 2 && (long)nch * typed_chan_stride(W) > budget) --W;
    return W;
}

// TYPED_S: the largest W <= kTypedSMaxW whose nch scalar channel windows fit the same budget
// (4 kTypedBudget floats): W = 30, 24, 20, 18, 17, 16, 15, 14 for 1..8 channels.
// Layout choice (measured): VSDOCK_TYPED_LAYOUT=quad|scalar overrides.
int typed_layout(int nch, int* W) {
    // (read at every pocket set-up, so one process can compare the two layouts)
    const char* e = getenv("VSDOCK_TYPED_LAYOUT");
    const int forced = !e ? -1 : strcmp(e, "scalar") == 0 ? kGridTypedS : strcmp(e, "quad") == 0 ? kGridTyped : -1;
    const int mode = forced >= 0 ? forced : (nch >= 2 ? kGridTypedS : kGridTyped);
    if (mode == kGridTyped) {
        *W = typed_window(nch);
        return mode;
    }
    int w = kTypedSMaxW;
    while (w > 2 && (long)nch * typeds_chan(w) > 4L * typed_budget()) --w;
    *W = w;
    return mode;
}

void grid_strides(int mode, int nx, int ny, int* rs, int* ps) {
    if (mode == kGridQuad) {   // in quads (16 bytes)
        *rs = kQuadRS;
        *ps = kQuadPS;
    } else if (mode != kGridRT) {
        *rs = dk::kFixRS;
        *ps = dk::kFixPS;
    } else {
        *rs = nx + 1;
        *ps = (nx + 1) * ny + 7;
    }
}

cudaError_t dock_kernel_attrs(int AC, int NW, int PPW, int gm, int K, cudaFuncAttributes* attr) {
    DockFn f = pick(AC, NW, PPW, gm, K);
    if (!f) return cudaErrorInvalidValue;
    return cudaFuncGetAttributes(attr, reinterpret_cast<const void*>(f));
}

cudaError_t dock_occupancy(int AC, int NW, int PPW, int gm, int K, size_t smem, int* blocks_per_sm) {
    DockFn f = pick(AC, NW, PPW, gm, K);
    if (!f) {   // no instantiation for this (class, warps, poses per warp, K): the policy skips it
        *blocks_per_sm = 0;
        return cudaSuccess;
    }
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(f));
    if (e != cudaSuccess) return e;
    if (smem + fa.sharedSizeBytes > (size_t)optin) {   // does not fit: no API call that must fail
        *blocks_per_sm = 0;
        return cudaSuccess;
    }
    e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        *blocks_per_sm = 0;
        cudaGetLastError();
        return cudaSuccess;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, reinterpret_cast<const void*>(f), NW * 32,
                                                         smem);
}

cudaError_t launch_dock(int AC, int NW, int PPW, const DockArgs& a, int grid, size_t smem, cudaStream_t st) {
    const bool ms = a.n_sites > 1;
    DockFn f = pick(AC, NW, PPW, a.pk[0].mode, a.K, ms);
    if (!f) return cudaErrorInvalidValue;
    if (a.n <= 0) return cudaSuccess;
    // the attribute is per function, and one instantiation can serve several grid layouts
    // (pockets of different sizes in one submit): set it for THIS launch's shared memory
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (!ms) {
        f<<<grid, NW * 32, smem, st>>>(a);
        return cudaGetLastError();
    }
    // fused multi-site: clusters of n_sites CTAs (grid = n_sites x clusters)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3((unsigned)(NW * 32), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)a.n_sites;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, f, a);
}

// Clusters of `sites` CTAs of the fused multi-site kernel that fit on the device at once
// (0: not available for this class / layout).
cudaError_t dock_cluster_occupancy(int AC, int NW, int PPW, int gmode, int K, size_t smem, int sites, int* clusters) {
    *clusters = 0;
    DockFn f = pick(AC, NW, PPW, gmode, K, true);
    if (!f || sites < 2 || sites > kMaxSites) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cudaSuccess;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)sites, 1, 1);
    cfg.blockDim = dim3((unsigned)(NW * 32), 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)sites;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaOccupancyMaxActiveClusters(clusters, reinterpret_cast<const void*>(f), &cfg);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *clusters = 0;
    }
    return cudaSuccess;
}

cudaError_t launch_score_points(const PocketDev& pk, const float* xyz, const uint8_t* types, int64_t n, float* out,
                                size_t smem, cudaStream_t st) {
    const void* f = pk.mode == kGridFix     ? reinterpret_cast<const void*>(dk::score_points_kernel<kGridFix>)
                    : pk.mode == kGridRT    ? reinterpret_cast<const void*>(dk::score_points_kernel<kGridRT>)
                    : pk.mode == kGridQuad  ? reinterpret_cast<const void*>(dk::score_points_kernel<kGridQuad>)
                    : pk.mode == kGridTyped ? reinterpret_cast<const void*>(dk::score_points_kernel<kGridTyped>)
                    : pk.mode == kGridTypedS ? reinterpret_cast<const void*>(dk::score_points_kernel<kGridTypedS>)
                                            : reinterpret_cast<const void*>(dk::score_points_kernel<kGridWin>);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (pk.mode == kGridFix) dk::score_points_kernel<kGridFix><<<148, 1024, smem, st>>>(pk, xyz, types, n, out);
    else if (pk.mode == kGridRT) dk::score_points_kernel<kGridRT><<<148, 1024, smem, st>>>(pk, xyz, types, n, out);
    else if (pk.mode == kGridQuad) dk::score_points_kernel<kGridQuad><<<148, 1024, smem, st>>>(pk, xyz, types, n, out);
    else if (pk.mode == kGridTyped) dk::score_points_kernel<kGridTyped><<<148, 1024, smem, st>>>(pk, xyz, types, n, out);
    else if (pk.mode == kGridTypedS) dk::score_points_kernel<kGridTypedS><<<148, 1024, smem, st>>>(pk, xyz, types, n, out);
    else dk::score_points_kernel<kGridWin><<<148, 1024, smem, st>>>(pk, xyz, types, n, out);
    return cudaGetLastError();
}

}  // namespace vsd
