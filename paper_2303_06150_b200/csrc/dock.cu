// dock.cu -- host-side dispatch of the dock / finalize kernels per atom class,
// shared-memory grid strides, occupancy queries, the score_points test hook.
// The kernels themselves are in dock_impl.cuh.
#include "dock_impl.cuh"

namespace vsd {

using dk::DockFn;

namespace {

DockFn pick(int AC, int NW, int PPW, int fix, int K) {
    switch (AC) {
        case 32: return dk::dock_pick_32(fix, NW, PPW, K);
        case 64: return dk::dock_pick_64(fix, NW, PPW, K);
        case 96: return dk::dock_pick_96(fix, NW, PPW, K);
        case 128: return dk::dock_pick_128(fix, NW, PPW, K);
        case 160: return dk::dock_pick_160(fix, NW, PPW, K);
        case 192: return dk::dock_pick_192(fix, NW, PPW, K);
        case 224: return dk::dock_pick_224(fix, NW, PPW, K);
        case 256: return dk::dock_pick_256(fix, NW, PPW, K);
        default: return nullptr;
    }
}

}  // namespace

// Padded shared-memory strides (tools/bank_sim3.py, the lane map of 4 poses x 8 angles:
// 3.06-way bank conflicts on the sweep's corner gathers instead of 3.21 at (33, 1063) and
// 7.5 unpadded; uniform random gathers give 3.5).  Grids of at most 32 x 32 per plane use
// the fixed layout (34, 1097) with compile-time strides; larger planes use
// (nx + 1, (nx + 1) * ny + 7).
void grid_strides(int nx, int ny, int* rs, int* ps) {
    if (nx <= 32 && ny <= 32) {
        *rs = dk::kFixRS;
        *ps = dk::kFixPS;
    } else {
        *rs = nx + 1;
        *ps = (nx + 1) * ny + 7;
    }
}

bool grid_fixed(int rs, int ps) { return rs == dk::kFixRS && ps == dk::kFixPS; }

cudaError_t dock_kernel_attrs(int AC, int NW, int PPW, int fix, int K, cudaFuncAttributes* attr) {
    DockFn f = pick(AC, NW, PPW, fix, K);
    if (!f) return cudaErrorInvalidValue;
    return cudaFuncGetAttributes(attr, reinterpret_cast<const void*>(f));
}

cudaError_t dock_occupancy(int AC, int NW, int PPW, int fix, int K, size_t smem, int* blocks_per_sm) {
    DockFn f = pick(AC, NW, PPW, fix, K);
    if (!f) {   // no instantiation for this (class, warps, poses per warp, K): the policy skips it
        *blocks_per_sm = 0;
        return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
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
    DockFn f = pick(AC, NW, PPW, grid_fixed(a.pk.rs, a.pk.ps), a.K);
    if (!f) return cudaErrorInvalidValue;
    if (a.n <= 0) return cudaSuccess;
    // the attribute is per function, and one instantiation can serve several grid layouts
    // (pockets of different sizes in one submit): set it for THIS launch's shared memory
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    f<<<grid, NW * 32, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_finalize(int AC, const DockArgs& a, const int64_t* atom_off, float* xyz_out, cudaStream_t st) {
    if (a.n <= 0) return cudaSuccess;
    switch (AC) {
        case 32: return dk::launch_finalize_32(a, atom_off, xyz_out, st);
        case 64: return dk::launch_finalize_64(a, atom_off, xyz_out, st);
        case 96: return dk::launch_finalize_96(a, atom_off, xyz_out, st);
        case 128: return dk::launch_finalize_128(a, atom_off, xyz_out, st);
        case 160: return dk::launch_finalize_160(a, atom_off, xyz_out, st);
        case 192: return dk::launch_finalize_192(a, atom_off, xyz_out, st);
        case 224: return dk::launch_finalize_224(a, atom_off, xyz_out, st);
        case 256: return dk::launch_finalize_256(a, atom_off, xyz_out, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_score_points(const PocketDev& pk, const float* xyz, int64_t n, float* out, size_t smem,
                                cudaStream_t st) {
    const bool fix = grid_fixed(pk.rs, pk.ps);
    const void* f = fix ? reinterpret_cast<const void*>(dk::score_points_kernel<true>)
                        : reinterpret_cast<const void*>(dk::score_points_kernel<false>);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (fix) dk::score_points_kernel<true><<<148, 1024, smem, st>>>(pk, xyz, n, out);
    else dk::score_points_kernel<false><<<148, 1024, smem, st>>>(pk, xyz, n, out);
    return cudaGetLastError();
}

}  // namespace vsd
