// dock_inst.cu -- instantiates the dock kernels of ONE atom class
// (compiled once per class with -DVSD_AC=<AC>; see build.py).
#include "dock_impl.cuh"

#ifndef VSD_AC
#error "compile with -DVSD_AC=<atom class capacity>"
#endif
#define VSD_CAT2(a, b) a##b
#define VSD_CAT(a, b) VSD_CAT2(a, b)

namespace vsd {
namespace dk {

DockFn VSD_CAT(dock_pick_, VSD_AC)(int gmode, int NW, int PPW, int K, bool ms) {
    return gmode == kGridQuad    ? pick_ac<VSD_AC, kGridQuad>(NW, PPW, K, ms)
           : gmode == kGridTyped ? pick_ac<VSD_AC, kGridTyped>(NW, PPW, K, ms)
           : gmode == kGridTypedS ? pick_ac<VSD_AC, kGridTypedS>(NW, PPW, K, ms)
           : gmode == kGridFix ? pick_ac<VSD_AC, kGridFix>(NW, PPW, K, ms)
           : gmode == kGridRT  ? pick_ac<VSD_AC, kGridRT>(NW, PPW, K, ms)
                               : pick_ac<VSD_AC, kGridWin>(NW, PPW, K, ms);
}

}  // namespace dk
}  // namespace vsd
