// Kernel instantiations for one (dimension, form, rational) triple; compiled as separate
// translation units so the build parallelises.  Exposes one pointer getter per triple.
#include "sg_assemble.cuh"
#include "sg_geom.cuh"
#include "sg_tile_mma.cuh"

#if !defined(SG_INST_NDIM) || !defined(SG_INST_FORM) || !defined(SG_INST_RAT)
#error "define SG_INST_NDIM, SG_INST_FORM and SG_INST_RAT"
#endif

namespace sg {

constexpr int kmax_for(int ndim) { return ndim == 3 ? 8 : 1; }
constexpr bool kRat = SG_INST_RAT != 0;

template <int P>
static void* simt_ptr() {
    if constexpr (SG_INST_FORM == BIHARMONIC && P < 2) return nullptr;
    else return (void*)&assemble_tiles<SG_INST_NDIM, P, SG_INST_FORM, kRat, kmax_for(SG_INST_NDIM)>;
}

template <int P>
static void* mma_ptr() {
    constexpr TileChoice tc = mma_tile(SG_INST_NDIM, P, SG_INST_FORM, kRat);
    constexpr bool fits = mma_geom(SG_INST_NDIM, P, SG_INST_FORM, kRat, tc.T0, tc.T1).total * 8 <= 227 * 1024;
    if constexpr ((SG_INST_FORM == BIHARMONIC && P < 2) || !fits) return nullptr;
    else return (void*)&assemble_mma<SG_INST_NDIM, P, SG_INST_FORM, kRat>;
}

#define SG_CAT2(a, b) a##b
#define SG_CAT(a, b) SG_CAT2(a, b)
#define SG_NAME SG_CAT(SG_CAT(SG_CAT(kernel_ptr_, SG_INST_NDIM), SG_CAT(_, SG_INST_FORM)), SG_CAT(_, SG_INST_RAT))

// which: 0 = SIMT tile kernel, 1 = DMMA tile kernel, 2 = geometry (K3), 3 = geometry of a polynomial map
void* SG_NAME(int which, int p, int* kmax) {
    if (kmax) *kmax = which == 1 ? 32 * mma_warps(SG_INST_NDIM, p, SG_INST_FORM, kRat) : kmax_for(SG_INST_NDIM);
    if (which == 2) return (void*)&geom_D_kernel<SG_INST_NDIM, SG_INST_FORM, kRat, false>;
    if (which == 3) return (void*)&geom_D_kernel<SG_INST_NDIM, SG_INST_FORM, kRat, true>;
    switch (p) {
        case 1: return which ? mma_ptr<1>() : simt_ptr<1>();
        case 2: return which ? mma_ptr<2>() : simt_ptr<2>();
        case 3: return which ? mma_ptr<3>() : simt_ptr<3>();
        case 4: return which ? mma_ptr<4>() : simt_ptr<4>();
    }
    return nullptr;
}

}  // namespace sg
