// Kernel instantiations of the tiled assembly kernel for one dimension (SG_INST_NDIM).
// Compiled once per dimension so the build parallelises.
#include "sg_assemble.cuh"
#include "sg_geom.cuh"

#if !defined(SG_INST_NDIM) || !defined(SG_INST_FORM)
#error "define SG_INST_NDIM and SG_INST_FORM"
#endif

namespace sg {

constexpr int kmax_for(int ndim) { return ndim == 3 ? 8 : 1; }

template <int P, int FORM, bool RAT>
static void* kptr() {
    if constexpr (FORM == BIHARMONIC && P < 2) return nullptr;
    else return (void*)&assemble_tiles<SG_INST_NDIM, P, FORM, RAT, kmax_for(SG_INST_NDIM)>;
}

template <int P>
static void* kptr_p(bool rat) {
    return rat ? kptr<P, SG_INST_FORM, true>() : kptr<P, SG_INST_FORM, false>();
}

#define SG_CAT2(a, b) a##b
#define SG_CAT(a, b) SG_CAT2(a, b)

void* SG_CAT(SG_CAT(assemble_kernel_, SG_INST_NDIM), SG_CAT(_, SG_INST_FORM))(int p, bool rat, int* kmax) {
    *kmax = kmax_for(SG_INST_NDIM);
    switch (p) {
        case 1: return kptr_p<1>(rat);
        case 2: return kptr_p<2>(rat);
        case 3: return kptr_p<3>(rat);
        case 4: return kptr_p<4>(rat);
#if SG_MAX_P >= 5
        case 5: return kptr_p<5>(rat);
#endif
    }
    return nullptr;
}

void* SG_CAT(SG_CAT(geom_kernel_, SG_INST_NDIM), SG_CAT(_, SG_INST_FORM))(bool rat) {
    return rat ? (void*)&geom_D_kernel<SG_INST_NDIM, SG_INST_FORM, true> : (void*)&geom_D_kernel<SG_INST_NDIM, SG_INST_FORM, false>;
}

}  // namespace sg
