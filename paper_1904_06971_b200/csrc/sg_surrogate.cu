// surrogate kernels (placeholder until the interpolation path lands)
#include "sg_internal.h"
extern "C" int sg_surrogate(const sg_problem*, const sg_surrogate_params*, const sg_exec*, sg_result** out,
                            sg_surrogate_stats*) {
    if (out) *out = nullptr;
    return sg::fail(-2, "surrogate path not built yet");
}
