// adi_fast.cu -- throughput-mode ADI kernels (placeholder until implemented).
#include "adi_kernels.h"

namespace pcgpu {

bool fast_supported(const DevProblem&) { return false; }
void launch_radial_fast(const DevProblem&, int, double, double, double, const double*,
                        const double*, const double*, const double*, double*, DevStatus*,
                        cudaStream_t) {}
void launch_explicit_axial_fast(const DevProblem&, const double*, double*, DevStatus*,
                                cudaStream_t) {}
void launch_axial_rhs_fast(const DevProblem&, double, double, const double*, const double*,
                           double*, double*, double*, DevStatus*, cudaStream_t) {}
void launch_axial_fast(const DevProblem&, int, double, const double*, const double*,
                       const double*, const double*, double*, DevStatus*, cudaStream_t) {}

}  // namespace pcgpu
