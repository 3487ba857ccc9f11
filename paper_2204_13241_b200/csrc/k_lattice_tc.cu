// k_lattice_tc.cu -- K3: lattice-plane amplitude on the tcgen05 tensor cores (placeholder until implemented).
#include "common.cuh"

namespace xpcs {

bool lattice_tc_supported(const LatticeGeom&) { return false; }

cudaError_t launch_lattice_tc(const uint4*, int64_t, int64_t, const LatticeGeom&, int64_t, int64_t, float2*,
                              cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace xpcs
