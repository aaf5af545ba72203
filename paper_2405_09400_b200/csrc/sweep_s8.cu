// sweep_s8.cu — sweep kernels for basic cells of 8 x 8 pixels (NX = 16).
#include "sweep_launch.cuh"

namespace dd {
template cudaError_t launch_sweep_nx<16>(const SweepParams&, const SweepClasses&, cudaStream_t, cudaStream_t);
template int sweep_occupancy_nx<16>(int, size_t);
template int cluster_capacity_nx<16>(int, size_t);
}  // namespace dd
