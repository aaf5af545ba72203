// sweep_s1.cu — sweep kernels for basic cells of 1 x 1 pixels (NX = 2).
#include "sweep_launch.cuh"

namespace dd {
template cudaError_t launch_sweep_nx<2>(const SweepParams&, const SweepClasses&, cudaStream_t, cudaStream_t);
template int sweep_occupancy_nx<2>(int, size_t);
template int cluster_capacity_nx<2>(int, size_t);
}  // namespace dd
