// sweep_s2.cu — sweep kernels for basic cells of 2 x 2 pixels (NX = 4).
#include "sweep_launch.cuh"

namespace dd {
template cudaError_t launch_sweep_nx<4>(const SweepParams&, const SweepClasses&, cudaStream_t, cudaStream_t);
template int sweep_occupancy_nx<4>(int, size_t);
template int cluster_capacity_nx<4>(int, size_t);
}  // namespace dd
