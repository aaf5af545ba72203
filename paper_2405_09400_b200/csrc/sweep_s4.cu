// sweep_s4.cu — sweep kernels for basic cells of 4 x 4 pixels (NX = 8).
#include "sweep_launch.cuh"

namespace dd {
template cudaError_t launch_sweep_nx<8>(const SweepParams&, const SweepClasses&, cudaStream_t, cudaStream_t);
template int sweep_occupancy_nx<8>(int, size_t);
template int cluster_capacity_nx<8>(int, size_t);
}  // namespace dd
