// sweep_launch.cuh — per-cell-size launch templates of the sweep (instantiated
// once per cell size in sweep_s*.cu so the translation units compile in
// parallel).  See sweep.cu for the size-class design.
#pragma once
#include "sweep.cuh"

namespace dd {

template <int NX, int C, bool PR>
cudaError_t launch_class(const SweepParams& p, const SweepClasses& cls, cudaStream_t st) {
  constexpr bool GS = C == 4;
  auto kern = sweep_kernel<NX, class_threads(NX, C), class_min_blocks(NX, C), PR, GS>;
  if (cls.smem[C] > 48 * 1024) {   // per-device attribute: set on every launch (cheap)
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cls.smem[C]);
    if (e != cudaSuccess) return e;
  }
  kern<<<cls.grid[C], class_threads(NX, C), cls.smem[C], st>>>(p, C, cls.ccap[C]);
  return cudaGetLastError();
}

template <int NX, bool PR>
cudaError_t launch_cluster(const SweepParams& p, const SweepClasses& cls, cudaStream_t st) {
  constexpr int NT = class_threads(NX, 4);
  auto kern = sweep_kernel_cl<NX, NT, PR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cls.cl_smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cls.cl_grid);
  cfg.blockDim = dim3((unsigned)NT);
  cfg.dynamicSmemBytes = cls.cl_smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cls.cl_size;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, p, 4, cls.ccap[4], (int)cls.cl_smem);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int NX>
int cluster_capacity_nx(int KC, size_t smem) {   // co-resident clusters (0: not launchable)
  constexpr int NT = class_threads(NX, 4);
  auto kern = sweep_kernel_cl<NX, NT, false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)KC);
  cfg.blockDim = dim3((unsigned)NT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)KC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  return cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess ? n : 0;
}

template <int NX, bool PR>
cudaError_t launch_all(const SweepParams& p, const SweepClasses& cls, cudaStream_t st, cudaStream_t aux) {
  cudaError_t e;
  // large classes on the auxiliary stream (biggest first), the bulk on the main one
  if ((e = cls.cl_size > 1 ? launch_cluster<NX, PR>(p, cls, aux) : launch_class<NX, 4, PR>(p, cls, aux)) !=
      cudaSuccess)
    return e;
  if ((e = launch_class<NX, 3, PR>(p, cls, aux)) != cudaSuccess) return e;
  if ((e = launch_class<NX, 2, PR>(p, cls, aux)) != cudaSuccess) return e;
  if ((e = launch_class<NX, 1, PR>(p, cls, aux)) != cudaSuccess) return e;
  return launch_class<NX, 0, PR>(p, cls, st);
}

template <int NX>
cudaError_t launch_sweep_nx(const SweepParams& p, const SweepClasses& cls, cudaStream_t st, cudaStream_t aux) {
  return p.ecell ? launch_all<NX, true>(p, cls, st, aux) : launch_all<NX, false>(p, cls, st, aux);
}

template <int NX, int C>
int occupancy_of(size_t smem) {
  auto kern = sweep_kernel<NX, class_threads(NX, C), class_min_blocks(NX, C), false, false>;
  if (smem > 48 * 1024 &&   // the query counts 0 CTAs above the opt-in limit
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return -1;
  int per = 0;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, class_threads(NX, C), smem) == cudaSuccess ? per
                                                                                                          : -1;
}

template <int NX>
int sweep_occupancy_nx(int C, size_t smem) {
  switch (C) {
    case 0: return occupancy_of<NX, 0>(smem);
    case 1: return occupancy_of<NX, 1>(smem);
    case 2: return occupancy_of<NX, 2>(smem);
    default: return occupancy_of<NX, 3>(smem);
  }
}

}  // namespace dd
