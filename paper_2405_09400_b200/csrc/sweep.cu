// sweep.cu — launch side of the domain-decomposition sweep (device code in
// sweep.cuh, per-cell-size kernels in sweep_s*.cu): size classes, binning,
// the class launches.
//
// Size classes (the device-side analogue of the paper's clustering of cells
// by bounding-box size).  A cell's shared-memory working
// set grows with its hull (24 B per hull entry), and hulls grow along a
// trajectory (low-mass cells, flow updates merging boxes: up to ~100 px at
// 1024^2 after 25 hybrid cycles, median ~27).  One launch configuration for
// all cells would either not fit the large hulls or run the common small
// ones at low occupancy, so k_bin appends each composite cell to the list of
// the smallest class whose capacity holds its hull side, and each class runs
// persistent CTAs (dynamic cell fetch) with a CTA size and occupancy matched
// to its hulls:
//   S  128 threads, 7 CTAs/SM   (the bulk of the cells)
//   M  256 threads, 3 CTAs/SM
//   L  512 threads, 2 CTAs/SM
//   X  512 threads, 1 CTA/SM    (largest hull that fits 227 KB)
// (s <= 2: S 64 x 14, M 128 x 7, L 256 x 3, X 512 x 1; internal.cuh)
//   H  512 threads, one CTA per SM on global-memory scratch (hull <= 1024; rare)
// The large classes run on an auxiliary stream concurrently with S (fork /
// join events), so their few long cells overlap the bulk instead of forming a
// serial tail.  No host synchronisation inside a sweep.
#include "sweep.cuh"
#include <algorithm>
#include <cstdlib>

namespace dd {

template <int NX>
cudaError_t launch_sweep_nx(const SweepParams& p, const SweepClasses& cls, cudaStream_t st, cudaStream_t aux);
template <int NX>
int sweep_occupancy_nx(int C, size_t smem);
template <int NX>
int cluster_capacity_nx(int KC, size_t smem);

namespace {


// Bin every composite cell by the side of its hull (warp-aggregated atomics).
__global__ void k_bin(const SweepParams p, const int4 caps) {
  const int J = blockIdx.x * blockDim.x + threadIdx.x;
  int cls = -1;
  if (J < p.ncells) {
    const CompCell cc = p.cells[J];
    int L1 = 1 << 30, L2 = 1 << 30, U1 = -(1 << 30), U2 = -(1 << 30);
    for (int k = 0; k < cc.nmem; ++k) {
      const int i = cc.mem[k];
      const int r = p.off_in[2 * i], c = p.off_in[2 * i + 1];
      L1 = min(L1, r);
      L2 = min(L2, c);
      U1 = max(U1, r + p.ext_in[2 * i]);
      U2 = max(U2, c + p.ext_in[2 * i + 1]);
    }
    const int side = max(U1 - L1, U2 - L2);
    cls = side <= caps.x ? 0 : side <= caps.y ? 1 : side <= caps.z ? 2 : side <= caps.w ? 3 : 4;
  }
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < kClasses; ++c) {
    const unsigned mask = __ballot_sync(0xffffffffu, cls == c);
    if (!mask) continue;
    const int leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&p.cls_count[c], __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (cls == c) p.cls_list[(size_t)c * p.ncells + base + __popc(mask & ((1u << lane) - 1u))] = J;
  }
}

int occupancy_s(int s, int C, size_t smem) {
  switch (s) {
    case 1: return sweep_occupancy_nx<2>(C, smem);
    case 2: return sweep_occupancy_nx<4>(C, smem);
    case 4: return sweep_occupancy_nx<8>(C, smem);
    default: return sweep_occupancy_nx<16>(C, smem);
  }
}

int cluster_capacity_s(int s, int KC, size_t smem) {
  switch (s) {
    case 1: return cluster_capacity_nx<2>(KC, smem);
    case 2: return cluster_capacity_nx<4>(KC, smem);
    case 4: return cluster_capacity_nx<8>(KC, smem);
    default: return cluster_capacity_nx<16>(KC, smem);
  }
}

}  // namespace

cudaError_t sweep_classes(int s, int N, int nsm, int ncells, SweepClasses* out, size_t* scratch_stride) {
  if (s != 1 && s != 2 && s != 4 && s != 8) return cudaErrorInvalidValue;
  // 228 KB of shared memory per SM, 1 KB reserved per CTA, <= 227 KB per CTA
  const size_t per_sm = 228 * 1024, max_cta = 227 * 1024;
  int prev = 0;
  for (int C = 0; C < kClasses - 1; ++C) {
    const int nt = class_threads(2 * s, C);
    size_t budget = per_sm / class_min_blocks(2 * s, C) - 1024;
    if (budget > max_cta) budget = max_cta;
    int cap = prev;
    while (cap < N && cell_layout(cap + 1, s, nt).total <= budget) ++cap;
    out->ccap[C] = cap;
    out->threads[C] = nt;
    out->smem[C] = cell_layout(cap > 0 ? cap : 1, s, nt).total;
    int occ = 1;
    if (cap > 0) {
      occ = occupancy_s(s, C, out->smem[C]);
      if (occ <= 0) return cudaErrorInvalidConfiguration;
    }
    long long g = (long long)nsm * occ;
    if (g > ncells) g = ncells;
    out->grid[C] = (int)(g > 0 ? g : 1);
    prev = cap;
  }
  // H: any hull up to 1024 px on global-memory scratch (24 B per entry,
  // 25 MB per CTA at 1024); one CTA per SM so that the few huge cells of a
  // refined multiscale layer run side by side instead of in waves of 16
  out->ccap[4] = N < 1024 ? N : 1024;
  out->threads[4] = class_threads(2 * s, 4);
  out->smem[4] = 0;
  out->grid[4] = nsm;
  *scratch_stride = ((size_t)cell_layout(out->ccap[4], s, out->threads[4]).total + 255) & ~size_t(255);
  // H on clusters of 8 CTAs (one per SM, 160 KB of shared memory each for the
  // rows of the cell; sweep_cluster.cuh), a cluster per 8 SMs.  Test knobs:
  // DD_H_CLUSTER = cluster size (0: the single-CTA path), DD_H_CLUSTER_KB =
  // shared memory per CTA (a small value sends every cell to the leader-only
  // fallback).
  out->cl_size = 0;
  out->cl_grid = 0;
  out->cl_smem = 0;
  const char* env = getenv("DD_H_CLUSTER");
  const char* envkb = getenv("DD_H_CLUSTER_KB");
  const int KC = env ? atoi(env) : 8;
  if (KC == 2 || KC == 4 || KC == 8) {
    const size_t sm = (size_t)(envkb && atoi(envkb) > 0 ? atoi(envkb) : 160) * 1024;
    const int active = cluster_capacity_s(s, KC, sm);   // co-resident clusters (placement limits)
    if (active > 0) {
      out->cl_size = KC;
      out->cl_grid = std::min(nsm / KC, active) * KC;
      out->cl_smem = sm;
    }
    cudaGetLastError();   // a failed capacity query is not an error of the caller
  }
  return cudaSuccess;
}

cudaError_t launch_sweep(const SweepParams& p, const SweepClasses& cls, cudaStream_t st, cudaStream_t aux,
                         cudaEvent_t fork, cudaEvent_t join) {
  cudaError_t e = cudaMemsetAsync(p.cls_count, 0, 2 * kClasses * sizeof(int), st);   // counts + fetch counters
  if (e == cudaSuccess) e = cudaMemsetAsync(p.pool_ctr, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  const int4 caps = make_int4(cls.ccap[0], cls.ccap[1], cls.ccap[2], cls.ccap[3]);
  k_bin<<<(p.ncells + 255) / 256, 256, 0, st>>>(p, caps);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const bool fork_join = aux && aux != st && fork && join;
  if (!fork_join) aux = st;
  if (fork_join) {
    if ((e = cudaEventRecord(fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(aux, fork, 0)) != cudaSuccess) return e;
  }
  switch (p.s) {
    case 1: e = launch_sweep_nx<2>(p, cls, st, aux); break;
    case 2: e = launch_sweep_nx<4>(p, cls, st, aux); break;
    case 4: e = launch_sweep_nx<8>(p, cls, st, aux); break;
    case 8: e = launch_sweep_nx<16>(p, cls, st, aux); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  if (fork_join) {
    if ((e = cudaEventRecord(join, aux)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(st, join, 0)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace dd
