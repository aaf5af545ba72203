// internal.cuh — device-side structures of libdomdec (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace dd {

// NVTX range over a C-ABI call (tracing: `ncu --nvtx --nvtx-include "dd:flow_update/dd:min-cost flow/"`
// selects the kernels a call launched; no cost without a tool attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Development timers (DD_MS_TIMERS=1): host time between checkpoints, with a
// device synchronisation at each checkpoint; no effect otherwise.
struct DevTimer {
  bool on = getenv("DD_MS_TIMERS") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[dd timer] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

constexpr float kNeg = -1.0e30f;     // log of zero weight (reading R19), never NaN
constexpr int kClasses = 5;          // size classes of the sweep (S, M, L, X, H)
// Threads and target CTAs per SM of each size class.  Cells of s <= 2
// (NX <= 4) carry a quarter of the work of s = 4 cells with the same per-cell
// overheads, so their classes use half the threads and twice the CTAs.
__host__ __device__ constexpr int class_threads(int NX, int C) {
  return NX <= 4 ? (C == 0 ? 64 : C == 1 ? 128 : C == 2 ? 256 : 512) : (C == 0 ? 128 : C == 1 ? 256 : 512);
}
__host__ __device__ constexpr int class_min_blocks(int NX, int C) {
  return NX <= 4 ? (C == 0 ? 14 : C == 1 ? 7 : C == 2 ? 3 : 1) : (C == 0 ? 7 : C == 1 ? 3 : C == 2 ? 2 : 1);
}

// One composite cell (Def. partitions).
struct CompCell {
  int r0, c0;       // pixel origin of the X-block X_J
  int n1, n2;       // X-block extent in pixels (s or 2s)
  int nmem;         // number of basic cells (1..4)
  int mem[4];       // basic cell indices, row-major order
  int quad[4];      // (h1 << 1) | h2: quadrant of the member inside the X-block
};

// Per composite-cell results of a sweep.
struct CellStats {
  int iters;
  int overflow;
  float e0;         // X-error after the first pass
  float e;          // X-error of the returned plan
  double dropped;   // truncated mass
};

// Device-side accumulators of one sweep (reset before each sweep).
struct SweepTotals {
  unsigned long long mufu;     // algorithmic ex2 + lg2
  unsigned long long bytes;    // algorithmic HBM bytes
  unsigned long long iters;
  unsigned long long cells;
  unsigned long long nonconv;
  unsigned long long overflow;
  int iters_max;
  int pad;
  double e0;
  double e;
  double dropped;
  unsigned long long invalid;  // output pool exhausted: the state is invalid (sticky in the
                               // cumulative totals, reported by every synchronising call)
};

struct SweepParams {
  int N1, N2, s;
  float w;              // log2(e) / eps'   (exponent scale, base-2 units)
  const float* __restrict__ mu;
  const float* __restrict__ log2mu;
  const CompCell* __restrict__ cells;
  int ncells;
  const double* __restrict__ pool_in;
  const long long* __restrict__ pos_in;   // [I] start of box i in pool_in
  const int* __restrict__ off_in;     // [I][2]
  const int* __restrict__ ext_in;     // [I][2]
  double* __restrict__ pool_out;
  long long* __restrict__ pos_out;
  int* __restrict__ off_out;
  int* __restrict__ ext_out;
  unsigned long long* __restrict__ pool_ctr;   // bump allocator of pool_out (elements used)
  long long pool_cap;                 // capacity of pool_out (elements)
  unsigned char* scratch;             // global scratch of the huge size class
  size_t scratch_stride;              // bytes per CTA
  float* __restrict__ alpha;          // [N1*N2] base-2 local-gauge potential of this partition
  int* __restrict__ gauge;            // [ncells][2] gauge origin used for alpha
  int alpha_valid;
  const double* __restrict__ m;       // basic-cell masses
  float tol;                          // Err
  int max_iter;
  int fixed_iter;
  double tau;
  CellStats* __restrict__ stats;
  SweepTotals* __restrict__ totals;
  SweepTotals* __restrict__ cum;      // cumulative over all sweeps (not reset)
  // size classes: k_bin appends every composite
  // cell to the list of the smallest class whose capacity holds its hull
  int* __restrict__ cls_count;        // [kClasses] cells per class
  int* __restrict__ cls_fetch;        // [kClasses] dynamic work counters
  int* __restrict__ cls_list;         // [kClasses][ncells]
  double* __restrict__ mom;           // [I][6] plan moments of the last sweep (reading R13):
                                      // M0, M1 (2), G0, G1, M2 about the cell centre, px units
  const double* __restrict__ nu;      // [N1*N2] global nu (primal score only)
  double* __restrict__ ecell;         // [ncells] primal score of each returned plan / h^2
  double eps_p;                       // eps' = eps / h^2
  double* __restrict__ pxm;           // [N1*N2][3] or NULL: per pixel PX(x) and E[y - x | x]
                                      // of the last sweep's plan (gluing candidates, f1)
};

// Launch configuration of the size classes (host side, per context).
struct SweepClasses {
  int ccap[kClasses];      // hull side capacity of each class (ccap[H] = the grid)
  int threads[kClasses];
  int grid[kClasses];      // persistent CTAs per class
  size_t smem[kClasses];   // dynamic shared memory per CTA (0 for H: global scratch)
  // H on thread-block clusters (sweep_cluster.cuh): cl_size CTAs per cell,
  // cl_grid CTAs, cl_smem bytes of dynamic shared memory each; 0 = off
  int cl_size, cl_grid;
  size_t cl_smem;
};
cudaError_t sweep_classes(int s, int N, int nsm, int ncells, SweepClasses* out, size_t* scratch_stride);
cudaError_t launch_sweep(const SweepParams& p, const SweepClasses& cls, cudaStream_t st, cudaStream_t aux,
                         cudaEvent_t fork, cudaEvent_t join);

}  // namespace dd
