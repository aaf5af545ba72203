// internal.cuh — device-side structures of libdomdec (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dd {

constexpr float kNeg = -1.0e30f;     // log of zero weight (reading R19), never NaN
constexpr int kSweepThreads = 128;

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
};

struct SweepParams {
  int N1, N2, s;
  float w;              // log2(e) / eps'   (exponent scale, base-2 units)
  const float* __restrict__ mu;
  const float* __restrict__ log2mu;
  const CompCell* __restrict__ cells;
  int ncells;
  const double* __restrict__ pool_in;
  const int* __restrict__ off_in;     // [I][2]
  const int* __restrict__ ext_in;     // [I][2]
  double* __restrict__ pool_out;
  int* __restrict__ off_out;
  int* __restrict__ ext_out;
  long long slot;                     // elements per basic-cell slot
  int ccap;                           // max composite box side
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
  int mode;                           // 0: one CTA per cell, defer cells with hull > ccap;
                                      // 1: persistent CTAs over the deferred list (large ccap)
  int* __restrict__ ovf_list;         // [ncells] deferred cells
  int* __restrict__ ovf_count;        // [1]
  double* __restrict__ mom;           // [I][6] plan moments of the last sweep (reading R13):
                                      // M0, M1 (2), G0, G1, M2 about the cell centre, px units
};

size_t sweep_smem_bytes(int ccap, int s);
cudaError_t launch_sweep(SweepParams p, int ccap_small, int ccap_big, cudaStream_t st);

}  // namespace dd
