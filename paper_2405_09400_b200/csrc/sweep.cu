// sweep.cu — the domain-decomposition sweep (sm_100a): two kernels per
// partition sweep, each batched over all composite cells (one CTA per cell,
// as the batched SinkhornGPU of App. A.1):
//
// solve_kernel (fp32 only, small register/shared footprint -> high occupancy)
//   a1 BasicToComposite   nu_J = sum_{i in J} nu_i on the hull box
//                         (Eq. get-composite-cell-marginal PAPER.md:1128-1133),
//                         needed here only as log2 nu_J
//   a2 log-domain separable Sinkhorn on X_J x box(nu_J),
//      base-2, in a per-cell local gauge, stopping
//      rule = L1 X-marginal error after the Y-update <= Err mu(X_J)
//      (per-cell reading R6), warm start from the previous
//      sweep on the same partition (reading R7); writes the plan's potential
//      (the warm start of the next sweep) and per-cell stats.
// split_kernel (fp64 marginals)
//   a1 nu_J again, in fp64
//   a3 CompositeToBasic   nu_i = nu_J exp(S_i - LSE_i' S_i') (share form of
//                         PAPER.md:1151-1193), plus
//                         the plan moments for the flow update (R13)
//   a4 Balance            (Alg. 4 l.6 PAPER.md:1231, reading R8)
//   a5 Truncate + minimal box (Alg. 4 l.7 PAPER.md:1233, tau PAPER.md:1265)
//   a6 per-cell stats for the sweep reductions.
// The linear-domain marginals are fp64 so that the global Y-marginal is
// preserved to fp64 rounding.  Cells whose hull
// exceeds the fast size class are queued on the device and handled by a
// second, large-shared-memory launch of each kernel.
#include <cstdio>

#include "internal.cuh"

#ifndef DD_SOLVE_MINB
#define DD_SOLVE_MINB 8
#endif
#ifndef DD_SPLIT_MINB
#define DD_SPLIT_MINB 4
#endif

namespace dd {

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x - 1 with relative accuracy near 0 (X-error of a nearly converged cell).
__device__ __forceinline__ float exp2m1f(float x) {
  if (fabsf(x) < 0.0625f) {
    const float t = x * 0.69314718055994531f;
    return t * (1.0f + t * (0.5f + t * (0.16666667f + t * 0.041666668f)));
  }
  return ex2f(x) - 1.0f;
}

// Deterministic block sum of one double (fixed tree); scratch >= 32 doubles.
__device__ __forceinline__ double block_sum1_d(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < nw; ++k) t += scratch[k];
  __syncthreads();
  return t;
}

// Deterministic block sum of the first 32 of N doubles per thread: a
// transpose butterfly leaves lane l with the warp total of value l (31
// shuffles of doubles instead of 160), then the warps are summed in a fixed
// order.  Fully unrolled so v stays in registers.  scratch >= 32 * nw.
// Generic deterministic block sum of NV (power of two <= 32) values of type T
// per thread: transpose butterfly inside the warp (NV - 1 + log2(32/NV)
// shuffles), then a fixed-order sum over the warps.  out[0..NV) in shared memory.
template <typename T, int NV>
__device__ __forceinline__ void block_xsum(T (&v)[NV], T* scratch, T* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int idx = 0, o = 16;
#pragma unroll
  for (int n = NV; n > 1; n >>= 1) {
    const int h = n >> 1;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const T send = up ? v[i] : v[i + h];
      const T keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    if (up) idx += h;
    o >>= 1;
  }
  T t = v[0];
  for (int oo = o; oo > 0; oo >>= 1) t += __shfl_xor_sync(0xffffffffu, t, oo);
  if ((lane & (32 / NV - 1)) == 0) scratch[wid * NV + idx] = t;   // one writer per output
  __syncthreads();
  if (threadIdx.x < NV) {
    T s = T(0);
    for (int q = 0; q < nw; ++q) s += scratch[q * NV + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

template <int N>
__device__ __forceinline__ void block_sum32_d(double (&v)[N], double* scratch, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int n = 32, o = 16; n > 1; n >>= 1, o >>= 1) {
    const int h = n >> 1;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? v[i] : v[i + h];
      const double keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  scratch[wid * 32 + lane] = v[0];   // lane l holds the total of value l
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (int q = 0; q < nw; ++q) t += scratch[q * 32 + threadIdx.x];
    out[threadIdx.x] = t;
  }
  __syncthreads();
}

__device__ __forceinline__ float block_max_f(float v, float* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  float t = scratch[0];
  for (int w = 1; w < nw; ++w) t = fmaxf(t, scratch[w]);
  __syncthreads();
  return t;
}

// Sum over the block; scratch must hold 2 * (blockDim / 32) floats and
// consecutive calls must alternate 'parity' (one barrier per call).
__device__ __forceinline__ float block_sum_f(float v, float* scratch, int parity) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  float* sc = scratch + (parity & 1) * nw;
  if (lane == 0) sc[wid] = v;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < nw; ++w) t += sc[w];
  return t;
}

// ---------------------------------------------------------------------------
// Shared-memory layouts.  BB = ccap^2 box entries, NX = 2 s.
// Byte offsets are 32-bit (the global-scratch class at ccap 1024 needs ~10 MB):
// cheaper to rematerialise than 64-bit offsets in the register-bound loops.
struct SolveLayout {
  unsigned B, LN, BK, U, V, X, fred, ints, dred, total;   // X: A2, A2n, LM, MU, AL
};
__host__ __device__ inline SolveLayout solve_layout(int ccap, int s) {
  SolveLayout L;
  const unsigned BB = (unsigned)ccap * (unsigned)ccap, NX = 2u * (unsigned)s;
  unsigned o = 0;
  auto take = [&](unsigned bytes) { unsigned r = o; o += (bytes + 15u) & ~15u; return r; };
  L.B = take(BB * 4);
  L.LN = take(BB * 4);
  L.BK = take(BB * 8);       // fp64 assembly scratch first, then BK (fp32)
  L.U = take(2 * NX * ccap * 4);
  L.V = take(2 * NX * ccap * 4);
  L.X = take((5 * NX * NX + 4) * 4);   // + scalars (mass defect rm1)
  L.fred = take(64 * 4);
  L.ints = take(64 * 4);
  // fp64 reduction scratch of the primal epilogue: the U/V stage buffers are
  // free after the Sinkhorn loop; a separate slot only if they are too small
  L.dred = (4 * NX * ccap * 4 >= 80 * 8) ? L.U : take(80 * 8);
  L.total = o;
  return L;
}
struct SplitLayout {
  unsigned nuJ, red, P0, P1, P2, P3, U, R, AL, ints, total;
};
__host__ __device__ inline SplitLayout split_layout(int ccap, int s) {
  SplitLayout L;
  const unsigned BB = (unsigned)ccap * (unsigned)ccap, NX = 2u * (unsigned)s;
  unsigned o = 0;
  auto take = [&](unsigned bytes) { unsigned r = o; o += (bytes + 15u) & ~15u; return r; };
  L.nuJ = take(BB * 8);
  L.red = take(288 * 8);
  L.P0 = take(BB * 4);
  L.P1 = take(BB * 4);
  L.P2 = take(BB * 4);
  L.P3 = take(BB * 4);
  L.U = take(2 * NX * ccap * 4);
  L.R = take(4 * NX * ccap * 4);
  L.AL = take(NX * NX * 4);
  L.ints = take(64 * 4);
  L.total = o;
  return L;
}
size_t sweep_smem_bytes(int ccap, int s) {
  const size_t a = solve_layout(ccap, s).total, b = split_layout(ccap, s).total;
  return a > b ? a : b;
}

// Member boxes and hull of composite cell J (a1).  ints[0..15] receive the
// member offsets/extents; returns (L1, L2, b1, b2).
__device__ __forceinline__ int4 cell_hull(const SweepParams& p, const CompCell& cc, int* ints) {
  const int tid = threadIdx.x;
  if (tid < cc.nmem) {
    const int i = cc.mem[tid];
    ints[tid] = p.off_in[2 * i];
    ints[4 + tid] = p.off_in[2 * i + 1];
    ints[8 + tid] = p.ext_in[2 * i];
    ints[12 + tid] = p.ext_in[2 * i + 1];
  }
  __syncthreads();
  int L1 = ints[0], L2 = ints[4], U1 = ints[0] + ints[8], U2 = ints[4] + ints[12];
  for (int k = 1; k < cc.nmem; ++k) {
    L1 = min(L1, ints[k]);
    L2 = min(L2, ints[4 + k]);
    U1 = max(U1, ints[k] + ints[8 + k]);
    U2 = max(U2, ints[4 + k] + ints[12 + k]);
  }
  return make_int4(L1, L2, U1 - L1, U2 - L2);
}

// nu_J = sum of the member boxes on the hull, fp64, member order (a1).
__device__ __forceinline__ void assemble(const SweepParams& p, const CompCell& cc, const int* ints, int L1, int L2,
                                         int b2, int BB, double* nuJ) {
  const int tid = threadIdx.x, T = blockDim.x;
  for (int t = tid; t < BB; t += T) nuJ[t] = 0.0;
  __syncthreads();
  for (int k = 0; k < cc.nmem; ++k) {
    const int i = cc.mem[k];
    const int e1 = ints[8 + k], e2 = ints[12 + k];
    const int d1 = ints[k] - L1, d2 = ints[4 + k] - L2;
    const double* src = p.pool_in + p.pos_in[i];
    for (int t = tid; t < e1 * e2; t += T) {
      const int r = t / e2, c = t - r * e2;
      nuJ[(d1 + r) * b2 + d2 + c] += src[t];
    }
    __syncthreads();
  }
}

// Primal score of the plan a solve returns (diagnostic):
// pi(k, l) = 2^(A(k) + B(l) - w |kappa - lt|^2) mu(k) nu_J(l) in the local
// gauge, k = K + kappa, l = G + lt, D = K - G.  Its Y-marginal is nu_J, its
// X-marginal PX = mu 2^(A - A').  With c = h^2 |k - l|^2 and eps = eps' h^2,
//   (<c, pi> + eps KL(pi | mu (x) nu) + eps sum pi) / h^2
//     = |D|^2 S0 + 2 D.(S_kappa - S_lt) + eps' (ln2 (S_A + S_B + S_L) - S0),
// S0 = sum nu_J, S_kappa = sum kappa PX, S_lt = sum lt nu_J, S_A = sum A PX,
// S_B = sum B nu_J, S_L = sum nu_J log2(nu_J / nu).
// nu_J is re-assembled in fp64 (the BK region is free after the loop).
template <int NX>
__device__ __forceinline__ void primal_terms(const SweepParams& p, const CompCell& cc, const int J, const int* ints,
                                          const int L1, const int L2, const int b1, const int b2, const int o1,
                                          const int o2, const int G1, const int G2, const float* A2,
                                          const float* A2n, const float* MU, const float* Bp, double* nuJ,
                                          double* red) {
  const int tid = threadIdx.x, T = blockDim.x;
  __syncthreads();
  assemble(p, cc, ints, L1, L2, b2, b1 * b2, nuJ);
  double v[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  constexpr int NXX = NX * NX;
  for (int t = tid; t < NXX; t += T) {
    const int k1 = t / NX, k2 = t % NX;
    if (k1 < cc.n1 && k2 < cc.n2) {
      const double a = (double)A2[t];
      const double px = (double)MU[t] * exp2(a - (double)A2n[t]);
      v[0] += a * px;
      v[1] += (double)k1 * px;
      v[2] += (double)k2 * px;
    }
  }
  for (int t = tid; t < b1 * b2; t += T) {
    const double nj = nuJ[t];
    if (nj > 0.0) {
      const int l1 = t / b2, l2 = t - l1 * b2;
      const double ng = p.nu[(long long)(L1 + l1) * p.N2 + L2 + l2];
      v[3] += nj;
      v[4] += (double)Bp[t] * nj;
      v[5] += ng > 0.0 ? nj * log2(nj / ng) : (double)INFINITY;   // pi not << mu (x) nu
      v[6] += (double)(l1 - o1) * nj;
      v[7] += (double)(l2 - o2) * nj;
    }
  }
  block_xsum<double, 8>(v, red, red + 64);
  if (tid == 0) {
    const double* S = red + 64;
    const double D1 = (double)(cc.r0 - G1), D2 = (double)(cc.c0 - G2);
    p.ecell[J] = (D1 * D1 + D2 * D2) * S[3] + 2.0 * (D1 * (S[1] - S[6]) + D2 * (S[2] - S[7])) +
                 p.eps_p * (0.69314718055994531 * (S[0] + S[4] + S[5]) - S[3]);
  }
}

// ===========================================================================
// solve_kernel: a1 (log2 nu_J) + a2 (Sinkhorn), one CTA per composite cell.
// GS: the cell's work arrays live in global scratch (huge size class); a
// separate instantiation so that the shared-memory classes see a pointer
// derived from the __shared__ array and compile to LDS/STS with 32-bit
// addresses instead of generic 64-bit loads.
template <int NX, bool PR, bool GS>
__device__ void solve_cell(const SweepParams& p, const int J, unsigned char* smem) {
  const int tid = threadIdx.x, T = blockDim.x;
  const SolveLayout Ls = solve_layout(p.ccap, p.s);
  float* P0 = (float*)(smem + Ls.B);       // B (Y potential)
  float* P1 = (float*)(smem + Ls.LN);      // log2 nu_J
  float* P2 = (float*)(smem + Ls.BK);      // BK
  double* nuJ = (double*)(smem + Ls.BK);   // assembly scratch (before the loop)
  float* Ub = (float*)(smem + Ls.U);
  float* Rb = Ub + NX * p.ccap;            // UK
  float* Vb = (float*)(smem + Ls.V);
  float* X = (float*)(smem + Ls.X);
  float* A2 = X;
  float* A2n = X + NX * NX;
  float* LM = X + 2 * NX * NX;
  float* MU = X + 3 * NX * NX;
  float* AL = X + 4 * NX * NX;
  float* fred = (float*)(smem + Ls.fred);
  int* ints = (int*)(smem + Ls.ints);

  const CompCell cc = p.cells[J];
  const int nmem = cc.nmem, n1 = cc.n1, n2 = cc.n2;
  const float w = p.w;
  const int4 hull = cell_hull(p, cc, ints);
  const int L1 = hull.x, L2 = hull.y, b1 = hull.z, b2 = hull.w, BB = b1 * b2;
  // gauge origin G = L + o, o = floor((b - n)/2)
  const int o1 = (b1 - n1) >> 1, o2 = (b2 - n2) >> 1;
  const int G1 = L1 + o1, G2 = L2 + o2;
  if (b1 > p.ccap || b2 > p.ccap) {
    if (tid == 0) {
      if (p.mode == 0) p.ovf_list[atomicAdd(p.ovf_count, 1)] = J;        // large class
      else if (p.mode == 1) p.ovf2_list[atomicAdd(p.ovf2_count, 1)] = J;  // huge class
      else p.stats[J].overflow = 1;   // cannot happen: the huge class covers the grid
    }
    return;
  }
  assemble(p, cc, ints, L1, L2, b2, BB, nuJ);
  double nsum = 0.0;
  for (int t = tid; t < BB; t += T) {
    const double v = nuJ[t];
    nsum += v;
    P1[t] = v > 0.0 ? lg2f((float)v) : kNeg;   // log2 nu_J (zeros -> kNeg, R19)
  }
  {
    // mass defect of the cell problem (truncation ledger, reading R9): after
    // a Y-update the plan has mass ||nu_J||, so its X-marginal is compared
    // with mu ||nu_J|| / mu(X_J) (reading R6')
    const double nuMass = block_sum1_d(nsum, (double*)(smem + Ls.dred));
    double mX = 0.0;
    for (int q = 0; q < nmem; ++q) mX += p.m[cc.mem[q]];
    if (tid == 0) X[5 * NX * NX] = (float)((nuMass - mX) / mX);
  }
  // ---- X-block data, warm start (R7) and re-gauge ------------------------
  // The X-block is padded to NX x NX (ragged B cells have n = s on an axis);
  // padded pixels carry log2 mu = kNeg, so their terms vanish.
  const int NN = n1 * n2;
  constexpr int NXX = NX * NX;
  float amax = kNeg;
  for (int t = tid; t < NXX; t += T) {
    const int k1 = t / NX, k2 = t % NX;
    float a = 0.f, lm = kNeg, mu = 0.f;
    if (k1 < n1 && k2 < n2) {
      const long long pix = (long long)(cc.r0 + k1) * p.N2 + cc.c0 + k2;
      if (p.alpha_valid) {
        const int g1 = p.gauge[2 * J], g2 = p.gauge[2 * J + 1];
        a = p.alpha[pix] + 2.f * w * ((float)(G1 - g1) * k1 + (float)(G2 - g2) * k2);
      } else {
        // first sweep: a = 0 in the global gauge (R7), i.e. A = -2 w D.kappa, D = K - G
        a = -2.f * w * ((float)(cc.r0 - G1) * k1 + (float)(cc.c0 - G2) * k2);
      }
      lm = p.log2mu[pix];
      mu = p.mu[pix];
      amax = fmaxf(amax, a);
    }
    A2[t] = a;
    LM[t] = lm;
    MU[t] = mu;
  }
  amax = block_max_f(amax, fred);
  for (int t = tid; t < NXX; t += T) {
    A2[t] -= amax;
    AL[t] = A2[t] + LM[t] - w * (float)((t % NX) * (t % NX));   // AK of the first pass
  }
  double muXJ = 0.0;
  for (int q = 0; q < nmem; ++q) muXJ += p.m[cc.mem[q]];
  const float tolJ = (float)(p.tol * muXJ);
  __syncthreads();

  // ---- a2: separable log-domain Sinkhorn ---------------------------------
  // Every term of every 1-D LSE stage is evaluated as
  //     z = fma(g, x, a) - c,   sum += ex2(z)
  // by expanding -w (k - l)^2 = -w k^2 + 2 w k l - w l^2, folding the
  // input-only part into a precomputed array (AK = AL, UK, BK, VK) and the
  // output-only part into the shift c.  After the first pass the shift is the
  // previous iterate of the same output.  Threads
  // own outputs; the long-axis stages (X1, X2) give each thread two outputs
  // that share every loaded input (two ex2 per shared-memory load), X2 also
  // splits its terms over SX lanes.  ~5 instructions per ex2.
  int it = 0;
  float e0 = 0.f, e = 0.f;
  bool first = true;
  float* UK = Rb;                     // [NX][b2]  U - w k1^2   (Rb is free during the loop)
  float* VK = Vb + NX * p.ccap;       // [b1][NX]  V - w l1^2
  float* BK = P2;                     // [b1][b2]  B + log2 nu_J - w l2^2
  const float w2 = 2.f * w;
  const float fo1 = (float)o1, fo2 = (float)o2;
  constexpr int HX = NX / 2;
  // Y2 mapping: thread -> (column l2, row group rg of RG)
  // (a hull wider than the CTA, huge class only: columns in chunks of T)
  const int RG = max(1, T / b2);
  const int y2_col = tid % b2, y2_rg = tid / b2;
  // X2 mapping: thread -> (pair qa in [0, HX), column k2, split h of SX)
  constexpr int SX = (kSweepThreads / (HX * NX)) > 8 ? 8 : (kSweepThreads / (HX * NX));
  const int x2_h = tid % SX, x2_pair = tid / SX;
  const int x2_k2 = x2_pair % NX, x2_qa = x2_pair / NX;
  const bool x2_valid = x2_pair < HX * NX;
  for (;;) {
    ++it;
    // Y-half stage 1: U(k1, l2) = LSE_k2 [A + log2 mu - w (k2 - l2~)^2]
    for (int o = tid, k1 = tid / b2, l2 = tid % b2; o < NX * b2;
         o += T, k1 += T / b2, l2 += T % b2, (l2 >= b2 ? (l2 -= b2, ++k1) : 0)) {
      const float x = (float)l2 - fo2;
      const float wx = w2 * x;   // term q: fma(q, w2 x, a_q) (immediate q, no per-q constants live)
      const float* ar = AL + k1 * NX;
      float a[NX];
#pragma unroll
      for (int q = 0; q < NX; ++q) a[q] = ar[q];
      float c;
      if (first) {
        c = kNeg;
#pragma unroll
        for (int q = 0; q < NX; ++q) c = fmaxf(c, fmaf((float)q, wx, a[q]));
      } else {
        c = Ub[o] + w * x * x;
      }
      float sum = 0.f;
#pragma unroll
      for (int q = 0; q < NX; ++q) sum += ex2f(fmaf((float)q, wx, a[q]) - c);
      if (!(sum > 0x1p-60f && sum < 0x1p60f)) {
        c = kNeg;
        for (int q = 0; q < NX; ++q) c = fmaxf(c, fmaf((float)q, wx, a[q]));
        sum = 0.f;
        for (int q = 0; q < NX; ++q) sum += ex2f(fmaf((float)q, wx, a[q]) - c);
      }
      const float U = c + lg2f(sum) - w * x * x;
      Ub[o] = U;
      UK[o] = U - w * (float)(k1 * k1);
    }
    __syncthreads();
    // Y-half stage 2: B(l1, l2) = -LSE_k1 [U(k1, l2) - w (k1 - l1~)^2]
    auto y2_column = [&](const int l2, const int l1_0, const int l1_step) {
      float u[NX];
#pragma unroll
      for (int q = 0; q < NX; ++q) u[q] = UK[q * b2 + l2];
      const float wl2 = w * (float)(l2 * l2);
      for (int l1 = l1_0; l1 < b1; l1 += l1_step) {
        const int o = l1 * b2 + l2;
        const float x = (float)l1 - fo1;
        const float wx = w2 * x;
        float c;
        if (first) {
          c = kNeg;
#pragma unroll
          for (int q = 0; q < NX; ++q) c = fmaxf(c, fmaf((float)q, wx, u[q]));
        } else {
          c = -P0[o] + w * x * x;
        }
        float sum = 0.f;
#pragma unroll
        for (int q = 0; q < NX; ++q) sum += ex2f(fmaf((float)q, wx, u[q]) - c);
        if (!(sum > 0x1p-60f && sum < 0x1p60f)) {
          c = kNeg;
          for (int q = 0; q < NX; ++q) c = fmaxf(c, fmaf((float)q, wx, u[q]));
          sum = 0.f;
          for (int q = 0; q < NX; ++q) sum += ex2f(fmaf((float)q, wx, u[q]) - c);
        }
        const float Bv = -(c + lg2f(sum) - w * x * x);
        P0[o] = Bv;
        BK[o] = Bv + P1[o] - wl2;
      }
    };
    if (b2 <= T) {
      if (y2_rg < RG) y2_column(y2_col, y2_rg, RG);
    } else {   // hull wider than the CTA (huge class only)
      for (int l2 = tid; l2 < b2; l2 += T) y2_column(l2, 0, 1);
    }
    __syncthreads();
    // X-half stage 1: V(l1, k2) = LSE_l2 [B + log2 nu_J - w (k2 - l2~)^2],
    // two outputs (k2 = qa, qa + HX) per thread sharing the loaded BK
    for (int t = tid; t < b1 * HX; t += T) {
      const int l1 = t / HX, qa = t % HX, qb = qa + HX;
      const float kta = (float)qa + fo2, ktb = (float)qb + fo2;   // k2 - l2~ = kt - l2
      const float ga = w2 * kta, gb = w2 * ktb;
      const float* br = BK + l1 * b2;
      float ca, cb;
      if (first) {
        ca = kNeg;
        cb = kNeg;
        float lf = 0.f;
        for (int l2 = 0; l2 < b2; ++l2, lf += 1.f) {
          const float bk = br[l2];
          ca = fmaxf(ca, fmaf(ga, lf, bk));
          cb = fmaxf(cb, fmaf(gb, lf, bk));
        }
      } else {
        ca = Vb[l1 * NX + qa] + w * kta * kta;
        cb = Vb[l1 * NX + qb] + w * ktb * ktb;
      }
      float sa = 0.f, sb = 0.f, sa1 = 0.f, sb1 = 0.f;
      float lf = 0.f;
      int l2 = 0;
      for (; l2 + 1 < b2; l2 += 2, lf += 2.f) {
        const float bk0 = br[l2], bk1 = br[l2 + 1];
        sa += ex2f(fmaf(ga, lf, bk0) - ca);
        sb += ex2f(fmaf(gb, lf, bk0) - cb);
        sa1 += ex2f(fmaf(ga, lf + 1.f, bk1) - ca);
        sb1 += ex2f(fmaf(gb, lf + 1.f, bk1) - cb);
      }
      if (l2 < b2) {
        const float bk0 = br[l2];
        sa += ex2f(fmaf(ga, lf, bk0) - ca);
        sb += ex2f(fmaf(gb, lf, bk0) - cb);
      }
      sa += sa1;
      sb += sb1;
      if (!(sa > 0x1p-60f && sa < 0x1p60f) || !(sb > 0x1p-60f && sb < 0x1p60f)) {
        ca = kNeg;
        cb = kNeg;
        float lg = 0.f;
        for (int q = 0; q < b2; ++q, lg += 1.f) {
          ca = fmaxf(ca, fmaf(ga, lg, br[q]));
          cb = fmaxf(cb, fmaf(gb, lg, br[q]));
        }
        sa = 0.f;
        sb = 0.f;
        lg = 0.f;
        for (int q = 0; q < b2; ++q, lg += 1.f) {
          sa += ex2f(fmaf(ga, lg, br[q]) - ca);
          sb += ex2f(fmaf(gb, lg, br[q]) - cb);
        }
      }
      const float Va = ca + lg2f(sa) - w * kta * kta;
      const float Vbv = cb + lg2f(sb) - w * ktb * ktb;
      const float wl1 = w * (float)(l1 * l1);
      Vb[l1 * NX + qa] = Va;
      Vb[l1 * NX + qb] = Vbv;
      VK[l1 * NX + qa] = Va - wl1;
      VK[l1 * NX + qb] = Vbv - wl1;
    }
    __syncthreads();
    // X-half stage 2: A'(k1, k2) = -LSE_l1 [V(l1, k2) - w (k1 - l1~)^2],
    // two outputs (k1 = qa, qa + HX) per thread, terms split over SX lanes
    float epart = 0.f;
    {
      const int qa = x2_qa, qb = qa + HX, k2 = x2_k2;
      const float kta = (float)qa + fo1, ktb = (float)qb + fo1;
      const float ga = w2 * kta, gb = w2 * ktb;
      float ca = 0.f, cb = 0.f;
      if (first) {
        ca = kNeg;
        cb = kNeg;
        if (x2_valid) {
          float lf = (float)x2_h;
          for (int l1 = x2_h; l1 < b1; l1 += SX, lf += (float)SX) {
            const float vk = VK[l1 * NX + k2];
            ca = fmaxf(ca, fmaf(ga, lf, vk));
            cb = fmaxf(cb, fmaf(gb, lf, vk));
          }
        }
#pragma unroll
        for (int off = SX >> 1; off > 0; off >>= 1) {
          ca = fmaxf(ca, __shfl_xor_sync(0xffffffffu, ca, off));
          cb = fmaxf(cb, __shfl_xor_sync(0xffffffffu, cb, off));
        }
      } else if (x2_valid) {
        ca = -A2[qa * NX + k2] + w * kta * kta;
        cb = -A2[qb * NX + k2] + w * ktb * ktb;
      }
      float sa = 0.f, sb = 0.f;
      if (x2_valid) {
        float lf = (float)x2_h;
        for (int l1 = x2_h; l1 < b1; l1 += SX, lf += (float)SX) {
          const float vk = VK[l1 * NX + k2];
          sa += ex2f(fmaf(ga, lf, vk) - ca);
          sb += ex2f(fmaf(gb, lf, vk) - cb);
        }
      }
#pragma unroll
      for (int off = SX >> 1; off > 0; off >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, off);
        sb += __shfl_xor_sync(0xffffffffu, sb, off);
      }
      const bool bad = x2_valid && (!(sa > 0x1p-60f && sa < 0x1p60f) || !(sb > 0x1p-60f && sb < 0x1p60f));
      if (__any_sync(0xffffffffu, bad)) {
        float ma = kNeg, mb = kNeg;
        if (x2_valid) {
          float lf = (float)x2_h;
          for (int l1 = x2_h; l1 < b1; l1 += SX, lf += (float)SX) {
            const float vk = VK[l1 * NX + k2];
            ma = fmaxf(ma, fmaf(ga, lf, vk));
            mb = fmaxf(mb, fmaf(gb, lf, vk));
          }
        }
#pragma unroll
        for (int off = SX >> 1; off > 0; off >>= 1) {
          ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, off));
          mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, off));
        }
        float ta = 0.f, tb = 0.f;
        if (x2_valid) {
          float lf = (float)x2_h;
          for (int l1 = x2_h; l1 < b1; l1 += SX, lf += (float)SX) {
            const float vk = VK[l1 * NX + k2];
            ta += ex2f(fmaf(ga, lf, vk) - ma);
            tb += ex2f(fmaf(gb, lf, vk) - mb);
          }
        }
#pragma unroll
        for (int off = SX >> 1; off > 0; off >>= 1) {
          ta += __shfl_xor_sync(0xffffffffu, ta, off);
          tb += __shfl_xor_sync(0xffffffffu, tb, off);
        }
        if (bad) { ca = ma; cb = mb; sa = ta; sb = tb; }
      }
      if (x2_valid && x2_h == 0) {
        const float wk2 = w * (float)(k2 * k2);
        const int oa = qa * NX + k2, ob = qb * NX + k2;
        const float ana = -(ca + lg2f(sa) - w * kta * kta);
        const float anb = -(cb + lg2f(sb) - w * ktb * ktb);
        A2n[oa] = ana;
        A2n[ob] = anb;
        // L1 X-marginal error of the plan (A, B): sum mu |1 - 2^(A - A')|
        const float rm1 = X[5 * NXX];   // (A2/A2n swap; X itself is fixed)
        epart += MU[oa] * fabsf(exp2m1f(A2[oa] - ana) - rm1) + MU[ob] * fabsf(exp2m1f(A2[ob] - anb) - rm1);
        AL[oa] = ana + LM[oa] - wk2;   // AK of the next pass
        AL[ob] = anb + LM[ob] - wk2;
      }
    }
    const float etot = block_sum_f(epart, fred, it);
    if (it == 1) e0 = etot;
    e = etot;
    const bool stop = p.fixed_iter > 0 ? (it >= p.fixed_iter) : (etot <= tolJ || it >= p.max_iter);
    if (stop) break;
    float* tmp = A2; A2 = A2n; A2n = tmp;   // A <- A'
    first = false;
  }
  if (PR)
    primal_terms<NX>(p, cc, J, ints, L1, L2, b1, b2, o1, o2, G1, G2, A2, A2n, MU, P0, nuJ,
                     (double*)(smem + Ls.dred));
  // ---- outputs: the plan's potential (next warm start, R7) and stats -----
  for (int t = tid; t < NN; t += T) {
    const int k1 = t / n2, k2 = t - k1 * n2;
    p.alpha[(long long)(cc.r0 + k1) * p.N2 + cc.c0 + k2] = A2[k1 * NX + k2];
  }
  if (tid == 0) {
    p.gauge[2 * J] = G1;
    p.gauge[2 * J + 1] = G2;
    CellStats st;
    st.iters = it;
    st.overflow = 0;
    st.e0 = e0;
    st.e = e;
    st.dropped = 0.0;
    p.stats[J] = st;
    // algorithmic MUFU count of the Sinkhorn passes: E_it + L_it
    // per pass plus NN for the X-error
    const unsigned long long E_it = (unsigned long long)n1 * n2 * b2 + (unsigned long long)b1 * b2 * n1 +
                                    (unsigned long long)b1 * n2 * b2 + (unsigned long long)n1 * n2 * b1;
    const unsigned long long L_it = (unsigned long long)n1 * b2 + BB + (unsigned long long)b1 * n2 + NN;
    const unsigned long long mufu = (unsigned long long)it * (E_it + L_it + NN) + BB;
    atomicAdd(&p.totals->mufu, mufu);
    atomicAdd(&p.cum->mufu, mufu);
    atomicAdd(&p.cum->iters, (unsigned long long)it);
    atomicAdd(&p.totals->iters, (unsigned long long)it);
    if (p.fixed_iter <= 0 && it >= p.max_iter && e > tolJ) atomicAdd(&p.totals->nonconv, 1ull);
    atomicMax(&p.totals->iters_max, it);
    atomicAdd(&p.totals->e0, (double)e0);
    atomicAdd(&p.totals->e, (double)e);
  }
}

template <int NX, bool PR>
__global__ void __launch_bounds__(kSweepThreads, DD_SOLVE_MINB) solve_kernel(SweepParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  // one call site, so the cell routine is inlined (two call sites made the
  // compiler emit it as a real call: ABI stack frame and spills, 3% slower)
  // (each instantiation has one call site, so it is inlined)
  const int n = p.mode == 0 ? p.ncells : (p.mode == 1 ? *p.ovf_count : *p.ovf2_count);
  const int* list = p.mode == 1 ? p.ovf_list : p.ovf2_list;
  if (p.mode == 2) {
    unsigned char* base = p.scratch + (size_t)blockIdx.x * p.scratch_stride;
    for (int k = blockIdx.x; k < n; k += gridDim.x) {
      solve_cell<NX, PR, true>(p, list[k], base);
      __syncthreads();
    }
  } else {
    for (int k = blockIdx.x; k < n; k += gridDim.x) {
      solve_cell<NX, PR, false>(p, p.mode == 0 ? k : list[k], smem);
      __syncthreads();
    }
  }
}

// ===========================================================================
// split_kernel: a1 (fp64) + a3 + a4 + a5 + a6, one CTA per composite cell.
// Final (balanced) value of every member at one box entry.  Explicit _rn
// intrinsics: bitwise identical in the truncation and the write pass.
// Balance (reading R8): blended overlap / own-shape transfer
//   v_k = parts_k + parts_k * (sum_j O_kj parts_j) / nu_J + sum_j P_kj parts_j
// (O: overlap-transfer coefficients f theta / T, P: own-shape coefficients
// f (1 - theta) / M_d; see oracle/domdec.py:balance for the definition).
// Balance coefficients live in shared memory: bc[0] = active flag,
// bc[1 + 4k + j] = O_kj, bc[17 + 4k + j] = P_kj.
__device__ __forceinline__ void member_values(double nuj, const float (&p)[4], int nmem, const double* bc,
                                              double (&out)[4]) {
  int am = 0;
  float pbest = p[0];   // running maximum: no dynamic index (keeps p in registers)
#pragma unroll
  for (int k = 1; k < 4; ++k)
    if (k < nmem && p[k] > pbest) { am = k; pbest = p[k]; }
  double parts[4];
  double rest = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    parts[k] = 0.0;
    if (k < nmem && k != am) {
      parts[k] = __dmul_rn(nuj, (double)p[k]);
      rest = __dadd_rn(rest, parts[k]);
    }
  }
  const double pa = __dsub_rn(nuj, rest);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k == am) parts[k] = pa > 0.0 ? pa : 0.0;
  if (bc[0] != 0.0 && nuj > 0.0) {
    const double inv = __drcp_rn(nuj);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double t = 0.0, u = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        t = __dadd_rn(t, __dmul_rn(bc[1 + 4 * k + j], parts[j]));
        u = __dadd_rn(u, __dmul_rn(bc[17 + 4 * k + j], parts[j]));
      }
      out[k] = __dadd_rn(__dadd_rn(parts[k], __dmul_rn(parts[k], __dmul_rn(t, inv))), u);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = parts[k];
  }
}

__device__ __forceinline__ int pair_id(int a, int b) {   // a < b, 4 members -> 6 pairs
  return a == 0 ? b - 1 : (a == 1 ? b + 1 : 5);
}

template <int NX, bool GS>
__device__ void split_cell(const SweepParams& p, const int J, unsigned char* smem) {
  const int tid = threadIdx.x, T = blockDim.x;
  const SplitLayout Ls = split_layout(p.ccap, p.s);
  double* nuJ = (double*)(smem + Ls.nuJ);
  double* red = (double*)(smem + Ls.red);
  float* P0 = (float*)(smem + Ls.P0);
  float* P1 = (float*)(smem + Ls.P1);
  float* P2 = (float*)(smem + Ls.P2);
  float* P3 = (float*)(smem + Ls.P3);
  float* Ub = (float*)(smem + Ls.U);
  float* Rb = (float*)(smem + Ls.R);
  float* AL = (float*)(smem + Ls.AL);
  int* ints = (int*)(smem + Ls.ints);

  const CompCell cc = p.cells[J];
  const int nmem = cc.nmem, n1 = cc.n1, n2 = cc.n2, s = p.s;
  const float w = p.w;
  const int4 hull = cell_hull(p, cc, ints);
  const int L1 = hull.x, L2 = hull.y, b1 = hull.z, b2 = hull.w, BB = b1 * b2;
  const int o1 = (b1 - n1) >> 1, o2 = (b2 - n2) >> 1;
  const float fo1 = (float)o1, fo2 = (float)o2;

  auto copy_unchanged = [&](int reason) {
    long long* base = (long long*)(ints + 48);
    if (tid == 0) {
      long long tot = 0;
      for (int k = 0; k < nmem; ++k) tot += (long long)ints[8 + k] * ints[12 + k];
      base[0] = (long long)atomicAdd(p.pool_ctr, (unsigned long long)tot);
      if (base[0] + tot > p.pool_cap) { base[0] = -1; atomicAdd(&p.totals->overflow, 1ull); }
    }
    __syncthreads();
    long long at = base[0];
    if (at < 0) return;
    for (int k = 0; k < nmem; ++k) {
      const int i = cc.mem[k];
      const long long len = (long long)ints[8 + k] * ints[12 + k];
      const double* src = p.pool_in + p.pos_in[i];
      double* dst = p.pool_out + at;
      for (long long t = tid; t < len; t += T) dst[t] = src[t];
      if (tid == 0) {
        p.pos_out[i] = at;
        p.off_out[2 * i] = ints[k];
        p.off_out[2 * i + 1] = ints[4 + k];
        p.ext_out[2 * i] = ints[8 + k];
        p.ext_out[2 * i + 1] = ints[12 + k];
      }
      at += len;
    }
    if (tid == 0) {
      p.stats[J].overflow = reason;
      atomicAdd(&p.totals->overflow, 1ull);
      atomicAdd(&p.totals->cells, 1ull);
    }
  };

  if (b1 > p.ccap || b2 > p.ccap) {
    if (p.mode == 2) copy_unchanged(1);
    return;   // handled by the next size class
  }
  if (p.stats[J].overflow) {
    copy_unchanged(1);
    return;
  }
  assemble(p, cc, ints, L1, L2, b2, BB, nuJ);
  // plan potential of this sweep (written by solve_kernel in the same gauge)
  constexpr int NXX = NX * NX;
  for (int t = tid; t < NXX; t += T) {
    const int k1 = t / NX, k2 = t % NX;
    float al = kNeg;
    if (k1 < n1 && k2 < n2) {
      const long long pix = (long long)(cc.r0 + k1) * p.N2 + cc.c0 + k2;
      al = p.alpha[pix] + p.log2mu[pix];
    }
    AL[t] = al;
  }
  double muXJ = 0.0;
  for (int q = 0; q < nmem; ++q) muXJ += p.m[cc.mem[q]];
  __syncthreads();

  // ---- a3: CompositeToBasic (share form) + plan moments (R13) --------------
  // Stage 1 split by column half h2: U_h2(k1, l2) = LSE over k2 in half h2,
  // plus the conditional moments of x2' = x2 - (centre column of the member).
  const int c2 = n2 / s;
  const float cen = 0.5f * (float)(s - 1);
  for (int o = tid; o < c2 * n1 * b2; o += T) {
    const int h2 = o / (n1 * b2);
    const int rem = o - h2 * n1 * b2;
    const int k1 = rem / b2, l2 = rem - k1 * b2;
    const float lt = (float)l2 - fo2;
    const float* ar = AL + k1 * NX;
    float sh = kNeg;
    for (int k2 = h2 * s; k2 < h2 * s + s; ++k2) { const float d = (float)k2 - lt; sh = fmaxf(sh, ar[k2] - w * d * d); }
    float sum = 0.f, m1 = 0.f, m2 = 0.f;
    for (int k2 = h2 * s; k2 < h2 * s + s; ++k2) {
      const float d = (float)k2 - lt;
      const float tt = ex2f(ar[k2] - w * d * d - sh);
      const float xq = (float)(k2 - h2 * s) - cen;
      sum += tt;
      m1 += tt * xq;
      m2 += tt * xq * xq;
    }
    const float inv = 1.0f / sum;
    Ub[o] = sh + lg2f(sum);
    Rb[o] = m1 * inv;
    Rb[c2 * n1 * b2 + o] = m2 * inv;
  }
  __syncthreads();
  int mq[4];
  for (int k = 0; k < 4; ++k) mq[k] = cc.quad[k];
  // acc[0..3]: split masses (= moment M0); acc[4 + 5k + .]: M1a, M1b, G0, G1,
  // M2 of member k; acc[24 + pair]: overlaps sum parts_a parts_b / nu_J (R8)
  // masses and overlaps need fp64 per thread (balance); the plan moments are
  // summed over only ~BB/128 entries per thread and are kept in fp32 until the
  // (fp64) cross-thread reduction.
  double da[16];    // per thread: masses [0..3], overlaps [4 + pair], fp64
  float mf[32];     // per thread: plan moments [5 q + c], fp32
#pragma unroll
  for (int q = 0; q < 16; ++q) da[q] = 0.0;
#pragma unroll
  for (int q = 0; q < 32; ++q) mf[q] = 0.f;
  for (int o = tid; o < BB; o += T) {
    const int l1 = o / b2, l2 = o - l1 * b2;
    const float lt = (float)l1 - fo1;
    float S[4], Ex1[4], Ex2[4], Exx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      S[k] = kNeg; Ex1[k] = 0.f; Ex2[k] = 0.f; Exx[k] = 0.f;
      if (k < nmem) {
        const int h1 = mq[k] >> 1, h2 = mq[k] & 1;
        const float* ur = Ub + (h2 * n1) * b2 + l2;
        const float* r1 = Rb + (h2 * n1) * b2 + l2;
        const float* r2 = Rb + c2 * n1 * b2 + (h2 * n1) * b2 + l2;
        float sh = kNeg;
        for (int k1 = h1 * s; k1 < h1 * s + s; ++k1) { const float d = (float)k1 - lt; sh = fmaxf(sh, ur[k1 * b2] - w * d * d); }
        float sum = 0.f, a1 = 0.f, a2 = 0.f, aq = 0.f;
        for (int k1 = h1 * s; k1 < h1 * s + s; ++k1) {
          const float d = (float)k1 - lt;
          const float tt = ex2f(ur[k1 * b2] - w * d * d - sh);
          const float xq = (float)(k1 - h1 * s) - cen;
          sum += tt;
          a1 += tt * xq;
          a2 += tt * r1[k1 * b2];
          aq += tt * (xq * xq + r2[k1 * b2]);
        }
        const float inv = 1.0f / sum;
        S[k] = sh + lg2f(sum);
        Ex1[k] = a1 * inv;
        Ex2[k] = a2 * inv;
        Exx[k] = aq * inv;
      }
    }
    float mx = S[0];
#pragma unroll
    for (int k = 1; k < 4; ++k) mx = fmaxf(mx, S[k]);
    float es[4], tot = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) { es[k] = k < nmem ? ex2f(S[k] - mx) : 0.f; tot += es[k]; }
    const float inv = 1.0f / tot;
    float pk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) pk[k] = es[k] * inv;
    P0[o] = pk[0];
    P1[o] = pk[1];
    P2[o] = pk[2];
    P3[o] = pk[3];
    const double nj = nuJ[o];
    if (nj > 0.0) {
      // identity split (the largest share takes the remainder: exact sum)
      double v[4];
      int am = 0;
      float pbest = pk[0];
#pragma unroll
      for (int q = 1; q < 4; ++q)
        if (q < nmem && pk[q] > pbest) { am = q; pbest = pk[q]; }
      double rest = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[q] = 0.0;
        if (q < nmem && q != am) { v[q] = __dmul_rn(nj, (double)pk[q]); rest = __dadd_rn(rest, v[q]); }
      }
      const double pa = __dsub_rn(nj, rest);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q == am) v[q] = pa > 0.0 ? pa : 0.0;
      // split masses and pairwise overlaps (balance, R8)
      const double invj = 1.0 / nj;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        da[a] += v[a];
#pragma unroll
        for (int b = a + 1; b < 4; ++b) da[4 + pair_id(a, b)] += v[a] * v[b] * invj;
      }
      // plan moments of the pre-balance marginals nu_k^pre = nu_J p_k (R13)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < nmem) {
          const int h1 = mq[q] >> 1, h2 = mq[q] & 1;
          const float vv = (float)nj * pk[q];
          const float y1 = (float)(L1 + l1 - cc.r0 - h1 * s) - cen;
          const float y2 = (float)(L2 + l2 - cc.c0 - h2 * s) - cen;
          mf[5 * q + 0] += vv * y1;
          mf[5 * q + 1] += vv * y2;
          mf[5 * q + 2] += vv * Exx[q];
          mf[5 * q + 3] += vv * (y1 * Ex1[q] + y2 * Ex2[q]);
          mf[5 * q + 4] += vv * (y1 * y1 + y2 * y2);
        }
      }
    }
  }
  __syncthreads();
  block_xsum<double, 16>(da, red, red + 160);
  block_xsum<float, 32>(mf, (float*)(red + 64), (float*)(red + 200));
  // reduced values live in shared memory: masses red[160..163], overlaps
  // red[164 + pair], plan moments (float) at red + 200
  const double* Rm = red + 160;
  const double* Rov = red + 164;
  const float* Rmom = (const float*)(red + 200);
  const double massJ = Rm[0] + Rm[1] + Rm[2] + Rm[3];
  // ---- a4: balance coefficients (reading R8), in shared memory -----------
  // Warp 0 computes them lane-parallel: lane 4 d + r -> O_dr, lane 16 + 4 k +
  // j -> P_kj (see oracle/domdec.py:balance for the definition).
  double* bc = red + 240;
  if (tid < 32) {
    double delta[4], Dsum = 0.0;
    bool any_d = false, any_r = false;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      delta[q] = 0.0;
      if (q < nmem) {
        delta[q] = Rm[q] - p.m[cc.mem[q]] * massJ / muXJ;
        if (delta[q] > 0) { any_d = true; Dsum += delta[q]; }
        if (delta[q] < 0) any_r = true;
      }
    }
    const bool active = any_d && any_r;
    // theta of every donor (redundant per lane, compile-time indices)
    double theta[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      theta[d] = 0.0;
      if (active && d < nmem && delta[d] > 0) {
        bool zeroT = false;
        double L = 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r < nmem && r != d && delta[r] < 0) {
            const double T = Rov[d < r ? pair_id(d, r) : pair_id(r, d)];
            if (!(T > 0.0)) zeroT = true;
            else L += delta[d] * (-delta[r]) / Dsum / T;
          }
        }
        const double l = delta[d] / Rm[d];
        theta[d] = zeroT ? 0.0 : (L <= 1.0 ? 1.0 : (1.0 - l) / (L - l));
      }
    }
    const int a = (tid & 15) >> 2, b = tid & 3;   // entry (a, b)
    double val = 0.0;
    if (active) {
#pragma unroll
      for (int d = 0; d < 4; ++d) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (d < nmem && r < nmem && delta[d] > 0 && delta[r] < 0) {
            const double f = delta[d] * (-delta[r]) / Dsum;
            if (tid < 16) {            // O: O_dr -= f theta / T, O_rd += f theta / T
              const double T = Rov[d < r ? pair_id(d, r) : pair_id(r, d)];
              if (theta[d] > 0.0) {
                const double x = f * theta[d] / T;
                if (a == d && b == r) val -= x;
                if (a == r && b == d) val += x;
              }
            } else {                   // P: P_dd -= f (1 - theta) / M_d, P_rd += same
              const double x = f * (1.0 - theta[d]) / Rm[d];
              if (a == d && b == d) val -= x;
              if (a == r && b == d) val += x;
            }
          }
        }
      }
    }
    bc[1 + tid] = val;   // tid < 16 -> O, tid >= 16 -> P (bc[17 + 4a + b])
    if (tid == 0) bc[0] = active ? 1.0 : 0.0;
  }
  __syncthreads();
  // ---- a5: truncate + minimal box -----------------------------------------
  // layout: ints[16 + 4k + 0] = min row, +1 = max row, +2 = min col, +3 = max col
  if (tid < 4) {
    ints[16 + 4 * tid + 0] = 1 << 30;
    ints[16 + 4 * tid + 1] = -1;
    ints[16 + 4 * tid + 2] = 1 << 30;
    ints[16 + 4 * tid + 3] = -1;
  }
  __syncthreads();
  double drop[1] = {0.0};
  double dloc = 0.0;
  // per-thread bounds in registers (static member indices), one warp
  // reduction and one shared atomic per warp and bound at the end
  int bmn1[4], bmx1[4], bmn2[4], bmx2[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { bmn1[k] = 1 << 30; bmx1[k] = -1; bmn2[k] = 1 << 30; bmx2[k] = -1; }
  for (int o = tid; o < BB; o += T) {
    const int l1 = o / b2, l2 = o - l1 * b2;
    const float pk[4] = {P0[o], P1[o], P2[o], P3[o]};
    double v[4];
    member_values(nuJ[o], pk, nmem, bc, v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k >= nmem) continue;
      if (v[k] >= p.tau) {
        bmn1[k] = min(bmn1[k], l1);
        bmx1[k] = max(bmx1[k], l1);
        bmn2[k] = min(bmn2[k], l2);
        bmx2[k] = max(bmx2[k], l2);
      } else if (v[k] > 0.0) {
        dloc += v[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int a = __reduce_min_sync(0xffffffffu, bmn1[k]);
    const int b = __reduce_max_sync(0xffffffffu, bmx1[k]);
    const int c = __reduce_min_sync(0xffffffffu, bmn2[k]);
    const int d = __reduce_max_sync(0xffffffffu, bmx2[k]);
    if ((tid & 31) == 0 && k < nmem && b >= 0) {
      atomicMin(&ints[16 + 4 * k + 0], a);
      atomicMax(&ints[16 + 4 * k + 1], b);
      atomicMin(&ints[16 + 4 * k + 2], c);
      atomicMax(&ints[16 + 4 * k + 3], d);
    }
  }
  drop[0] = block_sum1_d(dloc, red);
  // capacity check (uniform)
  bool ok = true;
  for (int k = 0; k < nmem; ++k) {
    const int mn1 = ints[16 + 4 * k], mx1 = ints[16 + 4 * k + 1];
    const int mn2 = ints[16 + 4 * k + 2], mx2 = ints[16 + 4 * k + 3];
    if (mx1 < mn1 || mx2 < mn2) { ok = false; break; }   // annihilated cell
  }
  if (!ok) {
    copy_unchanged(2);
    return;
  }
  // ---- write the new boxes: one pass over the union of the member boxes,
  // every entry evaluated once and scattered to the boxes containing it ----
  unsigned long long wbytes = 0;
  int bx[4][4];
  int umn1 = 1 << 30, umx1 = -1, umn2 = 1 << 30, umx2 = -1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    bx[q][0] = ints[16 + 4 * q]; bx[q][1] = ints[16 + 4 * q + 1];
    bx[q][2] = ints[16 + 4 * q + 2]; bx[q][3] = ints[16 + 4 * q + 3];
    if (q < nmem) {
      umn1 = min(umn1, bx[q][0]); umx1 = max(umx1, bx[q][1]);
      umn2 = min(umn2, bx[q][2]); umx2 = max(umx2, bx[q][3]);
      wbytes += (unsigned long long)(bx[q][1] - bx[q][0] + 1) * (bx[q][3] - bx[q][2] + 1) * 8ull;
    }
  }
  // allocate the member boxes consecutively in the output pool
  long long* pbase = (long long*)(ints + 48);
  if (tid == 0) {
    long long tot = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)   // static indices keep bx / mbase in registers
      if (q < nmem) tot += (long long)(bx[q][1] - bx[q][0] + 1) * (bx[q][3] - bx[q][2] + 1);
    long long b0 = (long long)atomicAdd(p.pool_ctr, (unsigned long long)tot);
    if (b0 + tot > p.pool_cap) { b0 = -1; atomicAdd(&p.totals->overflow, 1ull); }
    pbase[0] = b0;
  }
  __syncthreads();
  if (pbase[0] < 0) return;   // pool exhausted: reported as overflow (state invalid)
  long long mbase[4];
  {
    long long at = pbase[0];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      mbase[q] = at;
      if (q < nmem) at += (long long)(bx[q][1] - bx[q][0] + 1) * (bx[q][3] - bx[q][2] + 1);
    }
  }
  {
    const int ue2 = umx2 - umn2 + 1, un = (umx1 - umn1 + 1) * ue2;
    for (int t = tid; t < un; t += T) {
      const int l1 = umn1 + t / ue2, l2 = umn2 + t % ue2;
      const int o = l1 * b2 + l2;
      const float pk[4] = {P0[o], P1[o], P2[o], P3[o]};
      double v[4];
      member_values(nuJ[o], pk, nmem, bc, v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < nmem && l1 >= bx[q][0] && l1 <= bx[q][1] && l2 >= bx[q][2] && l2 <= bx[q][3]) {
          const int e2q = bx[q][3] - bx[q][2] + 1;
          p.pool_out[mbase[q] + (l1 - bx[q][0]) * e2q + (l2 - bx[q][2])] = v[q] >= p.tau ? v[q] : 0.0;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (tid == q && q < nmem) {
      const int i = cc.mem[q];
      p.pos_out[i] = mbase[q];
      p.off_out[2 * i] = L1 + bx[q][0];
      p.off_out[2 * i + 1] = L2 + bx[q][2];
      p.ext_out[2 * i] = bx[q][1] - bx[q][0] + 1;
      p.ext_out[2 * i + 1] = bx[q][3] - bx[q][2] + 1;
    }
  }
  if (tid == 0) {
    for (int q = 0; q < nmem; ++q)
    {
      p.mom[6 * cc.mem[q]] = Rm[q];
      for (int c = 0; c < 5; ++c) p.mom[6 * cc.mem[q] + 1 + c] = (double)Rmom[5 * q + c];
    }
  }
  if (tid == 0) {
    p.stats[J].dropped = drop[0];
    const int c2n = n2 / s;
    const unsigned long long E_c2b = (unsigned long long)n1 * n2 * b2 + (unsigned long long)nmem * s * BB +
                                     3ull * nmem * BB;
    const unsigned long long L_c2b = (unsigned long long)c2n * n1 * b2 + (unsigned long long)nmem * BB;
    atomicAdd(&p.totals->mufu, E_c2b + L_c2b);
    atomicAdd(&p.cum->mufu, E_c2b + L_c2b);
    atomicAdd(&p.cum->cells, 1ull);
    unsigned long long rbytes = 0;
    for (int k = 0; k < nmem; ++k) rbytes += (unsigned long long)ints[8 + k] * ints[12 + k] * 8ull;
    // pool read (twice: solve + split), pool write, metadata, mu/log2mu, alpha r/w, moments
    const unsigned long long byts = 2 * rbytes + wbytes + 16ull * nmem * 2 + (unsigned long long)n1 * n2 * 20ull + 48ull * nmem;
    atomicAdd(&p.totals->bytes, byts);
    atomicAdd(&p.cum->bytes, byts);
    atomicAdd(&p.totals->cells, 1ull);
    atomicAdd(&p.totals->dropped, drop[0]);
  }
}

template <int NX>
__global__ void __launch_bounds__(kSweepThreads, DD_SPLIT_MINB) split_kernel(SweepParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  // one call site, so the cell routine is inlined (two call sites made the
  // compiler emit it as a real call: ABI stack frame and spills, 3% slower)
  // (each instantiation has one call site, so it is inlined)
  const int n = p.mode == 0 ? p.ncells : (p.mode == 1 ? *p.ovf_count : *p.ovf2_count);
  const int* list = p.mode == 1 ? p.ovf_list : p.ovf2_list;
  if (p.mode == 2) {
    unsigned char* base = p.scratch + (size_t)blockIdx.x * p.scratch_stride;
    for (int k = blockIdx.x; k < n; k += gridDim.x) {
      split_cell<NX, true>(p, list[k], base);
      __syncthreads();
    }
  } else {
    for (int k = blockIdx.x; k < n; k += gridDim.x) {
      split_cell<NX, false>(p, p.mode == 0 ? k : list[k], smem);
      __syncthreads();
    }
  }
}

// Two size classes for each kernel (the device-side analogue of the paper's
// clustering by box size): pass 0 runs one CTA per
// composite cell with shared memory for hulls <= ccap_small and queues larger
// cells; pass 1 runs persistent CTAs with shared memory for hulls <= ccap_big
// over the queue.  No host synchronisation anywhere in the sweep.
template <int NX>
static cudaError_t launch_sweep_t(SweepParams p, int ccap_small, int ccap_big, int ccap_huge, cudaStream_t st) {
  static size_t conf_solve[2] = {0, 0}, conf_split = 0;
  // the primal-score epilogue is a separate instantiation so the timed
  // variant carries none of its code (options.track_primal)
  void (*solve)(SweepParams) = p.ecell ? solve_kernel<NX, true> : solve_kernel<NX, false>;
  const int pr = p.ecell ? 1 : 0;
  const size_t s0 = solve_layout(ccap_small, p.s).total, s1 = solve_layout(ccap_big, p.s).total;
  const size_t t0 = split_layout(ccap_small, p.s).total, t1 = split_layout(ccap_big, p.s).total;
  const size_t ns = s0 > s1 ? s0 : s1, nt = t0 > t1 ? t0 : t1;
  cudaError_t e;
  if (ns > 48 * 1024 && ns > conf_solve[pr]) {
    e = cudaFuncSetAttribute(solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ns);
    if (e != cudaSuccess) return e;
    conf_solve[pr] = ns;
  }
  if (nt > 48 * 1024 && nt > conf_split) {
    e = cudaFuncSetAttribute(split_kernel<NX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)nt);
    if (e != cudaSuccess) return e;
    conf_split = nt;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaMemsetAsync(p.ovf_count, 0, sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.ovf2_count, 0, sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.pool_ctr, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  const int nhuge = (int)(p.scratch_stride ? 16 : 0);
  // solve: small / large / huge
  p.mode = 0; p.ccap = ccap_small;
  solve<<<p.ncells, kSweepThreads, s0, st>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  p.mode = 1; p.ccap = ccap_big;
  solve<<<nsm, kSweepThreads, s1, st>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (nhuge) {
    p.mode = 2; p.ccap = ccap_huge;
    solve<<<nhuge, kSweepThreads, 0, st>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // split: small / large / huge
  p.mode = 0; p.ccap = ccap_small;
  split_kernel<NX><<<p.ncells, kSweepThreads, t0, st>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  p.mode = 1; p.ccap = ccap_big;
  split_kernel<NX><<<nsm, kSweepThreads, t1, st>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (nhuge) {
    p.mode = 2; p.ccap = ccap_huge;
    split_kernel<NX><<<nhuge, kSweepThreads, 0, st>>>(p);
    e = cudaGetLastError();
  }
  return e;
}

size_t sweep_scratch_bytes(int ccap, int s) {
  const size_t a = solve_layout(ccap, s).total, b = split_layout(ccap, s).total;
  return (a > b ? a : b) + 256;
}

cudaError_t launch_sweep(SweepParams p, int ccap_small, int ccap_big, int ccap_huge, cudaStream_t st) {
  switch (p.s) {
    case 1: return launch_sweep_t<2>(p, ccap_small, ccap_big, ccap_huge, st);
    case 2: return launch_sweep_t<4>(p, ccap_small, ccap_big, ccap_huge, st);
    case 4: return launch_sweep_t<8>(p, ccap_small, ccap_big, ccap_huge, st);
    case 8: return launch_sweep_t<16>(p, ccap_small, ccap_big, ccap_huge, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dd
