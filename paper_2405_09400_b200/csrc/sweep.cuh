// sweep.cuh — device code of the domain-decomposition sweep (sm_100a).
//
// One fused routine per composite cell J (one CTA per cell, as the batched
// SinkhornGPU of App. A.1), all steps of Alg. 4 l.3-7
// on the cell's shared-memory working set:
//   a1 BasicToComposite   nu_J = sum_{i in J} nu_i on the hull box, fp64
//                         (Eq. get-composite-cell-marginal PAPER.md:1128-1133)
//   a2 log-domain separable Sinkhorn on X_J x box(nu_J),
//      base-2, per-cell local gauge, stopping rule
//      L1 X-marginal error after the Y-update <= Err mu(X_J) (PAPER.md:1264,
//      readings R6/R6'), warm start from the previous sweep on the partition
//      (reading R7);
//   a3' plan moments for the flow update (reading R13) from one extra
//      moment-weighted X-half of the final plan: per pixel x the conditional
//      Y-moments E[y | x] and E[|y|^2 | x];
//   a3 CompositeToBasic   nu_i = nu_J exp(S_i - LSE_i' S_i') (share form of
//                         PAPER.md:1151-1193);
//   a4 Balance            (Alg. 4 l.6 PAPER.md:1231, reading R8);
//   a5 Truncate + minimal box (Alg. 4 l.7 PAPER.md:1233, tau PAPER.md:1265);
//   a6 per-cell stats for the sweep reductions.
// Linear-domain marginals are fp64 so the global Y-marginal is preserved to
// fp64 rounding (reading R16).  The cell's shared-memory footprint
// grows with its hull; cells are binned by hull side into size classes, each
// launched with its own CTA size and occupancy.
#pragma once
#include "internal.cuh"

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

// max(m, |v|), NaN-propagating (the Y stages' out-of-range flag: a shifted
// sum outside (2^-kLgRange, 2^kLgRange), an infinite or a NaN sum all give
// !(m < kLgRange))
__device__ __forceinline__ float fmax_nan_abs(float m, float v) {
  float y;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(y) : "f"(m), "f"(fabsf(v)));
  return y;
}
constexpr float kLgRange = 60.f;

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

// Deterministic block sum of NV (power of two <= 32) values of type T per
// thread: transpose butterfly inside the warp (NV - 1 + log2(32/NV)
// shuffles), then a fixed-order sum over the warps.  scratch >= NV * nwarps,
// out[0..NV) (distinct from scratch).
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
// Shared-memory layout of one cell.  BB = ccap^2 box entries, NX = 2 s,
// nt = threads per CTA.  Byte offsets are 32-bit.
//   nuJ  fp64 [BB]        a1, kept for the split
//   R2   16 B [BB]        Sinkhorn: B (Y potential), LN (log2 nu_J), BK;
//                         split: the member shares P0..P3
//   U    fp32 [2 NX ccap] Sinkhorn stage buffers Ub/UK; moments m1/m2; split stage 1
//   V    fp32 [2 NX ccap] Vb/VK
//   X    fp32 [5 NX^2+4]  A2, A2n, LM (log2 mu), MU, AL (+ mass defect)
//   fred fp32 [64], ints [64]
//   red  fp64             block reductions, per-pixel moments, balance coefficients
struct CellLayout {
  unsigned nuJ, R2, U, V, X, fred, ints, red, total;
};
__host__ __device__ constexpr unsigned red_doubles(int s, int nt) {
  const unsigned NXX = 4u * (unsigned)s * (unsigned)s, nw = (unsigned)nt / 32u;
  const unsigned a = 6u * NXX, b = 16u * nw + 16u;
  return (a > b ? a : b) + 64u;
}
__host__ __device__ inline CellLayout cell_layout(int ccap, int s, int nt) {
  CellLayout L;
  const unsigned BB = (unsigned)ccap * (unsigned)ccap, NX = 2u * (unsigned)s;
  unsigned o = 0;
  auto take = [&](unsigned bytes) { unsigned r = o; o += (bytes + 15u) & ~15u; return r; };
  L.nuJ = take(BB * 8);
  L.R2 = take(BB * 16);
  L.U = take(2 * NX * ccap * 4);
  L.V = take(2 * NX * ccap * 4);
  L.X = take((5 * NX * NX + 4) * 4);
  L.fred = take(64 * 4);
  L.ints = take(64 * 4);
  L.red = take(red_doubles(s, nt) * 8);
  L.total = o;
  return L;
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
      nuJ[(d1 + r) * b2 + d2 + c] += __ldg(src + t);
    }
    __syncthreads();
  }
}

// Final (balanced) value of every member at one box entry (a3 + a4).
// Explicit _rn intrinsics: bitwise identical in the truncation and the write
// pass.  Balance (reading R8): blended overlap / own-shape transfer
//   v_k = parts_k + parts_k * (sum_j O_kj parts_j) / nu_J + sum_j P_kj parts_j
// (O: overlap-transfer coefficients f theta / T, P: own-shape coefficients
// f (1 - theta) / M_d).  bc[0] = active flag, bc[1 + 4k + j] = O_kj,
// bc[17 + 4k + j] = P_kj.
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

// Cells whose hull exceeds the class capacity (cannot happen after binning
// unless the grid itself is larger than the huge class), or whose marginals
// would be annihilated, keep their previous marginals (copied to the output
// pool).  Pool exhaustion is counted in the sweep totals and the cumulative
// counters: the state is then invalid and every later synchronising call
// reports DD_ERR_NUMERIC (include/domdec.h).
__device__ __forceinline__ void copy_unchanged(const SweepParams& p, const CompCell& cc, const int J, int* ints,
                                               const int reason) {
  const int tid = threadIdx.x, T = blockDim.x, nmem = cc.nmem;
  long long* base = (long long*)(ints + 48);
  if (tid == 0) {
    long long tot = 0;
    for (int k = 0; k < nmem; ++k) tot += (long long)ints[8 + k] * ints[12 + k];
    base[0] = (long long)atomicAdd(p.pool_ctr, (unsigned long long)tot);
    if (base[0] + tot > p.pool_cap) {
      base[0] = -1;
      atomicAdd(&p.totals->overflow, 1ull);
      atomicAdd(&p.cum->invalid, 1ull);
    }
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
    atomicAdd(&p.cum->overflow, 1ull);
    atomicAdd(&p.totals->cells, 1ull);
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
template <int NX>
__device__ __forceinline__ void primal_terms(const SweepParams& p, const CompCell& cc, const int J, const int b1,
                                             const int b2, const int L1, const int L2, const int o1, const int o2,
                                             const int G1, const int G2, const float* A2, const float* A2n,
                                             const float* MU, const float* Bp, const double* nuJ, double* red) {
  const int tid = threadIdx.x, T = blockDim.x;
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
  const int nw = T >> 5;
  block_xsum<double, 8>(v, red, red + 8 * nw);
  if (tid == 0) {
    const double* S = red + 8 * nw;
    const double D1 = (double)(cc.r0 - G1), D2 = (double)(cc.c0 - G2);
    p.ecell[J] = (D1 * D1 + D2 * D2) * S[3] + 2.0 * (D1 * (S[1] - S[6]) + D2 * (S[2] - S[7])) +
                 p.eps_p * (0.69314718055994531 * (S[0] + S[4] + S[5]) - S[3]);
  }
  __syncthreads();
}

}  // namespace dd
#include "sweep_cluster.cuh"
namespace dd {

// ===========================================================================
// The fused cell routine.  NX = 2 s (X-block side), NT = threads per CTA,
// PR = record the primal score, GS = the working set lives in global scratch
// (huge class; a separate instantiation so that the shared-memory classes see
// a pointer derived from the __shared__ array and compile to LDS/STS),
// CL = the huge class on a thread-block cluster: every CTA of the cluster
// calls this routine for the same cell; the leader (rank 0) runs the setup
// and the epilogue on the global scratch, the Sinkhorn passes run on all KC
// CTAs (sweep_cluster.cuh).  loc = the CTA's own small shared buffers (ints,
// reductions), csm / cbudget = its shared-memory working set for the solve.
template <int NX, int NT, bool PR, bool GS, bool CL = false>
__device__ __forceinline__ void sweep_cell(const SweepParams& p, const int J, const int ccap, unsigned char* smem,
                                           unsigned char* loc = nullptr, float* csm = nullptr, int cbudget = 0,
                                           int rank = 0, int KC = 1) {
  const int tid = threadIdx.x;
  constexpr int T = NT;
  const CellLayout Ls = cell_layout(ccap, NX / 2, NT);
  double* nuJ = (double*)(smem + Ls.nuJ);
  float* P0 = (float*)(smem + Ls.R2);   // B (Y potential)
  const CompCell cc = p.cells[J];
  const int nmem = cc.nmem, n1 = cc.n1, n2 = cc.n2;
  const float w = p.w;
  int* ints = CL ? (int*)loc : (int*)(smem + Ls.ints);
  const bool lead = !CL || rank == 0;
  const int4 hull = cell_hull(p, cc, ints);
  const int L1 = hull.x, L2 = hull.y, b1 = hull.z, b2 = hull.w, BB = b1 * b2;
  const int b2p = b2 + (b2 & 1);        // even row stride of BK (8-byte aligned pairs)
  float* P1 = P0 + BB;                  // log2 nu_J - w lc2^2 (lc = l - o: centred hull column)
  float* P2 = P0 + 2 * BB;              // BK [b1][b2p] (may extend into the 4th R2 array)
  float* Ub = (float*)(smem + Ls.U);
  float* Rb = Ub + NX * ccap;           // UK
  float* Vb = (float*)(smem + Ls.V);
  float* X = (float*)(smem + Ls.X);
  float* A2 = X;
  float* A2n = X + NX * NX;
  float* LM = X + 2 * NX * NX;
  float* MU = X + 3 * NX * NX;
  float* AL = X + 4 * NX * NX;
  float* fred = CL ? (float*)(loc + 256) : (float*)(smem + Ls.fred);
  double* red = CL ? (double*)(loc + 512) : (double*)(smem + Ls.red);
  // gauge origin G = L + o, o = floor((b - n)/2)
  const int o1 = (b1 - n1) >> 1, o2 = (b2 - n2) >> 1;
  const int G1 = L1 + o1, G2 = L2 + o2;
  if (b1 > ccap || b2 > ccap) {   // cannot happen after binning (see copy_unchanged)
    if (lead) copy_unchanged(p, cc, J, ints, 1);
    return;
  }
  double muXJ = 0.0;
  for (int q = 0; q < nmem; ++q) muXJ += p.m[cc.mem[q]];
  const int NN = n1 * n2;
  constexpr int NXX = NX * NX;
  if (lead) {   // setup (a cluster's leader: on the global scratch)
  assemble(p, cc, ints, L1, L2, b2, BB, nuJ);
  double nsum = 0.0;
  for (int t = tid; t < BB; t += T) {
    const double v = nuJ[t];
    nsum += v;
    const float lc = (float)(t % b2 - o2);   // LNK = log2 nu_J - w lc^2 (zeros -> kNeg, R19)
    P1[t] = v > 0.0 ? lg2f((float)v) - w * lc * lc : kNeg;
  }
  {
    // mass defect of the cell problem (truncation ledger, reading R9): after
    // a Y-update the plan has mass ||nu_J||, so its X-marginal is compared
    // with mu ||nu_J|| / mu(X_J) (reading R6')
    const double nuMass = block_sum1_d(nsum, red);
    if (tid == 0) X[5 * NX * NX] = (float)((nuMass - muXJ) / muXJ);
  }
  // ---- X-block data, warm start (R7) and re-gauge ------------------------
  // The X-block is padded to NX x NX (ragged B cells have n = s on an axis);
  // padded pixels carry log2 mu = kNeg, so their terms vanish.
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
  }   // setup
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
  float* UK = Rb;                     // [NX][b2]  U - w k1^2
  float* VK = Vb + NX * ccap;         // [b1][NX]  V - w l1^2
  float* BK = P2;                     // [b1][b2p] B + log2 nu_J - w l2^2
  const float w2 = 2.f * w;
  const float fo1 = (float)o1, fo2 = (float)o2;
  constexpr int HX = NX / 2;
  // per-term slopes of the Y stages: z_q = x * (2 w) k_q + input, k_q = 2q, 2q+1
  float2 gq[HX];
#pragma unroll
  for (int q = 0; q < HX; ++q) gq[q] = make_float2(w2 * (float)(2 * q), w2 * (float)(2 * q + 1));
  auto single_loop = [&]() {
  if (b2 & 1)                         // padding column: a zero-weight term for X1's pairs
    for (int l1 = tid; l1 < b1; l1 += T) BK[l1 * b2p + b2] = kNeg;
  // Y2 mapping: thread -> (column l2, row group rg of RG)
  // (a hull wider than the CTA: columns in chunks of T)
  const int RG = max(1, T / b2);
  const int y2_col = tid % b2, y2_rg = tid / b2;
  // X2 mapping: thread -> (pair qa in [0, HX), column k2, split h of SX)
  constexpr int SX0 = T / (HX * NX);
  constexpr int SX = SX0 > 8 ? 8 : (SX0 < 1 ? 1 : SX0);
  const int x2_h = tid % SX, x2_pair = tid / SX;
  const int x2_k2 = x2_pair % NX, x2_qa = x2_pair / NX;
  const bool x2_valid = x2_pair < HX * NX;
  for (;;) {
    ++it;
    // Y-half stage 1: U(k1, l2) = LSE_k2 [A + log2 mu - w (k2 - l2~)^2].
    // Terms in pairs (FFMA2 / FADD2 on {q, q+1}); the shift c is the max
    // (first pass) or the previous output; a shifted sum outside
    // [2^-60, 2^60] only sets a flag, and a thread with a flagged output
    // recomputes all its outputs of the stage with a max shift (cold path).
    {
      // out-of-range flag: max over the thread's outputs of |lg2 sum| (NaN
      // propagating), tested once per pass: one FMNMX per output
      float lgmax = 0.f;
      auto y1_out = [&](const int o, const int k1, const int l2, const bool maxpass) {
        const float x = (float)l2 - fo2;
        const float2* ar = reinterpret_cast<const float2*>(AL + k1 * NX);
        float2 a[HX];
#pragma unroll
        for (int q = 0; q < HX; ++q) a[q] = ar[q];
        const float2 x2 = make_float2(x, x);
        float2 z[HX];
#pragma unroll
        for (int q = 0; q < HX; ++q) z[q] = __ffma2_rn(x2, gq[q], a[q]);
        float s0;   // U = s0 + lg2(sum) - w x^2 ... with c = s0' + w x^2 (see below)
        float c;
        if (maxpass) {
          c = kNeg;
#pragma unroll
          for (int q = 0; q < HX; ++q) c = fmaxf(c, fmaxf(z[q].x, z[q].y));
          s0 = c - w * x * x;
        } else {
          s0 = Ub[o];               // previous U: the shift is U_old + w x^2
          const float K = __fmul_rn(__fmul_rn(w, x), x);   // see Y2: s0 <- (s0 + K) - K
          c = __fadd_rn(s0, K);
          s0 = __fsub_rn(c, K);
        }
        const float2 nc = make_float2(-c, -c);
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < HX; ++q) {
          const float2 t = __fadd2_rn(z[q], nc);
          acc = __fadd2_rn(acc, make_float2(ex2f(t.x), ex2f(t.y)));
        }
        const float lg = lg2f(acc.x + acc.y);
        lgmax = fmax_nan_abs(lgmax, lg);
        const float U = s0 + lg;
        Ub[o] = U;
        UK[o] = U - w * (float)(k1 * k1);
      };
      // pass 1 (cold, flagged threads only): the outputs again with a true
      // max shift; one call site keeps the stage's code compact (i-cache)
      for (int pass = 0; pass < 2 && (pass == 0 || !(lgmax < kLgRange)); ++pass) {
        const bool mp = first || pass == 1;
        for (int o = tid, k1 = tid / b2, l2 = tid % b2; o < NX * b2;
             o += T, k1 += T / b2, l2 += T % b2, (l2 >= b2 ? (l2 -= b2, ++k1) : 0))
          y1_out(o, k1, l2, mp);
      }
    }
    __syncthreads();
    // Y-half stage 2: B(l1, l2) = -LSE_k1 [U(k1, l2) - w (k1 - l1~)^2]; the
    // thread's column inputs stay in registers as pairs; BK rows have the
    // even stride b2p (row b2p-1 of an odd b2 holds kNeg for X1's pairs).
    {
      float lgmax = 0.f;   // out-of-range flag as in Y1
      auto y2_column = [&](const int l2, const int l1_0, const int l1_step, const bool maxpass) {
        float2 u[HX];
#pragma unroll
        for (int q = 0; q < HX; ++q) u[q] = make_float2(UK[(2 * q) * b2 + l2], UK[(2 * q + 1) * b2 + l2]);
        float x = (float)l1_0 - fo1;
        const float xstep = (float)l1_step;
        for (int l1 = l1_0; l1 < b1; l1 += l1_step, x += xstep) {
          const int o = l1 * b2 + l2;
          const float2 x2 = make_float2(x, x);
          float2 z[HX];
#pragma unroll
          for (int q = 0; q < HX; ++q) z[q] = __ffma2_rn(x2, gq[q], u[q]);
          float s0, c;
          if (maxpass) {
            c = kNeg;
#pragma unroll
            for (int q = 0; q < HX; ++q) c = fmaxf(c, fmaxf(z[q].x, z[q].y));
            s0 = c - w * x * x;
          } else {
            s0 = -P0[o];            // previous B: the shift is -B_old + w x^2
            // shift c = s0 + K; s0 <- c - K (exact) carries the rounding of
            // the shift into the output (the output is c + lg2 sum - K)
            const float K = __fmul_rn(__fmul_rn(w, x), x);
            c = __fadd_rn(s0, K);
            s0 = __fsub_rn(c, K);
          }
          const float2 nc = make_float2(-c, -c);
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < HX; ++q) {
            const float2 t = __fadd2_rn(z[q], nc);
            acc = __fadd2_rn(acc, make_float2(ex2f(t.x), ex2f(t.y)));
          }
          const float lg = lg2f(acc.x + acc.y);
          lgmax = fmax_nan_abs(lgmax, lg);
          const float Bv = -s0 - lg;
          P0[o] = Bv;
          BK[l1 * b2p + l2] = Bv + P1[o];   // P1 = log2 nu_J - w lc2^2
        }
      };
      // columns in chunks of T when the hull is wider than the CTA; pass 1
      // (cold, flagged threads only) with a true max shift; one call site
      const int c0 = b2 <= T ? y2_col : tid, cstep = b2 <= T ? b2 : T;
      const int r0 = b2 <= T ? y2_rg : 0, rstep = b2 <= T ? RG : 1;
      if (b2 > T || y2_rg < RG)
        for (int pass = 0; pass < 2 && (pass == 0 || !(lgmax < kLgRange)); ++pass)
          for (int l2 = c0; l2 < b2; l2 += cstep) y2_column(l2, r0, rstep, first || pass == 1);
    }
    __syncthreads();
    // X-half stage 1: V(l1, k2) = LSE_l2 [B + log2 nu_J - w (k2 - lc2)^2],
    // two outputs (k2 = qa, qa + HX) per thread sharing every loaded BK pair
    // (LDS.64 of {l2, l2+1}, FFMA2 / FADD2 on the pair).  Hull coordinates
    // are centred on the X-block (lc = l - o): the expanded terms
    // BK + 2 w k2 lc then stay O(w b k2) instead of O(w b^2), which keeps
    // fp32 exponents of wide hulls accurate.
    for (int t = tid; t < b1 * HX; t += T) {
      const int l1 = t / HX, qa = t % HX, qb = qa + HX;
      const float kta = (float)qa, ktb = (float)qb;
      const float ga = w2 * kta, gb = w2 * ktb;
      const float Ka = __fmul_rn(__fmul_rn(w, kta), kta), Kb = __fmul_rn(__fmul_rn(w, ktb), ktb);
      const float2* br = reinterpret_cast<const float2*>(BK + l1 * b2p);
      const int np = b2p >> 1;
      float ca, cb;
      const bool maxpass = first;
      auto maxshift = [&]() {
        ca = kNeg;
        cb = kNeg;
        float2 lf = make_float2(-fo2, 1.f - fo2);
        for (int k = 0; k < np; ++k) {
          const float2 bk = br[k];
          const float2 za = __ffma2_rn(make_float2(ga, ga), lf, bk), zb = __ffma2_rn(make_float2(gb, gb), lf, bk);
          ca = fmaxf(ca, fmaxf(za.x, za.y));
          cb = fmaxf(cb, fmaxf(zb.x, zb.y));
          lf = __fadd2_rn(lf, make_float2(2.f, 2.f));
        }
      };
      ca = cb = 0.f;
      auto sums = [&](float2& sa, float2& sb) {
        const float2 nca = make_float2(-ca, -ca), ncb = make_float2(-cb, -cb);
        const float2 g2a = make_float2(ga, ga), g2b = make_float2(gb, gb);
        sa = make_float2(0.f, 0.f);
        sb = make_float2(0.f, 0.f);
        float2 lf = make_float2(-fo2, 1.f - fo2);
#pragma unroll 2
        for (int k = 0; k < np; ++k) {
          const float2 bk = br[k];
          const float2 ta = __fadd2_rn(__ffma2_rn(g2a, lf, bk), nca);
          const float2 tb = __fadd2_rn(__ffma2_rn(g2b, lf, bk), ncb);
          sa = __fadd2_rn(sa, make_float2(ex2f(ta.x), ex2f(ta.y)));
          sb = __fadd2_rn(sb, make_float2(ex2f(tb.x), ex2f(tb.y)));
          lf = __fadd2_rn(lf, make_float2(2.f, 2.f));
        }
      };
      float2 s2a, s2b;
      float sa = 0.f, sb = 0.f;
      for (int pass = 0; pass < 2; ++pass) {   // pass 1: max shift after an out-of-range sum
        if (maxpass || pass == 1) {
          maxshift();
        } else {
          ca = __fadd_rn(Vb[l1 * NX + qa], Ka);
          cb = __fadd_rn(Vb[l1 * NX + qb], Kb);
        }
        sums(s2a, s2b);
        sa = s2a.x + s2a.y;
        sb = s2b.x + s2b.y;
        if ((sa > 0x1p-60f && sa < 0x1p60f) && (sb > 0x1p-60f && sb < 0x1p60f)) break;
      }
      // (c - K) + lg2 sum: c - K is exact, so the output carries no rounding
      // of the large shift K = w kt^2 (wide hulls)
      const float Va = __fsub_rn(ca, Ka) + lg2f(sa);
      const float Vbv = __fsub_rn(cb, Kb) + lg2f(sb);
      const float lc1 = (float)l1 - fo1;
      const float wl1 = w * lc1 * lc1;
      Vb[l1 * NX + qa] = Va;
      Vb[l1 * NX + qb] = Vbv;
      VK[l1 * NX + qa] = Va - wl1;
      VK[l1 * NX + qb] = Vbv - wl1;
    }
    __syncthreads();
    // X-half stage 2: A'(k1, k2) = -LSE_l1 [V(l1, k2) - w (k1 - lc1)^2],
    // two outputs (k1 = qa, qa + HX) per thread, terms split over SX lanes
    // (centred rows, as in X1)
    float epart = 0.f;
    {
      const int qa = x2_qa, qb = qa + HX, k2 = x2_k2;
      const float kta = (float)qa, ktb = (float)qb;
      const float ga = w2 * kta, gb = w2 * ktb;
      const float Ka = __fmul_rn(__fmul_rn(w, kta), kta), Kb = __fmul_rn(__fmul_rn(w, ktb), ktb);
      float ca = 0.f, cb = 0.f;
      if (first) {
        ca = kNeg;
        cb = kNeg;
        if (x2_valid) {
          float lf = (float)x2_h - fo1;
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
        ca = __fadd_rn(-A2[qa * NX + k2], Ka);
        cb = __fadd_rn(-A2[qb * NX + k2], Kb);
      }
      float sa = 0.f, sb = 0.f;
      if (x2_valid) {   // the two outputs as a pair (FFMA2 / FADD2)
        const float2 g2 = make_float2(ga, gb), nc2 = make_float2(-ca, -cb);
        float2 s2 = make_float2(0.f, 0.f);
        float lf = (float)x2_h - fo1;
#pragma unroll 4
        for (int l1 = x2_h; l1 < b1; l1 += SX, lf += (float)SX) {
          const float vk = VK[l1 * NX + k2];
          const float2 z = __fadd2_rn(__ffma2_rn(make_float2(lf, lf), g2, make_float2(vk, vk)), nc2);
          s2 = __fadd2_rn(s2, make_float2(ex2f(z.x), ex2f(z.y)));
        }
        sa = s2.x;
        sb = s2.y;
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
          float lf = (float)x2_h - fo1;
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
          float lf = (float)x2_h - fo1;
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
        const float ana = -(__fsub_rn(ca, Ka) + lg2f(sa));   // (c - K) exact, as in X1
        const float anb = -(__fsub_rn(cb, Kb) + lg2f(sb));
        A2n[oa] = ana;
        A2n[ob] = anb;
        // L1 X-marginal error of the plan (A, B): sum mu |r - 2^(A - A')| (R6')
        // (padded pixels of ragged B cells carry mu = 0 and would give 0 * inf)
        const float rm1 = X[5 * NXX];   // (A2/A2n swap; X itself is fixed)
        if (MU[oa] > 0.f) epart += MU[oa] * fabsf(exp2m1f(A2[oa] - ana) - rm1);
        if (MU[ob] > 0.f) epart += MU[ob] * fabsf(exp2m1f(A2[ob] - anb) - rm1);
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
  };   // single_loop
  if constexpr (CL) {
    cluster_sync_all();   // the leader's setup is in the global scratch
    if (cluster_floats(b1, b2, NX, KC) * 4u <= (unsigned)cbudget) {
      const ClusterSolveOut co =
          cluster_solve<NX, NT>(p, b1, b2, w, fo1, fo2, tolJ, P1, P0, BK, Vb, VK, X, csm, fred, rank, KC);
      it = co.it;
      e0 = co.e0;
      e = co.e;
      A2 = X;
      A2n = X + NXX;
    } else if (lead) {   // too large for the cluster's shared memory: the leader alone
      single_loop();
    }
    cluster_sync_all();
    if (!lead) return;
  } else {
    single_loop();
  }
  __syncthreads();
  if (PR) primal_terms<NX>(p, cc, J, b1, b2, L1, L2, o1, o2, G1, G2, A2, A2n, MU, P0, nuJ, red);

  // ---- outputs of the solve: the plan's potential (next warm start, R7) ---
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
    // per pass plus NN for the X-error, BB for log2 nu_J
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

  // ---- a3': plan moments for the flow update (reading R13) ----------------
  // The final plan pi(x, y) = 2^(A(x) + B(y) - w |kappa - lt|^2) mu(x) nu_J(y)
  // has X-marginal PX = mu 2^(A - A') and, for each x, a conditional law over
  // y whose weights are exactly the terms of the last X-half.  One more
  // X-half with moment weights gives, with d = lt - kappa (local Y minus
  // local X), E[d | x] and E[|d|^2 | x]:
  //   X1m: m1(l1, k2) = E[d2 | l1, k2], m2(l1, k2) = E[d2^2 | l1, k2] over l2
  //        (shift = the last V, so the sum is ~1);
  //   X2m: over l1 with weights 2^(V(l1, k2) - w (k1 - l1~)^2 - shift).
  // Per basic cell i (member quadrant) about its centre z_i, with u = x - z_i
  // and the displacement e = y - x = d - D (D = K - G):
  //   M0 = sum PX, M1 = sum PX (u + E e), G0 = sum PX |u|^2,
  //   G1 = sum PX u.(u + E e), M2 = sum PX E|u + e|^2.
  {
    float* m1 = Ub;                 // [b1][NX] (the U region is free now)
    float* m2 = Ub + NX * ccap;
    for (int t = tid; t < b1 * NX; t += T) {
      const int l1 = t / NX, k2 = t % NX;
      const float kt = (float)k2 + fo2;   // lt2 - k2 = l2 - kt
      const float g = w2 * (float)k2;     // centred columns (X1)
      const float c = Vb[t] + w * (float)(k2 * k2);
      const float* br = BK + l1 * b2p;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f;
      float lf = -fo2, d = -kt;
      for (int l2 = 0; l2 < b2; ++l2, lf += 1.f, d += 1.f) {
        const float ev = ex2f(fmaf(g, lf, br[l2]) - c);
        s0 += ev;
        s1 = fmaf(ev, d, s1);
        s2 = fmaf(ev * d, d, s2);
      }
      const float inv = s0 > 0.f ? 1.0f / s0 : 0.f;
      m1[t] = s1 * inv;
      m2[t] = s2 * inv;
    }
    __syncthreads();
    const float cen = 0.5f * (float)(NX / 2 - 1);
    double* pm = red;   // [6][NXX] per-pixel contributions (fp64)
    for (int t = tid; t < NXX; t += T) {
      const int k1 = t / NX, k2 = t % NX;
      double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      if (k1 < n1 && k2 < n2) {
        const float kt = (float)k1 + fo1;
        const float g = w2 * (float)k1;   // centred rows (X2)
        const float c = -A2n[t] + w * (float)(k1 * k1);
        float t0 = 0.f, t1 = 0.f, t2 = 0.f, u1 = 0.f, u2 = 0.f;
        float lf = -fo1, d = -kt;
        for (int l1 = 0; l1 < b1; ++l1, lf += 1.f, d += 1.f) {
          const float ev = ex2f(fmaf(g, lf, VK[l1 * NX + k2]) - c);
          t0 += ev;
          t1 = fmaf(ev, d, t1);
          t2 = fmaf(ev * d, d, t2);
          u1 = fmaf(ev, m1[l1 * NX + k2], u1);
          u2 = fmaf(ev, m2[l1 * NX + k2], u2);
        }
        const double inv = t0 > 0.f ? 1.0 / (double)t0 : 0.0;
        const double Ed1 = t1 * inv, Ed2 = u1 * inv, Edd = (t2 + u2) * inv;
        const double D1 = (double)(cc.r0 - G1), D2 = (double)(cc.c0 - G2);
        const double Ee1 = Ed1 - D1, Ee2 = Ed2 - D2;                       // E[y - x | x]
        const double Eee = Edd - 2.0 * (D1 * Ed1 + D2 * Ed2) + D1 * D1 + D2 * D2;   // E|y - x|^2
        const int s = NX / 2;
        const double uu1 = (double)(k1 % s) - cen, uu2 = (double)(k2 % s) - cen;   // x - z_i
        const double px = (double)MU[t] * exp2((double)A2[t] - (double)A2n[t]);
        const double uu = uu1 * uu1 + uu2 * uu2;
        if (p.pxm) {   // per pixel record for the gluing candidates (f1)
          const long long pix = (long long)(cc.r0 + k1) * p.N2 + cc.c0 + k2;
          p.pxm[3 * pix] = px;
          p.pxm[3 * pix + 1] = Ee1;
          p.pxm[3 * pix + 2] = Ee2;
        }
        v[0] = px;
        v[1] = px * (uu1 + Ee1);
        v[2] = px * (uu2 + Ee2);
        v[3] = px * uu;
        v[4] = px * (uu + uu1 * Ee1 + uu2 * Ee2);
        v[5] = px * (uu + 2.0 * (uu1 * Ee1 + uu2 * Ee2) + Eee);
      }
#pragma unroll
      for (int q = 0; q < 6; ++q) pm[q * NXX + t] = v[q];
    }
    __syncthreads();
    // member k (quadrant (h1, h2)) sums its s x s pixels in a fixed order
    if (tid < 24) {
      const int k = tid / 6, q = tid % 6;
      if (k < nmem) {
        const int s = NX / 2, h1 = cc.quad[k] >> 1, h2 = cc.quad[k] & 1;
        double acc = 0.0;
        for (int a = 0; a < s; ++a)
          for (int b = 0; b < s; ++b) acc += pm[q * NXX + (h1 * s + a) * NX + h2 * s + b];
        p.mom[6 * cc.mem[k] + q] = acc;
      }
    }
    __syncthreads();
  }

  // ---- a3: CompositeToBasic (share form) ----------------------------------
  // Stage 1 split by column half h2: U_h2(k1, l2) = LSE over k2 in half h2
  // of A + log2 mu - w (k2 - l2~)^2.
  const int s = NX / 2;
  const int c2 = n2 / s;
  float* Us = Ub;   // [c2][n1][b2]
  for (int o = tid; o < c2 * n1 * b2; o += T) {
    const int h2 = o / (n1 * b2);
    const int rem = o - h2 * n1 * b2;
    const int k1 = rem / b2, l2 = rem - k1 * b2;
    const float lt = (float)l2 - fo2;
    float sh = kNeg;
    for (int k2 = h2 * s; k2 < h2 * s + s; ++k2) {
      const float d = (float)k2 - lt;
      sh = fmaxf(sh, A2[k1 * NX + k2] + LM[k1 * NX + k2] - w * d * d);
    }
    float sum = 0.f;
    for (int k2 = h2 * s; k2 < h2 * s + s; ++k2) {
      const float d = (float)k2 - lt;
      sum += ex2f(A2[k1 * NX + k2] + LM[k1 * NX + k2] - w * d * d - sh);
    }
    Us[o] = sh + lg2f(sum);
  }
  __syncthreads();
  // Stage 2 per box entry: member log-weights S_k, shares p_k (stored), the
  // exact fp64 split (the largest share takes the remainder: sum = nu_J), the
  // split masses and the pairwise overlaps sum v_a v_b / nu_J (balance, R8).
  float* S0 = P0;   // shares P0..P3 overwrite B, LN, BK (dead now)
  float* S1 = P0 + BB;
  float* S2 = P0 + 2 * BB;
  float* S3 = P0 + 3 * BB;
  int mq[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) mq[k] = cc.quad[k];
  double da[8], db[2];   // masses [0..3], overlaps [4 + pair] (pairs 0..3 in da, 4..5 in db)
#pragma unroll
  for (int q = 0; q < 8; ++q) da[q] = 0.0;
  db[0] = 0.0;
  db[1] = 0.0;
  for (int o = tid; o < BB; o += T) {
    const int l1 = o / b2, l2 = o - l1 * b2;
    const float lt = (float)l1 - fo1;
    float S[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      S[k] = kNeg;
      if (k < nmem) {
        const int h1 = mq[k] >> 1, h2 = mq[k] & 1;
        const float* ur = Us + (h2 * n1) * b2 + l2;
        float sh = kNeg;
        for (int k1 = h1 * s; k1 < h1 * s + s; ++k1) {
          const float d = (float)k1 - lt;
          sh = fmaxf(sh, ur[k1 * b2] - w * d * d);
        }
        float sum = 0.f;
        for (int k1 = h1 * s; k1 < h1 * s + s; ++k1) {
          const float d = (float)k1 - lt;
          sum += ex2f(ur[k1 * b2] - w * d * d - sh);
        }
        S[k] = sh + lg2f(sum);
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
    S0[o] = pk[0];
    S1[o] = pk[1];
    S2[o] = pk[2];
    S3[o] = pk[3];
    const double nj = nuJ[o];
    if (nj > 0.0) {
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
      const double invj = 1.0 / nj;
#pragma unroll
      for (int a = 0; a < 4; ++a) da[a] += v[a];
      da[4] += v[0] * v[1] * invj;   // pair (0,1)
      da[5] += v[0] * v[2] * invj;   // (0,2)
      da[6] += v[0] * v[3] * invj;   // (0,3)
      da[7] += v[1] * v[2] * invj;   // (1,2)
      db[0] += v[1] * v[3] * invj;   // (1,3)
      db[1] += v[2] * v[3] * invj;   // (2,3)
    }
  }
  __syncthreads();
  const int nw = T >> 5;
  // reduced values: masses Rv[0..3], overlaps Rv[4 + pair]
  double* Rv = red + 16 * nw;   // [10]
  block_xsum<double, 8>(da, red, Rv);
  block_xsum<double, 2>(db, red, Rv + 8);
  const double* Rm = Rv;
  const double* Rov = Rv + 4;
  const double massJ = Rm[0] + Rm[1] + Rm[2] + Rm[3];
  // ---- a4: balance coefficients (reading R8), in shared memory -----------
  // Warp 0 computes them lane-parallel: lane 4 d + r -> O_dr, lane 16 + 4 k +
  // j -> P_kj.
  double* bc = Rv + 16;   // [33]
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
        double Lsum = 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r < nmem && r != d && delta[r] < 0) {
            const double Tdr = Rov[d < r ? pair_id(d, r) : pair_id(r, d)];
            if (!(Tdr > 0.0)) zeroT = true;
            else Lsum += delta[d] * (-delta[r]) / Dsum / Tdr;
          }
        }
        const double l = delta[d] / Rm[d];
        theta[d] = zeroT ? 0.0 : (Lsum <= 1.0 ? 1.0 : (1.0 - l) / (Lsum - l));
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
              const double Tdr = Rov[d < r ? pair_id(d, r) : pair_id(r, d)];
              if (theta[d] > 0.0) {
                const double x = f * theta[d] / Tdr;
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
  // ---- a5: truncate + minimal box -----------------------------------------
  // layout: ints[16 + 4k + 0] = min row, +1 = max row, +2 = min col, +3 = max col
  if (tid < 4) {
    ints[16 + 4 * tid + 0] = 1 << 30;
    ints[16 + 4 * tid + 1] = -1;
    ints[16 + 4 * tid + 2] = 1 << 30;
    ints[16 + 4 * tid + 3] = -1;
  }
  __syncthreads();
  double dloc = 0.0;
  // per-thread bounds in registers (static member indices), one warp
  // reduction and one shared atomic per warp and bound at the end
  int bmn1[4], bmx1[4], bmn2[4], bmx2[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { bmn1[k] = 1 << 30; bmx1[k] = -1; bmn2[k] = 1 << 30; bmx2[k] = -1; }
  for (int o = tid; o < BB; o += T) {
    const int l1 = o / b2, l2 = o - l1 * b2;
    const float pk[4] = {S0[o], S1[o], S2[o], S3[o]};
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
  const double dropped = block_sum1_d(dloc, red);
  // an annihilated member (no entry above tau) keeps its previous marginal
  bool ok = true;
  for (int k = 0; k < nmem; ++k) {
    const int mn1 = ints[16 + 4 * k], mx1 = ints[16 + 4 * k + 1];
    const int mn2 = ints[16 + 4 * k + 2], mx2 = ints[16 + 4 * k + 3];
    if (mx1 < mn1 || mx2 < mn2) { ok = false; break; }
  }
  if (!ok) {
    copy_unchanged(p, cc, J, ints, 2);
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
    if (b0 + tot > p.pool_cap) {
      b0 = -1;
      atomicAdd(&p.totals->overflow, 1ull);
      atomicAdd(&p.cum->invalid, 1ull);
    }
    pbase[0] = b0;
  }
  __syncthreads();
  if (pbase[0] < 0) return;   // pool exhausted: reported (state invalid, include/domdec.h)
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
      const float pk[4] = {S0[o], S1[o], S2[o], S3[o]};
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
    p.stats[J].dropped = dropped;
    // algorithmic MUFU count of the split (C2B) and of the moment X-half
    const unsigned long long E_c2b = (unsigned long long)n1 * n2 * b2 + (unsigned long long)nmem * s * BB +
                                     (unsigned long long)nmem * BB;
    const unsigned long long L_c2b = (unsigned long long)c2 * n1 * b2 + (unsigned long long)nmem * BB;
    const unsigned long long E_mom = (unsigned long long)b1 * n2 * b2 + (unsigned long long)n1 * n2 * b1;
    const unsigned long long mufu = E_c2b + L_c2b + E_mom;
    atomicAdd(&p.totals->mufu, mufu);
    atomicAdd(&p.cum->mufu, mufu);
    // algorithmic HBM bytes (with the fp64 marginals of reading
    // R16): member boxes read once + written once, metadata, mu / log2 mu,
    // alpha read + write, plan moments
    unsigned long long rbytes = 0;
    for (int k = 0; k < nmem; ++k) rbytes += (unsigned long long)ints[8 + k] * ints[12 + k] * 8ull;
    const unsigned long long byts = rbytes + wbytes + 32ull * nmem + (unsigned long long)NN * 16ull + 48ull * nmem;
    atomicAdd(&p.totals->bytes, byts);
    atomicAdd(&p.cum->bytes, byts);
    atomicAdd(&p.cum->cells, 1ull);
    atomicAdd(&p.totals->cells, 1ull);
    atomicAdd(&p.totals->dropped, dropped);
  }
}

// Persistent CTAs of one size class: cells are fetched dynamically from the
// class list (load balance across cells of different hull and iteration
// count).
template <int NX, int NT, int MINB, bool PR, bool GS>
__global__ void __launch_bounds__(NT, MINB) sweep_kernel(SweepParams p, const int cls, const int ccap) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int job;
  unsigned char* base = GS ? p.scratch + (size_t)blockIdx.x * p.scratch_stride : smem;
  const int n = p.cls_count[cls];
  const int* list = p.cls_list + (size_t)cls * p.ncells;
  for (;;) {
    if (threadIdx.x == 0) job = atomicAdd(&p.cls_fetch[cls], 1);
    __syncthreads();
    const int k = job;
    __syncthreads();
    if (k >= n) break;
    sweep_cell<NX, NT, PR, GS>(p, list[k], ccap, base);
    __syncthreads();
  }
}

// The huge class on thread-block clusters: each cluster fetches one cell at
// a time (the leader's fetch is read by all CTAs through DSMEM) and solves it
// with sweep_cell<..., CL> on the cluster's slot of the global scratch.
template <int NX, int NT, bool PR>
__global__ void __launch_bounds__(NT, 1) sweep_kernel_cl(SweepParams p, const int cls, const int ccap,
                                                         const int cbudget) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(16) unsigned char loc[512 + 8 * red_doubles(NX / 2, NT)];
  __shared__ int job;
  cgc::cluster_group cl = cgc::this_cluster();
  const int rank = (int)cl.block_rank(), KC = (int)cl.num_blocks();
  unsigned char* base = p.scratch + (size_t)(blockIdx.x / KC) * p.scratch_stride;
  const int n = p.cls_count[cls];
  const int* list = p.cls_list + (size_t)cls * p.ncells;
  for (;;) {
    if (rank == 0 && threadIdx.x == 0) job = atomicAdd(&p.cls_fetch[cls], 1);
    cl.sync();
    const int k = *cl.map_shared_rank(&job, 0);
    cl.sync();   // every CTA has read the job before the leader fetches again
    if (k >= n) break;
    sweep_cell<NX, NT, PR, true, true>(p, list[k], ccap, base, loc, (float*)smem, cbudget, rank, KC);
    __syncthreads();
  }
}

}  // namespace dd
