// sweep_cluster.cuh — the Sinkhorn loop (a2) of one composite cell spread
// over a thread-block cluster (sm_100a, distributed shared memory).
//
// Composite cells whose Y-hull exceeds what one CTA can hold in shared
// memory (the huge size class H) are rare, but on
// refined multiscale layers they are the critical path of a sweep: their
// Y-boxes are a few hundred pixels wide (strong expansion of the transport
// map) and they need hundreds of Sinkhorn passes, each of ~0.5M ex2 terms.
// One CTA on global-memory scratch runs them at a small fraction of the MUFU
// peak.  Here a cluster of KC CTAs (one per SM) solves one such cell:
//   * rows l1 of the Y-hull are split into KC contiguous chunks; each CTA
//     keeps its rows of B, log2 nu_J and BK, and V of its rows, in its own
//     shared memory for the whole solve;
//   * the X-block data (A, A', log2 mu, mu: NX^2 values) is replicated;
//   * Y-half stage 1 (U(k1, l2), no row dependence, NX^2 b2 terms) is
//     computed for all columns by every CTA: a column split with a DSMEM
//     exchange cost one more cluster barrier per pass and measured 15% slower
//     (profiles/r02_ncu_cluster.txt);
//   * Y-half stage 2 and X-half stage 1 are row-local;
//   * X-half stage 2 (A' = -LSE over all rows) adds per-CTA partial sums of
//     the same shift (the previous A', or the cluster-wide maximum on the
//     first pass): partials in shared memory, cluster barrier, every CTA sums
//     the KC partials in rank order, so all CTAs hold bit-identical A' and
//     X-errors and take the same stopping decision.
// One cluster barrier per pass (two on the first).  The arithmetic of
// every term is the one of the single-CTA loop (sweep.cuh, "Shift trick");
// only the fp32 summation order of the row sums differs.  On exit the CTAs
// write their rows of B, BK, V back to the cell's global scratch, where the
// leader CTA continues with the moments, the split, balance and truncation.
// (Included by sweep.cuh after its helpers: ex2f, lg2f, exp2m1f, block_sum_f.)
#pragma once
#include <cooperative_groups.h>

#include "internal.cuh"

namespace dd {

namespace cgc = cooperative_groups;

__device__ __forceinline__ void cluster_sync_all() {
  __threadfence();   // global-scratch writes of this CTA visible to the cluster
  cgc::this_cluster().sync();
}

// Float count of a CTA's shared-memory working set for a b1 x b2 hull.
__host__ __device__ inline unsigned cluster_floats(int b1, int b2, int NX, int KC) {
  const unsigned Rm = (unsigned)((b1 + KC - 1) / KC);
  const unsigned b2p = (unsigned)(b2 + (b2 & 1));
  const unsigned NXX = (unsigned)(NX * NX);
  return (unsigned)NX * b2   // UK of all columns, transposed [b2][NX] (first: float4 rows)
         + Rm * b2p          // BK (8-byte aligned pairs)
         + 2 * Rm * b2       // B, log2 nu_J - w l2^2
         + 2 * Rm * NX       // V, VK
         + (unsigned)NX * b2 // U of every column (shifts; Y-stage 1 is replicated)
         + 5 * NXX + 4       // A, A', log2 mu, mu, AL, mass defect
         + 4 * NXX + 4;      // shifts, partial sums (two buffers), partial maxima
}

struct ClusterSolveOut {
  int it;
  float e0, e;
};

// Runs the Sinkhorn passes of one cell on the cluster.  Global scratch (the
// single-CTA layout of sweep_cell, written by the leader's setup):
//   P1g [b1][b2] log2 nu_J - w l2^2; Xg: A (re-gauged), -, log2 mu, mu, AL,
//   mass defect.  Written back: P0g [b1][b2] B, BKg [b1][b2p] BK, Vbg /
//   VKg [b1][NX] V and VK, Xg[0..NXX) the plan's A, Xg[NXX..2NXX) A'.
template <int NX, int NT>
__device__ ClusterSolveOut cluster_solve(const SweepParams& p, const int b1, const int b2, const float w,
                                         const float fo1, const float fo2, const float tolJ, const float* P1g,
                                         float* P0g, float* BKg, float* Vbg, float* VKg, float* Xg, float* csm,
                                         float* fred, const int rank, const int KC) {
  cgc::cluster_group cl = cgc::this_cluster();
  const int tid = threadIdx.x;
  constexpr int T = NT, NXX = NX * NX, HX = NX / 2;
  const int b2p = b2 + (b2 & 1);
  const int Rm = (b1 + KC - 1) / KC;
  const int r0 = min(b1, rank * Rm), R = min(b1, r0 + Rm) - r0;   // own rows [r0, r0 + R)
  // Y-stage 1 (NX^2 b2 terms) is computed by every CTA for all columns: cheaper
  // than a DSMEM exchange and its cluster barrier on every pass
  // shared-memory carve-up (see cluster_floats)
  float* UKt = csm;                   // [b2][NX]
  float* BK = UKt + NX * b2;
  float* B = BK + Rm * b2p;
  float* LN = B + Rm * b2;
  float* Vb = LN + Rm * b2;
  float* VK = Vb + Rm * NX;
  float* Ub = VK + Rm * NX;           // [NX][b2]
  float* Xl = Ub + NX * b2;
  float* A2 = Xl;
  float* A2n = Xl + NXX;
  float* LM = Xl + 2 * NXX;
  float* MU = Xl + 3 * NXX;
  float* AL = Xl + 4 * NXX;
  float* csh = Xl + 5 * NXX + 4;      // per-output shift of X-stage 2
  float* part2 = csh + NXX;           // partial sums, by pass parity (read remotely)
  float* pmx = part2 + 2 * NXX;       // partial maxima (read remotely)
  for (int t = tid; t < R * b2; t += T) LN[t] = __ldcg(P1g + (size_t)r0 * b2 + t);
  for (int t = tid; t < 5 * NXX + 1; t += T) Xl[t] = __ldcg(Xg + t);
  if (b2 & 1)
    for (int l = tid; l < R; l += T) BK[l * b2p + b2] = kNeg;
  __syncthreads();
  const float rm1 = Xl[5 * NXX];
  const float w2 = 2.f * w;
  ClusterSolveOut out{0, 0.f, 0.f};
  bool first = true;
  // X-stage 1 mapping: task (row l, pair qa) on SXX lanes splitting the terms
  const int ntask1 = R * HX;
  int SXX = 1;
  while (SXX < 16 && 2 * SXX * max(ntask1, 1) <= T) SXX *= 2;
  // X-stage 2 mapping: output o on SX2 lanes splitting the own rows
  constexpr int SX2 = T / NXX >= 8 ? 8 : (T / NXX >= 1 ? T / NXX : 1);
  for (;;) {
    ++out.it;
    // ---- Y-half stage 1 (every column, replicated in every CTA) ------------
    {
      bool bad = false;
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1 && !bad) break;
        const bool mp = first || pass == 1;
        for (int o = tid; o < NX * b2; o += T) {
          const int k1 = o / b2, l2 = o - (o / b2) * b2;
          const float x = (float)l2 - fo2;
          const float wx = w2 * x;
          float z[NX];
#pragma unroll
          for (int q = 0; q < NX; ++q) z[q] = fmaf((float)q, wx, AL[k1 * NX + q]);
          float s0, c;
          if (mp) {
            c = kNeg;
#pragma unroll
            for (int q = 0; q < NX; ++q) c = fmaxf(c, z[q]);
            s0 = c - w * x * x;
          } else {
            s0 = Ub[o];
            // shift c = s0 + K; s0 <- c - K (exact) carries the rounding of
            // the shift into the output (the output is c + lg2 sum - K)
            const float K = __fmul_rn(__fmul_rn(w, x), x);
            c = __fadd_rn(s0, K);
            s0 = __fsub_rn(c, K);
          }
          float sum = 0.f;
#pragma unroll
          for (int q = 0; q < NX; ++q) sum += ex2f(z[q] - c);
          bad |= !(sum > 0x1p-60f && sum < 0x1p60f);
          const float U = s0 + lg2f(sum);
          Ub[o] = U;
          UKt[l2 * NX + k1] = U - w * (float)(k1 * k1);
        }
      }
    }
    __syncthreads();
    // ---- Y-half stage 2 on the own rows: B(l1, l2) = -LSE_k1 [...] --------
    {
      bool bad = false;
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1 && !bad) break;
        const bool mp = first || pass == 1;
        for (int o = tid; o < R * b2; o += T) {
          const int l = o / b2, l2 = o - l * b2;
          const float x = (float)(r0 + l) - fo1;
          const float wx = w2 * x;
          float u[NX];
          if constexpr (NX % 4 == 0) {
            const float4* up = reinterpret_cast<const float4*>(UKt + l2 * NX);
#pragma unroll
            for (int q = 0; q < NX / 4; ++q) {
              const float4 v = up[q];
              u[4 * q] = v.x; u[4 * q + 1] = v.y; u[4 * q + 2] = v.z; u[4 * q + 3] = v.w;
            }
          } else {
            const float2* up = reinterpret_cast<const float2*>(UKt + l2 * NX);
#pragma unroll
            for (int q = 0; q < NX / 2; ++q) {
              const float2 v = up[q];
              u[2 * q] = v.x; u[2 * q + 1] = v.y;
            }
          }
          float z[NX];
#pragma unroll
          for (int q = 0; q < NX; ++q) z[q] = fmaf((float)q, wx, u[q]);
          float s0, c;
          if (mp) {
            c = kNeg;
#pragma unroll
            for (int q = 0; q < NX; ++q) c = fmaxf(c, z[q]);
            s0 = c - w * x * x;
          } else {
            s0 = -B[o];
            // shift c = s0 + K; s0 <- c - K (exact) carries the rounding of
            // the shift into the output (the output is c + lg2 sum - K)
            const float K = __fmul_rn(__fmul_rn(w, x), x);
            c = __fadd_rn(s0, K);
            s0 = __fsub_rn(c, K);
          }
          float sum = 0.f;
#pragma unroll
          for (int q = 0; q < NX; ++q) sum += ex2f(z[q] - c);
          bad |= !(sum > 0x1p-60f && sum < 0x1p60f);
          const float Bv = -(s0 + lg2f(sum));
          B[o] = Bv;
          BK[l * b2p + l2] = Bv + LN[o];
        }
      }
    }
    __syncthreads();
    // ---- X-half stage 1 on the own rows: V(l1, k2) = LSE_l2 [...] ---------
    for (int gbase = 0; gbase < ntask1; gbase += T / SXX) {   // warp-uniform trip count
      const int g = gbase + tid / SXX, h = tid - (tid / SXX) * SXX;
      const bool valid = g < ntask1;
      const int l = valid ? g / HX : 0, qa = valid ? g % HX : 0, qb = qa + HX;
      const float kta = (float)qa, ktb = (float)qb;   // centred columns (sweep.cuh X1)
      const float ga = w2 * kta, gb = w2 * ktb;
      const float Ka = __fmul_rn(__fmul_rn(w, kta), kta), Kb = __fmul_rn(__fmul_rn(w, ktb), ktb);
      const float2* br = reinterpret_cast<const float2*>(BK + l * b2p);
      const int np = b2p >> 1;
      float ca = 0.f, cb = 0.f, sa = 0.f, sb = 0.f;
      bool need_max = first;
      for (int pass = 0; pass < 2; ++pass) {
        if (need_max) {
          ca = kNeg;
          cb = kNeg;
          if (valid)
            for (int k = h; k < np; k += SXX) {
              const float2 bk = br[k];
              const float lf = (float)(2 * k) - fo2;
              ca = fmaxf(ca, fmaxf(fmaf(ga, lf, bk.x), fmaf(ga, lf + 1.f, bk.y)));
              cb = fmaxf(cb, fmaxf(fmaf(gb, lf, bk.x), fmaf(gb, lf + 1.f, bk.y)));
            }
          for (int off = SXX >> 1; off > 0; off >>= 1) {
            ca = fmaxf(ca, __shfl_xor_sync(0xffffffffu, ca, off));
            cb = fmaxf(cb, __shfl_xor_sync(0xffffffffu, cb, off));
          }
        } else if (valid) {
          ca = __fadd_rn(Vb[l * NX + qa], Ka);
          cb = __fadd_rn(Vb[l * NX + qb], Kb);
        }
        float2 s2a = make_float2(0.f, 0.f), s2b = make_float2(0.f, 0.f);
        if (valid) {
          const float2 nca = make_float2(-ca, -ca), ncb = make_float2(-cb, -cb);
          const float2 g2a = make_float2(ga, ga), g2b = make_float2(gb, gb);
          for (int k = h; k < np; k += SXX) {
            const float2 bk = br[k];
            const float2 lf = make_float2((float)(2 * k) - fo2, (float)(2 * k + 1) - fo2);
            const float2 ta = __fadd2_rn(__ffma2_rn(g2a, lf, bk), nca);
            const float2 tb = __fadd2_rn(__ffma2_rn(g2b, lf, bk), ncb);
            s2a = __fadd2_rn(s2a, make_float2(ex2f(ta.x), ex2f(ta.y)));
            s2b = __fadd2_rn(s2b, make_float2(ex2f(tb.x), ex2f(tb.y)));
          }
        }
        sa = s2a.x + s2a.y;
        sb = s2b.x + s2b.y;
        for (int off = SXX >> 1; off > 0; off >>= 1) {
          sa += __shfl_xor_sync(0xffffffffu, sa, off);
          sb += __shfl_xor_sync(0xffffffffu, sb, off);
        }
        const bool bad = valid && (!(sa > 0x1p-60f && sa < 0x1p60f) || !(sb > 0x1p-60f && sb < 0x1p60f));
        // warp-uniform retry with the max shift (shuffles need the whole warp)
        if (need_max || !__any_sync(0xffffffffu, bad)) break;
        need_max = true;
      }
      if (valid && h == 0) {
        const float Va = __fsub_rn(ca, Ka) + lg2f(sa);   // (c - K) exact, see sweep.cuh
        const float Vbv = __fsub_rn(cb, Kb) + lg2f(sb);
        const float lc1 = (float)(r0 + l) - fo1;
        const float wl1 = w * lc1 * lc1;
        Vb[l * NX + qa] = Va;
        Vb[l * NX + qb] = Vbv;
        VK[l * NX + qa] = Va - wl1;
        VK[l * NX + qb] = Vbv - wl1;
      }
    }
    __syncthreads();
    // ---- X-half stage 2: A'(k1, k2) = -LSE over all rows -----------------
    const int o2 = tid / SX2, h2 = tid - (tid / SX2) * SX2;
    const bool ov = o2 < NXX;
    const int k1 = ov ? o2 / NX : 0, k2 = ov ? o2 % NX : 0;
    const float g = w2 * (float)k1;   // centred rows (sweep.cuh X2)
    // One cluster barrier per pass (in partial_sum): a CTA may start the next
    // pass's partial sums while another still reads this pass's, hence two
    // buffers by pass parity.
    float* part = part2 + (out.it & 1) * NXX;
    auto partial_max = [&]() {
      float m = kNeg;
      if (ov)
        for (int l = h2; l < R; l += SX2) m = fmaxf(m, fmaf(g, (float)(r0 + l) - fo1, VK[l * NX + k2]));
      for (int off = SX2 >> 1; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      if (ov && h2 == 0) pmx[o2] = m;
      cl.sync();
      if (tid < NXX) {
        float mm = kNeg;
        for (int r = 0; r < KC; ++r) mm = fmaxf(mm, cl.map_shared_rank(pmx, r)[tid]);
        csh[tid] = mm;
      }
      __syncthreads();
    };
    auto partial_sum = [&]() {
      float s = 0.f;
      if (ov) {
        const float c = csh[o2];
        for (int l = h2; l < R; l += SX2) s += ex2f(fmaf(g, (float)(r0 + l) - fo1, VK[l * NX + k2]) - c);
      }
      for (int off = SX2 >> 1; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (ov && h2 == 0) part[o2] = s;
      cl.sync();
    };
    if (first) {
      partial_max();
    } else {
      if (tid < NXX) {
        const float kq = (float)(tid / NX);
        csh[tid] = __fadd_rn(-A2[tid], __fmul_rn(__fmul_rn(w, kq), kq));
      }
      __syncthreads();
    }
    partial_sum();
    float tot = 0.f;
    if (tid < NXX)
      for (int r = 0; r < KC; ++r) tot += cl.map_shared_rank(part, r)[tid];
    const bool badt = tid < NXX && !(tot > 0x1p-60f && tot < 0x1p60f);
    if (__syncthreads_or(badt)) {   // same totals in every CTA: a cluster-uniform decision
      partial_max();
      partial_sum();
      tot = 0.f;
      if (tid < NXX)
        for (int r = 0; r < KC; ++r) tot += cl.map_shared_rank(part, r)[tid];
    }
    float epart = 0.f;
    if (tid < NXX) {
      const float kq = (float)(tid / NX);
      const int kk2 = tid % NX;
      const float an = -(__fsub_rn(csh[tid], __fmul_rn(__fmul_rn(w, kq), kq)) + lg2f(tot));   // (c - K) exact
      A2n[tid] = an;
      // L1 X-marginal error (R6'); padded pixels carry mu = 0
      if (MU[tid] > 0.f) epart = MU[tid] * fabsf(exp2m1f(A2[tid] - an) - rm1);
      AL[tid] = an + LM[tid] - w * (float)(kk2 * kk2);
    }
    const float etot = block_sum_f(epart, fred, out.it);
    if (out.it == 1) out.e0 = etot;
    out.e = etot;
    const bool stop = p.fixed_iter > 0 ? (out.it >= p.fixed_iter) : (etot <= tolJ || out.it >= p.max_iter);
    if (stop) break;
    float* tmp = A2; A2 = A2n; A2n = tmp;
    first = false;
    __syncthreads();
  }
  // ---- write back the own rows; the leader writes the X-block ---------------
  for (int t = tid; t < R * b2; t += T) P0g[(size_t)r0 * b2 + t] = B[t];
  for (int t = tid; t < R * b2p; t += T) BKg[(size_t)r0 * b2p + t] = BK[t];
  for (int t = tid; t < R * NX; t += T) {
    Vbg[(size_t)r0 * NX + t] = Vb[t];
    VKg[(size_t)r0 * NX + t] = VK[t];
  }
  if (rank == 0)
    for (int t = tid; t < NXX; t += T) {
      Xg[t] = A2[t];
      Xg[NXX + t] = A2n[t];
    }
  return out;
}

}  // namespace dd
