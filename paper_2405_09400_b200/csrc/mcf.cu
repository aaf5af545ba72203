// mcf.cu — exact min-cost flow on the basic-cell grid graph (flow update
// step 2, §5.1; Eq. MinCostFlow PAPER.md:378-381 with the
// divergence constraints PAPER.md:350-354).
//
// The LP is a transportation problem: sources S_i with supply q_i, sinks T_j
// with demand q_j, arcs S_i -> T_j for j in N(i) (self + 4 neighbours) with
// integer cost C_ij (reading R11).  It is solved exactly on the GPU by
// Goldberg-Tarjan cost scaling with synchronous push/relabel rounds inside ONE
// cooperative persistent kernel (grid-wide barriers, no host round trips):
//   * costs are scaled by SC = 2I + 1 (> number of nodes), so an eps-optimal
//     flow with eps = 1 is optimal;
//   * refine(eps): saturate every residual arc with negative reduced cost,
//     then rounds of {push (prices frozen; each arc pair is touched by at most
//     one endpoint because admissibility is antisymmetric), merge excess,
//     relabel (p(v) = max over residual arcs of p(u) - c(v,u) - eps, computed
//     from the previous round's prices: simultaneous relabels only lower
//     prices and keep eps-optimality)} until no node has excess;
//   * before scaling, a Bellman-Ford negative-cycle test on (I, 4-nbr arcs, C)
//     certifies stationarity (no negative cycle <=> the stationary flow is
//     optimal); near the optimum it passes
//     in one round.
// Every decision depends only on the previous round's state and integer
// atomics commute, so the result is deterministic.
#include <cooperative_groups.h>

#include <cstdlib>
#include <string>

#include "../../include/domdec.h"
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace dd {

struct McfArgs {
  int n1, n2, I;
  const long long* q;     // [I]
  const long long* C;     // [I][5] original integer costs
  long long* w;           // [I][5] flow (output)
  long long* cs;          // [I][5] scaled costs
  long long* eS;          // [I] excess of sources
  long long* eT;          // [I] excess of sinks
  unsigned long long* addS;   // [I] incoming excess of this round (two's complement adds)
  unsigned long long* addT;
  long long* pS[2];       // prices, double-buffered by round parity
  long long* pT[2];
  long long* dist[2];     // Bellman-Ford labels (certificate) / source labels (price update)
  long long* distT[2];    // sink labels (price update)
  unsigned long long* ctr;  // [16] counters
  long long* info;        // [16] results: 0 objective, 1 stationary, 2 certificate, 3 refines, 4 rounds, 6 error
  int bf_rounds;
  int max_rounds;
  int gu_every;           // push/relabel rounds between global price updates
  int tiled;              // 1: checkerboard tile phases instead of grid-wide rounds
  int tile_rounds;        // local rounds per tile phase
  int gu_tiled;           // tile phases between global price updates
  int alpha;              // cost-scaling factor between refine phases
  int bf_sweeps;          // local sweeps per grid round of the tiled Bellman-Ford
  int pr_cap;             // grid rounds allowed to a price refinement (0: 64 + (n1 + n2) / 8)
  // warm start (flow_update of a context): the supplies q are static across
  // flow updates (q_i = m_i 2^E), so the previous optimal flow is feasible
  // for the next instance and its prices are a good start; only the costs
  // change (reading R11)
  int warm;               // 1: start from (wW, wpS, wpT) when *wvalid, and store the result there
  long long warm_div;     // first phase runs at eps = ceil(violation / warm_div)
  long long* wW;          // [I][5] last optimal flow
  long long* wpS;         // [I] its prices (scaled costs)
  long long* wpT;         // [I]
  long long* wvalid;      // [1]
  // stationarity certificate warm start: the labels of the last certificate
  // that converged are a feasible potential d (d_j <= d_i + C_ij on every
  // 4-neighbour arc).  If they still are for the new costs, the stationary
  // flow is certified optimal in one pass; otherwise the Bellman-Ford starts
  // from them (any finite start converges to a feasible potential iff there
  // is no negative cycle), which near the optimum takes a few rounds instead
  // of O(n1 + n2).
  long long* certd;       // [I]
  long long* cvalid;      // [1]
};

__device__ __forceinline__ int nbr(int i, int a, int n1, int n2) {
  const int i1 = i / n2, i2 = i - (i / n2) * n2;
  switch (a) {
    case 0: return i;
    case 1: return i1 > 0 ? i - n2 : -1;
    case 2: return i1 + 1 < n1 ? i + n2 : -1;
    case 3: return i2 > 0 ? i - 1 : -1;
    default: return i2 + 1 < n2 ? i + 1 : -1;
  }
}

// incoming arc k (0..4) of sink T_j: source index and its arc number
__device__ __forceinline__ int in_arc(int j, int k, int n1, int n2, int* a_out) {
  const int j1 = j / n2, j2 = j - (j / n2) * n2;
  switch (k) {
    case 0: *a_out = 0; return j;
    case 1: *a_out = 2; return j1 > 0 ? j - n2 : -1;       // from up, its 'down' arc
    case 2: *a_out = 1; return j1 + 1 < n1 ? j + n2 : -1;  // from down, its 'up' arc
    case 3: *a_out = 4; return j2 > 0 ? j - 1 : -1;        // from left, its 'right' arc
    default: *a_out = 3; return j2 + 1 < n2 ? j + 1 : -1;  // from right, its 'left' arc
  }
}

constexpr long long kInf = (1LL << 60);

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ long long floor_div(long long a, long long b) {   // b > 0
  long long q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}

// ---------------------------------------------------------------------------
// Tiled Bellman-Ford.  All label computations of the solver (certificate,
// global price update, price refinement) are shortest-path fixpoints, which
// are unique whatever the relaxation order, so they run as chaotic
// relaxation: each CTA owns a TH x TW tile of cells (both nodes S_i and T_i of
// a cell), keeps the tile's labels plus a one-cell halo in shared memory,
// precomputes its arc lengths in registers and relaxes in place for up to
// kSweeps local sweeps (block barriers only) before one grid-wide barrier.
// Labels only decrease and are always lengths of real paths, so the result
// equals synchronous Bellman-Ford; a grid round in which no tile changed a
// label proves the fixpoint.  Paths cross a tile in one grid round instead of
// one hop per round.
//   mode 0 (price update): d(v) = distance from v to a deficit node along
//     residual arcs v -> u with l = max(0, floor(c_p/eps) + 1);
//   mode 1 (price refinement): d(u) = distance from a virtual source (0 at
//     every node) along residual arcs v -> u with l = c_p + epsT;
//   mode 2 (certificate): one node per cell, d(j) over the 4-neighbour arcs
//     i -> j with the integer costs C (no negative cycle <=> converges).
// tile height: 8 x 32 cells per CTA (at 1024^2: 256 tiles, 128 working per
// checkerboard phase on 148 SMs) — 4.5% faster warm solves than 16 x 32
// (128 tiles, 64 working per phase) and 16% faster than 4 x 32 on the bench
// trajectory (profiles/r02_mcf_experiments.txt)
#ifndef DD_MCF_TH
#define DD_MCF_TH 8
#endif
constexpr int TH = DD_MCF_TH, TW = 32, TP = TW + 2, kSweeps = 16;   // (sweeps per grid round: tuned on the bench trajectory, tools/mcf_knobs.py)

__device__ __noinline__ bool tiled_bf(const McfArgs& A, cg::grid_group& grid, const int mode, const int par, const long long eps,
                         const int cap, long long gt, long long gs, int* rounds_used) {
  const int n1 = A.n1, n2 = A.n2, I = A.I;
  const long long* pS = A.pS[par];
  const long long* pT = A.pT[par];
  long long* dS = A.dist[0];
  long long* dT = A.distT[0];
  __shared__ long long sS[(TH + 2) * TP], sT[(TH + 2) * TP];
  const int nt2 = (n2 + TW - 1) / TW, ntiles = ((n1 + TH - 1) / TH) * nt2;
  const int ty = threadIdx.x / TW, tx = threadIdx.x % TW;
  const int offs[5] = {0, -TP, TP, -1, 1};   // self, up, down, left, right (arc order of nbr / in_arc)
  for (long long i = gt; i < I; i += gs) {
    if (mode == 0) {
      dS[i] = A.eS[i] < 0 ? 0 : kInf;
      dT[i] = A.eT[i] < 0 ? 0 : kInf;
    } else {
      dS[i] = (mode == 2 && A.warm && *A.cvalid) ? A.certd[i] : 0;
      dT[i] = mode == 1 ? 0 : kInf;
    }
  }
  if (gt == 0) { A.ctr[10] = 0; A.ctr[11] = 0; A.ctr[12] = 0; }
  grid.sync();
  // One tile per CTA (the usual case): arc lengths stay in registers and the
  // tile interior stays in shared memory across grid rounds (only this CTA
  // writes it); only the halo is re-read.  Otherwise CTAs loop over tiles and
  // reload everything per tile.
  const bool single = ntiles <= (int)gridDim.x;
  long long LS[5], LT[5];
  bool conv = false;
  int r = 0;
  for (; r < cap; ++r) {
    if (gt == 0) A.ctr[10 + (r + 1) % 3] = 0;
    bool changed_any = false;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int r0 = (tile / nt2) * TH, c0 = (tile % nt2) * TW;
      const bool full = !single || r == 0;
      for (int e = threadIdx.x; e < (TH + 2) * TP; e += blockDim.x) {
        const int ey = e / TP, ex = e % TP;
        if (!full && ey > 0 && ey < TH + 1 && ex > 0 && ex < TP - 1) continue;   // interior kept
        const int y = ey - 1 + r0, x = ex - 1 + c0;
        long long vs = kInf, vt = kInf;
        if (y >= 0 && y < n1 && x >= 0 && x < n2) {
          const long long g = (long long)y * n2 + x;
          vs = __ldcg(dS + g);
          vt = __ldcg(dT + g);
        }
        sS[e] = vs;
        sT[e] = vt;
      }
      const int y = r0 + ty, x = c0 + tx;
      const bool mine = y < n1 && x < n2;
      const long long i = (long long)y * n2 + x;
      if (full) {
#pragma unroll
        for (int a = 0; a < 5; ++a) { LS[a] = kInf; LT[a] = kInf; }
        if (mine) {
#pragma unroll
          for (int a = 0; a < 5; ++a) {
            const int j = nbr((int)i, a, n1, n2);
            if (j >= 0) {
              if (mode == 0) {
                if (A.q[i] - A.w[5 * i + a] > 0) {
                  long long l = floor_div(A.cs[5 * i + a] + pS[i] - pT[j], eps) + 1;
                  LS[a] = l < 0 ? 0 : (l > (1LL << 40) ? (1LL << 40) : l);
                }
              } else if (mode == 1) {
                if (A.w[5 * i + a] > 0) LS[a] = -(A.cs[5 * i + a] + pS[i] - pT[j]) + eps;
              }
            }
            int b;
            const int src = in_arc((int)i, a, n1, n2, &b);
            if (src >= 0) {
              if (mode == 0) {
                if (A.w[5LL * src + b] > 0) {
                  long long l = floor_div(-(A.cs[5LL * src + b] + pS[src] - pT[i]), eps) + 1;
                  LT[a] = l < 0 ? 0 : (l > (1LL << 40) ? (1LL << 40) : l);
                }
              } else if (mode == 1) {
                if (A.q[src] - A.w[5LL * src + b] > 0) LT[a] = A.cs[5LL * src + b] + pS[src] - pT[i] + eps;
              } else if (a > 0) {
                LS[a] = A.C[5LL * src + b];   // certificate: arc src -> i, label of S only
              }
            }
          }
        }
      }
      __syncthreads();
      const int c = (ty + 1) * TP + tx + 1;
      bool ch_tile = false;
      for (int sw = 0; sw < A.bf_sweeps; ++sw) {
        bool ch = false;
        if (mine) {
          long long bs = sS[c], bt = sT[c];
#pragma unroll
          for (int a = 0; a < 5; ++a) {
            if (LS[a] < kInf) {
              const long long u = mode == 2 ? sS[c + offs[a]] : sT[c + offs[a]];
              if (u < kInf && u + LS[a] < bs) bs = u + LS[a];
            }
            if (LT[a] < kInf) {
              const long long u = sS[c + offs[a]];
              if (u < kInf && u + LT[a] < bt) bt = u + LT[a];
            }
          }
          if (bs < sS[c]) { sS[c] = bs; ch = true; }
          if (bt < sT[c]) { sT[c] = bt; ch = true; }
        }
        if (!__syncthreads_or(ch)) break;
        ch_tile = true;
      }
      if (mine && ch_tile) {
        dS[i] = sS[c];
        dT[i] = sT[c];
      }
      changed_any |= ch_tile;
      __syncthreads();
    }
    if (threadIdx.x == 0 && changed_any) atomicAdd(&A.ctr[10 + r % 3], 1ull);
    grid.sync();
    if (A.ctr[10 + r % 3] == 0) { conv = true; ++r; break; }
  }
  *rounds_used = r;
  // every CTA must have read the last round's counter before anyone reuses
  // ctr[10..12] (a following call resets them)
  grid.sync();
  if (gt == 0) A.ctr[14] += r;
  return conv;
}

// Global price update (Goldberg's set-relabel): d(v) = length of the
// shortest residual path from v to a deficit node with arc lengths
// l(v,u) = floor(c_p(v,u)/eps) + 1; then p(v) -= eps * d(v).  Keeps
// eps-optimality and makes every shortest path admissible.  Applied only if
// the labels converged within the round cap.  Uniform control flow.
__device__ void price_update(const McfArgs& A, cg::grid_group& grid, int par, long long eps, long long gt,
                             long long gs, int cap_rounds) {
  const int I = A.I;
  int r = 0;
  if (gt == 0) A.ctr[13] = 0;
  const bool conv = tiled_bf(A, grid, 0, par, eps, cap_rounds, gt, gs, &r);
  if (!conv) return;
  long long* pS = A.pS[par];
  long long* pT = A.pT[par];
  const long long* dS = A.dist[0];
  const long long* dT = A.distT[0];
  for (long long i = gt; i < I; i += gs) {
    if (dS[i] < kInf) atomicMax(&A.ctr[13], (unsigned long long)dS[i]);
    if (dT[i] < kInf) atomicMax(&A.ctr[13], (unsigned long long)dT[i]);
  }
  grid.sync();
  const long long Dmax = (long long)A.ctr[13];
  for (long long i = gt; i < I; i += gs) {
    const long long a = dS[i] < kInf ? dS[i] : Dmax;
    const long long b = dT[i] < kInf ? dT[i] : Dmax;
    pS[i] -= eps * a;
    pT[i] -= eps * b;
  }
  grid.sync();
}

// Price refinement (Goldberg's CS2 heuristic): if the current flow admits
// prices that make it epsT-optimal (no residual cycle of mean reduced cost
// < -epsT), Bellman-Ford from a virtual source (d = 0 at every node) with
// arc lengths c_p(v,u) + epsT converges and p += d achieves it; otherwise the
// labels keep decreasing and the cap stops the attempt with the prices
// unchanged.  With epsT = 1 on costs scaled by SC = 2I + 1 a success proves
// the current flow optimal.  Uniform control flow.
__device__ bool price_refine(const McfArgs& A, cg::grid_group& grid, int par, long long epsT, long long gt,
                             long long gs, int cap_rounds) {
  const int I = A.I;
  int r = 0;
  if (!tiled_bf(A, grid, 1, par, epsT, cap_rounds, gt, gs, &r)) return false;
  long long* pS = A.pS[par];
  long long* pT = A.pT[par];
  for (long long i = gt; i < I; i += gs) {
    pS[i] += A.dist[0][i];
    pT[i] += A.distT[0][i];
  }
  grid.sync();
  return true;
}

// ---------------------------------------------------------------------------
// Checkerboard tile discharge.  The cell grid is cut into TH x TW tiles
// coloured like a checkerboard; edge-adjacent tiles have different colours
// and every arc joins edge-adjacent (or equal) cells, so while the tiles of
// one colour work, the nodes, prices and incident arcs they touch are touched
// by no other working tile.  A working tile runs up to R synchronous
// push / merge+relabel rounds (the same rounds as the grid-wide loop) on its
// own nodes with block barriers only; neighbours outside the tile are frozen:
// their prices are read once, pushes into them go to their global excess
// (atomics), and the arcs between a working and a frozen tile are written by
// the working side only.  Every operation is therefore a valid push or
// relabel of the generic algorithm and eps-optimality is kept exactly as in
// the grid-wide rounds; one grid barrier per colour phase instead of two per
// round.
struct TileSmem {
  long long *pSa, *pTa, *pSb, *pTb;   // prices with halo, two buffers [(TH + 2) * TP]
  long long *w;                       // [TH * TW][5] out-arc flows of the tile's sources
  long long *cin;                     // [TH * TW][5] scaled costs of the sinks' in-arcs
  long long *win;                     // [TH * TW][5] flows of in-arcs from sources outside the tile
  long long *eS, *eT, *addS, *addT;   // [TH * TW]
};

__device__ __forceinline__ TileSmem tile_smem(unsigned char* base) {
  TileSmem t;
  long long* p = (long long*)base;
  const int H = (TH + 2) * TP, C = TH * TW;
  t.pSa = p; p += H;
  t.pTa = p; p += H;
  t.pSb = p; p += H;
  t.pTb = p; p += H;
  t.w = p; p += 5 * C;
  t.cin = p; p += 5 * C;
  t.win = p; p += 5 * C;
  t.eS = p; p += C;
  t.eT = p; p += C;
  t.addS = p; p += C;
  t.addT = p; p += C;
  return t;
}
constexpr size_t kTileSmemBytes = sizeof(long long) * (4 * (TH + 2) * TP + 19 * TH * TW);

// returns the number of local rounds run (block-uniform)
__device__ __noinline__ int tile_discharge(const McfArgs& A, const int tile, const int par, const long long eps, const int R,
                              unsigned char* smem_raw) {
  const int n1 = A.n1, n2 = A.n2;
  TileSmem S = tile_smem(smem_raw);
  const int nt2 = (n2 + TW - 1) / TW;
  const int r0 = (tile / nt2) * TH, c0 = (tile % nt2) * TW;
  const int t = threadIdx.x, ty = t / TW, tx = t % TW;
  const long long* gpS = A.pS[par];
  const long long* gpT = A.pT[par];
  for (int e = t; e < (TH + 2) * TP; e += blockDim.x) {
    const int y = e / TP - 1 + r0, x = e % TP - 1 + c0;
    long long vs = 0, vt = 0;
    if (y >= 0 && y < n1 && x >= 0 && x < n2) {
      const long long g = (long long)y * n2 + x;
      vs = __ldcg(gpS + g);
      vt = __ldcg(gpT + g);
    }
    S.pSa[e] = vs; S.pTa[e] = vt; S.pSb[e] = vs; S.pTb[e] = vt;
  }
  const int y = r0 + ty, x = c0 + tx;
  const bool mine = y < n1 && x < n2;
  const long long i = (long long)y * n2 + x;
  const int c = (ty + 1) * TP + tx + 1;
  const int offs[5] = {0, -TP, TP, -1, 1};
  const int toff[5] = {0, -TW, TW, -1, 1};
  long long qi = 0, csr[5];
  bool inS[5];   // neighbour cell of arc a lies inside the tile
#pragma unroll
  for (int a = 0; a < 5; ++a) {
    csr[a] = 0;
    const int yy = ty + (a == 1 ? -1 : a == 2 ? 1 : 0), xx = tx + (a == 3 ? -1 : a == 4 ? 1 : 0);
    inS[a] = yy >= 0 && yy < TH && xx >= 0 && xx < TW && r0 + yy < n1 && c0 + xx < n2;
  }
  if (mine) {
    qi = A.q[i];
#pragma unroll
    for (int a = 0; a < 5; ++a) {
      csr[a] = A.cs[5 * i + a];
      S.w[5 * t + a] = __ldcg(A.w + 5 * i + a);
    }
    S.eS[t] = __ldcg(A.eS + i);
    S.eT[t] = __ldcg(A.eT + i);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      int b;
      const int src = in_arc((int)i, k, n1, n2, &b);
      S.cin[5 * t + k] = src >= 0 ? A.cs[5LL * src + b] : 0;
      S.win[5 * t + k] = (src >= 0 && !inS[k]) ? __ldcg(A.w + 5LL * src + b) : 0;
    }
  } else {
    S.eS[t] = 0;
    S.eT[t] = 0;
  }
  S.addS[t] = 0;
  S.addT[t] = 0;
  __syncthreads();
  long long *pS = S.pSa, *pT = S.pTa, *pSn = S.pSb, *pTn = S.pTb;
  int rr = 0;
  for (; rr < R; ++rr) {
    // phase A: push (prices frozen)
    if (mine) {
      long long e = S.eS[t];
      if (e > 0) {
        for (int a = 0; a < 5 && e > 0; ++a) {
          const int j = nbr((int)i, a, n1, n2);
          if (j < 0) continue;
          const long long r = qi - S.w[5 * t + a];
          if (r <= 0) continue;
          if (csr[a] + pS[c] - pT[c + offs[a]] < 0) {
            const long long d = e < r ? e : r;
            S.w[5 * t + a] += d;
            e -= d;
            if (inS[a]) atomicAdd((unsigned long long*)&S.addT[t + toff[a]], (unsigned long long)d);
            else atomicAdd((unsigned long long*)&A.eT[j], (unsigned long long)d);
          }
        }
        S.eS[t] = e;
      }
      long long f = S.eT[t];
      if (f > 0) {
        for (int k = 0; k < 5 && f > 0; ++k) {
          int b;
          const int src = in_arc((int)i, k, n1, n2, &b);
          if (src < 0) continue;
          long long* wp = inS[k] ? &S.w[5 * (t + toff[k]) + b] : &S.win[5 * t + k];
          const long long r = *wp;
          if (r <= 0) continue;
          if (S.cin[5 * t + k] + pS[c + offs[k]] - pT[c] > 0) {   // reverse arc admissible
            const long long d = f < r ? f : r;
            *wp = r - d;
            f -= d;
            if (inS[k]) atomicAdd((unsigned long long*)&S.addS[t + toff[k]], (unsigned long long)d);
            else atomicAdd((unsigned long long*)&A.eS[src], (unsigned long long)d);
          }
        }
        S.eT[t] = f;
      }
    }
    __syncthreads();
    // phase B: merge, relabel active nodes without admissible arcs (from the
    // frozen prices of this round), count
    bool act = false;
    long long ps = pS[c], pt = pT[c];
    if (mine) {
      const long long es = S.eS[t] + S.addS[t];
      const long long et = S.eT[t] + S.addT[t];
      S.addS[t] = 0;
      S.addT[t] = 0;
      S.eS[t] = es;
      S.eT[t] = et;
      if (es > 0) {
        act = true;
        bool adm = false;
        long long best = LLONG_MIN;
        for (int a = 0; a < 5; ++a) {
          if (nbr((int)i, a, n1, n2) < 0) continue;
          if (qi - S.w[5 * t + a] <= 0) continue;
          const long long cp = csr[a] + pS[c] - pT[c + offs[a]];
          if (cp < 0) { adm = true; break; }
          const long long cand = pT[c + offs[a]] - csr[a];
          if (cand > best) best = cand;
        }
        if (!adm && best != LLONG_MIN) ps = best - eps;
      }
      if (et > 0) {
        act = true;
        bool adm = false;
        long long best = LLONG_MIN;
        for (int k = 0; k < 5; ++k) {
          int b;
          const int src = in_arc((int)i, k, n1, n2, &b);
          if (src < 0) continue;
          const long long wv = inS[k] ? S.w[5 * (t + toff[k]) + b] : S.win[5 * t + k];
          if (wv <= 0) continue;
          const long long cs = S.cin[5 * t + k];
          const long long cp = cs + pS[c + offs[k]] - pT[c];
          if (cp > 0) { adm = true; break; }
          const long long cand = pS[c + offs[k]] + cs;
          if (cand > best) best = cand;
        }
        if (!adm && best != LLONG_MIN) pt = best - eps;
      }
    }
    pSn[c] = ps;
    pTn[c] = pt;
    const int nact = __syncthreads_count(act);
    long long* tmp = pS; pS = pSn; pSn = tmp;
    tmp = pT; pT = pTn; pTn = tmp;
    if (nact == 0) { ++rr; break; }
  }
  // write back (no other working tile touches these nodes or arcs)
  if (mine) {
    A.pS[par][i] = pS[c];
    A.pT[par][i] = pT[c];
    A.eS[i] = S.eS[t];
    A.eT[i] = S.eT[t];
#pragma unroll
    for (int a = 0; a < 5; ++a) A.w[5 * i + a] = S.w[5 * t + a];
#pragma unroll
    for (int k = 1; k < 5; ++k) {
      if (inS[k]) continue;
      int b;
      const int src = in_arc((int)i, k, n1, n2, &b);
      if (src >= 0) A.w[5LL * src + b] = S.win[5 * t + k];
    }
  }
  __syncthreads();
  return rr;
}

__global__ void __launch_bounds__(512, 1) mcf_kernel(McfArgs A) {
  extern __shared__ __align__(16) unsigned char dsmem[];
  long long local_rounds = 0;
  unsigned long long tm_refine = 0, tm_update = 0, tm_phase = 0, tm_wait = 0;
  const unsigned long long tm_start = gtimer();
  cg::grid_group grid = cg::this_grid();
  const int n1 = A.n1, n2 = A.n2, I = A.I;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gs = (long long)gridDim.x * blockDim.x;
  const long long SC = 2LL * I + 1;

  // ---- init: stationary flow, scaled costs, max |C| -------------------------
  const bool warm = A.warm && *A.wvalid;
  const bool cwarm = A.warm && *A.cvalid;
  for (long long i = gt; i < I; i += gs) {
    for (int a = 0; a < 5; ++a) {
      const int j = nbr((int)i, a, n1, n2);
      A.w[5 * i + a] = warm ? A.wW[5 * i + a] : ((a == 0) ? A.q[i] : 0);
      const long long c = (j >= 0 && a > 0) ? A.C[5 * i + a] : 0;
      A.cs[5 * i + a] = c * SC;
      if (j >= 0 && a > 0) {
        const unsigned long long ab = (unsigned long long)(c < 0 ? -c : c);
        atomicMax(&A.ctr[0], ab);
        if (c < 0) atomicAdd(&A.ctr[1], 1ull);
        if (cwarm && c + A.certd[i] - A.certd[j] < 0) atomicAdd(&A.ctr[2], 1ull);
      }
    }
    A.dist[0][i] = 0;
    A.pS[0][i] = warm ? A.wpS[i] : 0;
    A.pT[0][i] = warm ? A.wpT[i] : 0;
    A.eS[i] = 0;
    A.eT[i] = 0;
    A.addS[i] = 0;
    A.addT[i] = 0;
  }
  grid.sync();
  // The stationary flow (w_ii = q_i) is the result of every early exit: A.w
  // holds the warm flow at this point and must not be applied again.
  // The certificate's labels d (d_j <= d_i + C_ij on every 4-neighbour arc;
  // d = 0 when no cost is negative) price the stationary flow optimally:
  // with p_S = p_T = SC d every arc has reduced cost SC (C_ij + d_i - d_j) >= 0
  // and the self arcs 0.  A warm context keeps that pair, so the next
  // non-stationary update starts from the optimum of this instance instead
  // of the last moving flow, however old.
  auto stationary_exit = [&](int bf_rounds, const long long* labels) {
    for (long long i = gt; i < I; i += gs) {
      for (int a = 0; a < 5; ++a) A.w[5 * i + a] = (a == 0) ? A.q[i] : 0;
      if (A.warm) {
        for (int a = 0; a < 5; ++a) A.wW[5 * i + a] = (a == 0) ? A.q[i] : 0;
        const long long pr = labels ? labels[i] * SC : 0;
        A.wpS[i] = pr;
        A.wpT[i] = pr;
      }
    }
    if (A.warm && gt == 0) *A.wvalid = 1;
    if (gt == 0) {
      A.info[0] = 0; A.info[1] = 1; A.info[2] = 1; A.info[3] = 0; A.info[4] = 0; A.info[5] = bf_rounds;
      A.info[6] = 0; A.info[12] = (long long)(gtimer() - tm_start);
    }
  };
  const bool any_negative = A.ctr[1] > 0;
  // no negative arc cost, or the last certificate's labels are still a
  // feasible potential: no negative cycle, the stationary flow is optimal
  if (!any_negative || (cwarm && A.ctr[2] == 0)) {
    stationary_exit(0, any_negative ? A.certd : nullptr);
    return;
  }
  // ---- Bellman-Ford certificate on (I, 4-nbr arcs, C) -----------------------
  // Warm-started updates get a short certificate: near the optimum (the only
  // case where it passes) it converges within a few rounds (all C_ij >= 0
  // passes in one); a failing certificate otherwise runs to
  // its cap (~2(n1+n2) rounds at ~26 us each) before cost scaling starts.
  // Exactness is unaffected: a certificate that does not converge only
  // means that cost scaling decides.
  int rb = 0;
  const int cert_cap = warm ? (A.bf_rounds < 64 ? A.bf_rounds : 64) : A.bf_rounds;
  const int cert = tiled_bf(A, grid, 2, 0, 0, cert_cap, gt, gs, &rb) ? 1 : 0;
  if (cert) {
    if (A.warm) {   // keep the labels (a feasible potential) for the next certificate
      for (long long i = gt; i < I; i += gs) A.certd[i] = A.dist[0][i];
      if (gt == 0) *A.cvalid = 1;
    }
    stationary_exit(rb, A.warm ? A.certd : nullptr);
    return;
  }
  // ---- cost scaling -----------------------------------------------------------
  long long eps = (long long)A.ctr[0] * SC;
  long long warm_eps = 0;
  if (warm) {
    // smallest eps for which the warm (flow, prices) pair is eps-optimal
    for (long long i = gt; i < I; i += gs) {
      for (int a = 1; a < 5; ++a) {
        const int j = nbr((int)i, a, n1, n2);
        if (j < 0) continue;
        const long long cp = A.cs[5 * i + a] + A.pS[0][i] - A.pT[0][j];
        unsigned long long v = 0;
        if (A.q[i] - A.w[5 * i + a] > 0 && cp < 0) v = (unsigned long long)(-cp);
        if (A.w[5 * i + a] > 0 && cp > 0 && (unsigned long long)cp > v) v = (unsigned long long)cp;
        if (v) atomicMax(&A.ctr[15], v);
      }
    }
    grid.sync();
    const long long viol = (long long)A.ctr[15];
    warm_eps = (viol + A.warm_div - 1) / A.warm_div;
    if (warm_eps < 1) warm_eps = 1;
  }
  bool first_phase = true;
  int refines = 0, rounds = 0, par = 0;
  // a feasible refinement converges in a few dozen tiled rounds; a failing one
  // runs to the cap, so keep it small
  const int pr_cap = A.pr_cap > 0 ? A.pr_cap : 64 + (n1 + n2) / 8;
  bool failed = false;
  while (eps >= 1 && !failed) {
    if (first_phase && warm) {
      eps = warm_eps;
    } else {
      eps = (eps + A.alpha - 1) / A.alpha;   // cost-scaling factor
      if (eps < 1) eps = 1;
    }
    first_phase = false;
    ++refines;
    // price refinement: after the first phase the flow is often already
    // optimal (degenerate instances) or eps-optimal for the next eps; then
    // the phase is skipped instead of rebuilt from saturated arcs
    if (refines > 1) {
      const unsigned long long t0 = gtimer();
      const bool opt = price_refine(A, grid, par, 1, gt, gs, pr_cap);
      tm_refine += gtimer() - t0;
      if (opt) break;
      const unsigned long long t1 = gtimer();
      const bool ok = price_refine(A, grid, par, eps, gt, gs, pr_cap);
      tm_refine += gtimer() - t1;
      if (ok) {
        if (eps == 1) break;
        continue;
      }
    }
    const long long* pSo = A.pS[par];
    const long long* pTo = A.pT[par];
    // saturate arcs with negative reduced cost (both directions)
    for (long long i = gt; i < I; i += gs) {
      for (int a = 0; a < 5; ++a) {
        const int j = nbr((int)i, a, n1, n2);
        if (j < 0) continue;
        const long long cp = A.cs[5 * i + a] + pSo[i] - pTo[j];
        if (cp < 0) A.w[5 * i + a] = A.q[i];
        else if (cp > 0) A.w[5 * i + a] = 0;
      }
    }
    grid.sync();
    for (long long i = gt; i < I; i += gs) {
      long long out = 0;
      for (int a = 0; a < 5; ++a) out += A.w[5 * i + a];
      A.eS[i] = A.q[i] - out;
      long long in = 0;
      for (int k = 0; k < 5; ++k) {
        int a;
        const int src = in_arc((int)i, k, n1, n2, &a);
        if (src >= 0) in += A.w[5LL * src + a];
      }
      A.eT[i] = in - A.q[i];
    }
    grid.sync();
    const int gu_every = A.gu_every;
    const int gu_cap = 8 * (n1 + n2) + 256;
    price_update(A, grid, par, eps, gt, gs, gu_cap);
    int since_gu = 0;
    if (A.tiled) {
      // checkerboard tile phases (see tile_discharge); one grid barrier per
      // phase.  The active-node count taken at the start of phase g is read
      // at the start of phase g + 1: zero means phase g had nothing to do.
      const int nt2 = (n2 + TW - 1) / TW, ntiles = ((n1 + TH - 1) / TH) * nt2;
      for (int g = 0;; ++g) {
        if (g > 0 && A.ctr[5 + (g - 1) % 3] == 0) break;
        if (rounds >= A.max_rounds) { failed = true; break; }
        ++rounds;
        if (++since_gu >= A.gu_tiled) {
          since_gu = 0;
          const unsigned long long t0 = gtimer();
          price_update(A, grid, par, eps, gt, gs, gu_cap);
          tm_update += gtimer() - t0;
        }
        const unsigned long long t2 = gtimer();
        if (gt == 0) A.ctr[5 + (g + 1) % 3] = 0;
        unsigned int act = 0;
        for (long long i = gt; i < I; i += gs) act += (A.eS[i] > 0) + (A.eT[i] > 0);
        act = __reduce_add_sync(0xffffffffu, act);
        if ((threadIdx.x & 31) == 0 && act) atomicAdd(&A.ctr[5 + g % 3], (unsigned long long)act);
        grid.sync();   // counts complete, and no tile starts before every count has read the state
        if (A.ctr[5 + g % 3] != 0) {
          const int color = g & 1;
          for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            if ((((tile / nt2) + (tile % nt2)) & 1) != color) continue;
            local_rounds += tile_discharge(A, tile, par, eps, A.tile_rounds, dsmem);
          }
        }
        const unsigned long long t3 = gtimer();
        grid.sync();
        tm_phase += t3 - t2;
        tm_wait += gtimer() - t3;
      }
      if (eps == 1) break;
      continue;
    }
    for (;;) {
      if (rounds >= A.max_rounds) { failed = true; break; }
      ++rounds;
      if (++since_gu >= gu_every) {
        since_gu = 0;
        price_update(A, grid, par, eps, gt, gs, gu_cap);
      }
      const long long* pS = A.pS[par];
      const long long* pT = A.pT[par];
      long long* pSn = A.pS[par ^ 1];
      long long* pTn = A.pT[par ^ 1];
      if (gt == 0) A.ctr[5 + (rounds + 1) % 3] = 0;   // counter of the next round
      // phase A: push (prices frozen)
      for (long long i = gt; i < I; i += gs) {
        long long e = A.eS[i];
        if (e > 0) {
          for (int a = 0; a < 5 && e > 0; ++a) {
            const int j = nbr((int)i, a, n1, n2);
            if (j < 0) continue;
            const long long r = A.q[i] - A.w[5 * i + a];
            if (r <= 0) continue;
            if (A.cs[5 * i + a] + pS[i] - pT[j] < 0) {
              const long long d = e < r ? e : r;
              A.w[5 * i + a] += d;
              e -= d;
              atomicAdd(&A.addT[j], (unsigned long long)d);
            }
          }
          A.eS[i] = e;
        }
        long long f = A.eT[i];
        if (f > 0) {
          for (int k = 0; k < 5 && f > 0; ++k) {
            int a;
            const int src = in_arc((int)i, k, n1, n2, &a);
            if (src < 0) continue;
            const long long r = A.w[5LL * src + a];
            if (r <= 0) continue;
            if (A.cs[5LL * src + a] + pS[src] - pT[i] > 0) {   // reverse arc has negative reduced cost
              const long long d = f < r ? f : r;
              A.w[5LL * src + a] -= d;
              f -= d;
              atomicAdd(&A.addS[src], (unsigned long long)d);
            }
          }
          A.eT[i] = f;
        }
      }
      grid.sync();
      // phase B: merge incoming excess, count active nodes, relabel the
      // active nodes without admissible arcs (new prices from the frozen ones)
      unsigned int act = 0;
      for (long long i = gt; i < I; i += gs) {
        const long long es = A.eS[i] + (long long)A.addS[i];
        const long long et = A.eT[i] + (long long)A.addT[i];
        A.addS[i] = 0;
        A.addT[i] = 0;
        A.eS[i] = es;
        A.eT[i] = et;
        long long ps = pS[i];
        if (es > 0) {
          ++act;
          bool adm = false;
          long long best = LLONG_MIN;
          for (int a = 0; a < 5; ++a) {
            const int j = nbr((int)i, a, n1, n2);
            if (j < 0) continue;
            if (A.q[i] - A.w[5 * i + a] <= 0) continue;
            const long long cp = A.cs[5 * i + a] + pS[i] - pT[j];
            if (cp < 0) { adm = true; break; }
            const long long cand = pT[j] - A.cs[5 * i + a];
            if (cand > best) best = cand;
          }
          if (!adm && best != LLONG_MIN) ps = best - eps;
        }
        pSn[i] = ps;
        long long pt = pT[i];
        if (et > 0) {
          ++act;
          bool adm = false;
          long long best = LLONG_MIN;
          for (int k = 0; k < 5; ++k) {
            int a;
            const int src = in_arc((int)i, k, n1, n2, &a);
            if (src < 0) continue;
            if (A.w[5LL * src + a] <= 0) continue;
            const long long cp = A.cs[5LL * src + a] + pS[src] - pT[i];
            if (cp > 0) { adm = true; break; }
            const long long cand = pS[src] + A.cs[5LL * src + a];
            if (cand > best) best = cand;
          }
          if (!adm && best != LLONG_MIN) pt = best - eps;
        }
        pTn[i] = pt;
      }
      act = __reduce_add_sync(0xffffffffu, act);
      if ((threadIdx.x & 31) == 0 && act) atomicAdd(&A.ctr[5 + rounds % 3], (unsigned long long)act);
      grid.sync();
      par ^= 1;
      if (A.ctr[5 + rounds % 3] == 0) break;
    }
    if (eps == 1) break;
  }
  // ---- objective (original integer costs) -------------------------------------
  if (gt == 0) A.ctr[8] = 0;
  grid.sync();
  for (long long i = gt; i < I; i += gs) {
    long long acc = 0;
    for (int a = 1; a < 5; ++a)
      if (nbr((int)i, a, n1, n2) >= 0) acc += A.w[5 * i + a] * A.C[5 * i + a];
    atomicAdd(&A.ctr[8], (unsigned long long)acc);
  }
  grid.sync();
  const long long obj = (long long)A.ctr[8];
  if (A.warm && !failed) {   // keep the optimal flow and its prices for the next flow update
    for (long long i = gt; i < I; i += gs) {
      for (int a = 0; a < 5; ++a) A.wW[5 * i + a] = A.w[5 * i + a];
      A.wpS[i] = A.pS[par][i];
      A.wpT[i] = A.pT[par][i];
    }
    if (gt == 0) *A.wvalid = 1;
    grid.sync();
  }
  if (obj >= 0 && !failed) {   // stationary flow is optimal: keep it exactly
    for (long long i = gt; i < I; i += gs)
      for (int a = 0; a < 5; ++a) A.w[5 * i + a] = (a == 0) ? A.q[i] : 0;
  }
  if (gt == 0) {
    A.info[0] = obj >= 0 ? 0 : obj;
    A.info[1] = obj >= 0 ? 1 : 0;
    A.info[2] = 0;
    A.info[3] = refines;
    A.info[4] = rounds;
    A.info[5] = (long long)A.ctr[14];
    A.info[7] = local_rounds;   // thread 0's CTA only (diagnostic)
    A.info[8] = (long long)tm_refine;   // ns, thread 0 (diagnostic timers)
    A.info[9] = (long long)tm_update;
    A.info[10] = (long long)tm_phase;
    A.info[11] = (long long)tm_wait;
    A.info[12] = (long long)(gtimer() - tm_start);
    A.info[6] = failed ? 1 : 0;
  }
  if (failed) {
    for (long long i = gt; i < I; i += gs)
      for (int a = 0; a < 5; ++a) A.w[5 * i + a] = (a == 0) ? A.q[i] : 0;
  }
}

static size_t ws_size(int I) {
  // cs, w handled by caller for w; workspace: cs[5I] eS eT addS addT pS0 pS1 pT0 pT1 d0 d1 ctr[16],
  // info[16], warm state wW[5I] wpS[I] wpT[I] wvalid
  return sizeof(long long) * (5ull * I + 12ull * I) + 16 * sizeof(unsigned long long) + 16 * sizeof(long long) +
         sizeof(long long) * (7ull * I + 1) + sizeof(long long) * (I + 1) + 256;
}

dd_status mcf_solve_device(int n1, int n2, const int64_t* d_q, const int64_t* d_C, int64_t* d_w, void** d_ws,
                           size_t* ws_bytes, int warm, cudaStream_t st, std::string& err) {
  const int I = n1 * n2;
  const size_t need = ws_size(I);
  if (*ws_bytes < need) {
    if (*d_ws) cudaFreeAsync(*d_ws, st);
    *d_ws = nullptr;
    if (cudaMallocAsync(d_ws, need, st) != cudaSuccess) {
      err = "mcf workspace allocation failed";
      return DD_ERR_OOM;
    }
    *ws_bytes = need;
    if (cudaMemsetAsync(*d_ws, 0, need, st) != cudaSuccess) {   // warm state invalid
      err = "mcf workspace init failed";
      return DD_ERR_CUDA;
    }
  }
  char* base = (char*)*d_ws;
  McfArgs A;
  A.n1 = n1;
  A.n2 = n2;
  A.I = I;
  A.q = (const long long*)d_q;
  A.C = (const long long*)d_C;
  A.w = (long long*)d_w;
  long long* p = (long long*)base;
  A.cs = p; p += 5LL * I;
  A.eS = p; p += I;
  A.eT = p; p += I;
  A.addS = (unsigned long long*)p; p += I;
  A.addT = (unsigned long long*)p; p += I;
  A.pS[0] = p; p += I;
  A.pS[1] = p; p += I;
  A.pT[0] = p; p += I;
  A.pT[1] = p; p += I;
  A.dist[0] = p; p += I;
  A.dist[1] = p; p += I;
  A.distT[0] = p; p += I;
  A.distT[1] = p; p += I;
  A.ctr = (unsigned long long*)p; p += 16;
  A.info = p; p += 16;
  A.wW = p; p += 5LL * I;
  A.wpS = p; p += I;
  A.wpT = p; p += I;
  A.wvalid = p; p += 1;
  A.certd = p; p += I;
  A.cvalid = p;
  A.warm = warm;
  A.warm_div = 1LL << 40;   // warm start: one eps = 1 phase (tools/mcf_sim.cpp: 3x fewer rounds than cold)
  if (const char* env = getenv("DD_MCF_WDIV")) A.warm_div = atoll(env) > 0 ? atoll(env) : A.warm_div;
  if (const char* env = getenv("DD_MCF_WARM")) A.warm = warm && atoi(env);
  A.bf_rounds = 2 * (n1 + n2) + 8;
  A.max_rounds = 2000000;
  // rounds between global price updates: tuned on dumped flow-update
  // instances (tools/mcf_time.py); DD_MCF_GU overrides (development knob)
  A.gu_every = 50;
  A.tiled = 1;
  A.tile_rounds = 16;
  A.gu_tiled = 8;    // tile phases between global price updates (profiles/r02_mcf_experiments.txt)
  A.alpha = 16;
  A.bf_sweeps = kSweeps;
  A.pr_cap = 0;
  if (const char* env = getenv("DD_MCF_PRCAP")) A.pr_cap = atoi(env);
  if (const char* env = getenv("DD_MCF_ALPHA")) A.alpha = atoi(env) > 1 ? atoi(env) : A.alpha;
  if (const char* env = getenv("DD_MCF_SWEEPS")) A.bf_sweeps = atoi(env) > 0 ? atoi(env) : A.bf_sweeps;
  if (const char* env = getenv("DD_MCF_GU")) A.gu_every = atoi(env) > 0 ? atoi(env) : A.gu_every;
  if (const char* env = getenv("DD_MCF_TILED")) A.tiled = atoi(env);
  if (const char* env = getenv("DD_MCF_MAXR")) A.max_rounds = atoi(env) > 0 ? atoi(env) : A.max_rounds;
  if (const char* env = getenv("DD_MCF_R")) A.tile_rounds = atoi(env) > 0 ? atoi(env) : A.tile_rounds;
  if (const char* env = getenv("DD_MCF_GUT")) A.gu_tiled = atoi(env) > 0 ? atoi(env) : A.gu_tiled;
  cudaError_t e = cudaMemsetAsync(A.ctr, 0, 32 * sizeof(long long), st);
  if (e != cudaSuccess) { err = cudaGetErrorString(e); return DD_ERR_CUDA; }
  int dev = 0;
  cudaGetDevice(&dev);
  int nsm = 0, per = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // one CTA per tile (TH x TW cells, one thread per cell), at most the
  // co-resident CTAs of the device
  const int threads = TH * TW;
  // per-device function attribute: set on every launch (cheap)
  e = cudaFuncSetAttribute(mcf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmemBytes);
  if (e != cudaSuccess) { err = std::string("mcf smem: ") + cudaGetErrorString(e); return DD_ERR_CUDA; }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, mcf_kernel, threads, kTileSmemBytes);
  if (per <= 0) { err = "mcf kernel cannot be resident"; return DD_ERR_CUDA; }
  long long want = (I + threads - 1) / threads;
  long long blocks = (long long)nsm * (TH < 16 ? per : 1);
  if (want < blocks) blocks = want;
  if (blocks < 1) blocks = 1;
  void* args[] = {&A};
  e = cudaLaunchCooperativeKernel((void*)mcf_kernel, dim3((unsigned)blocks), dim3(threads), args, kTileSmemBytes, st);
  if (e != cudaSuccess) { err = std::string("mcf launch: ") + cudaGetErrorString(e); return DD_ERR_CUDA; }
  return DD_OK;
}

long long* mcf_info_ptr(void* ws, int I) {
  char* base = (char*)ws;
  return (long long*)(base + sizeof(long long) * (17ull * I) + 16 * sizeof(unsigned long long));
}

}  // namespace dd
