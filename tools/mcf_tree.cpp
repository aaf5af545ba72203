// mcf_tree.cpp — CPU emulation of cost scaling with "shortest-path forest"
// augmentation (development aid, not part of the library).  Each iteration:
// (1) distances to the nearest deficit in the price-update metric, ties
// broken by hop count (key = d * 2^20 + hops), with parent pointers; (2)
// prices p -= eps * d; (3) excess is routed down the forest in decreasing key
// order, each node forwarding min(accumulated, residual cap) to its parent.
// g++ -O3 -o /tmp/mcf_tree tools/mcf_tree.cpp
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
typedef long long ll;
int n1, n2, I;
std::vector<ll> q, C, w, cs, pS, pT;
inline int nbr(int i, int a) {
  int i1 = i / n2, i2 = i % n2;
  switch (a) { case 0: return i; case 1: return i1 > 0 ? i - n2 : -1; case 2: return i1 + 1 < n1 ? i + n2 : -1;
    case 3: return i2 > 0 ? i - 1 : -1; default: return i2 + 1 < n2 ? i + 1 : -1; }
}
inline int in_arc(int j, int k, int* a) {
  int j1 = j / n2, j2 = j % n2;
  switch (k) { case 0: *a = 0; return j; case 1: *a = 2; return j1 > 0 ? j - n2 : -1;
    case 2: *a = 1; return j1 + 1 < n1 ? j + n2 : -1; case 3: *a = 4; return j2 > 0 ? j - 1 : -1;
    default: *a = 3; return j2 + 1 < n2 ? j + 1 : -1; }
}
const ll kInf = 1LL << 62;
ll fdiv(ll a, ll b) { ll r = a / b; if ((a % b) && a < 0) --r; return r; }
void load(const char* fn) {
  FILE* f = fopen(fn, "rb");
  ll nn[2]; if (fread(nn, 8, 2, f) != 2) exit(1); n1 = nn[0]; n2 = nn[1]; I = n1 * n2;
  q.resize(I); C.resize(5 * I);
  if (fread(q.data(), 8, I, f) != (size_t)I || fread(C.data(), 8, 5 * I, f) != (size_t)5 * I) exit(1);
  fclose(f);
}
// node v < I: S_v ; v >= I: T_{v-I}
std::vector<ll> ex, key, d;
std::vector<int> par, para;  // parent node and arc id (5*i+a), sign via node type
long long bf_rounds_total = 0, iters_total = 0;
void excesses() {
  ex.assign(2 * I, 0);
  for (int i = 0; i < I; ++i) {
    ll out = 0; for (int a = 0; a < 5; ++a) out += w[5 * i + a];
    ex[i] = q[i] - out;
    ll in = 0; for (int k = 0; k < 5; ++k) { int a; int s = in_arc(i, k, &a); if (s >= 0) in += w[5LL * s + a]; }
    ex[I + i] = in - q[i];
  }
}
// lexicographic (d, hops) shortest distances to deficits; synchronous rounds
// counted like the GPU's Bellman-Ford (Jacobi) for a round estimate
#include <queue>
int forest(ll eps) {   // multi-source Dijkstra backwards from the deficits on key = (d << 20) + hops
  key.assign(2 * I, kInf); par.assign(2 * I, -1); para.assign(2 * I, -1);
  typedef std::pair<ll, int> P;
  std::priority_queue<P, std::vector<P>, std::greater<P>> pq;
  for (int v = 0; v < 2 * I; ++v) if (ex[v] < 0) { key[v] = 0; pq.push(P(0, v)); }
  while (!pq.empty()) {
    P t = pq.top(); pq.pop();
    const int u = t.second; if (t.first != key[u]) continue;
    if (u >= I) {             // T_j: residual arcs S_i -> T_j
      const int j = u - I;
      for (int k = 0; k < 5; ++k) { int a; int i = in_arc(j, k, &a); if (i < 0 || q[i] - w[5LL * i + a] <= 0) continue;
        ll cp = cs[5LL * i + a] + pS[i] - pT[j]; ll l = fdiv(cp, eps) + 1; if (l < 0) l = 0;
        ll kk = key[u] + (l << 20) + 1;
        if (kk < key[i]) { key[i] = kk; par[i] = u; para[i] = 5 * i + a; pq.push(P(kk, i)); } }
    } else {                  // S_i: residual arcs T_j -> S_i (reverse of S_i -> T_j with w > 0)
      const int i = u;
      for (int a = 0; a < 5; ++a) { int j = nbr(i, a); if (j < 0 || w[5LL * i + a] <= 0) continue;
        ll cp = cs[5LL * i + a] + pS[i] - pT[j]; ll l = fdiv(-cp, eps) + 1; if (l < 0) l = 0;
        ll kk = key[u] + (l << 20) + 1;
        if (kk < key[I + j]) { key[I + j] = kk; par[I + j] = i; para[I + j] = 5 * i + a; pq.push(P(kk, I + j)); } }
    }
  }
  return 0;
}
#include <deque>
// price refinement: prices making the current flow eps-optimal, if any (SPFA
// from a virtual source, lengths cp + eps on residual arcs; a path longer
// than 2I arcs proves a cycle of mean reduced cost < -eps)
bool refine_prices(ll eps, std::vector<ll>& nS, std::vector<ll>& nT) {
  std::vector<ll> dd(2 * I, 0); std::vector<int> len(2 * I, 0); std::vector<char> inq(2 * I, 1);
  std::deque<int> dq; for (int v = 0; v < 2 * I; ++v) dq.push_back(v);
  while (!dq.empty()) {
    int v = dq.front(); dq.pop_front(); inq[v] = 0;
    if (v < I) {            // S_i -> T_j forward residual
      for (int a = 0; a < 5; ++a) { int j = nbr(v, a); if (j < 0 || q[v] - w[5LL * v + a] <= 0) continue;
        ll l = cs[5LL * v + a] + pS[v] - pT[j] + eps; int u = I + j;
        if (dd[v] + l < dd[u]) { dd[u] = dd[v] + l; len[u] = len[v] + 1; if (len[u] > 2 * I) return false; if (!inq[u]) { inq[u] = 1; dq.push_back(u); } } }
    } else {                // T_j -> S_i reverse residual
      int j = v - I;
      for (int k = 0; k < 5; ++k) { int a; int i = in_arc(j, k, &a); if (i < 0 || w[5LL * i + a] <= 0) continue;
        ll l = -(cs[5LL * i + a] + pS[i] - pT[j]) + eps; int u = i;
        if (dd[v] + l < dd[u]) { dd[u] = dd[v] + l; len[u] = len[v] + 1; if (len[u] > 2 * I) return false; if (!inq[u]) { inq[u] = 1; dq.push_back(u); } } }
    }
  }
  nS.resize(I); nT.resize(I);
  for (int i = 0; i < I; ++i) { nS[i] = pS[i] + dd[i]; nT[i] = pT[i] + dd[I + i]; }
  return true;
}
int main(int argc, char** argv) {
  // usage: mcf_tree alpha warm_alpha inst1.bin [inst2.bin ...] (later instances warm-started)
  const int alpha0 = atoi(argv[1]), walpha = atoi(argv[2]);
  load(argv[3]);
  int alpha = alpha0;
  const ll SC = 2LL * I + 1;
  w.assign(5 * I, 0); pS.assign(I, 0); pT.assign(I, 0); cs.assign(5 * I, 0);
  ll cmax = 0;
  for (int i = 0; i < I; ++i) for (int a = 0; a < 5; ++a) { int j = nbr(i, a); w[5 * i + a] = a == 0 ? q[i] : 0;
    ll c = (j >= 0 && a > 0) ? C[5 * i + a] : 0; cs[5 * i + a] = c * SC; if (j >= 0 && a > 0) cmax = std::max(cmax, std::llabs(c)); }
  bool warm = false;
  for (int inst = 3; inst < argc; ++inst) {
    if (inst > 3) {
      load(argv[inst]);
      for (int i = 0; i < I; ++i) for (int a = 0; a < 5; ++a) { int j = nbr(i, a);
        cs[5 * i + a] = (j >= 0 && a > 0) ? C[5 * i + a] * SC : 0; }
      alpha = walpha;
    }
    ll eps = cmax * SC;
    if (warm) {
      ll viol = 0;
      for (int i = 0; i < I; ++i) for (int a = 0; a < 5; ++a) { int j = nbr(i, a); if (j < 0) continue;
        ll cp = cs[5 * i + a] + pS[i] - pT[j];
        if (q[i] - w[5 * i + a] > 0) viol = std::max(viol, -cp);
        if (w[5 * i + a] > 0) viol = std::max(viol, cp); }
      eps = viol * alpha;
      if (getenv("REFIT")) {   // smallest power-of-two eps for which the warm flow is eps-optimal
        std::vector<ll> nS, nT; ll lo = 0, e = 1;
        while (e < viol && !refine_prices(e, nS, nT)) e *= 2;
        refine_prices(e, nS, nT); pS = nS; pT = nT;
        printf("warm: violation %lld (%.1f cost units); flow is eps-optimal at eps %lld (%.3f cost units)\n", viol, viol / (double)SC, e, e / (double)SC);
        eps = e * alpha;
      }
    }
    int refines = 0; long long iters = 0; bf_rounds_total = 0;
    std::vector<int> order(2 * I);
    while (eps >= 1) {
      eps = (eps + alpha - 1) / alpha; if (eps < 1) eps = 1; ++refines;
      for (int i = 0; i < I; ++i) for (int a = 0; a < 5; ++a) { int j = nbr(i, a); if (j < 0) continue;
        ll cp = cs[5 * i + a] + pS[i] - pT[j]; if (cp < -eps) w[5 * i + a] = q[i]; else if (cp > eps) w[5 * i + a] = 0; }
      excesses();
      int it = 0; long long maxdepth = 0;
      for (;;) {
        ll tot = 0; for (int v = 0; v < 2 * I; ++v) if (ex[v] > 0) tot += ex[v];
        if (!tot) break;
        ++it;
        forest(eps);
        ll D = 0; for (int v = 0; v < 2 * I; ++v) if (key[v] < kInf) D = std::max(D, key[v] >> 20);
        for (int i = 0; i < I; ++i) {
          pS[i] -= eps * (key[i] < kInf ? key[i] >> 20 : D);
          pT[i] -= eps * (key[I + i] < kInf ? key[I + i] >> 20 : D);
        }
        for (int v = 0; v < 2 * I; ++v) order[v] = v;
        std::sort(order.begin(), order.end(), [&](int x, int y) { return key[x] > key[y]; });
        std::vector<ll> acc(2 * I, 0);
        for (int v : order) {
          if (key[v] >= kInf) continue;
          maxdepth = std::max(maxdepth, key[v] & ((1 << 20) - 1));
          ll tot2 = acc[v] + (ex[v] > 0 ? ex[v] : 0);
          if (ex[v] < 0) {  // deficit root
            ll take = std::min(tot2, -ex[v]); ex[v] += take; tot2 -= take;
            // leftover stays as excess at v (ex >= 0 now)
            ex[v] += tot2; continue;
          }
          if (par[v] < 0) { continue; }
          int e = para[v]; ll cap = v < I ? q[v] - w[e] : w[e];
          ll f = std::min(tot2, cap);
          // only admissible-forward if reduced cost < 0 after price change (always on the forest)
          if (v < I) w[e] += f; else w[e] -= f;
          ex[v] = tot2 - f;     // what could not pass stays
          acc[par[v]] += f;
        }
        // nodes never in the forest keep their excess (unreachable)
        if (it > 100000) { printf("cap\n"); break; }
      }
      iters += it;
      printf("refine %d eps %lld iters %d bf %lld maxhops %lld\n", refines, eps, it, bf_rounds_total, maxdepth);
      if (eps == 1) break;
    }
    ll obj = 0; for (int i = 0; i < I; ++i) for (int a = 1; a < 5; ++a) if (nbr(i, a) >= 0) obj += w[5 * i + a] * C[5 * i + a];
    printf("%s objective %lld iters %lld bf %lld refines %d\n", argv[inst], obj, iters, bf_rounds_total, refines);
    warm = true;
  }
}
