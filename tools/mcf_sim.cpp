// mcf_sim.cpp — CPU emulation of the GPU min-cost-flow kernel's synchronous
// rounds (development aid for tuning round counts on dumped instances; not
// part of the library).  g++ -O3 -fopenmp -o /tmp/mcf_sim tools/mcf_sim.cpp
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <climits>
#include <vector>
#include <algorithm>
typedef long long ll;
int n1, n2, I;
std::vector<ll> q, C, w, cs, eS, eT, addS, addT, pS, pT, pS2, pT2, dS, dT, dS2, dT2;
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
const ll kInf = 1LL << 60;
ll fdiv(ll a, ll b) { ll q = a / b; if ((a % b) && a < 0) --q; return q; }
long long bf_total = 0;
bool price_update(ll eps, int cap) {
  for (int i = 0; i < I; ++i) { dS[i] = eS[i] < 0 ? 0 : kInf; dT[i] = eT[i] < 0 ? 0 : kInf; }
  bool conv = false;
  for (int r = 0; r < cap; ++r) {
    ll ch = 0;
#pragma omp parallel for reduction(+:ch)
    for (int i = 0; i < I; ++i) {
      ll best = dS[i];
      if (best > 0) for (int a = 0; a < 5; ++a) { int j = nbr(i, a); if (j < 0 || q[i] - w[5*i+a] <= 0) continue;
        ll du = dT[j]; if (du >= kInf) continue; ll l = fdiv(cs[5*i+a] + pS[i] - pT[j], eps) + 1; if (l < 0) l = 0;
        if (du + l < best) best = du + l; }
      dS2[i] = best;
      ll bt = dT[i];
      if (bt > 0) for (int k = 0; k < 5; ++k) { int a; int s = in_arc(i, k, &a); if (s < 0 || w[5LL*s+a] <= 0) continue;
        ll du = dS[s]; if (du >= kInf) continue; ll l = fdiv(-(cs[5LL*s+a] + pS[s] - pT[i]), eps) + 1; if (l < 0) l = 0;
        if (du + l < bt) bt = du + l; }
      dT2[i] = bt;
      if (best != dS[i] || bt != dT[i]) ch++;
    }
    std::swap(dS, dS2); std::swap(dT, dT2);
    ++bf_total;
    if (!ch) { conv = true; break; }
  }
  if (!conv) return false;
  ll D = 0;
  for (int i = 0; i < I; ++i) { if (dS[i] < kInf) D = std::max(D, dS[i]); if (dT[i] < kInf) D = std::max(D, dT[i]); }
  for (int i = 0; i < I; ++i) { pS[i] -= eps * (dS[i] < kInf ? dS[i] : D); pT[i] -= eps * (dT[i] < kInf ? dT[i] : D); }
  return true;
}
int alpha = 16, gu_every = -1;
void load(const char* fn) {
  FILE* f = fopen(fn, "rb");
  ll nn[2]; fread(nn, 8, 2, f); n1 = nn[0]; n2 = nn[1]; I = n1 * n2;
  q.resize(I); C.resize(5 * I); fread(q.data(), 8, I, f); fread(C.data(), 8, 5 * I, f); fclose(f);
}
void solve(bool warm) {
  if (!warm) { w.assign(5*I,0); pS.assign(I,0); pT.assign(I,0); }
  cs.assign(5*I,0); eS.assign(I,0); eT.assign(I,0); addS.assign(I,0); addT.assign(I,0);
  pS2=pS; pT2=pT; dS.assign(I,0); dT=dS; dS2=dS; dT2=dS; bf_total = 0;
  ll SC = 2LL * I + 1, cmax = 0;
  for (int i = 0; i < I; ++i) for (int a = 0; a < 5; ++a) { int j = nbr(i, a); if (!warm) w[5*i+a] = a == 0 ? q[i] : 0;
    ll c = (j >= 0 && a > 0) ? C[5*i+a] : 0; cs[5*i+a] = c * SC; if (j >= 0 && a > 0) cmax = std::max(cmax, std::llabs(c)); }
  if (gu_every < 0) gu_every = 2 * (n1 + n2) + 32;
  int gu_cap = 8 * (n1 + n2) + 256;
  ll eps = cmax * SC; long long rounds = 0; int refines = 0;
  if (warm) {   // smallest eps for which (w, p) is eps-optimal
    ll viol = 0;
    for (int i = 0; i < I; ++i) for (int a = 0; a < 5; ++a) { int j = nbr(i, a); if (j < 0) continue;
      ll cp = cs[5*i+a] + pS[i] - pT[j];
      if (q[i] - w[5*i+a] > 0) viol = std::max(viol, -cp);
      if (w[5*i+a] > 0) viol = std::max(viol, cp); }
    if (getenv("WALPHA")) alpha = atoi(getenv("WALPHA"));
    eps = viol * alpha;  // first refine runs at viol
    printf("warm start: initial violation %lld (cold eps %lld)\n", viol, cmax * SC);
  }
  while (eps >= 1) {
    eps = (eps + alpha - 1) / alpha; if (eps < 1) eps = 1; ++refines;
    for (int i = 0; i < I; ++i) for (int a = 0; a < 5; ++a) { int j = nbr(i, a); if (j < 0) continue;
      ll cp = cs[5*i+a] + pS[i] - pT[j]; ll th = getenv("SAT0") ? 0 : eps; if (cp < -th) w[5*i+a] = q[i]; else if (cp > th) w[5*i+a] = 0; }
    for (int i = 0; i < I; ++i) { ll out = 0; for (int a = 0; a < 5; ++a) out += w[5*i+a]; eS[i] = q[i] - out;
      ll in = 0; for (int k = 0; k < 5; ++k) { int a; int s = in_arc(i, k, &a); if (s >= 0) in += w[5LL*s+a]; } eT[i] = in - q[i]; }
    price_update(eps, gu_cap);
    long long r0 = rounds, bf0 = bf_total; int since = 0;
    for (;;) {
      ++rounds;
      if (++since >= gu_every) { since = 0; price_update(eps, gu_cap); }
      // push
      for (int i = 0; i < I; ++i) {
        ll e = eS[i];
        if (e > 0) {
          int ord[5] = {0,1,2,3,4};
          if (getenv("ORDER")) { ll key[5]; for (int a = 0; a < 5; ++a) { int j = nbr(i, a); key[a] = j < 0 ? LLONG_MAX : cs[5*i+a] + pS[i] - pT[j]; }
            std::sort(ord, ord + 5, [&](int x, int y){ return key[x] < key[y]; }); }
          for (int t = 0; t < 5 && e > 0; ++t) { int a = ord[t]; int j = nbr(i, a); if (j < 0) continue; ll r = q[i] - w[5*i+a];
          if (r <= 0) continue; if (cs[5*i+a] + pS[i] - pT[j] < 0) { ll d = std::min(e, r); w[5*i+a] += d; e -= d; addT[j] += d; } } eS[i] = e; }
        ll fe = eT[i];
        if (fe > 0) { for (int k = 0; k < 5 && fe > 0; ++k) { int a; int s = in_arc(i, k, &a); if (s < 0) continue; ll r = w[5LL*s+a];
          if (r <= 0) continue; if (cs[5LL*s+a] + pS[s] - pT[i] > 0) { ll d = std::min(fe, r); w[5LL*s+a] -= d; fe -= d; addS[s] += d; } } eT[i] = fe; }
      }
      ll active = 0;
      for (int i = 0; i < I; ++i) { eS[i] += addS[i]; eT[i] += addT[i]; addS[i] = addT[i] = 0; active += (eS[i] > 0) + (eT[i] > 0); }
      if (getenv("TRACE") && refines == atoi(getenv("TRACE")) && ((rounds - r0) < 10 || (rounds - r0) % 250 == 0)) {
        ll ex = 0; for (int i = 0; i < I; ++i) ex += std::max(0LL, eS[i]) + std::max(0LL, eT[i]);
        printf("  r %lld active %lld excess %lld\n", rounds - r0, active, ex);
      }
      if (!active) break;
      for (int i = 0; i < I; ++i) {
        ll ps = pS[i];
        if (eS[i] > 0) { bool adm = false; ll best = LLONG_MIN; for (int a = 0; a < 5; ++a) { int j = nbr(i, a); if (j < 0) continue;
          if (q[i] - w[5*i+a] <= 0) continue; ll cp = cs[5*i+a] + pS[i] - pT[j]; if (cp < 0) { adm = true; break; }
          best = std::max(best, pT[j] - cs[5*i+a]); } if (!adm && best != LLONG_MIN) ps = best - eps; }
        pS2[i] = ps;
        ll pt = pT[i];
        if (eT[i] > 0) { bool adm = false; ll best = LLONG_MIN; for (int k = 0; k < 5; ++k) { int a; int s = in_arc(i, k, &a); if (s < 0) continue;
          if (w[5LL*s+a] <= 0) continue; ll cp = cs[5LL*s+a] + pS[s] - pT[i]; if (cp > 0) { adm = true; break; }
          best = std::max(best, pS[s] + cs[5LL*s+a]); } if (!adm && best != LLONG_MIN) pt = best - eps; }
        pT2[i] = pt;
      }
      std::swap(pS, pS2); std::swap(pT, pT2);
      if (rounds - r0 > 3000000) { printf("cap\n"); break; }
    }
    printf("refine %d eps %lld rounds %lld bf %lld\n", refines, eps, rounds - r0, bf_total - bf0);
    if (eps == 1) break;
  }
  ll obj = 0; for (int i = 0; i < I; ++i) for (int a = 1; a < 5; ++a) if (nbr(i, a) >= 0) obj += w[5*i+a] * C[5*i+a];
  printf("objective %lld rounds %lld bf %lld refines %d\n", obj, rounds, bf_total, refines);
}
int main(int argc, char** argv) {
  if (argc > 3) alpha = atoi(argv[3]);
  if (argc > 4) gu_every = atoi(argv[4]);
  load(argv[1]); solve(false);
  if (argc > 2 && argv[2][0] == 'p') {   // restart from stationary flow with (perturbed) optimal prices
    double noise = atof(argv[2] + 1);
    ll SC = 2LL * I + 1;
    srand(1);
    for (int i = 0; i < I; ++i) { pS[i] += (ll)(noise * SC * ((rand() / (double)RAND_MAX) - 0.5)); pT[i] += (ll)(noise * SC * ((rand() / (double)RAND_MAX) - 0.5)); }
    if (!getenv("KEEPW")) for (int i = 0; i < I; ++i) for (int a = 0; a < 5; ++a) w[5*i+a] = a == 0 ? q[i] : 0;
    solve(true);
  } else if (argc > 2 && argv[2][0] != '-') { load(argv[2]); solve(true); }
}
