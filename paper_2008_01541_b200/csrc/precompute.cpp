// Host-side precompute of the constant global system (scene setup; NOT on the
// per-frame hot path). Replaces the reference's partial_cholesky
// (/root/reference/pkg/src/schurpd/linalg.py:329-382), fill_ordering (:280-292,
// AMD in _amd.py) and the numba up-looking Cholesky (:107-200).
//
// What it computes, for the symmetric scalar block A already permuted x1-first
// (partition.py:67-71), is exactly the reference's PartialFactor:
//     P1 A11 P1^T = L1 L1^T,  C = A21 P1^T L1^-T,  sigma0 = A22 - C C^T,
// via ONE multifrontal supernodal factorization of the whole matrix with the
// x2 block pinned last: the x2 rows of the supernodal panels are C and the
// assembled root front is sigma0 (ordering independent, as the reference notes).
//
// B200-first choices:
//   * fill ordering = nested dissection (geometric bisection on rest
//     coordinates when the caller has them, BFS level-set bisection otherwise),
//     then an elimination-tree postorder so every supernode is contiguous;
//   * relaxed supernode amalgamation so the device solves run on dense blocks;
//   * a PARTITIONED-INVERSE panel per supernode, M_s = [inv(L_ss); L_below inv(L_ss)],
//     so each supernode of the device forward/backward solve is ONE dense
//     GEMV (no intra-supernode dependency chain); the chain that remains is
//     the supernodal elimination-tree height.
// Dense kernels go through the host BLAS/LAPACK whose function pointers the
// Python side registers (scipy's cython_blas/cython_lapack capsules).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "spb_internal.h"

#include <chrono>
#include <cstdio>

namespace spb {
// SPB_PRECOMPUTE_TIMING=1: per-phase wall times of Factor::build on stderr
struct PhaseTimer {
  bool on = getenv("SPB_PRECOMPUTE_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[precompute] %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};


// ----------------------------------------------------------------- host BLAS
typedef void (*dgemm_t)(const char*, const char*, const int*, const int*, const int*, const double*,
                        const double*, const int*, const double*, const int*, const double*, double*,
                        const int*);
typedef void (*dsyrk_t)(const char*, const char*, const int*, const int*, const double*, const double*,
                        const int*, const double*, double*, const int*);
typedef void (*dtrsm_t)(const char*, const char*, const char*, const char*, const int*, const int*,
                        const double*, const double*, const int*, double*, const int*);
typedef void (*dpotrf_t)(const char*, const int*, double*, const int*, int*);
typedef void (*dtrtri_t)(const char*, const char*, const int*, double*, const int*, int*);

static dgemm_t g_dgemm = nullptr;
static dsyrk_t g_dsyrk = nullptr;
static dtrsm_t g_dtrsm = nullptr;
static dpotrf_t g_dpotrf = nullptr;
static dtrtri_t g_dtrtri = nullptr;

// ------------------------------------------------------------- small helpers
static inline int as_int(int64_t v) { return static_cast<int>(v); }

// Undirected adjacency (CSR, no diagonal) of the x1 block of an upper-CSC matrix.
static void x1_graph(int64_t n1, const int64_t* Ap, const int64_t* Ai, std::vector<int64_t>& gp,
                     std::vector<int64_t>& gi) {
  std::vector<int64_t> deg(n1 + 1, 0);
  for (int64_t j = 0; j < n1; ++j)
    for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) {
      int64_t i = Ai[p];
      if (i < j) { deg[i]++; deg[j]++; }
    }
  gp.assign(n1 + 1, 0);
  for (int64_t i = 0; i < n1; ++i) gp[i + 1] = gp[i] + deg[i];
  gi.resize(gp[n1]);
  std::vector<int64_t> fill(gp.begin(), gp.end() - 1);
  for (int64_t j = 0; j < n1; ++j)
    for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) {
      int64_t i = Ai[p];
      if (i < j) { gi[fill[i]++] = j; gi[fill[j]++] = i; }
    }
}

// ------------------------------------------------------- nested dissection
struct NDState {
  const std::vector<int64_t>* gp;
  const std::vector<int64_t>* gi;
  const double* xyz;  // (n1,3) or null
  std::vector<int32_t> mark;  // subset membership tag
  std::vector<int32_t> side;
  std::vector<int64_t> vis;
  int64_t vstamp = 0;
  int32_t tag = 0;
  std::vector<int64_t> order;
  int64_t leaf = 48;
};

// Vertex separator from a 2-way split: nodes of the smaller boundary side.
static void split_separator(NDState& st, const std::vector<int64_t>& nodes, std::vector<int64_t>& L,
                            std::vector<int64_t>& R, std::vector<int64_t>& S) {
  const auto& gp = *st.gp;
  const auto& gi = *st.gi;
  // side[] holds 1 for L, 2 for R (only valid for nodes of this subset).
  std::vector<int64_t> bl, br;
  for (int64_t v : nodes) {
    bool cross = false;
    for (int64_t p = gp[v]; p < gp[v + 1] && !cross; ++p) {
      int64_t u = gi[p];
      if (st.mark[u] == st.tag && st.side[u] != st.side[v]) cross = true;
    }
    if (cross) (st.side[v] == 1 ? bl : br).push_back(v);
  }
  std::vector<int64_t>& sep = (bl.size() <= br.size()) ? bl : br;
  int32_t sep_side = (bl.size() <= br.size()) ? 1 : 2;
  for (int64_t v : sep) st.side[v] = 3;
  L.clear(); R.clear(); S.clear();
  for (int64_t v : nodes) {
    if (st.side[v] == 1) L.push_back(v);
    else if (st.side[v] == 2) R.push_back(v);
    else S.push_back(v);
  }
  (void)sep_side;
}

static bool geometric_split(NDState& st, std::vector<int64_t>& nodes) {
  // bisect along the widest coordinate at a median plane
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t v : nodes)
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], st.xyz[3 * v + a]);
      hi[a] = std::max(hi[a], st.xyz[3 * v + a]);
    }
  int ax = 0;
  for (int a = 1; a < 3; ++a)
    if (hi[a] - lo[a] > hi[ax] - lo[ax]) ax = a;
  if (!(hi[ax] > lo[ax])) return false;
  std::vector<double> c(nodes.size());
  for (size_t k = 0; k < nodes.size(); ++k) c[k] = st.xyz[3 * nodes[k] + ax];
  std::vector<double> cs = c;
  size_t mid = cs.size() / 2;
  std::nth_element(cs.begin(), cs.begin() + mid, cs.end());
  double med = cs[mid];
  // nodes strictly below the median plane go left; choose <= or < for balance
  size_t nlt = 0, nle = 0;
  for (double v : c) { nlt += (v < med); nle += (v <= med); }
  bool use_le = (std::llabs((long long)(2 * nle) - (long long)c.size()) <
                 std::llabs((long long)(2 * nlt) - (long long)c.size()));
  if ((use_le ? nle : nlt) == 0 || (use_le ? nle : nlt) == c.size()) use_le = !use_le;
  size_t nleft = use_le ? nle : nlt;
  if (nleft == 0 || nleft == c.size()) return false;
  for (size_t k = 0; k < nodes.size(); ++k) st.side[nodes[k]] = ((use_le ? c[k] <= med : c[k] < med) ? 1 : 2);
  return true;
}

static bool bfs_split(NDState& st, std::vector<int64_t>& nodes) {
  // George-Liu pseudo-peripheral start, then split the BFS level structure at
  // the median node; split_separator() carves the vertex separator.
  const auto& gp = *st.gp;
  const auto& gi = *st.gi;
  std::vector<int64_t> lvl, seq;
  auto bfs = [&](int64_t root) -> int64_t {
    st.vstamp++;
    seq.clear();
    lvl.clear();
    seq.push_back(root);
    lvl.push_back(0);
    st.vis[root] = st.vstamp;
    for (size_t h = 0; h < seq.size(); ++h) {
      int64_t v = seq[h];
      for (int64_t p = gp[v]; p < gp[v + 1]; ++p) {
        int64_t u = gi[p];
        if (st.mark[u] == st.tag && st.vis[u] != st.vstamp) {
          st.vis[u] = st.vstamp;
          seq.push_back(u);
          lvl.push_back(lvl[h] + 1);
        }
      }
    }
    return lvl.back();
  };
  int64_t root = nodes[0];
  int64_t ecc = bfs(root);
  if (seq.size() < nodes.size()) {
    // disconnected: the root's component against the rest (empty separator)
    for (int64_t v : nodes) st.side[v] = 2;
    for (int64_t v : seq) st.side[v] = 1;
    return true;
  }
  for (int it = 0; it < 4; ++it) {
    int64_t far = seq.back();
    int64_t e2 = bfs(far);
    if (e2 <= ecc) { bfs(root); break; }
    ecc = e2;
    root = far;
  }
  if (ecc < 2) return false;
  int64_t cut = lvl[seq.size() / 2];
  for (size_t k = 0; k < seq.size(); ++k) st.side[seq[k]] = (lvl[k] <= cut ? 1 : 2);
  size_t nl = 0;
  for (int64_t v : nodes) nl += (st.side[v] == 1);
  return nl > 0 && nl < nodes.size();
}

static void nd_recurse(NDState& st, std::vector<int64_t> nodes) {
  if ((int64_t)nodes.size() <= st.leaf) {
    st.order.insert(st.order.end(), nodes.begin(), nodes.end());
    return;
  }
  st.tag++;
  for (int64_t v : nodes) st.mark[v] = st.tag;
  bool ok = st.xyz ? geometric_split(st, nodes) : bfs_split(st, nodes);
  if (!ok) {
    st.order.insert(st.order.end(), nodes.begin(), nodes.end());
    return;
  }
  std::vector<int64_t> L, R, S;
  split_separator(st, nodes, L, R, S);
  nodes.clear();
  nodes.shrink_to_fit();
  nd_recurse(st, std::move(L));
  nd_recurse(st, std::move(R));
  st.order.insert(st.order.end(), S.begin(), S.end());
}

// ------------------------------------------------------------------ Factor

// Elimination tree of a symmetric matrix given by a CSR-of-lower adjacency:
// for each k, rows i<k with a_ik != 0 (Liu's algorithm with path compression).
static void etree_from_lower(int64_t n, const std::vector<int64_t>& lp, const std::vector<int64_t>& li,
                             std::vector<int64_t>& parent) {
  parent.assign(n, -1);
  std::vector<int64_t> anc(n, -1);
  for (int64_t k = 0; k < n; ++k) {
    for (int64_t p = lp[k]; p < lp[k + 1]; ++p) {
      int64_t i = li[p];
      while (i != -1 && i < k) {
        int64_t nxt = anc[i];
        anc[i] = k;
        if (nxt == -1) parent[i] = k;
        i = nxt;
      }
    }
  }
}

int Factor::build(int64_t n_, int64_t n1_, const int64_t* Ap, const int64_t* Ai, const double* Ax,
                  const double* coords, int ordering, int relax) {
  n = n_;
  n1 = n1_;
  n2 = n - n1;
  if (n1 < 0 || n1 > n) { set_error("n1 out of range"); return SPB_ERR_ARG; }
  if (!g_dgemm || !g_dsyrk || !g_dtrsm || !g_dpotrf || !g_dtrtri) {
    set_error("host BLAS/LAPACK pointers not registered (call spb_set_host_blas first)");
    return SPB_ERR_SETUP;
  }
  // validate upper storage
  for (int64_t j = 0; j < n; ++j)
    for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p)
      if (Ai[p] < 0 || Ai[p] > j) { set_error("input must be the upper triangle in CSC"); return SPB_ERR_ARG; }

  PhaseTimer ptimer;
  // ---- 1. fill ordering of x1 (fperm: new -> old within x1)
  std::vector<int64_t> gp, gi;
  x1_graph(n1, Ap, Ai, gp, gi);
  std::vector<int64_t> fperm(n1);
  if (ordering == 1 && n1 > 1) {
    NDState st;
    st.gp = &gp;
    st.gi = &gi;
    st.xyz = coords;
    st.mark.assign(n1, 0);
    st.side.assign(n1, 0);
    st.vis.assign(n1, 0);
    std::vector<int64_t> all(n1);
    std::iota(all.begin(), all.end(), 0);
    st.order.reserve(n1);
    nd_recurse(st, std::move(all));
    fperm = std::move(st.order);
  } else {
    std::iota(fperm.begin(), fperm.end(), 0);
  }

  // full ordering q: new -> old (x1 by fperm, x2 untouched)
  auto lower_pattern = [&](const std::vector<int64_t>& q, std::vector<int64_t>& lp, std::vector<int64_t>& li,
                           std::vector<double>* lx) {
    // rows = new index, list of (col < row) entries for the etree; plus, if lx,
    // a column-oriented lower CSC (rows >= col) with values for assembly
    std::vector<int64_t> qinv(n);
    for (int64_t k = 0; k < n; ++k) qinv[q[k]] = k;
    std::vector<int64_t> cnt(n + 1, 0);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) {
        int64_t a = qinv[Ai[p]], b = qinv[j];
        int64_t hi = std::max(a, b);
        cnt[hi + 1]++;
      }
    lp.assign(n + 1, 0);
    for (int64_t k = 0; k < n; ++k) lp[k + 1] = lp[k] + cnt[k + 1];
    li.resize(lp[n]);
    if (lx) lx->resize(lp[n]);
    std::vector<int64_t> fill(lp.begin(), lp.end() - 1);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) {
        int64_t a = qinv[Ai[p]], b = qinv[j];
        int64_t hi = std::max(a, b), lo = std::min(a, b);
        int64_t d = fill[hi]++;
        li[d] = lo;
        if (lx) (*lx)[d] = Ax[p];
      }
  };

  std::vector<int64_t> q(n);
  for (int64_t k = 0; k < n1; ++k) q[k] = fperm[k];
  for (int64_t k = n1; k < n; ++k) q[k] = k;
  std::vector<int64_t> rp, ri;  // row-wise lower: row k lists columns < k (and k itself)
  lower_pattern(q, rp, ri, nullptr);
  std::vector<int64_t> parent;
  etree_from_lower(n, rp, ri, parent);

  ptimer.mark("ordering");
  // ---- 2. postorder of the x1 forest (parents >= n1 are virtual roots)
  if (ordering == 1 && n1 > 1) {
    std::vector<int64_t> head(n1, -1), next(n1, -1), stack, post;
    post.reserve(n1);
    for (int64_t j = n1 - 1; j >= 0; --j) {
      int64_t p = parent[j];
      if (p >= 0 && p < n1) { next[j] = head[p]; head[p] = j; }
    }
    for (int64_t j = 0; j < n1; ++j) {
      int64_t p = parent[j];
      if (p >= 0 && p < n1) continue;
      stack.push_back(j);
      while (!stack.empty()) {
        int64_t top = stack.back();
        int64_t child = head[top];
        if (child == -1) { stack.pop_back(); post.push_back(top); }
        else { head[top] = next[child]; stack.push_back(child); }
      }
    }
    std::vector<int64_t> f2(n1);
    for (int64_t k = 0; k < n1; ++k) f2[k] = fperm[post[k]];
    fperm.swap(f2);
    for (int64_t k = 0; k < n1; ++k) q[k] = fperm[k];
    lower_pattern(q, rp, ri, nullptr);
    etree_from_lower(n, rp, ri, parent);
  }
  fill_perm = fperm;

  // column-wise lower pattern with values (rows >= col) for assembly
  std::vector<int64_t> cp, ci;
  std::vector<double> cx;
  {
    // transpose row-wise lists into column-wise, with values
    std::vector<int64_t> qinv(n);
    for (int64_t k = 0; k < n; ++k) qinv[q[k]] = k;
    std::vector<int64_t> cnt(n + 1, 0);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) cnt[std::min(qinv[Ai[p]], qinv[j]) + 1]++;
    cp.assign(n + 1, 0);
    for (int64_t k = 0; k < n; ++k) cp[k + 1] = cp[k] + cnt[k + 1];
    ci.resize(cp[n]);
    cx.resize(cp[n]);
    std::vector<int64_t> fill(cp.begin(), cp.end() - 1);
    for (int64_t j = 0; j < n; ++j)
      for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) {
        int64_t a = qinv[Ai[p]], b = qinv[j];
        int64_t lo = std::min(a, b), hi = std::max(a, b);
        int64_t d = fill[lo]++;
        ci[d] = hi;
        cx[d] = Ax[p];
      }
  }

  ptimer.mark("postorder");
  // ---- 3. column counts of L (columns < n1, all rows) via row subtrees
  std::vector<int64_t> colcount(n1, 1);
  {
    std::vector<int64_t> w(n, -1);
    for (int64_t k = 0; k < n; ++k) {
      w[k] = k;
      for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
        int64_t i = ri[p];
        if (i >= k) continue;
        while (i < n1 && w[i] != k) {
          colcount[i]++;
          w[i] = k;
          i = parent[i];
          if (i < 0) break;
        }
      }
    }
  }
  maxdiag = 0.0;
  for (int64_t j = 0; j < n1; ++j)
    for (int64_t p = cp[j]; p < cp[j + 1]; ++p)
      if (ci[p] == j) maxdiag = std::max(maxdiag, cx[p]);

  ptimer.mark("column counts");
  // ---- 4. fundamental supernodes (+ relaxed amalgamation)
  std::vector<int64_t> nchild(n1, 0);
  for (int64_t j = 0; j < n1; ++j)
    if (parent[j] >= 0 && parent[j] < n1) nchild[parent[j]]++;
  std::vector<int64_t> first;  // supernode first columns
  for (int64_t j = 0; j < n1; ++j) {
    bool start = (j == 0) || !(parent[j - 1] == j && colcount[j - 1] == colcount[j] + 1 && nchild[j] == 1);
    if (start) first.push_back(j);
  }
  first.push_back(n1);
  int64_t ns0 = (int64_t)first.size() - 1;
  std::vector<int64_t> col2sn(n1);
  for (int64_t s = 0; s < ns0; ++s)
    for (int64_t j = first[s]; j < first[s + 1]; ++j) col2sn[j] = s;
  std::vector<int64_t> snparent(ns0, -1);
  for (int64_t s = 0; s < ns0; ++s) {
    int64_t p = parent[first[s + 1] - 1];
    snparent[s] = (p >= 0 && p < n1) ? col2sn[p] : -1;
  }
  // row counts of each fundamental supernode = colcount of its first column
  std::vector<int64_t> snrows(ns0);
  for (int64_t s = 0; s < ns0; ++s) snrows[s] = colcount[first[s]];
  if (relax && ordering == 1) {
    // merge s into its parent p when s is p's contiguous (last) child; the
    // merged block keeps p's rows plus s's columns. Zero-fill limits follow
    // the usual relaxed-supernode rule: always for <= 4 columns, <= 80 % zeros
    // up to 16, <= 10 % up to 48, <= 5 % beyond.
    std::vector<int64_t> zeros(ns0, 0), ncolv(ns0);
    std::vector<int64_t> newfirst(ns0);
    for (int64_t s = 0; s < ns0; ++s) { ncolv[s] = first[s + 1] - first[s]; newfirst[s] = first[s]; }
    std::vector<char> merged(ns0, 0);
    for (int64_t s = 0; s < ns0; ++s) {
      int64_t p = snparent[s];
      if (p < 0 || p != s + 1) continue;
      int64_t nc_s = ncolv[s], nc_p = ncolv[p];
      int64_t nr_p = snrows[p];
      int64_t nc = nc_s + nc_p;
      // merged block rows = cols(s) + rows(p); s's columns gain nr_m - nr_s zeros each
      int64_t nr_m = nc_s + nr_p;
      int64_t extra = nc_s * (nr_m - snrows[s]);
      int64_t z = zeros[s] + zeros[p] + extra;
      double stored = (double)nc * nr_m - 0.5 * (double)nc * (nc - 1);
      double frac = stored > 0 ? (double)z / stored : 0.0;
      bool ok = (nc <= 4) || (nc <= 16 && frac < 0.8) || (nc <= 48 && frac < 0.1) || (frac < 0.05);
      if (ok) {
        merged[s] = 1;
        zeros[p] = z;
        ncolv[p] = nc;
        newfirst[p] = newfirst[s];
        snrows[p] = nc_s + nr_p;
      }
    }
    std::vector<int64_t> f3;
    for (int64_t s = 0; s < ns0; ++s)
      if (!merged[s]) f3.push_back(newfirst[s]);
    f3.push_back(n1);
    first.swap(f3);
  }
  nsuper = (int64_t)first.size() - 1;
  sn_first = first;
  col2sn.assign(n1, 0);
  for (int64_t s = 0; s < nsuper; ++s)
    for (int64_t j = first[s]; j < first[s + 1]; ++j) col2sn[j] = s;
  sn_parent.assign(nsuper, -1);
  for (int64_t s = 0; s < nsuper; ++s) {
    int64_t p = parent[first[s + 1] - 1];
    sn_parent[s] = (p >= 0 && p < n1) ? col2sn[p] : -1;
  }

  ptimer.mark("supernodes");
  // ---- 5. supernodal row structures (children before parents: s ascending)
  std::vector<std::vector<int64_t>> children(nsuper);
  for (int64_t s = 0; s < nsuper; ++s)
    if (sn_parent[s] >= 0) children[sn_parent[s]].push_back(s);
  sn_rowptr.assign(nsuper + 1, 0);
  std::vector<std::vector<int64_t>> st(nsuper);
  {
    std::vector<int64_t> mark(n, -1);
    for (int64_t s = 0; s < nsuper; ++s) {
      int64_t f = first[s], l = first[s + 1];
      std::vector<int64_t>& rows = st[s];
      for (int64_t j = f; j < l; ++j) { rows.push_back(j); mark[j] = s; }
      for (int64_t j = f; j < l; ++j)
        for (int64_t p = cp[j]; p < cp[j + 1]; ++p) {
          int64_t i = ci[p];
          if (i >= l && mark[i] != s) { mark[i] = s; rows.push_back(i); }
        }
      for (int64_t c : children[s]) {
        const auto& cr = st[c];
        int64_t ncc = first[c + 1] - first[c];
        for (size_t k = ncc; k < cr.size(); ++k) {
          int64_t i = cr[k];
          if (i >= l && mark[i] != s) { mark[i] = s; rows.push_back(i); }
        }
      }
      std::sort(rows.begin() + (l - f), rows.end());
      sn_rowptr[s + 1] = sn_rowptr[s] + (int64_t)rows.size();
    }
  }
  sn_rows.resize(sn_rowptr[nsuper]);
  for (int64_t s = 0; s < nsuper; ++s) std::copy(st[s].begin(), st[s].end(), sn_rows.begin() + sn_rowptr[s]);
  st.clear();
  st.shrink_to_fit();
  sn_valptr.assign(nsuper + 1, 0);
  for (int64_t s = 0; s < nsuper; ++s) {
    int64_t nr = sn_rowptr[s + 1] - sn_rowptr[s];
    int64_t nc = first[s + 1] - first[s];
    sn_valptr[s + 1] = sn_valptr[s] + nr * nc;
  }
  Lval.assign(sn_valptr[nsuper], 0.0);
  Mval.assign(sn_valptr[nsuper], 0.0);

  ptimer.mark("row structures");
  // ---- 6. numeric multifrontal factorization
  sigma0.assign((size_t)n2 * n2, 0.0);
  for (int64_t j = n1; j < n; ++j)  // A22 (lower)
    for (int64_t p = cp[j]; p < cp[j + 1]; ++p) {
      int64_t i = ci[p];
      sigma0[(size_t)(i - n1) * n2 + (j - n1)] += cx[p];  // row-major (i >= j)
    }
  std::vector<std::vector<double>> upd(nsuper);
  std::vector<int64_t> pos(n, -1);
  double blas_ms = 0.0;
  auto timed = [&](auto&& fn) {
    if (!ptimer.on) return fn();
    auto t0 = std::chrono::steady_clock::now();
    fn();
    blas_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  const double one = 1.0, mone = -1.0;
  bad_column = -1;
  for (int64_t s = 0; s < nsuper; ++s) {
    int64_t f = first[s], l = first[s + 1];
    int64_t nc = l - f;
    int64_t r0 = sn_rowptr[s], nr = sn_rowptr[s + 1] - r0;
    int64_t nb = nr - nc;
    const int64_t* rows = sn_rows.data() + r0;
    for (int64_t k = 0; k < nr; ++k) pos[rows[k]] = k;
    std::vector<double> F((size_t)nr * nr, 0.0);  // column-major, lower used
    for (int64_t j = f; j < l; ++j)
      for (int64_t p = cp[j]; p < cp[j + 1]; ++p) F[(size_t)(j - f) * nr + pos[ci[p]]] += cx[p];
    for (int64_t c : children[s]) {
      int64_t cr0 = sn_rowptr[c], cnr = sn_rowptr[c + 1] - cr0;
      int64_t cnc = first[c + 1] - first[c];
      int64_t cnb = cnr - cnc;
      const int64_t* crows = sn_rows.data() + cr0 + cnc;
      std::vector<double>& U = upd[c];
      for (int64_t b = 0; b < cnb; ++b) {
        int64_t pb = pos[crows[b]];
        for (int64_t a = b; a < cnb; ++a) F[(size_t)pb * nr + pos[crows[a]]] += U[(size_t)b * cnb + a];
      }
      std::vector<double>().swap(U);
    }
    // partial factorization of the front
    int inc = as_int(nc), inr = as_int(nr), info = 0;
    timed([&] { g_dpotrf("L", &inc, F.data(), &inr, &info); });
    if (info > 0) { bad_column = f + info - 1; break; }
    for (int64_t k = 0; k < nc; ++k) {
      double d = F[(size_t)k * nr + k];
      if (d * d <= PIVOT_TOL * maxdiag) { bad_column = f + k; break; }
    }
    if (bad_column >= 0) break;
    if (nb > 0) {
      int inb = as_int(nb);
      timed([&] { g_dtrsm("R", "L", "T", "N", &inb, &inc, &one, F.data(), &inr, F.data() + nc, &inr); });
      std::vector<double>& U = upd[s];
      U.assign((size_t)nb * nb, 0.0);
      for (int64_t b = 0; b < nb; ++b)
        for (int64_t a = b; a < nb; ++a) U[(size_t)b * nb + a] = F[(size_t)(nc + b) * nr + nc + a];
      timed([&] { g_dsyrk("L", "N", &inb, &inc, &mone, F.data() + nc, &inr, &one, U.data(), &inb); });
      if (sn_parent[s] < 0) {
        // root of the x1 forest: all below rows are x2 -> extend-add into sigma0
        for (int64_t b = 0; b < nb; ++b) {
          int64_t gb = rows[nc + b] - n1;
          for (int64_t a = b; a < nb; ++a) {
            int64_t ga = rows[nc + a] - n1;  // ga >= gb (rows sorted)
            sigma0[(size_t)ga * n2 + gb] += U[(size_t)b * nb + a];
          }
        }
        std::vector<double>().swap(U);
      }
    }
    // store L panel (column-major nr x nc; strict upper of the diagonal block = 0)
    double* Ls = Lval.data() + sn_valptr[s];
    double* Ms = Mval.data() + sn_valptr[s];
    for (int64_t c = 0; c < nc; ++c)
      for (int64_t r = 0; r < nr; ++r) Ls[(size_t)c * nr + r] = (r < c) ? 0.0 : F[(size_t)c * nr + r];
    // partitioned inverse: Minv = inv(L_ss), W = L_below Minv
    std::memcpy(Ms, Ls, sizeof(double) * (size_t)nr * nc);
    timed([&] { g_dtrtri("L", "N", &inc, Ms, &inr, &info); });
    if (nb > 0) {
      // W = L_below * Minv  ==  solve W * L_ss = L_below
      int inb = as_int(nb);
      timed([&] { g_dtrsm("R", "L", "N", "N", &inb, &inc, &one, Ls, &inr, Ms + nc, &inr); });
    }
    for (int64_t k = 0; k < nr; ++k) pos[rows[k]] = -1;
  }
  if (bad_column >= 0) {
    set_error("non-positive pivot in the leading block");
    return SPB_ERR_INDEFINITE;
  }
  // symmetrize sigma0 (lower -> full)
  for (int64_t i = 0; i < n2; ++i)
    for (int64_t j = 0; j < i; ++j) sigma0[(size_t)j * n2 + i] = sigma0[(size_t)i * n2 + j];

  ptimer.mark("numeric factorization");
  if (ptimer.on) fprintf(stderr, "[precompute]   of which host BLAS/LAPACK   %8.1f ms\n", blas_ms);
  // ---- 7. schedule metadata for the device solves
  sn_level.assign(nsuper, 0);
  nlevels = 0;
  for (int64_t s = 0; s < nsuper; ++s) {
    for (int64_t c : children[s]) sn_level[s] = std::max(sn_level[s], sn_level[c] + 1);
    nlevels = std::max(nlevels, sn_level[s] + 1);
  }
  nnz_l1 = 0;
  nnz_c = 0;
  for (int64_t s = 0; s < nsuper; ++s) {
    int64_t nc = first[s + 1] - first[s];
    for (int64_t k = sn_rowptr[s]; k < sn_rowptr[s + 1]; ++k) {
      int64_t r = sn_rows[k];
      int64_t off = k - sn_rowptr[s];
      int64_t cnt = std::min(off + 1, nc);  // columns of s that reach row r
      if (r < n1) nnz_l1 += cnt; else nnz_c += cnt;
    }
  }
  return SPB_OK;
}

void Factor::export_l1(int64_t* indptr, int64_t* indices, double* data) const {
  // CSC of L1 (diagonal first in each column), fill-ordered basis
  int64_t nz = 0;
  indptr[0] = 0;
  for (int64_t s = 0; s < nsuper; ++s) {
    int64_t f = sn_first[s], nc = sn_first[s + 1] - f;
    int64_t r0 = sn_rowptr[s], nr = sn_rowptr[s + 1] - r0;
    const double* Ls = Lval.data() + sn_valptr[s];
    for (int64_t c = 0; c < nc; ++c) {
      for (int64_t k = c; k < nr; ++k) {
        int64_t r = sn_rows[r0 + k];
        if (r >= n1) break;
        indices[nz] = r;
        data[nz] = Ls[(size_t)c * nr + k];
        nz++;
      }
      indptr[f + c + 1] = nz;
    }
  }
}

void Factor::export_coupling(int64_t* indptr, int64_t* indices, double* data) const {
  // CSR (n2 x n1): row r-n1 lists columns j (ascending) with L[r, j] stored
  std::vector<int64_t> cnt(n2 + 1, 0);
  for (int64_t s = 0; s < nsuper; ++s) {
    int64_t nc = sn_first[s + 1] - sn_first[s];
    for (int64_t k = sn_rowptr[s] + nc; k < sn_rowptr[s + 1]; ++k)
      if (sn_rows[k] >= n1) cnt[sn_rows[k] - n1 + 1] += nc;
  }
  indptr[0] = 0;
  for (int64_t r = 0; r < n2; ++r) indptr[r + 1] = indptr[r] + cnt[r + 1];
  std::vector<int64_t> fill(indptr, indptr + n2);
  for (int64_t s = 0; s < nsuper; ++s) {  // s ascending => columns ascending per row
    int64_t f = sn_first[s], nc = sn_first[s + 1] - f;
    int64_t r0 = sn_rowptr[s], nr = sn_rowptr[s + 1] - r0;
    const double* Ls = Lval.data() + sn_valptr[s];
    for (int64_t k = nc; k < nr; ++k) {
      int64_t r = sn_rows[r0 + k];
      if (r < n1) continue;
      for (int64_t c = 0; c < nc; ++c) {
        int64_t d = fill[r - n1]++;
        indices[d] = f + c;
        data[d] = Ls[(size_t)c * nr + k];
      }
    }
  }
}

}  // namespace spb

// ------------------------------------------------------------------- C ABI
using spb::Factor;

extern "C" {

int spb_set_host_blas(void* dgemm, void* dsyrk, void* dtrsm, void* dpotrf, void* dtrtri) {
  spb::g_dgemm = (spb::dgemm_t)dgemm;
  spb::g_dsyrk = (spb::dsyrk_t)dsyrk;
  spb::g_dtrsm = (spb::dtrsm_t)dtrsm;
  spb::g_dpotrf = (spb::dpotrf_t)dpotrf;
  spb::g_dtrtri = (spb::dtrtri_t)dtrtri;
  return SPB_OK;
}

int spb_factor_create(int64_t n, int64_t n1, const int64_t* Ap, const int64_t* Ai, const double* Ax,
                      const double* coords, int32_t ordering, int32_t relax, spb_factor** out,
                      int64_t* bad_column) {
  SPB_GUARD_BEGIN
  if (!out || !Ap || (n > 0 && (!Ai || !Ax))) { spb::set_error("null argument"); return SPB_ERR_ARG; }
  auto* f = new Factor();
  int rc = f->build(n, n1, Ap, Ai, Ax, coords, ordering, relax);
  if (bad_column) *bad_column = f->bad_column >= 0 ? f->fill_perm[f->bad_column] : -1;
  if (rc != SPB_OK) { delete f; *out = nullptr; return rc; }
  *out = reinterpret_cast<spb_factor*>(f);
  return SPB_OK;
  SPB_GUARD_END
}

void spb_factor_destroy(spb_factor* f) { delete reinterpret_cast<Factor*>(f); }

int spb_factor_info(const spb_factor* fp, int64_t* info) {
  const Factor* f = reinterpret_cast<const Factor*>(fp);
  info[0] = f->n1;
  info[1] = f->n2;
  info[2] = f->nsuper;
  info[3] = f->nnz_l1;
  info[4] = f->nnz_c;
  info[5] = f->nlevels;
  info[6] = f->sn_valptr.empty() ? 0 : f->sn_valptr.back();
  info[7] = f->sn_rowptr.empty() ? 0 : f->sn_rowptr.back();
  return SPB_OK;
}

int spb_factor_fill_perm(const spb_factor* fp, int64_t* out) {
  const Factor* f = reinterpret_cast<const Factor*>(fp);
  std::copy(f->fill_perm.begin(), f->fill_perm.end(), out);
  return SPB_OK;
}

int spb_factor_export_l1(const spb_factor* fp, int64_t* indptr, int64_t* indices, double* data) {
  reinterpret_cast<const Factor*>(fp)->export_l1(indptr, indices, data);
  return SPB_OK;
}

int spb_factor_export_coupling(const spb_factor* fp, int64_t* indptr, int64_t* indices, double* data) {
  reinterpret_cast<const Factor*>(fp)->export_coupling(indptr, indices, data);
  return SPB_OK;
}

int spb_factor_sigma0(const spb_factor* fp, double* out) {
  const Factor* f = reinterpret_cast<const Factor*>(fp);
  std::copy(f->sigma0.begin(), f->sigma0.end(), out);
  return SPB_OK;
}

int spb_factor_supernodes(const spb_factor* fp, int64_t* first, int64_t* rowptr, int64_t* rows, int64_t* parent,
                          int64_t* level) {
  const Factor* f = reinterpret_cast<const Factor*>(fp);
  if (first) std::copy(f->sn_first.begin(), f->sn_first.end(), first);
  if (rowptr) std::copy(f->sn_rowptr.begin(), f->sn_rowptr.end(), rowptr);
  if (rows) std::copy(f->sn_rows.begin(), f->sn_rows.end(), rows);
  if (parent) std::copy(f->sn_parent.begin(), f->sn_parent.end(), parent);
  if (level) std::copy(f->sn_level.begin(), f->sn_level.end(), level);
  return SPB_OK;
}

}  // extern "C"

// ------------------------------------------------------------ public helpers
extern "C" {

// Fill-reducing ordering of a symmetric pattern given by its upper CSC
// (linalg.fill_ordering, linalg.py:280-292): nested dissection; out[new] = old.
int spb_fill_ordering(int64_t n, const int64_t* Ap, const int64_t* Ai, const double* coords, int64_t* out) {
  SPB_GUARD_BEGIN
  std::vector<int64_t> gp, gi;
  spb::x1_graph(n, Ap, Ai, gp, gi);
  spb::NDState st;
  st.gp = &gp;
  st.gi = &gi;
  st.xyz = coords;
  st.mark.assign(n, 0);
  st.side.assign(n, 0);
  st.vis.assign(n, 0);
  std::vector<int64_t> all(n);
  std::iota(all.begin(), all.end(), 0);
  if (n > 1) spb::nd_recurse(st, std::move(all));
  else st.order = all;
  std::copy(st.order.begin(), st.order.end(), out);
  return SPB_OK;
  SPB_GUARD_END
}

// nnz of the Cholesky factor of a symmetric pattern (upper CSC), incl. the
// diagonal (partition.py:113-120 _symbolic_factor_nnz).
int spb_symbolic_nnz(int64_t n, const int64_t* Ap, const int64_t* Ai, int64_t* nnz) {
  SPB_GUARD_BEGIN
  // row-wise lower lists == column-wise upper lists
  std::vector<int64_t> lp(n + 1), li;
  for (int64_t j = 0; j < n; ++j) lp[j + 1] = lp[j] + (Ap[j + 1] - Ap[j]);
  li.assign(Ai, Ai + Ap[n]);
  std::vector<int64_t> parent;
  spb::etree_from_lower(n, lp, li, parent);
  std::vector<int64_t> w(n, -1);
  int64_t total = n;
  for (int64_t k = 0; k < n; ++k) {
    w[k] = k;
    for (int64_t p = lp[k]; p < lp[k + 1]; ++p) {
      int64_t i = li[p];
      while (i != -1 && i < k && w[i] != k) {
        total++;
        w[i] = k;
        i = parent[i];
      }
    }
  }
  *nnz = total;
  return SPB_OK;
  SPB_GUARD_END
}

}  // extern "C"
