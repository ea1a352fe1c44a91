// Host symbolic analysis (see symbolic.hpp).  PAPER.md P:108-113.
#include "symbolic.hpp"

#include <algorithm>
#include <queue>
#include <set>

namespace sdpc {

std::vector<int32_t> minimum_degree(int32_t n, const std::vector<std::pair<int32_t, int32_t>>& edges) {
  // Elimination game: eliminate the vertex of minimum current degree (ties -> smallest id),
  // then make its remaining neighbours a clique ("appropriate order like
  // approximation minimum ordering"; exact MD here, SURVEY §8(c) reading #5).
  std::vector<std::vector<int32_t>> adj(n);
  for (auto& e : edges) {
    if (e.first == e.second) continue;
    adj[e.first].push_back(e.second);
    adj[e.second].push_back(e.first);
  }
  for (auto& a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  using Item = std::pair<int64_t, int32_t>;
  std::priority_queue<Item, std::vector<Item>, std::greater<Item>> pq;
  for (int32_t v = 0; v < n; ++v) pq.push({(int64_t)adj[v].size(), v});
  std::vector<char> done(n, 0);
  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<int32_t> tmp;
  while (!pq.empty()) {
    auto [d, v] = pq.top();
    pq.pop();
    if (done[v] || d != (int64_t)adj[v].size()) continue;
    done[v] = 1;
    order.push_back(v);
    const std::vector<int32_t> nb = adj[v];
    for (int32_t u : nb) {
      auto& au = adj[u];
      tmp.clear();
      std::set_union(au.begin(), au.end(), nb.begin(), nb.end(), std::back_inserter(tmp));
      tmp.erase(std::remove_if(tmp.begin(), tmp.end(), [&](int32_t x) { return x == u || x == v; }), tmp.end());
      au.swap(tmp);
      pq.push({(int64_t)au.size(), u});
    }
    adj[v].clear();
  }
  return order;
}

std::string analyse(Symbolic& S, int32_t n, int32_t m, const int64_t* a_ptr, const int32_t* a_row,
                    const int32_t* a_col, const int32_t* perm_in) {
  S.n = n;
  S.m = m;
  const int64_t ntrip = a_ptr[m + 1];
  std::vector<std::pair<int32_t, int32_t>> edges;  // original ids, off-diagonal
  for (int64_t e = 0; e < ntrip; ++e) {
    int32_t r = a_row[e], c = a_col[e];
    if (r < 0 || r >= n || c < 0 || c >= n) return "triplet index out of range";
    if (r < c) return "triplet with row < col";
    if (r != c) edges.push_back({c, r});
  }
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());

  if (perm_in) {
    S.perm.assign(perm_in, perm_in + n);
  } else {
    S.perm = minimum_degree(n, edges);
  }
  S.iperm.assign(n, -1);
  for (int32_t k = 0; k < n; ++k) {
    int32_t o = S.perm[k];
    if (o < 0 || o >= n || S.iperm[o] != -1) return "perm is not a permutation";
    S.iperm[o] = k;
  }

  // lower pattern by rows in elimination order: lowrow[k] = {i < k : A(k,i) != 0}
  std::vector<int64_t> rp(n + 1, 0);
  for (auto& e : edges) {
    int32_t a = S.iperm[e.first], b = S.iperm[e.second];
    rp[std::max(a, b) + 1]++;
  }
  for (int32_t k = 0; k < n; ++k) rp[k + 1] += rp[k];
  std::vector<int32_t> rc(rp[n]);
  {
    std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
    for (auto& e : edges) {
      int32_t a = S.iperm[e.first], b = S.iperm[e.second];
      rc[fill[std::max(a, b)]++] = std::min(a, b);
    }
  }

  // elimination tree (Liu, path compression)
  S.parent.assign(n, -1);
  {
    std::vector<int32_t> anc(n, -1);
    for (int32_t k = 0; k < n; ++k) {
      for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
        int32_t i = rc[p];
        while (i != -1 && i < k) {
          int32_t nx = anc[i];
          anc[i] = k;
          if (nx == -1) S.parent[i] = k;
          i = nx;
        }
      }
    }
  }

  // row structure of L by etree reach; append row k to each column -> ascending columns
  std::vector<std::vector<int32_t>> cols(n);
  {
    std::vector<int32_t> mark(n, -1);
    for (int32_t k = 0; k < n; ++k) {
      mark[k] = k;
      for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
        for (int32_t i = rc[p]; i != -1 && mark[i] != k; i = S.parent[i]) {
          mark[i] = k;
          cols[i].push_back(k);
        }
      }
    }
  }
  S.colptr.assign(n + 1, 0);
  for (int32_t j = 0; j < n; ++j) S.colptr[j + 1] = S.colptr[j] + 1 + (int64_t)cols[j].size();
  const int64_t nnz = S.colptr[n];
  if (nnz >= (int64_t(1) << 31)) return "nnz(E) too large for int32 offsets";
  S.rowind.resize(nnz);
  for (int32_t j = 0; j < n; ++j) {
    int64_t p = S.colptr[j];
    S.rowind[p++] = j;
    for (int32_t i : cols[j]) S.rowind[p++] = i;
    if (!cols[j].empty() && cols[j][0] != S.parent[j]) return "internal: etree/structure mismatch";
  }
  std::vector<int64_t> cc(n);
  for (int32_t j = 0; j < n; ++j) cc[j] = (int64_t)cols[j].size();
  cols.clear();
  cols.shrink_to_fit();

  // fundamental supernodes: j+1 joins j iff parent(j) = j+1, j+1 has one child, cc_j = cc_{j+1}+1
  std::vector<int32_t> nchild(n, 0);
  for (int32_t j = 0; j < n; ++j)
    if (S.parent[j] >= 0) nchild[S.parent[j]]++;
  S.super_ptr.clear();
  S.super_ptr.push_back(0);
  for (int32_t j = 0; j + 1 < n; ++j) {
    bool same = S.parent[j] == j + 1 && nchild[j + 1] == 1 && cc[j] == cc[j + 1] + 1;
    if (!same) S.super_ptr.push_back(j + 1);
  }
  S.super_ptr.push_back(n);
  S.nsuper = (int32_t)S.super_ptr.size() - 1;
  const int32_t ns = S.nsuper;
  S.sn_of_col.assign(n, 0);
  S.snc.assign(ns, 0);
  S.sns.assign(ns, 0);
  S.sparent.assign(ns, -1);
  for (int32_t r = 0; r < ns; ++r) {
    int32_t f = S.super_ptr[r], l = S.super_ptr[r + 1];
    for (int32_t j = f; j < l; ++j) S.sn_of_col[j] = r;
    S.sns[r] = l - f;
    S.snc[r] = (int32_t)(cc[f] + 1);
  }
  for (int32_t r = 0; r < ns; ++r) {
    int32_t last = S.super_ptr[r + 1] - 1;
    int32_t p = S.parent[last];
    S.sparent[r] = p < 0 ? -1 : S.sn_of_col[p];
    if (p >= 0 && S.super_ptr[S.sparent[r]] != p) return "internal: parent column not first of supernode";
  }
  // children CSR
  S.child_ptr.assign(ns + 1, 0);
  for (int32_t r = 0; r < ns; ++r)
    if (S.sparent[r] >= 0) S.child_ptr[S.sparent[r] + 1]++;
  for (int32_t r = 0; r < ns; ++r) S.child_ptr[r + 1] += S.child_ptr[r];
  S.child_list.assign(S.child_ptr[ns], 0);
  {
    std::vector<int32_t> fill(S.child_ptr.begin(), S.child_ptr.end() - 1);
    for (int32_t r = 0; r < ns; ++r)
      if (S.sparent[r] >= 0) S.child_list[fill[S.sparent[r]]++] = r;
  }

  // panels
  S.panel_off.assign(ns + 1, 0);
  for (int32_t r = 0; r < ns; ++r) S.panel_off[r + 1] = S.panel_off[r] + (int64_t)S.snc[r] * S.sns[r];
  S.panel_total = S.panel_off[ns];
  if (S.panel_total >= (int64_t(1) << 31)) return "panel storage too large for int32 map";
  S.e2p.resize(nnz);
  for (int32_t j = 0; j < n; ++j) {
    int32_t r = S.sn_of_col[j];
    int32_t t = j - S.super_ptr[r];
    int64_t base = S.panel_off[r] + (int64_t)t * S.snc[r] + t;
    for (int64_t p = S.colptr[j]; p < S.colptr[j + 1]; ++p) S.e2p[p] = (int32_t)(base + (p - S.colptr[j]));
  }

  // Algorithm 1 gather maps for U_r x U_r (lower, packed column-major)
  S.umap_off.assign(ns + 1, 0);
  for (int32_t r = 0; r < ns; ++r) {
    int64_t u = S.snc[r] - S.sns[r];
    S.umap_off[r + 1] = S.umap_off[r] + u * (u + 1) / 2;
  }
  S.umap.resize(S.umap_off[ns]);
  for (int32_t r = 0; r < ns; ++r) {
    const int32_t f = S.super_ptr[r], s = S.sns[r], c = S.snc[r], u = c - s;
    const int32_t* C = &S.rowind[S.colptr[f]];
    int64_t o = S.umap_off[r];
    for (int32_t b = 0; b < u; ++b) {
      int32_t col = C[s + b];
      int64_t p = S.colptr[col], pe = S.colptr[col + 1];
      for (int32_t a = b; a < u; ++a) {
        int32_t row = C[s + a];
        while (p < pe && S.rowind[p] < row) ++p;
        if (p >= pe || S.rowind[p] != row) return "internal: clique entry outside E";
        S.umap[o++] = (int32_t)p;
      }
    }
  }

  // multifrontal relative indices and update buffers
  S.relind_off.assign(ns + 1, 0);
  S.upd_off.assign(ns + 1, 0);
  for (int32_t r = 0; r < ns; ++r) {
    int64_t u = S.snc[r] - S.sns[r];
    S.relind_off[r + 1] = S.relind_off[r] + u;
    S.upd_off[r + 1] = S.upd_off[r] + u * u;
  }
  S.upd_total = S.upd_off[ns];
  S.relind.resize(S.relind_off[ns]);
  for (int32_t r = 0; r < ns; ++r) {
    int32_t R = S.sparent[r];
    const int32_t f = S.super_ptr[r], s = S.sns[r], u = S.snc[r] - s;
    if (u == 0) continue;
    if (R < 0) return "internal: supernode with U but no parent";
    const int32_t* U = &S.rowind[S.colptr[f] + s];
    const int32_t* CR = &S.rowind[S.colptr[S.super_ptr[R]]];
    int32_t cR = S.snc[R], p = 0;
    for (int32_t q = 0; q < u; ++q) {
      while (p < cR && CR[p] < U[q]) ++p;
      if (p >= cR || CR[p] != U[q]) return "internal: U_r not inside parent clique";
      S.relind[S.relind_off[r] + q] = p;
    }
  }

  // schedules: height (leaves 0) and depth (roots 0)
  S.height.assign(ns, 0);
  for (int32_t r = 0; r < ns; ++r)
    if (S.sparent[r] >= 0) S.height[S.sparent[r]] = std::max(S.height[S.sparent[r]], S.height[r] + 1);
  S.depth.assign(ns, 0);
  for (int32_t r = ns - 1; r >= 0; --r)
    if (S.sparent[r] >= 0) S.depth[r] = S.depth[S.sparent[r]] + 1;
  auto group = [&](const std::vector<int32_t>& lev, std::vector<int32_t>& ptr, std::vector<int32_t>& list) {
    int32_t L = 0;
    for (int32_t v : lev) L = std::max(L, v + 1);
    ptr.assign(L + 1, 0);
    for (int32_t v : lev) ptr[v + 1]++;
    for (int32_t i = 0; i < L; ++i) ptr[i + 1] += ptr[i];
    list.assign(lev.size(), 0);
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    for (int32_t r = 0; r < (int32_t)lev.size(); ++r) list[fill[lev[r]]++] = r;
  };
  group(S.height, S.hlev_ptr, S.hlev_sn);
  group(S.depth, S.dlev_ptr, S.dlev_sn);
  // preorder of the supernodal forest (roots in index order, children in index order)
  S.preorder.clear();
  {
    std::vector<int32_t> stack;
    for (int32_t r = ns - 1; r >= 0; --r)
      if (S.sparent[r] < 0) stack.push_back(r);
    while (!stack.empty()) {
      int32_t r = stack.back();
      stack.pop_back();
      S.preorder.push_back(r);
      for (int32_t q = S.child_ptr[r + 1] - 1; q >= S.child_ptr[r]; --q) stack.push_back(S.child_list[q]);
    }
  }
  // backward task decomposition: subtree work w(r) = sum over the subtree of s*u + s^2/2.
  // Subtree roots: w(r) <= wmax < w(parent).  Everything above is "top".
  {
    std::vector<int64_t> w(ns, 0);
    for (int32_t r = 0; r < ns; ++r) {
      w[r] += (int64_t)S.sns[r] * (S.snc[r] - S.sns[r]) + (int64_t)S.sns[r] * (S.sns[r] + 1) / 2;
      if (S.sparent[r] >= 0) w[S.sparent[r]] += w[r];
    }
    int64_t total = 0;
    for (int32_t r = 0; r < ns; ++r)
      if (S.sparent[r] < 0) total += w[r];
    const int64_t wmax = std::max<int64_t>(1, total / 96);
    // top = heavy subtrees (CTA-wide tensor-core path, level order); the rest are subtrees, one warp
    // each (a wide supernode alone in a light subtree, e.g. a block-arrow leaf, stays on a warp: many
    // such leaves run in parallel that way)
    std::vector<char> is_top(ns, 0);
    std::vector<int32_t> roots;
    for (int32_t r = 0; r < ns; ++r) {
      const int32_t p = S.sparent[r];
      if (w[r] > wmax) is_top[r] = 1;
      else if (p < 0 || w[p] > wmax) roots.push_back(r);
    }
    S.border.clear();
    for (size_t lv = 0; lv + 1 < S.dlev_ptr.size(); ++lv) {
      std::vector<int32_t> tops;
      for (int32_t q = S.dlev_ptr[lv]; q < S.dlev_ptr[lv + 1]; ++q)
        if (is_top[S.dlev_sn[q]]) tops.push_back(S.dlev_sn[q]);
      std::stable_sort(tops.begin(), tops.end(), [&](int32_t x, int32_t y) { return w[x] > w[y]; });
      S.border.insert(S.border.end(), tops.begin(), tops.end());
    }
    S.ntop = (int32_t)S.border.size();
    std::stable_sort(roots.begin(), roots.end(), [&](int32_t x, int32_t y) { return w[x] > w[y]; });
    S.sub_ptr.assign(1, S.ntop);
    std::vector<int32_t> stack;
    for (int32_t rt : roots) {
      stack.assign(1, rt);
      while (!stack.empty()) {
        const int32_t r = stack.back();
        stack.pop_back();
        S.border.push_back(r);
        for (int32_t q = S.child_ptr[r + 1] - 1; q >= S.child_ptr[r]; --q) stack.push_back(S.child_list[q]);
      }
      S.sub_ptr.push_back((int32_t)S.border.size());
    }
    if ((int32_t)S.border.size() != ns) return "internal: backward task order incomplete";
  }
  // within a depth level, the most work first (backward solve: one warp per supernode)
  for (size_t lv = 0; lv + 1 < S.dlev_ptr.size(); ++lv) {
    auto b = S.dlev_sn.begin() + S.dlev_ptr[lv], e = S.dlev_sn.begin() + S.dlev_ptr[lv + 1];
    std::stable_sort(b, e, [&](int32_t x, int32_t y) {
      const int64_t wx = (int64_t)S.sns[x] * (S.snc[x] - S.sns[x]) + (int64_t)S.sns[x] * S.sns[x] / 2;
      const int64_t wy = (int64_t)S.sns[y] * (S.snc[y] - S.sns[y]) + (int64_t)S.sns[y] * S.sns[y] / 2;
      return wx > wy;
    });
  }
  return "";
}

}  // namespace sdpc
