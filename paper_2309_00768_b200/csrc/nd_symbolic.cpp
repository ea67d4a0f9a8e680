// Host symbolic analysis for the nested-dissection supernodal LU (see nd.hpp).
#include <cstdlib>
#include <algorithm>
#include <numeric>
#include <queue>

#include "nd.hpp"

namespace stmhd {

namespace {

struct Graph {
  std::vector<int64_t> ptr;
  std::vector<int> adj;
};

// Symmetrised adjacency without self loops.
Graph symmetrize(int64_t n, const int32_t *rowptr, const int32_t *col) {
  std::vector<std::vector<int>> nb(n);
  for (int64_t i = 0; i < n; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      int j = col[e];
      if (j == i) continue;
      nb[i].push_back(j);
      nb[j].push_back((int)i);
    }
  Graph g;
  g.ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    auto &v = nb[i];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    g.ptr[i + 1] = g.ptr[i] + (int64_t)v.size();
  }
  g.adj.resize(g.ptr[n]);
  for (int64_t i = 0; i < n; ++i) std::copy(nb[i].begin(), nb[i].end(), g.adj.begin() + g.ptr[i]);
  return g;
}

struct TreeNode {
  std::vector<int> cols;
  std::vector<int> children;
};

class Dissector {
 public:
  Dissector(const Graph &g, const int32_t *gx, const int32_t *gy, int leaf)
      : g_(g), gx_(gx), gy_(gy), leaf_(std::max(leaf, 1)), mark_(g.ptr.size() - 1, 0) {}

  int build(std::vector<int> nodes) {
    int id = (int)tree.size();
    tree.emplace_back();
    if ((int)nodes.size() <= leaf_) {
      std::sort(nodes.begin(), nodes.end());
      tree[id].cols = std::move(nodes);
      return id;
    }
    std::vector<int> L, R, S;
    bool ok = gx_ ? split_coords(nodes, L, R, S) : false;
    if (!ok) split_graph(nodes, L, R, S);
    if (L.empty() && R.empty()) {  // could not split: dense leaf
      std::sort(nodes.begin(), nodes.end());
      tree[id].cols = std::move(nodes);
      return id;
    }
    std::vector<int> kids;
    if (!L.empty()) kids.push_back(build(std::move(L)));
    if (!R.empty()) kids.push_back(build(std::move(R)));
    std::sort(S.begin(), S.end());
    tree[id].cols = std::move(S);
    tree[id].children = kids;
    return id;
  }

  std::vector<TreeNode> tree;

 private:
  // Separator = nodes on an axis-aligned grid line, plus any left node still
  // coupled to the right side (wide stencils).  Tries the lines around the
  // middle of the longer extent and keeps the smallest separator.
  bool split_coords(const std::vector<int> &nodes, std::vector<int> &L, std::vector<int> &R,
                    std::vector<int> &S) {
    int x0 = INT32_MAX, x1 = INT32_MIN, y0 = INT32_MAX, y1 = INT32_MIN;
    for (int v : nodes) {
      x0 = std::min(x0, gx_[v]); x1 = std::max(x1, gx_[v]);
      y0 = std::min(y0, gy_[v]); y1 = std::max(y1, gy_[v]);
    }
    bool found = false;
    size_t best = SIZE_MAX;
    for (int axis = 0; axis < 2; ++axis) {
      int lo = axis == 0 ? x0 : y0, hi = axis == 0 ? x1 : y1;
      if (hi - lo < 2) continue;
      int mid = lo + (hi - lo) / 2;
      for (int d = -2; d <= 2; ++d) {
        int line = mid + d;
        if (line <= lo || line >= hi) continue;
        std::vector<int> l, r, s;
        const int32_t *c = axis == 0 ? gx_ : gy_;
        for (int v : nodes) {
          if (c[v] < line) l.push_back(v);
          else if (c[v] > line) r.push_back(v);
          else s.push_back(v);
        }
        for (int v : r) mark_[v] = 2;
        std::vector<int> l2;
        for (int v : l) {
          bool cross = false;
          for (int64_t e = g_.ptr[v]; e < g_.ptr[v + 1] && !cross; ++e) cross = mark_[g_.adj[e]] == 2;
          (cross ? s : l2).push_back(v);
        }
        for (int v : r) mark_[v] = 0;
        if (l2.empty() || r.empty()) continue;
        // balance penalty: separator size dominates, imbalance breaks ties
        size_t imb = (size_t)std::abs((long)l2.size() - (long)r.size());
        size_t score = s.size() * 4 * nodes.size() + imb;
        if (score < best) {
          best = score;
          L.swap(l2); R.swap(r); S.swap(s);
          found = true;
        }
      }
    }
    return found;
  }

  // BFS level-structure bisection from a pseudo-peripheral node.
  void split_graph(const std::vector<int> &nodes, std::vector<int> &L, std::vector<int> &R,
                   std::vector<int> &S) {
    for (int v : nodes) mark_[v] = 1;
    auto bfs = [&](int src, std::vector<int> &lev_of, std::vector<int> &order) {
      order.clear();
      std::queue<int> q;
      q.push(src);
      lev_of[src] = 0;
      mark_[src] = 3;
      while (!q.empty()) {
        int v = q.front(); q.pop();
        order.push_back(v);
        for (int64_t e = g_.ptr[v]; e < g_.ptr[v + 1]; ++e) {
          int w = g_.adj[e];
          if (mark_[w] == 1) { mark_[w] = 3; lev_of[w] = lev_of[v] + 1; q.push(w); }
        }
      }
      for (int v : order) mark_[v] = 1;
    };
    std::vector<int> lev(mark_.size(), 0), order;
    int src = nodes[0];
    for (int it = 0; it < 2; ++it) {
      bfs(src, lev, order);
      src = order.back();
    }
    bfs(src, lev, order);
    int maxlev = lev[order.back()];
    for (int v : nodes) mark_[v] = 0;
    if (maxlev < 2) return;  // no useful separator
    // median level by node count
    std::vector<int> cnt(maxlev + 1, 0);
    for (int v : order) cnt[lev[v]]++;
    int half = (int)order.size() / 2, acc = 0, cut = 1;
    for (int l = 0; l <= maxlev; ++l) { acc += cnt[l]; if (acc >= half) { cut = std::max(1, std::min(l, maxlev - 1)); break; } }
    std::vector<char> seen(mark_.size(), 0);
    for (int v : order) {
      seen[v] = 1;
      if (lev[v] < cut) L.push_back(v);
      else if (lev[v] > cut) R.push_back(v);
      else S.push_back(v);
    }
    for (int v : nodes) if (!seen[v]) R.push_back(v);  // other components
  }

  const Graph &g_;
  const int32_t *gx_, *gy_;
  int leaf_;
  std::vector<int> mark_;
};

}  // namespace

NDPlan nd_analyze(int64_t n, const int32_t *rowptr, const int32_t *col, const int32_t *gx,
                  const int32_t *gy, int leaf_max, const int32_t *value_map, unsigned merge_mask) {
  require(n > 0, "nd_analyze: empty matrix");
  Graph g = symmetrize(n, rowptr, col);
  Dissector dis(g, gx, gy, leaf_max);
  std::vector<int> all(n);
  std::iota(all.begin(), all.end(), 0);
  int root = dis.build(std::move(all));
  auto &tree = dis.tree;

  // Amalgamation of tree levels (bit d of merge_mask: depth d): every separator at such a
  // depth absorbs its two child separators -- one supernode whose columns are the
  // children's then its own, whose children are the grandchildren (up to four).  The
  // time sweeps pay a synchronised step per tree level, so a level fewer is worth the
  // larger front (explicit zeros between the two absorbed separators).  Depths in the
  // mask are at least two apart (an absorbed node is never a merge root itself).
  require((merge_mask & (merge_mask << 1)) == 0, "nd_analyze: adjacent depths in the merge mask");
  if (merge_mask) {
    std::vector<int> depth(tree.size(), -1), order{root};
    depth[root] = 0;
    for (size_t i = 0; i < order.size(); ++i)
      for (int c : tree[order[i]].children) {
        depth[c] = depth[order[i]] + 1;
        order.push_back(c);
      }
    for (int t : order) {
      if (depth[t] > 31 || !(merge_mask >> depth[t] & 1u) || tree[t].children.size() != 2) continue;
      bool ok = true;
      std::vector<int> grand;
      for (int c : tree[t].children) {
        ok = ok && tree[c].children.size() == 2;
        for (int gc : tree[c].children) grand.push_back(gc);
      }
      if (!ok) continue;
      std::vector<int> cols;
      for (int c : tree[t].children) cols.insert(cols.end(), tree[c].cols.begin(), tree[c].cols.end());
      cols.insert(cols.end(), tree[t].cols.begin(), tree[t].cols.end());
      tree[t].cols = std::move(cols);
      tree[t].children = std::move(grand);
    }
  }

  // postorder
  std::vector<int> post;
  post.reserve(tree.size());
  {
    std::vector<std::pair<int, int>> st{{root, 0}};
    while (!st.empty()) {
      auto &[t, i] = st.back();
      if (i < (int)tree[t].children.size()) {
        int c = tree[t].children[i++];
        st.push_back({c, 0});
      } else {
        post.push_back(t);
        st.pop_back();
      }
    }
  }
  std::vector<int> sn_of_tree(tree.size());
  for (size_t i = 0; i < post.size(); ++i) sn_of_tree[post[i]] = (int)i;

  NDPlan p;
  p.n = n;
  p.nsn = (int)post.size();
  int S = p.nsn;
  p.level.assign(S, 0);
  p.ns.assign(S, 0);
  p.nb.assign(S, 0);
  p.parent.assign(S, -1);
  p.first.assign(S, 0);
  std::vector<int64_t> pos(n, -1);
  std::vector<int> sn_of(n, -1);
  std::vector<std::vector<int>> kids(S);
  int64_t cursor = 0;
  for (int s = 0; s < S; ++s) {
    const TreeNode &t = tree[post[s]];
    p.first[s] = cursor;
    p.ns[s] = (int)t.cols.size();
    for (int v : t.cols) { pos[v] = cursor++; sn_of[v] = s; }
    for (int c : t.children) {
      int cs = sn_of_tree[c];
      kids[s].push_back(cs);
      p.parent[cs] = s;
      p.level[s] = std::max(p.level[s], p.level[cs] + 1);
    }
  }
  require(cursor == n, "nd_analyze: ordering does not cover all unknowns");

  // boundary sets, bottom-up
  std::vector<std::vector<int>> bnd(S);
  std::vector<char> in(n, 0);
  for (int s = 0; s < S; ++s) {
    const TreeNode &t = tree[post[s]];
    int64_t last = p.first[s] + p.ns[s] - 1;
    std::vector<int> b;
    auto add = [&](int v) {
      if (pos[v] > last && !in[v]) { in[v] = 1; b.push_back(v); }
    };
    for (int v : t.cols)
      for (int64_t e = g.ptr[v]; e < g.ptr[v + 1]; ++e) add(g.adj[e]);
    for (int c : kids[s])
      for (int v : bnd[c]) add(v);
    for (int v : b) in[v] = 0;
    std::sort(b.begin(), b.end(), [&](int a, int c) { return pos[a] < pos[c]; });
    bnd[s] = std::move(b);
    p.nb[s] = (int)bnd[s].size();
  }

  // front index lists, offsets
  p.idx_off.assign(S + 1, 0);
  p.fl_off.assign(S, 0);
  p.fu_off.assign(S, 0);
  p.sfl_off.assign(S, 0);
  p.sfu_off.assign(S, 0);
  p.rf.assign(S, 1);
  p.rb.assign(S, 1);
  p.bsz_f.assign(S, 0);
  p.bsz_b.assign(S, 0);
  // rows per chunk: the largest power of two <= 32 whose block fits kChunkMax doubles
  // (STMHD_CHUNK_MAX; default 640 doubles, 512 for the large 64^2 velocity blocks,
  // whose sweeps run grid-wide: smaller TMA slots leave shared memory for deeper
  // CTA-local subtrees -- C4/C3 P_T^-1 -7 %, measured)
  static const int64_t chunk_env = [] {
    const char *e = getenv("STMHD_CHUNK_MAX");
    return e ? (int64_t)atoi(e) : (int64_t)0;
  }();
  const int64_t kChunkMax = chunk_env > 0 ? chunk_env : (n > 20000 ? 512 : 640);
  auto rows_per_chunk = [&](int64_t K) {
    int R = 32;
    while (R > 1 && (int64_t)R * K > kChunkMax) R >>= 1;
    return R;
  };
  p.front_off.assign(S, 0);
  p.cbv_off.assign(S, 0);
  for (int s = 0; s < S; ++s) {
    int64_t f = p.ns[s] + p.nb[s];
    p.idx_off[s + 1] = p.idx_off[s] + f;
    const int64_t ns64 = p.ns[s];
    p.sfl_off[s] = p.stage_size;
    p.stage_size += f * ns64;
    p.sfu_off[s] = p.stage_size;
    p.stage_size += f * ns64;
    p.rf[s] = rows_per_chunk(ns64);
    p.rb[s] = rows_per_chunk(f);
    p.bsz_f[s] = ((int64_t)p.rf[s] * ns64 + 1) & ~int64_t(1);
    p.bsz_b[s] = ((int64_t)p.rb[s] * f + 1) & ~int64_t(1);
    const int64_t ncf = (f + p.rf[s] - 1) / p.rf[s], ncb = (ns64 + p.rb[s] - 1) / p.rb[s];
    p.fl_off[s] = p.factor_size;
    p.factor_size += ncf * p.bsz_f[s];
    p.fu_off[s] = p.factor_size;
    p.factor_size += ncb * p.bsz_b[s];
    p.front_off[s] = p.front_size;
    p.front_size += f * f;
    p.cbv_off[s] = p.cbv_size;
    p.cbv_size += p.nb[s];
    p.max_front = std::max<int>(p.max_front, (int)f);
    int64_t ns = p.ns[s];
    p.sym_nnz += ns * ns + 2 * ns * p.nb[s];
  }
  p.idx.resize(p.idx_off[S]);
  for (int s = 0; s < S; ++s) {
    const TreeNode &t = tree[post[s]];
    int64_t o = p.idx_off[s];
    for (int v : t.cols) p.idx[o++] = v;
    for (int v : bnd[s]) p.idx[o++] = v;
  }

  // children CSR + extend-add maps (child bnd -> parent front position)
  p.child_ptr.assign(S + 1, 0);
  for (int s = 0; s < S; ++s) p.child_ptr[s + 1] = p.child_ptr[s] + (int)kids[s].size();
  p.child_list.resize(p.child_ptr[S]);
  for (int s = 0; s < S; ++s)
    std::copy(kids[s].begin(), kids[s].end(), p.child_list.begin() + p.child_ptr[s]);
  p.emap_off.assign(S + 1, 0);
  for (int s = 0; s < S; ++s) p.emap_off[s + 1] = p.emap_off[s] + p.nb[s];
  p.emap.assign(p.emap_off[S], -1);
  std::vector<int> fpos(n, -1);
  for (int s = 0; s < S; ++s) {
    int64_t f = p.ns[s] + p.nb[s];
    for (int64_t t = 0; t < f; ++t) fpos[p.idx[p.idx_off[s] + t]] = (int)t;
    for (int c : kids[s])
      for (int a = 0; a < p.nb[c]; ++a) {
        int v = bnd[c][a];
        require(fpos[v] >= 0, "nd_analyze: child boundary not in parent front");
        p.emap[p.emap_off[c] + a] = fpos[v];
      }
    for (int64_t t = 0; t < f; ++t) fpos[p.idx[p.idx_off[s] + t]] = -1;
  }

  // scatter of original entries into the owning front
  std::vector<std::vector<std::pair<int64_t, int64_t>>> sc(S);
  {
    // front position lookup per supernode computed lazily per row owner
    std::vector<int> lpos(n, -1);
    // group entries by owner supernode
    std::vector<std::vector<std::pair<int64_t, int64_t>>> raw(S);  // (entry, other)
    for (int64_t i = 0; i < n; ++i)
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        int j = col[e];
        int owner = pos[i] <= pos[j] ? sn_of[i] : sn_of[j];
        raw[owner].push_back({e, i});
      }
    for (int s = 0; s < S; ++s) {
      int64_t f = p.ns[s] + p.nb[s];
      for (int64_t t = 0; t < f; ++t) lpos[p.idx[p.idx_off[s] + t]] = (int)t;
      for (auto &pr : raw[s]) {
        int64_t e = pr.first, i = pr.second;
        int j = col[e];
        require(lpos[i] >= 0 && lpos[j] >= 0, "nd_analyze: entry outside its front");
        int64_t src = value_map ? (int64_t)value_map[e] : e;
        sc[s].push_back({src, (int64_t)lpos[i] * f + lpos[j]});
      }
      for (int64_t t = 0; t < f; ++t) lpos[p.idx[p.idx_off[s] + t]] = -1;
    }
  }
  p.scat_ptr.assign(S + 1, 0);
  for (int s = 0; s < S; ++s) p.scat_ptr[s + 1] = p.scat_ptr[s] + (int64_t)sc[s].size();
  p.scat_src.resize(p.scat_ptr[S]);
  p.scat_dst.resize(p.scat_ptr[S]);
  for (int s = 0; s < S; ++s) {
    std::sort(sc[s].begin(), sc[s].end(), [](auto &a, auto &b) { return a.second < b.second; });
    for (size_t t = 0; t < sc[s].size(); ++t) {
      p.scat_src[p.scat_ptr[s] + t] = sc[s][t].first;
      p.scat_dst[p.scat_ptr[s] + t] = sc[s][t].second;
    }
  }

  p.nlevels = 0;
  for (int s = 0; s < S; ++s) p.nlevels = std::max(p.nlevels, p.level[s] + 1);
  p.level_sn.assign(p.nlevels, {});
  for (int s = 0; s < S; ++s) p.level_sn[p.level[s]].push_back(s);
  for (int s = 0; s < S; ++s) {
    require(p.child_ptr[s + 1] - p.child_ptr[s] <= 4, "nd_analyze: supernode with more than four children");
    p.nwide += p.wide(s);
  }
  return p;
}

}  // namespace stmhd
