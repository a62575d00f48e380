// Host-side setup, once per grid.  See analysis.hpp.
//
// * validation (R24, R25)
// * index maps of x and p (R3, R5)
// * bus -> incident line CSR (adjacency A(i))
// * J pattern: row P_i / Q_i meets column theta_j / v_j iff j = i or j in A(i)
// * minimum-degree ordering of the bus graph (REF removed), expanded to the
//   (theta, v) variables of each bus; J's pattern is structurally symmetric
//   under the pairing P_i <-> theta_i, Q_i <-> v_i, so a symmetric ordering with
//   static diagonal pivots keeps a fixed fill pattern (PAPER.md:764-767,
//   cuSOLVER_RF reuses the host's pivot order; R15)
// * symbolic factorization via the elimination tree (L pattern = U^T pattern)
// * level sets of the forward (L, U^T) and backward (U, L^T) sweeps
#include "analysis.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <set>
#include <sstream>

#include "../../include/redhess.h"

namespace rh {

namespace {

template <class T>
void sort_unique(std::vector<T> &v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

// Minimum degree on an undirected graph given by sorted adjacency lists.
// Exact elimination graph; ties broken by lowest index (R19).
std::vector<int32_t> minimum_degree(std::vector<std::vector<int32_t>> adj) {
  const int n = (int)adj.size();
  std::set<std::pair<int, int>> pq;
  for (int u = 0; u < n; ++u) pq.insert({(int)adj[u].size(), u});
  std::vector<char> done(n, 0);
  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<int32_t> merged;
  while (!pq.empty()) {
    const int u = pq.begin()->second;
    pq.erase(pq.begin());
    done[u] = 1;
    order.push_back(u);
    const std::vector<int32_t> nb = adj[u];
    for (int a : nb) {
      pq.erase({(int)adj[a].size(), a});
      // adj[a] = (adj[a] u nb) \ {a, u}
      merged.clear();
      merged.reserve(adj[a].size() + nb.size());
      std::set_union(adj[a].begin(), adj[a].end(), nb.begin(), nb.end(), std::back_inserter(merged));
      std::vector<int32_t> out;
      out.reserve(merged.size());
      for (int w : merged)
        if (w != a && w != u) out.push_back(w);
      adj[a].swap(out);
      pq.insert({(int)adj[a].size(), a});
    }
    adj[u].clear();
  }
  return order;
}

}  // namespace

std::string analyze(const ::rh_grid &g, Analysis &A) {
  std::ostringstream err;
  const int n = g.n_bus, m = g.n_line, ng = g.n_gen;
  if (n < 2) return "grid needs at least 2 buses";
  if (m < 1) return "grid needs at least 1 line";
  if (ng < 0) return "n_gen < 0";
  if (!g.bus_type || !g.G_ii || !g.B_ii || !g.Pd || !g.Qd || !g.line_f || !g.line_t || !g.G_ft ||
      !g.B_ft || !g.G_tf || !g.B_tf || (ng > 0 && (!g.gen_bus || !g.c2 || !g.c1 || !g.c0)))
    return "null array in rh_grid";
  A = Analysis();
  A.n_bus = n;
  A.n_line = m;
  A.n_gen = ng;
  A.theta_ref = g.theta_ref;
  A.bus_type.assign(g.bus_type, g.bus_type + n);
  A.G_ii.assign(g.G_ii, g.G_ii + n);
  A.B_ii.assign(g.B_ii, g.B_ii + n);
  A.Pd.assign(g.Pd, g.Pd + n);
  A.Qd.assign(g.Qd, g.Qd + n);
  A.line_f.assign(g.line_f, g.line_f + m);
  A.line_t.assign(g.line_t, g.line_t + m);
  A.G_ft.assign(g.G_ft, g.G_ft + m);
  A.B_ft.assign(g.B_ft, g.B_ft + m);
  A.G_tf.assign(g.G_tf, g.G_tf + m);
  A.B_tf.assign(g.B_tf, g.B_tf + m);

  int nref = 0;
  for (int b = 0; b < n; ++b) {
    const int t = A.bus_type[b];
    if (t != RH_PQ && t != RH_PV && t != RH_REF) {
      err << "bus " << b << " has invalid type " << t;
      return err.str();
    }
    if (t == RH_REF) {
      ++nref;
      A.ref = b;
    }
  }
  if (nref != 1) {
    err << "exactly one REF bus required, found " << nref;
    return err.str();
  }
  for (int l = 0; l < m; ++l) {
    const int f = A.line_f[l], t = A.line_t[l];
    if (f < 0 || f >= n || t < 0 || t >= n) {
      err << "line " << l << " has a bus index out of range";
      return err.str();
    }
    if (f == t) {
      err << "line " << l << " has f == t";
      return err.str();
    }
  }
  A.c2b.assign(n, 0.0);
  A.c1b.assign(n, 0.0);
  A.c0b.assign(n, 0.0);
  A.has_gen.assign(n, 0);
  for (int k = 0; k < ng; ++k) {
    const int b = g.gen_bus[k];
    if (b < 0 || b >= n) {
      err << "generator " << k << " bus index out of range";
      return err.str();
    }
    if (A.bus_type[b] == RH_PQ) {
      err << "generator " << k << " sits on PQ bus " << b;
      return err.str();
    }
    if (A.has_gen[b]) {
      err << "more than one generator on bus " << b << " (R25)";
      return err.str();
    }
    A.has_gen[b] = 1;
    A.c2b[b] = g.c2[k];
    A.c1b[b] = g.c1[k];
    A.c0b[b] = g.c0[k];
  }

  // bus -> line CSR
  A.bl_ptr.assign(n + 1, 0);
  for (int l = 0; l < m; ++l) {
    A.bl_ptr[A.line_f[l] + 1]++;
    A.bl_ptr[A.line_t[l] + 1]++;
  }
  for (int b = 0; b < n; ++b) A.bl_ptr[b + 1] += A.bl_ptr[b];
  A.bl_line.assign(2 * m, 0);
  A.bl_other.assign(2 * m, 0);
  A.bl_end.assign(2 * m, 0);
  {
    std::vector<int32_t> fill(A.bl_ptr.begin(), A.bl_ptr.end() - 1);
    for (int l = 0; l < m; ++l) {
      int s = fill[A.line_f[l]]++;
      A.bl_line[s] = l;
      A.bl_other[s] = A.line_t[l];
      A.bl_end[s] = 0;
      s = fill[A.line_t[l]]++;
      A.bl_line[s] = l;
      A.bl_other[s] = A.line_f[l];
      A.bl_end[s] = 1;
    }
  }
  // connectivity
  {
    std::vector<char> seen(n, 0);
    std::vector<int> stack{0};
    seen[0] = 1;
    int cnt = 1;
    while (!stack.empty()) {
      int b = stack.back();
      stack.pop_back();
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
        int o = A.bl_other[s];
        if (!seen[o]) {
          seen[o] = 1;
          ++cnt;
          stack.push_back(o);
        }
      }
    }
    if (cnt != n) {
      err << "grid graph is not connected (" << cnt << " of " << n << " buses reachable)";
      return err.str();
    }
  }

  // ---------------- index maps (R5) ----------------
  A.th_x.assign(n, -1);
  A.v_x.assign(n, -1);
  A.v_p.assign(n, -1);
  A.pg_p.assign(n, -1);
  for (int pass = 0; pass < 3; ++pass) {
    for (int b = 0; b < n; ++b) {
      const int t = A.bus_type[b];
      if (pass == 0 && t == RH_PV) {
        A.th_x[b] = (int)A.x_bus.size();
        A.x_bus.push_back(b);
        A.x_kind.push_back(RH_KIND_THETA);
      } else if (pass == 1 && t == RH_PQ) {
        A.th_x[b] = (int)A.x_bus.size();
        A.x_bus.push_back(b);
        A.x_kind.push_back(RH_KIND_THETA);
      } else if (pass == 2 && t == RH_PQ) {
        A.v_x[b] = (int)A.x_bus.size();
        A.x_bus.push_back(b);
        A.x_kind.push_back(RH_KIND_V);
      }
    }
  }
  for (int b = 0; b < n; ++b)
    if (A.bus_type[b] == RH_PV) {
      A.pg_p[b] = (int)A.p_bus.size();
      A.p_bus.push_back(b);
      A.p_kind.push_back(RH_KIND_PG);
    }
  for (int b = 0; b < n; ++b)
    if (A.bus_type[b] != RH_PQ) {
      A.v_p[b] = (int)A.p_bus.size();
      A.p_bus.push_back(b);
      A.p_kind.push_back(RH_KIND_V);
    }
  A.n_x = (int)A.x_bus.size();
  A.n_p = (int)A.p_bus.size();
  const int nx = A.n_x;

  // ---------------- natural J pattern ----------------
  A.J_rowptr.assign(nx + 1, 0);
  {
    std::vector<std::vector<int32_t>> rows(nx);
    for (int r = 0; r < nx; ++r) {
      const int b = A.x_bus[r];
      auto &c = rows[r];
      c.push_back(A.th_x[b]);
      if (A.v_x[b] >= 0) c.push_back(A.v_x[b]);
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
        const int o = A.bl_other[s];
        if (A.th_x[o] >= 0) c.push_back(A.th_x[o]);
        if (A.v_x[o] >= 0) c.push_back(A.v_x[o]);
      }
      sort_unique(c);
    }
    for (int r = 0; r < nx; ++r) A.J_rowptr[r + 1] = A.J_rowptr[r] + (int)rows[r].size();
    A.J_col.reserve(A.J_rowptr[nx]);
    for (auto &c : rows) A.J_col.insert(A.J_col.end(), c.begin(), c.end());
    A.nnz_J = A.J_rowptr[nx];
  }

  // ---------------- ordering: MD on the bus graph without REF ----------------
  std::vector<int32_t> nonref;
  std::vector<int32_t> bidx(n, -1);
  for (int b = 0; b < n; ++b)
    if (b != A.ref) {
      bidx[b] = (int)nonref.size();
      nonref.push_back(b);
    }
  {
    std::vector<std::vector<int32_t>> adj(nonref.size());
    for (size_t u = 0; u < nonref.size(); ++u) {
      const int b = nonref[u];
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
        const int o = A.bl_other[s];
        if (o != A.ref) adj[u].push_back(bidx[o]);
      }
      sort_unique(adj[u]);
    }
    std::vector<int32_t> border = minimum_degree(adj);
    A.perm.clear();
    for (int u : border) {
      const int b = nonref[u];
      A.perm.push_back(A.th_x[b]);
      if (A.v_x[b] >= 0) A.perm.push_back(A.v_x[b]);
    }
    A.pinv.assign(nx, -1);
    for (int i = 0; i < nx; ++i) A.pinv[A.perm[i]] = i;
  }

  // ---------------- symbolic factorization ----------------
  std::vector<std::vector<int32_t>> Ls(nx);   // strict-lower rows of column k (= U row k cols)
  {
    std::vector<std::vector<int32_t>> children(nx);
    for (int k = 0; k < nx; ++k) {
      const int r = A.perm[k];
      std::vector<int32_t> s;
      for (int e = A.J_rowptr[r]; e < A.J_rowptr[r + 1]; ++e) {
        const int i = A.pinv[A.J_col[e]];
        if (i > k) s.push_back(i);
      }
      for (int c : children[k])
        for (int i : Ls[c])
          if (i != k) s.push_back(i);
      sort_unique(s);
      Ls[k].swap(s);
      if (!Ls[k].empty()) children[Ls[k][0]].push_back(k);
      std::vector<int32_t>().swap(children[k]);
    }
  }
  std::vector<std::vector<int32_t>> Lrow(nx);
  for (int k = 0; k < nx; ++k)
    for (int i : Ls[k]) Lrow[i].push_back(k);
  A.F_rowptr.assign(nx + 1, 0);
  for (int i = 0; i < nx; ++i) A.F_rowptr[i + 1] = A.F_rowptr[i] + (int)(Lrow[i].size() + 1 + Ls[i].size());
  A.F_col.resize(A.F_rowptr[nx]);
  A.F_diag.resize(nx);
  for (int i = 0; i < nx; ++i) {
    int p = A.F_rowptr[i];
    for (int k : Lrow[i]) A.F_col[p++] = k;
    A.F_diag[i] = p;
    A.F_col[p++] = i;
    for (int k : Ls[i]) A.F_col[p++] = k;
  }
  auto fpos = [&](int i, int j) -> int {
    auto b = A.F_col.begin() + A.F_rowptr[i], e = A.F_col.begin() + A.F_rowptr[i + 1];
    auto it = std::lower_bound(b, e, j);
    if (it == e || *it != j) return -1;
    return (int)(it - A.F_col.begin());
  };

  // ---------------- levels ----------------
  A.lev_fwd.assign(nx, 0);
  A.lev_bwd.assign(nx, 0);
  for (int i = 0; i < nx; ++i) {
    int lv = 0;
    for (int k : Lrow[i]) lv = std::max(lv, A.lev_fwd[k] + 1);
    A.lev_fwd[i] = lv;
  }
  for (int i = nx - 1; i >= 0; --i) {
    int lv = 0;
    for (int k : Ls[i]) lv = std::max(lv, A.lev_bwd[k] + 1);
    A.lev_bwd[i] = lv;
  }
  A.nlev_fwd = nx ? 1 + *std::max_element(A.lev_fwd.begin(), A.lev_fwd.end()) : 0;
  A.nlev_bwd = nx ? 1 + *std::max_element(A.lev_bwd.begin(), A.lev_bwd.end()) : 0;

  auto level_order = [&](const std::vector<int32_t> &lev, int nlev, std::vector<int32_t> &lev_ptr,
                         std::vector<int32_t> &rows) {
    lev_ptr.assign(nlev + 1, 0);
    for (int i = 0; i < nx; ++i) lev_ptr[lev[i] + 1]++;
    for (int l = 0; l < nlev; ++l) lev_ptr[l + 1] += lev_ptr[l];
    rows.assign(nx, 0);
    std::vector<int32_t> fill(lev_ptr.begin(), lev_ptr.end() - 1);
    for (int i = 0; i < nx; ++i) rows[fill[lev[i]]++] = i;
  };
  auto build_sweep = [&](Sweep &S, bool fwd, bool transposed, bool unit) {
    level_order(fwd ? A.lev_fwd : A.lev_bwd, fwd ? A.nlev_fwd : A.nlev_bwd, S.lev_ptr, S.rows);
    S.rptr.assign(nx + 1, 0);
    S.col.clear();
    S.src.clear();
    S.diag_src.assign(nx, -1);
    for (int q = 0; q < nx; ++q) {
      const int i = S.rows[q];
      const std::vector<int32_t> &deps = fwd ? Lrow[i] : Ls[i];
      for (int k : deps) {
        S.col.push_back(k);
        S.src.push_back(transposed ? fpos(k, i) : fpos(i, k));
      }
      S.rptr[q + 1] = (int)S.col.size();
      if (!unit) S.diag_src[q] = A.F_diag[i];
    }
  };
  build_sweep(A.sL, true, false, true);
  build_sweep(A.sU, false, false, false);
  build_sweep(A.sUt, true, true, false);
  build_sweep(A.sLt, false, true, true);
  A.max_level_rows = 0;
  for (int l = 0; l < A.nlev_fwd; ++l)
    A.max_level_rows = std::max(A.max_level_rows, A.sL.lev_ptr[l + 1] - A.sL.lev_ptr[l]);
  A.fact_order = A.sL.rows;

  // ---------------- assembly positions ----------------
  A.diag_pos.assign(4 * n, -1);
  A.slot_pos.assign(8 * m, -1);
  for (int b = 0; b < n; ++b) {
    if (b == A.ref) continue;
    const int rP = A.pinv[A.th_x[b]];
    const int rQ = A.v_x[b] >= 0 ? A.pinv[A.v_x[b]] : -1;
    const int cth = rP, cv = rQ;
    A.diag_pos[4 * b + 0] = fpos(rP, cth);
    if (cv >= 0) A.diag_pos[4 * b + 1] = fpos(rP, cv);
    if (rQ >= 0) {
      A.diag_pos[4 * b + 2] = fpos(rQ, cth);
      A.diag_pos[4 * b + 3] = fpos(rQ, cv);
    }
    for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
      const int o = A.bl_other[s];
      const int oth = A.th_x[o] >= 0 ? A.pinv[A.th_x[o]] : -1;
      const int ov = A.v_x[o] >= 0 ? A.pinv[A.v_x[o]] : -1;
      if (oth >= 0) A.slot_pos[4 * s + 0] = fpos(rP, oth);
      if (ov >= 0) A.slot_pos[4 * s + 1] = fpos(rP, ov);
      if (rQ >= 0 && oth >= 0) A.slot_pos[4 * s + 2] = fpos(rQ, oth);
      if (rQ >= 0 && ov >= 0) A.slot_pos[4 * s + 3] = fpos(rQ, ov);
    }
  }
  for (int e : A.diag_pos)
    if (e < -1) return "internal: diag position";
  for (int b = 0; b < n; ++b) {
    if (b == A.ref) continue;
    for (int q = 0; q < 4; ++q)
      if ((q == 0 || A.v_x[b] >= 0) && A.diag_pos[4 * b + q] < 0) return "internal: missing diagonal entry";
  }

  // ---------------- G_p pattern (permuted rows) ----------------
  {
    std::vector<std::vector<int32_t>> rows(nx);
    for (int b = 0; b < n; ++b) {
      if (b == A.ref) continue;
      const int rP = A.pinv[A.th_x[b]];
      const int rQ = A.v_x[b] >= 0 ? A.pinv[A.v_x[b]] : -1;
      if (A.pg_p[b] >= 0) rows[rP].push_back(A.pg_p[b]);
      if (A.v_p[b] >= 0) rows[rP].push_back(A.v_p[b]);
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
        const int o = A.bl_other[s];
        if (A.v_p[o] >= 0) {
          rows[rP].push_back(A.v_p[o]);
          if (rQ >= 0) rows[rQ].push_back(A.v_p[o]);
        }
      }
    }
    A.gp_rptr.assign(nx + 1, 0);
    for (int r = 0; r < nx; ++r) {
      sort_unique(rows[r]);
      A.gp_rptr[r + 1] = A.gp_rptr[r] + (int)rows[r].size();
    }
    A.gp_col.clear();
    for (auto &c : rows) A.gp_col.insert(A.gp_col.end(), c.begin(), c.end());
    auto gpos = [&](int r, int c) -> int {
      auto bb = A.gp_col.begin() + A.gp_rptr[r], ee = A.gp_col.begin() + A.gp_rptr[r + 1];
      auto it = std::lower_bound(bb, ee, c);
      if (it == ee || *it != c) return -1;
      return (int)(it - A.gp_col.begin());
    };
    A.gp_self_pos.assign(n, -1);
    A.gp_pg_pos.assign(n, -1);
    A.gp_slot_pos.assign(4 * m, -1);
    for (int b = 0; b < n; ++b) {
      if (b == A.ref) continue;
      const int rP = A.pinv[A.th_x[b]];
      const int rQ = A.v_x[b] >= 0 ? A.pinv[A.v_x[b]] : -1;
      if (A.pg_p[b] >= 0) A.gp_pg_pos[b] = gpos(rP, A.pg_p[b]);
      if (A.v_p[b] >= 0) A.gp_self_pos[b] = gpos(rP, A.v_p[b]);
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
        const int o = A.bl_other[s];
        if (A.v_p[o] >= 0) {
          A.gp_slot_pos[2 * s + 0] = gpos(rP, A.v_p[o]);
          if (rQ >= 0) A.gp_slot_pos[2 * s + 1] = gpos(rQ, A.v_p[o]);
        }
      }
    }
    // CSC
    const int np_ = A.n_p;
    A.gpc_ptr.assign(np_ + 1, 0);
    for (int c : A.gp_col) A.gpc_ptr[c + 1]++;
    for (int c = 0; c < np_; ++c) A.gpc_ptr[c + 1] += A.gpc_ptr[c];
    A.gpc_pos.assign(A.gp_col.size(), 0);
    A.gpc_row.assign(A.gp_col.size(), 0);
    std::vector<int32_t> fill(A.gpc_ptr.begin(), A.gpc_ptr.end() - 1);
    for (int r = 0; r < nx; ++r)
      for (int e = A.gp_rptr[r]; e < A.gp_rptr[r + 1]; ++e) {
        const int q = fill[A.gp_col[e]]++;
        A.gpc_pos[q] = e;
        A.gpc_row[q] = r;
      }
  }

  // ---------------- FoR sources / destinations ----------------
  A.dth_src.assign(n, -1);
  A.dv_src.assign(n, -1);
  A.yth_dst.assign(n, -1);
  A.yv_dst.assign(n, -1);
  for (int b = 0; b < n; ++b) {
    if (b != A.ref) A.dth_src[b] = A.yth_dst[b] = A.pinv[A.th_x[b]];
    if (A.v_x[b] >= 0)
      A.dv_src[b] = A.yv_dst[b] = A.pinv[A.v_x[b]];
    else
      A.dv_src[b] = A.yv_dst[b] = -(A.v_p[b] + 2);
  }
  A.near_ref.push_back(A.ref);
  for (int s = A.bl_ptr[A.ref]; s < A.bl_ptr[A.ref + 1]; ++s) A.near_ref.push_back(A.bl_other[s]);
  sort_unique(A.near_ref);
  return "";
}

}  // namespace rh
