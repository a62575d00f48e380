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
#include <array>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <set>
#include <sstream>
#include <stdexcept>
#include <unordered_map>

#include "../../include/redhess.h"

namespace rh {

namespace {

constexpr int kSchedWarps = 16;  // warps of the block sweep kernel (512 threads)
constexpr int kMaxTops = 32;      // cap on a block's densely inverted top rows

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


// Subtree-to-warp split of one block.  Lanes own
// columns, so a warp needs no synchronization between rows it computes
// itself.  The block's forest is cut into <= ~nw "pieces" (whole subtrees) of
// balanced cost packed onto warps (LPT); the removed roots ("tops", <= max_tops,
// a near-dense chain at the top of the block) are not chained row by row:
// their diagonal block is inverted once per state (k_tops_inverse) and applied
// as a dense product, so every sweep of a block needs only 2-3 CTA barriers.
// The same split serves both directions and the refactorization.
//
// Nodes are bus UNITS (the 1 or 2 rows of a bus, see UnitSweep): a unit's rows
// always land in the same piece (or both in the tops), so the bus-unit sweeps
// can process them together.  A unit's parent is the unit holding the
// elimination-tree parent of its highest row.
//
// Unit sweeps (dual = true): the cut goes on while the largest piece exceeds
// `cut` x (remaining pieces' cost / nw), and the pieces are packed onto the
// warps twice, once per pattern direction with that direction's unit cost (a
// fixed per-unit latency plus one per dependency unit): warp_rows for the
// forward sweeps (L, U^T), warp_rows_b for the backward ones (U, L^T).
BlockSplit split_block(const std::vector<int32_t> &rows, const std::vector<int32_t> &unit_lo,
                       const std::vector<std::vector<int32_t>> &Ls, const std::vector<std::vector<int32_t>> &Lrow,
                       int nw, int max_tops, bool dual = false, double cut = 1.25) {
  const int n = (int)rows.size();   // ascending permuted rows
  std::vector<int> uofr(n), ubeg;   // unit of each local row, first local row of each unit
  for (int i = 0; i < n; ++i) {
    if (i == 0 || unit_lo[rows[i]] != unit_lo[rows[i - 1]]) ubeg.push_back(i);
    uofr[i] = (int)ubeg.size() - 1;
  }
  const int nu = (int)ubeg.size();
  ubeg.push_back(n);
  std::unordered_map<int, int> li;
  li.reserve(n * 2);
  for (int i = 0; i < n; ++i) li[rows[i]] = i;
  std::vector<int> par(nu, -1);
  std::vector<std::vector<int>> kids(nu);
  std::vector<double> cost(nu, 0.0), sc(nu);
  std::vector<int> usize(nu);
  for (int u = 0; u < nu; ++u) {
    usize[u] = ubeg[u + 1] - ubeg[u];
    const int hi = rows[ubeg[u + 1] - 1];
    if (!Ls[hi].empty()) {
      auto it = li.find(Ls[hi][0]);
      if (it != li.end()) par[u] = uofr[it->second];
    }
    for (int i = ubeg[u]; i < ubeg[u + 1]; ++i) cost[u] += 8.0 + (double)(Lrow[rows[i]].size() + Ls[rows[i]].size());
  }
  for (int u = 0; u < nu; ++u)
    if (par[u] >= 0) kids[par[u]].push_back(u);
  for (int u = 0; u < nu; ++u) {  // children precede parents (ascending rows)
    sc[u] = cost[u];
    for (int k : kids[u]) sc[u] += sc[k];
  }
  double total = 0;
  std::vector<int> pieces;
  for (int u = 0; u < nu; ++u)
    if (par[u] < 0) {
      pieces.push_back(u);
      total += sc[u];
    }
  const double target = total / nw;
  std::vector<char> is_top(nu, 0);
  int ntop = 0, ntop_units = 0;
  double rem = total;
  while (true) {
    int best = -1;
    for (int k = 0; k < (int)pieces.size(); ++k)
      if (best < 0 || sc[pieces[k]] > sc[pieces[best]]) best = k;
    if (best < 0 || kids[pieces[best]].empty()) break;
    if (sc[pieces[best]] <= (dual ? cut * rem / nw : cut * target)) break;
    const int p = pieces[best];
    if (ntop + usize[p] > max_tops || ntop_units >= UnitSweep::kMaxTopUnits) break;
    pieces.erase(pieces.begin() + best);
    is_top[p] = 1;
    ntop += usize[p];
    ++ntop_units;
    rem -= cost[p];
    for (int k : kids[p]) pieces.push_back(k);
  }
  std::sort(pieces.begin(), pieces.end(), [&](int x, int y) { return sc[x] > sc[y]; });
  if (getenv("RH_DEBUG_SCHED") && nw == UnitSweep::kWarps) {
    static double s_big = 0, s_tgt = 0;
    static int nblk_seen = 0;
    double rp = 0;
    for (int p : pieces) rp += sc[p];
    s_big += pieces.empty() ? 0 : sc[pieces[0]];
    s_tgt += rp / nw;
    if (++nblk_seen % 10 == 0)
      fprintf(stderr, "split: %d blocks: sum largest piece %.0f, sum remaining/nw %.0f; this block: %zu pieces, tops %d units %d rows\n",
              nblk_seen, s_big, s_tgt, pieces.size(), ntop_units, ntop);
  }
  BlockSplit B;
  // LPT of the pieces onto the warps by subtree cost w (per unit)
  auto pack = [&](const std::vector<double> &w, std::vector<std::vector<int32_t>> &out, bool post = false) {
    std::vector<double> sw(nu);
    for (int u = 0; u < nu; ++u) {
      sw[u] = w[u];
      for (int k : kids[u]) sw[u] += sw[k];
    }
    std::vector<int> pc(pieces);
    std::stable_sort(pc.begin(), pc.end(), [&](int x, int y) { return sw[x] > sw[y]; });
    std::vector<double> load(nw, 0.0);
    out.assign(nw, {});
    for (int p : pc) {
      const int wi = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      load[wi] += sw[p];
      if (post) {   // depth-first postorder: every parent right after its last child
        std::vector<std::pair<int, int>> st{{p, 0}};
        while (!st.empty()) {
          auto &[x, ci] = st.back();
          if (ci < (int)kids[x].size()) {
            const int k = kids[x][ci++];
            st.push_back({k, 0});
          } else {
            for (int i = ubeg[x]; i < ubeg[x + 1]; ++i) out[wi].push_back(rows[i]);
            st.pop_back();
          }
        }
        continue;
      }
      std::vector<int> st{p};
      while (!st.empty()) {
        const int x = st.back();
        st.pop_back();
        for (int i = ubeg[x]; i < ubeg[x + 1]; ++i) out[wi].push_back(rows[i]);
        for (int k : kids[x]) st.push_back(k);
      }
    }
    if (!post)
      for (auto &v : out) std::sort(v.begin(), v.end());  // ascending = forward topological
  };
  if (!dual) {
    pack(cost, B.warp_rows);
  } else {
    // direction costs: a fixed per-unit latency + its dependency units (fwd: L row, bwd: U row)
    constexpr double kUnitLat = 6.0;
    std::vector<double> cf(nu), cb(nu);
    std::vector<int32_t> du;
    for (int u = 0; u < nu; ++u)
      for (int dir = 0; dir < 2; ++dir) {
        du.clear();
        for (int i = ubeg[u]; i < ubeg[u + 1]; ++i)
          for (int k : dir == 0 ? Lrow[rows[i]] : Ls[rows[i]])
            if (unit_lo[k] != unit_lo[rows[ubeg[u]]]) du.push_back(unit_lo[k]);
        sort_unique(du);
        (dir == 0 ? cf : cb)[u] = kUnitLat + (double)du.size();
      }
    // unit sweeps: pieces in depth-first postorder (forward sweeps: a parent right
    // after its last child; the backward sweeps walk it reversed: a parent right
    // before one of its children), so most units forward a dependency from the
    // unit solved just before (build_units)
    const bool post = !getenv("RH_NO_POSTORDER");
    pack(cf, B.warp_rows, post);
    pack(cb, B.warp_rows_b, post);
  }
  for (int u = 0; u < nu; ++u)
    if (is_top[u])
      for (int i = ubeg[u]; i < ubeg[u + 1]; ++i) B.tops.push_back(rows[i]);
  std::sort(B.tops.begin(), B.tops.end());
  return B;
}

// ---------------------------------------------------------------------------
// Bus-unit schedule of the block sweeps of one pattern direction (UnitSweep;
// DESIGN.md "Block sweeps").  fwd: rows ascending, deps = L row (sweeps L and
// U^T); bwd: rows descending, deps = U row (sweeps U and L^T).  Sweep a takes
// the coefficient (i, k) from F(i, k), sweep b from F(k, i).
// ---------------------------------------------------------------------------
template <class FPos>
void build_units(Analysis &A, bool fwd, const std::vector<std::vector<int32_t>> &Ls,
                 const std::vector<std::vector<int32_t>> &Lrow, FPos fpos) {
  UnitSweep &U = fwd ? A.ufwd : A.ubwd;
  const SegSweep &S = fwd ? A.fwd : A.bwd;
  const int nb = A.nblk;
  U = UnitSweep();
  U.unit_off.assign(1, 0);
  U.tmeta_off.assign(1, 0);
  U.rec_off.assign(1, 0);
  U.doff_off.assign(1, 0);
  auto deps = [&](int i) -> const std::vector<int32_t> & { return fwd ? Lrow[i] : Ls[i]; };
  auto coef = [&](bool b, int i, int k) -> int {   // src code of the coefficient (row i, dep k)
    const auto &d = deps(i);
    if (!std::binary_search(d.begin(), d.end(), k)) return -1;
    return b ? fpos(k, i) : fpos(i, k);
  };
  for (int s = 0; s < nb; ++s) {
    const int r0 = A.seg_row_off[s], nr = A.seg_row_off[s + 1] - r0;
    const int x0 = S.ext_off[s], nxr = S.ext_off[s + 1] - x0;
    U.max_rows = std::max(U.max_rows, nr + nxr);
    std::unordered_map<int, int> ext_pos;   // separator row -> tile row
    for (int k = 0; k < nxr; ++k) ext_pos[S.ext_rows[x0 + k]] = nr + k;
    auto tile_row = [&](int k) { return A.seg_of[k] == s ? A.loc_of[k] : ext_pos.at(k); };
    const BlockSplit &B = A.usplit[s];
    std::vector<char> top(nr, 0);
    for (int r : B.tops) top[A.loc_of[r]] = 1;
    // units in schedule order: pieces (warp by warp, sweep order), then tops
    std::vector<std::vector<int>> units;   // rows in sweep order (first, second)
    std::vector<int> lvl;
    auto add_units = [&](std::vector<int32_t> rows) {
      if (!fwd) std::reverse(rows.begin(), rows.end());
      for (size_t i = 0; i < rows.size(); ++i) {
        const int r = rows[i];
        if (i + 1 < rows.size() && A.unit_lo[rows[i + 1]] == A.unit_lo[r]) {
          units.push_back({r, rows[i + 1]});
          ++i;
        } else {
          units.push_back({r});
        }
      }
    };
    for (int w = 0; w < UnitSweep::kWarps; ++w) {
      lvl.push_back((int)units.size());
      add_units(fwd ? B.warp_rows[w] : B.warp_rows_b[w]);
    }
    lvl.push_back((int)units.size());
    const int tu0 = (int)units.size();
    add_units(B.tops);
    const int tu1 = (int)units.size();
    lvl.push_back(tu0);
    lvl.push_back(tu1);
    lvl.push_back((int)B.tops.size());   // tops rows
    while ((int)lvl.size() < UnitSweep::kLvl) lvl.push_back(0);
    U.lvl.insert(U.lvl.end(), lvl.begin(), lvl.end());
    const int rec0 = (int)U.src_a.size() / 2, off0 = (int)U.doff.size();
    // dependency units: (first tile row, number of values)
    auto dep_units = [&](const std::vector<int> &u, bool tops_only, bool skip_tops) {
      std::vector<std::pair<int, int>> du;   // (first dependency row (permuted), values)
      std::set<int> seen;
      for (int i : u)
        for (int k : deps(i)) {
          if (std::find(u.begin(), u.end(), k) != u.end()) continue;
          const bool kt = A.seg_of[k] == s && top[A.loc_of[k]];
          if ((tops_only && !kt) || (skip_tops && kt)) continue;
          int lo = A.unit_lo[k], nv = (lo + 1 < A.n_x && A.unit_lo[lo + 1] == lo) ? 2 : 1;
          if (A.seg_of[k] != s) {   // staged separator rows: two values only if both are staged
            if (nv == 2 && !(ext_pos.count(lo) && ext_pos.count(lo + 1))) {
              lo = k;
              nv = 1;
            }
          }
          if (seen.insert(lo).second) du.push_back({lo, nv});
        }
      std::stable_sort(du.begin(), du.end(), [&](const std::pair<int, int> &a, const std::pair<int, int> &b) {
        return tile_row(a.first) < tile_row(b.first);
      });
      return du;
    };
    // emit one dependency list; returns the int4 meta; `hdr`: piece unit header
    // records.  Every dependency is a pair of tile rows (o0, o1) (byte offsets;
    // a one-value dependency repeats its row with a zero second coefficient);
    // lists hold the unit's dependencies padded to an even count (slots of two).
    auto emit = [&](const std::vector<int> &u, std::vector<std::pair<int, int>> du, bool hdr,
                    std::vector<int> *pos_rows, std::vector<int32_t> *pos_out, const std::vector<int> *prev) {
      const bool two = u.size() == 2;
      // forwarding: a dependency on the unit solved just before (same warp) is read
      // from that unit's results in registers; its coefficients go to the header
      int fw_k0 = -1, fw_nv = 0;
      bool fw_swap = false;
      if (prev && hdr) {
        const int plo = A.unit_lo[(*prev)[0]];
        for (size_t i = 0; i < du.size(); ++i)
          if (du[i].first == plo && A.seg_of[plo] == s) {
            fw_k0 = plo;
            fw_nv = du[i].second;
            fw_swap = (*prev)[0] != plo;   // the previous unit's first row is the pair's second
            du.erase(du.begin() + i);
            break;
          }
      }
      // the list starts at an even dependency (offset pairs are read as int4 per two dependencies)
      if (((int)U.doff.size() - off0) % 4) {
        U.doff.push_back(0);
        U.doff.push_back(0);
      }
      const int cbeg = (int)U.src_a.size() / 2 - rec0, obeg = (int)U.doff.size() - off0;
      auto rec = [&](int a0, int a1, int b0, int b1) {
        U.src_a.push_back(a0);
        U.src_a.push_back(a1);
        U.src_b.push_back(b0);
        U.src_b.push_back(b1);
      };
      if (hdr) {
        // (dinv_f, dinv_s): sweep a = fwd L (unit) / bwd U; sweep b = fwd U^T / bwd L^T (unit)
        auto inv = [&](int i) { return -2 - A.F_diag[i]; };
        const int f = u[0], sr = two ? u[1] : -1;
        rec(fwd ? -1 : inv(f), (!fwd && two) ? inv(sr) : -1, fwd ? inv(f) : -1, (fwd && two) ? inv(sr) : -1);
        if (two) rec(coef(false, sr, f), -1, coef(true, sr, f), -1);
        if (fw_k0 >= 0) {   // the forwarded dependency's coefficient records (as a list entry's)
          const int k0 = fw_k0, k1 = fw_nv == 2 ? fw_k0 + 1 : -1;
          auto cf = [&](bool b, int i, int k) { return k < 0 ? -1 : coef(b, i, k); };
          rec(cf(false, u[0], k0), cf(false, u[0], k1), cf(true, u[0], k0), cf(true, u[0], k1));
          if (two) rec(cf(false, u[1], k0), cf(false, u[1], k1), cf(true, u[1], k0), cf(true, u[1], k1));
        }
      }
      const int nd = (int)du.size();   // no padding to 4 (r02: lists were padded to chunks of 4)
      const int ndp = nd;               // slots of two, an odd last one alone (dep_slots)
      const int rowb = UnitSweep::kCols * 8;
      for (int di = 0; di < ndp; ++di) {
        if (di >= nd) {   // padding: zero coefficients on the unit's own (finite) row
          U.doff.push_back(A.loc_of[u[0]] * rowb);
          U.doff.push_back(A.loc_of[u[0]] * rowb);
          rec(-1, -1, -1, -1);
          if (two) rec(-1, -1, -1, -1);
          continue;
        }
        const int k0 = du[di].first, nv = du[di].second, k1 = nv == 2 ? k0 + 1 : -1;
        U.doff.push_back(tile_row(k0) * rowb);
        U.doff.push_back(tile_row(nv == 2 ? k1 : k0) * rowb);   // one-value dependency: its row again, zero coefficient
        const size_t at = U.src_a.size();
        auto cf = [&](bool b, int i, int k) { return k < 0 ? -1 : coef(b, i, k); };
        rec(cf(false, u[0], k0), cf(false, u[0], k1), cf(true, u[0], k0), cf(true, u[0], k1));
        if (two) rec(cf(false, u[1], k0), cf(false, u[1], k1), cf(true, u[1], k0), cf(true, u[1], k1));
        if (pos_rows) {   // dense tops list: record where M(row, dep) lives
          const std::vector<int> &T = *pos_rows;
          auto ti = [&](int r) { return (int)(std::lower_bound(T.begin(), T.end(), r) - T.begin()); };
          const int nt = (int)T.size();
          for (int ri = 0; ri < (int)u.size(); ++ri)
            for (int v = 0; v < nv; ++v) (*pos_out)[ti(u[ri]) * nt + ti(k0 + v)] = (int)(at + 2 * ri + v);
        }
      }
      // (x, y) tile byte offsets of the rows; z record byte offset; w offsets' byte
      // offset | ndeps << 16 | two << 30
      if (obeg * 4 >= (1 << 16) || ndp >= (1 << 13)) U.overflow = true;
      return std::array<int, 4>{A.loc_of[u[0]] * rowb, two ? A.loc_of[u[1]] * rowb : 0, cbeg * 16,
                                obeg * 4 | ndp << 16 | (fw_swap ? 1 << 29 : 0) | (two ? 1 << 30 : 0) |
                                    (fw_k0 >= 0 ? (int)(1u << 31) : 0)};
    };
    const bool fwd_prev = !getenv("RH_NO_FORWARD");
    for (int ui = 0; ui < (int)units.size(); ++ui) {
      const auto &u = units[ui];
      const bool is_top = ui >= tu0;
      bool first_of_warp = false;   // the warp's first unit has no predecessor in registers
      for (int w = 0; w <= UnitSweep::kWarps; ++w) first_of_warp |= lvl[w] == ui;
      const std::vector<int> *prev = fwd_prev && !is_top && !first_of_warp ? &units[ui - 1] : nullptr;
      const auto m = emit(u, dep_units(u, false, is_top), !is_top, nullptr, nullptr, prev);
      U.meta.insert(U.meta.end(), m.begin(), m.end());
    }
    {  // tops (dense product on the fp64 tensor cores): tile rows of the block's tops, ascending
      const std::vector<int32_t> &T = B.tops;
      for (int a = 0; a < UnitSweep::kTopRows; ++a)
        U.top_rows.push_back(T.empty() ? 0 : A.loc_of[T[a < (int)T.size() ? a : 0]]);
    }
    while (((int)U.doff.size() - off0) % 4) U.doff.push_back(0);   // 16-byte bulk copies
    U.unit_off.push_back((int)(U.meta.size() / 4));
    U.tmeta_off.push_back((int)(U.tmeta.size() / 4));
    U.rec_off.push_back((int)U.src_a.size() / 2);
    U.doff_off.push_back((int)U.doff.size());
    const int nrec = (int)U.src_a.size() / 2 - rec0, noff = (int)U.doff.size() - off0;
    U.max_units = std::max(U.max_units, (int)units.size());
    U.max_tunits = std::max(U.max_tunits, tu1 - tu0);
    U.max_rec = std::max(U.max_rec, nrec);
    U.max_doff = std::max(U.max_doff, noff);
    // scheduling weight ~ shared-memory wavefronts of one 32-column tile
    U.cost.push_back(std::max(1, 3 * nrec + noff / 8 + 6 * nr + 4 * nxr));
  }
  if (getenv("RH_DEBUG_SCHED")) {
    long long tot = 0;
    for (int c : U.cost) tot += c;
    for (int s = 0; s < nb && s < 6; ++s) {   // per-warp chain: units and records
      const int *lv = U.lvl.data() + s * UnitSweep::kLvl;
      const int ub = U.unit_off[s];
      int mu = 0, mr = 0, sr = 0;
      for (int w = 0; w < UnitSweep::kWarps; ++w) {
        int r = 0;
        for (int u = lv[w]; u < lv[w + 1]; ++u) {
          const int *m = U.meta.data() + 4 * (ub + u);
          r += ((m[3] >> 16) & 0x1fff) * ((m[3] >> 30) & 1 ? 2 : 1);
        }
        mu = std::max(mu, lv[w + 1] - lv[w]);
        mr = std::max(mr, r);
        sr += r;
      }
      fprintf(stderr, "  %s blk %d: units %d, warp max units %d, warp max records %d (mean %d), tops units %d\n",
              fwd ? "fwd" : "bwd", s, U.unit_off[s + 1] - ub, mu, mr, sr / UnitSweep::kWarps,
              lv[UnitSweep::kWarps + 2] - lv[UnitSweep::kWarps + 1]);
    }
    {  // warp balance of the pieces phase, unit cost = 6 + dependencies (latency-bound units)
      double smax = 0, smean = 0;
      for (int s = 0; s < nb; ++s) {
        const int *lv = U.lvl.data() + s * UnitSweep::kLvl;
        const int ub = U.unit_off[s];
        double mx = 0, sm = 0;
        for (int w = 0; w < UnitSweep::kWarps; ++w) {
          double c = 0;
          for (int u = lv[w]; u < lv[w + 1]; ++u) c += 6 + ((U.meta[4 * (ub + u) + 3] >> 16) & 0x1fff);
          mx = std::max(mx, c);
          sm += c;
        }
        smax += mx;
        smean += sm / UnitSweep::kWarps;
      }
      fprintf(stderr, "  %s pieces balance: sum over blocks of max-warp cost %.0f, of mean-warp cost %.0f (ratio %.3f)\n",
              fwd ? "fwd" : "bwd", smax, smean, smax / smean);
    }
    fprintf(stderr, "units %s: blocks %d max rows %d units %d tops-units %d rec %d doff %d; records %zu, cost sum %lld\n",
            fwd ? "fwd" : "bwd", nb, U.max_rows, U.max_units, U.max_tunits, U.max_rec, U.max_doff,
            U.src_a.size() / 2, tot);
    // shared-memory wavefronts of one 32-column tile (X loads 2, broadcast loads 1), mean over blocks
    long long wf_piece = 0, wf_tops = 0, deps = 0, real = 0;
    for (size_t u = 0; u < U.meta.size() / 4; ++u) {
      const int *m = U.meta.data() + 4 * u;
      const int nd = (m[3] >> 16) & 0x1fff, two = (m[3] >> 30) & 1;
      wf_piece += nd * 4 + nd * (two ? 2 : 1) + (nd + 1) / 2 + (two ? 2 : 1) + 4 * (two ? 2 : 1) + 1;
      deps += nd;
    }
    wf_tops = 16 * 2 * 8 * 4;   // DMMA: 16 output tiles x 8 k-steps x (A + B fragments)
    for (size_t i = 0; i < U.doff.size(); i += 2) real += U.doff[i] != U.doff[i + 1] || true;
    fprintf(stderr, "  smem wavefronts per tile: units+gather %lld, tops dense %lld; dep slots %lld\n",
            wf_piece / std::max(nb, 1), wf_tops / std::max(nb, 1), deps / std::max(nb, 1));
  }
}

// ---------------------------------------------------------------------------
// Tiles of the staged tensor projection (ForGroups): every bus is an output of
// the group of its theta row's segment (the REF bus, which has no theta row,
// goes with its lowest neighbour); separator buses in chunks of kMaxOut.
// ---------------------------------------------------------------------------
void build_for_groups(Analysis &A) {
  ForGroups &F = A.fg;
  F = ForGroups();
  const int n = A.n_bus, nb = A.nblk;
  std::vector<int> gseg(n, -1);   // segment of each bus
  for (int b = 0; b < n; ++b)
    if (b != A.ref) gseg[b] = A.seg_of[A.pinv[A.th_x[b]]];
  {
    int lo = -1;
    for (int s = A.bl_ptr[A.ref]; s < A.bl_ptr[A.ref + 1]; ++s)
      if (lo < 0 || A.bl_other[s] < lo) lo = A.bl_other[s];
    gseg[A.ref] = lo >= 0 ? gseg[lo] : nb;
  }
  std::vector<std::vector<int>> seg_bus(nb + 1);
  for (int b = 0; b < n; ++b) seg_bus[gseg[b]].push_back(b);
  auto theta_row = [&](int b) { return b == A.ref ? -1 : A.pinv[A.th_x[b]]; };
  for (auto &v : seg_bus)
    std::stable_sort(v.begin(), v.end(), [&](int x, int y) { return theta_row(x) < theta_row(y); });
  // greedy: a segment's buses (theta-row order) while outputs + halo fit kMaxLoc
  std::vector<std::vector<int>> groups;
  {
    std::vector<int> mark(n, -1);
    int gid = 0;
    for (int s = 0; s <= nb; ++s) {
      std::vector<int> cur;
      int nloc = 0;
      auto close = [&]() {
        if (!cur.empty()) groups.push_back(cur);
        cur.clear();
        nloc = 0;
        ++gid;
      };
      for (int b : seg_bus[s]) {
        int add = mark[b] == gid ? 0 : 1;
        for (int q = A.bl_ptr[b]; q < A.bl_ptr[b + 1]; ++q) add += mark[A.bl_other[q]] == gid ? 0 : 1;
        if (!cur.empty() && nloc + add + (int)A.near_ref.size() > ForGroups::kMaxLoc) close();
        cur.push_back(b);
        if (mark[b] != gid) ++nloc;
        mark[b] = gid;
        for (int q = A.bl_ptr[b]; q < A.bl_ptr[b + 1]; ++q)
          if (mark[A.bl_other[q]] != gid) {
            mark[A.bl_other[q]] = gid;
            ++nloc;
          }
      }
      close();
    }
  }
  std::vector<char> near(n, 0);
  for (int b : A.near_ref) near[b] = 1;
  F.grp_off.assign(1, 0);
  F.grp_obase.assign(1, 0);
  F.grp_ref.assign(1, 0);
  F.grp_sbase.assign(1, 0);
  std::vector<int> lidx(n, -1);
  for (const auto &out : groups) {
    std::vector<int> locs(out);
    for (int i = 0; i < (int)locs.size(); ++i) lidx[locs[i]] = i;
    bool has_ref = false;
    for (int b : out) {
      has_ref = has_ref || near[b];
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
        const int o = A.bl_other[s];
        if (lidx[o] < 0) {
          lidx[o] = (int)locs.size();
          locs.push_back(o);
        }
      }
    }
    if (has_ref)
      for (int o : A.near_ref)
        if (lidx[o] < 0) {
          lidx[o] = (int)locs.size();
          locs.push_back(o);
        }
    int zrows = 0;
    for (int b : locs) {
      F.loc.push_back(A.dth_src[b]);
      F.loc.push_back(A.dv_src[b]);
      F.loc.push_back(b);
      F.loc.push_back(0);
      zrows += (A.dth_src[b] >= 0) + (A.dv_src[b] >= 0);
    }
    const int sbase = (int)F.slots.size() / 2;
    for (int b : out) {
      const int first = (int)F.slots.size() / 2 - sbase;
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
        F.slots.push_back(A.bl_line[s]);
        F.slots.push_back(lidx[A.bl_other[s]] * 2 + (A.bl_end[s] ? 1 : 0));
      }
      F.out_bus.push_back(b);
      F.out_dst.push_back(A.yth_dst[b]);
      F.out_dst.push_back(A.yv_dst[b]);
      F.out_dst.push_back(first);
      F.out_dst.push_back(A.bl_ptr[b + 1] - A.bl_ptr[b]);
    }
    while ((F.slots.size() / 2) % 4) {   // pad the group's slot range to a multiple of 4
      F.slots.push_back(-1);
      F.slots.push_back(0);
    }
    F.grp_sbase.push_back((int)F.slots.size() / 2);
    F.max_slots = std::max(F.max_slots, F.grp_sbase.back() - sbase);
    if (has_ref)
      for (int o : A.near_ref) F.ref_loc.push_back(lidx[o]);
    for (int b : locs) lidx[b] = -1;
    F.grp_off.push_back(F.grp_off.back() + (int)locs.size());
    F.grp_nout.push_back((int)out.size());
    F.grp_obase.push_back(F.grp_obase.back() + (int)out.size());
    F.grp_zrows.push_back(zrows);
    F.grp_ref.push_back((int)F.ref_loc.size());
    F.max_loc = std::max(F.max_loc, (int)locs.size());
    F.max_nout = std::max(F.max_nout, (int)out.size());
  }
  if (getenv("RH_DEBUG_SCHED"))
    fprintf(stderr, "for groups %zu: max locals %d, max outputs %d, locals %zu (buses %d)\n", F.grp_nout.size(),
            F.max_loc, F.max_nout, F.loc.size() / 4, n);
}

// ---------------------------------------------------------------------------
// Elimination-tree segments (blocks of whole subtrees + the separator), the
// per-segment level schedules of the four sweeps, and the refactorization
// schedule (DESIGN.md "Sweeps" and "Refactorization").
// ---------------------------------------------------------------------------
template <class FPos>
void build_segments(Analysis &A, const std::vector<std::vector<int32_t>> &Ls,
                    const std::vector<std::vector<int32_t>> &Lrow, FPos fpos, int rmax) {
  const int nx = A.n_x;
  A.rmax = rmax;
  std::vector<int32_t> parent(nx, -1), size(nx, 1);
  for (int k = 0; k < nx; ++k)
    if (!Ls[k].empty()) parent[k] = Ls[k][0];
  for (int k = 0; k < nx; ++k)
    if (parent[k] >= 0) size[parent[k]] += size[k];
  // maximal subtrees of <= rmax rows
  std::vector<int32_t> roots;
  for (int k = 0; k < nx; ++k)
    if (size[k] <= rmax && (parent[k] < 0 || size[parent[k]] > rmax)) roots.push_back(k);
  // first-fit decreasing bin packing of the subtrees into blocks of <= rmax rows
  std::vector<int32_t> rord(roots);
  std::stable_sort(rord.begin(), rord.end(), [&](int a, int b) { return size[a] > size[b]; });
  std::vector<int32_t> bin_fill;
  std::vector<int32_t> root_bin(nx, -1);
  for (int r : rord) {
    int b = -1;
    for (size_t q = 0; q < bin_fill.size(); ++q)
      if (bin_fill[q] + size[r] <= rmax) {
        b = (int)q;
        break;
      }
    if (b < 0) {
      b = (int)bin_fill.size();
      bin_fill.push_back(0);
    }
    bin_fill[b] += size[r];
    root_bin[r] = b;
  }
  const int nb = (int)bin_fill.size();
  A.nblk = nb;
  A.seg_of.assign(nx, nb);
  for (int k = nx - 1; k >= 0; --k) {
    if (root_bin[k] >= 0)
      A.seg_of[k] = root_bin[k];
    else if (parent[k] >= 0 && A.seg_of[parent[k]] < nb)
      A.seg_of[k] = A.seg_of[parent[k]];
  }
  const int nseg = nb + 1;
  // bus units: consecutive permuted rows of one bus in one segment (theta_b, v_b)
  A.unit_lo.assign(nx, 0);
  for (int k = 0; k < nx; ++k)
    A.unit_lo[k] = (k > 0 && A.x_bus[A.perm[k]] == A.x_bus[A.perm[k - 1]] && A.seg_of[k] == A.seg_of[k - 1])
                       ? A.unit_lo[k - 1] : k;
  A.seg_row_off.assign(nseg + 1, 0);
  for (int k = 0; k < nx; ++k) A.seg_row_off[A.seg_of[k] + 1]++;
  for (int s = 0; s < nseg; ++s) A.seg_row_off[s + 1] += A.seg_row_off[s];
  A.row_global.assign(nx, 0);
  A.loc_of.assign(nx, 0);
  {
    std::vector<int32_t> fill(A.seg_row_off.begin(), A.seg_row_off.end() - 1);
    for (int k = 0; k < nx; ++k) {
      const int s = A.seg_of[k];
      A.loc_of[k] = fill[s] - A.seg_row_off[s];
      A.row_global[fill[s]++] = k;
    }
  }
  A.max_seg_rows = 0;
  for (int s = 0; s < nb; ++s) A.max_seg_rows = std::max(A.max_seg_rows, A.seg_row_off[s + 1] - A.seg_row_off[s]);
  A.sep_rows = A.seg_row_off[nseg] - A.seg_row_off[nb];

  auto build = [&](SegSweep &S, bool fwd) {
    // local levels: deps within the same segment only
    std::vector<int32_t> lv(nx, 0);
    if (fwd) {
      for (int i = 0; i < nx; ++i) {
        int l = 0;
        for (int k : Lrow[i])
          if (A.seg_of[k] == A.seg_of[i]) l = std::max(l, lv[k] + 1);
        lv[i] = l;
      }
    } else {
      for (int i = nx - 1; i >= 0; --i) {
        int l = 0;
        for (int k : Ls[i])
          if (A.seg_of[k] == A.seg_of[i]) l = std::max(l, lv[k] + 1);
        lv[i] = l;
      }
    }
    S.seg_lvl.assign(nseg + 1, 0);
    S.lvl_ptr.clear();
    S.order.clear();
    S.rptr.assign(1, 0);
    S.rext.clear();
    S.dep.clear();
    S.src_a.clear();
    S.src_b.clear();
    S.dsrc.clear();
    S.ext_off.assign(nseg + 1, 0);
    S.ext_rows.clear();
    S.max_levels = 0;
    for (int s = 0; s < nseg; ++s) {
      S.seg_lvl[s] = (int)S.lvl_ptr.size();
      std::vector<int32_t> rows(A.row_global.begin() + A.seg_row_off[s],
                                A.row_global.begin() + A.seg_row_off[s + 1]);
      const int nr_s = (int)rows.size();
      std::vector<int32_t> ext;  // blocks only: separator rows this segment depends on
      if (s < nb) {
        for (int r : rows)
          for (int k : (fwd ? Lrow[r] : Ls[r]))
            if (A.seg_of[k] != s) ext.push_back(k);
        sort_unique(ext);
      }
      S.ext_off[s] = (int)S.ext_rows.size();
      S.ext_rows.insert(S.ext_rows.end(), ext.begin(), ext.end());
      auto ext_local = [&](int k) -> int {
        auto it = std::lower_bound(ext.begin(), ext.end(), k);
        return nr_s + (int)(it - ext.begin());
      };
      std::stable_sort(rows.begin(), rows.end(), [&](int a, int b) { return lv[a] < lv[b]; });
      int nl = 0;
      for (int r : rows) nl = std::max(nl, lv[r] + 1);
      S.max_levels = std::max(S.max_levels, nl);
      const int qbase = (int)S.order.size();
      std::vector<char> top_row;  // blocks: membership in the block's tops, by local index
      if (s < nb) {
        // blocks: [warp pieces] + [tops] (forward) or [tops] + [warp pieces] (backward);
        // lvl entries: nw + 1 piece bounds, then the tops' [begin, end)
        const BlockSplit &B = A.split[s];
        std::vector<int32_t> ord;
        std::vector<int32_t> pb(kSchedWarps + 1, 0), tb(2, 0);
        auto add_pieces = [&]() {
          for (int w = 0; w < kSchedWarps; ++w) {
            pb[w] = (int)ord.size();
            if (fwd)
              ord.insert(ord.end(), B.warp_rows[w].begin(), B.warp_rows[w].end());
            else
              ord.insert(ord.end(), B.warp_rows[w].rbegin(), B.warp_rows[w].rend());
          }
          pb[kSchedWarps] = (int)ord.size();
        };
        auto add_tops = [&]() {
          tb[0] = (int)ord.size();
          ord.insert(ord.end(), B.tops.begin(), B.tops.end());   // dense phase: any order
          tb[1] = (int)ord.size();
        };
        if (fwd) {
          add_pieces();
          add_tops();
        } else {
          add_tops();
          add_pieces();
        }
        rows = ord;
        for (int b : pb) S.lvl_ptr.push_back(qbase + b);
        for (int b : tb) S.lvl_ptr.push_back(qbase + b);
        top_row.assign(nr_s, 0);
        for (int r : B.tops) top_row[A.loc_of[r]] = 1;
      } else {
        std::vector<int32_t> cnt(nl + 1, 0);
        for (int r : rows) cnt[lv[r] + 1]++;
        for (int l = 0; l < nl; ++l) cnt[l + 1] += cnt[l];
        for (int l = 0; l <= nl; ++l) S.lvl_ptr.push_back(qbase + cnt[l]);
      }
      if (fwd) {  // level order of every segment for the refactorization (R_A)
        A.fact_seg_lvl.push_back((int)A.fact_lvl_ptr.size());
        std::vector<int32_t> lrows(rows);
        std::stable_sort(lrows.begin(), lrows.end(), [&](int a, int b) { return lv[a] < lv[b]; });
        std::vector<int32_t> cnt(nl + 1, 0);
        for (int r : lrows) cnt[lv[r] + 1]++;
        for (int l = 0; l < nl; ++l) cnt[l + 1] += cnt[l];
        const int fb = (int)A.fact_order.size();
        for (int l = 0; l <= nl; ++l) A.fact_lvl_ptr.push_back(fb + cnt[l]);
        for (int r : lrows) A.fact_order.push_back(A.loc_of[r]);
      }
      auto pad4 = [&](int r) {  // blocks: pad to a multiple of 4 entries (coefficient 0, own row)
        while ((S.dep.size() - S.rptr.back()) % 4 != 0) {
          S.dep.push_back(A.loc_of[r]);
          S.src_a.push_back(-1);
          S.src_b.push_back(-1);
        }
      };
      for (int r : rows) {
        S.order.push_back(A.loc_of[r]);
        const std::vector<int32_t> &deps = fwd ? Lrow[r] : Ls[r];
        const bool is_top = s < nb && top_row[A.loc_of[r]];
        if (s < nb) {
          // blocks: local (and staged separator) entries; a top row keeps only its entries
          // outside the tops, then gets one dense entry per top row (values: k_tops_inverse)
          for (int k : deps) {
            if (is_top && A.seg_of[k] == s && top_row[A.loc_of[k]]) continue;
            S.dep.push_back(A.seg_of[k] == s ? A.loc_of[k] : ext_local(k));
            S.src_a.push_back(fpos(r, k));   // fwd: L[r,k]  bwd: U[r,k]
            S.src_b.push_back(fpos(k, r));   // fwd: U[k,r]  bwd: L[k,r]
          }
          pad4(r);
          S.rext.push_back((int)S.dep.size());   // blocks: start of the dense (tops) entries
          if (is_top) {
            (fwd ? A.top_fwd_base : A.top_bwd_base).push_back((int)S.dep.size());
            for (int j : A.split[s].tops) {
              S.dep.push_back(A.loc_of[j]);
              S.src_a.push_back(-1);
              S.src_b.push_back(-1);
            }
            pad4(r);
          }
        } else {
          // separator: external entries first (grouped by block, then row: a Cartesian
          // batch's gather skips whole blocks), then local
          std::vector<int32_t> ord(deps.begin(), deps.end());
          std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
            return A.seg_of[a] != A.seg_of[b] ? A.seg_of[a] < A.seg_of[b] : a < b;
          });
          for (int pass = 0; pass < 2; ++pass) {
            for (int k : ord) {
              const bool local = A.seg_of[k] == s;
              if (local != (pass == 1)) continue;
              S.dep.push_back(local ? A.loc_of[k] : k);
              S.src_a.push_back(fpos(r, k));
              S.src_b.push_back(fpos(k, r));
            }
            if (pass == 0) S.rext.push_back((int)S.dep.size());
          }
        }
        S.rptr.push_back((int)S.dep.size());
        S.dsrc.push_back(A.F_diag[r]);
      }
    }
    S.seg_lvl[nseg] = (int)S.lvl_ptr.size();
    S.ext_off[nseg] = (int)S.ext_rows.size();
    if (fwd) A.fact_seg_lvl.push_back((int)A.fact_lvl_ptr.size());
  };
  A.fact_seg_lvl.clear();
  A.fact_lvl_ptr.clear();
  A.fact_order.clear();
  // subtree-to-warp split of every block (shared by both directions and R_A)
  A.split.assign(nb, BlockSplit());
  int tops_cap = kMaxTops;
  if (const char *env = getenv("RH_TOPS")) tops_cap = std::max(0, std::min(kMaxTops, atoi(env)));  // tuning override
  for (int s = 0; s < nb; ++s) {
    std::vector<int32_t> rows(A.row_global.begin() + A.seg_row_off[s], A.row_global.begin() + A.seg_row_off[s + 1]);
    A.split[s] = split_block(rows, A.unit_lo, Ls, Lrow, kSchedWarps, tops_cap);
  }
  A.usplit.assign(nb, BlockSplit());
  double ucut = 1.0;
  if (const char *env = getenv("RH_CUT")) ucut = atof(env);   // tuning override
  for (int s = 0; s < nb; ++s) {
    std::vector<int32_t> rows(A.row_global.begin() + A.seg_row_off[s], A.row_global.begin() + A.seg_row_off[s + 1]);
    A.usplit[s] = split_block(rows, A.unit_lo, Ls, Lrow, UnitSweep::kWarps, tops_cap, true, ucut);
  }
  A.top_fwd_base.clear();
  A.top_bwd_base.clear();
  build(A.fwd, true);
  build(A.bwd, false);
  if (getenv("RH_DEBUG_SCHED")) {  // tuning aid: per-block chain lengths (rows, 4-entry groups)
    for (const SegSweep *S : {&A.fwd, &A.bwd}) {
      long long worst = 0, sum = 0;
      for (int s = 0; s < nb; ++s) {
        const int *lv = S->lvl_ptr.data() + S->seg_lvl[s];
        int mr = 0, mg = 0;
        for (int w = 0; w < kSchedWarps; ++w) {
          int g = 0;
          for (int q = lv[w]; q < lv[w + 1]; ++q) g += (S->rext[q] - S->rptr[q]) / 4;
          mr = std::max(mr, lv[w + 1] - lv[w]);
          mg = std::max(mg, g);
        }
        const int nt = lv[kSchedWarps + 2] - lv[kSchedWarps + 1];
        int tg = 0;
        for (int q = lv[kSchedWarps + 1]; q < lv[kSchedWarps + 2]; ++q) tg = std::max(tg, (S->rext[q] - S->rptr[q]) / 4);
        const long long est = 60LL * mr + 40LL * mg + (nt ? 1000 + 40LL * tg + 40LL * ((nt + 3) / 4) * ((nt + 15) / 16) : 0);
        // shared-memory wavefronts at 64 columns: per row meta + ldx(4) + stx(4) + dinv; per group 4 ent + 16 X
        const int qa = A.seg_row_off[s], qz = A.seg_row_off[s + 1];
        const long long wf = 10LL * (qz - qa) + 20LL * (S->rptr[qz] - S->rptr[qa]) / 4;
        worst = std::max(worst, est);
        sum += est;
        if (s < 4 || getenv("RH_DEBUG_SCHED")[0] == '2')
          fprintf(stderr, "%s blk %d rows %d: warp max rows %d groups %d | tops %d outer-groups %d | est %lld cyc | smem wavefronts %lld (entries %d)\n",
                  S == &A.fwd ? "fwd" : "bwd", s, qz - qa, mr, mg, nt, tg, est, wf, S->rptr[qz] - S->rptr[qa]);
      }
      fprintf(stderr, "%s: est worst %lld mean %lld cycles\n", S == &A.fwd ? "fwd" : "bwd", worst, sum / std::max(nb, 1));
    }
  }
  build_units(A, true, Ls, Lrow, fpos);
  build_units(A, false, Ls, Lrow, fpos);
  // tops of every block for k_tops_inverse: rows and F positions of T x T
  A.top_ptr.assign(nb + 1, 0);
  A.top_rows.clear();
  A.top_fpos.clear();
  A.top_fpos_ptr.assign(nb + 1, 0);
  A.max_tops = 0;
  for (int s = 0; s < nb; ++s) {
    const auto &T = A.usplit[s].tops;
    A.top_rows.insert(A.top_rows.end(), T.begin(), T.end());
    A.top_ptr[s + 1] = (int)A.top_rows.size();
    for (int x : T)
      for (int y : T) A.top_fpos.push_back(fpos(x, y));
    A.top_fpos_ptr[s + 1] = (int)A.top_fpos.size();
    A.max_tops = std::max(A.max_tops, (int)T.size());
  }
  A.blk_gp_ptr.assign(nb + 1, 0);
  A.blk_gp_loc.clear();
  for (int s = 0; s < nb; ++s) {
    for (int q = A.seg_row_off[s]; q < A.seg_row_off[s + 1]; ++q) {
      const int r = A.row_global[q];
      if (A.gp_rptr[r + 1] > A.gp_rptr[r]) A.blk_gp_loc.push_back(q - A.seg_row_off[s]);
    }
    A.blk_gp_ptr[s + 1] = (int)A.blk_gp_loc.size();
  }
  A.gpe_off.assign(1, 0);
  A.gpe_row.clear();
  A.gpe_col.clear();
  A.gpe_src.clear();
  A.gpe_split.clear();
  A.max_gpe = 0;
  for (int s = 0; s < nb; ++s) {
    const int e0 = (int)A.gpe_src.size();
    std::vector<int> row_start;   // block-relative entry index of every row's first entry
    for (int q = A.seg_row_off[s]; q < A.seg_row_off[s + 1]; ++q) {
      const int r = A.row_global[q];
      if (A.gp_rptr[r + 1] == A.gp_rptr[r]) continue;
      row_start.push_back((int)A.gpe_src.size() - e0);
      for (int e = A.gp_rptr[r]; e < A.gp_rptr[r + 1]; ++e) {
        A.gpe_row.push_back((q - A.seg_row_off[s]) * UnitSweep::kCols * 8);
        A.gpe_col.push_back(A.gp_col[e]);
        A.gpe_src.push_back(e);
      }
    }
    const int ne = (int)A.gpe_src.size() - e0;
    A.max_gpe = std::max(A.max_gpe, ne);
    // 8 warp ranges, balanced by entries, split at row starts
    std::vector<int> sp(UnitSweep::kWarps + 1, ne);
    sp[0] = 0;
    for (int w = 1; w < UnitSweep::kWarps; ++w) {
      const int target = (int)((long long)ne * w / UnitSweep::kWarps);
      auto it = std::lower_bound(row_start.begin(), row_start.end(), target);
      sp[w] = it == row_start.end() ? ne : *it;
      sp[w] = std::max(sp[w], sp[w - 1]);
    }
    for (int w = 0; w <= UnitSweep::kWarps; ++w) A.gpe_split.push_back(sp[w]);
    while (A.gpe_split.size() % 12) A.gpe_split.push_back(0);
    A.gpe_off.push_back((int)A.gpe_src.size());
  }

  // ---------------- refactorization schedule ----------------
  // R_A: block rows staged in shared memory (local order), up-looking per row.
  A.blk_fo_off.assign(nb + 1, 0);
  A.fo.clear();
  A.max_blk_fnnz = 0;
  std::vector<int32_t> fo_of(nx, -1);
  for (int s = 0; s < nb; ++s) {
    A.blk_fo_off[s] = (int)A.fo.size();
    int off = 0;
    for (int q = A.seg_row_off[s]; q < A.seg_row_off[s + 1]; ++q) {
      const int r = A.row_global[q];
      fo_of[r] = off;
      A.fo.push_back(off);
      off += A.F_rowptr[r + 1] - A.F_rowptr[r];
    }
    A.fo.push_back(off);
    A.max_blk_fnnz = std::max(A.max_blk_fnnz, off);
  }
  A.blk_fo_off[nb] = (int)A.fo.size();
  // k-steps in SEGMENT order (q = position in row_global): a block's k-steps and
  // target offsets are contiguous, so R_A stages them in shared memory
  A.ks_ptr.assign(nx + 1, 0);
  A.ks4.clear();
  A.ks_k.clear();
  A.tgt16.clear();
  A.max_blk_ks = A.max_blk_tgt = 0;
  for (int q = 0; q < nx; ++q) {
    const int i = A.row_global[q];
    const int si = A.seg_of[i];
    const int rb = A.F_rowptr[i];
    for (int k : Lrow[i]) {
      const int sk = A.seg_of[k];
      if (si == nb && sk == nb) continue;  // separator x separator: dense Gauss-Jordan
      const int ub = A.F_diag[k] + 1, ue = A.F_rowptr[k + 1];
      const int kf = si < nb ? fo_of[k] + (A.F_diag[k] - A.F_rowptr[k]) : A.F_diag[k];
      A.ks4.push_back(fpos(i, k) - rb);
      A.ks4.push_back(kf);
      A.ks4.push_back(ue - ub);
      A.ks4.push_back((int)A.tgt16.size());
      A.ks_k.push_back(si < nb ? A.loc_of[k] : k);
      for (int u = ub; u < ue; ++u) A.tgt16.push_back((uint16_t)(fpos(i, A.F_col[u]) - rb));
    }
    A.ks_ptr[q + 1] = (int)A.ks_k.size();
  }
  for (int s = 0; s < nb; ++s) {
    const int q0 = A.seg_row_off[s], q1 = A.seg_row_off[s + 1];
    const int k0 = A.ks_ptr[q0], k1 = A.ks_ptr[q1];
    A.max_blk_ks = std::max(A.max_blk_ks, k1 - k0);
    if (k1 > k0) {
      const int t0 = A.ks4[4 * k0 + 3];
      const int t1 = A.ks4[4 * (k1 - 1) + 3] + A.ks4[4 * (k1 - 1) + 2];
      A.max_blk_tgt = std::max(A.max_blk_tgt, t1 - t0);
    }
  }
  // R_B2: separator x separator entries, right-looking in separator order
  const int sb0 = A.seg_row_off[nb];
  const int ns = A.sep_rows;
  std::vector<std::vector<std::pair<int, int>>> srow(ns);  // (global col, slot)
  A.sb_src.clear();
  for (int a = 0; a < ns; ++a) {
    const int i = A.row_global[sb0 + a];
    for (int e = A.F_rowptr[i]; e < A.F_rowptr[i + 1]; ++e) {
      const int j = A.F_col[e];
      if (A.seg_of[j] == nb) {
        srow[a].push_back({j, (int)A.sb_src.size()});
        A.sb_src.push_back(e);
      }
    }
  }
  // dense position (row-major, ns x ns) of every separator x separator entry
  A.sb_dense.assign(A.sb_src.size(), 0);
  for (int a = 0; a < ns; ++a)
    for (auto &pr : srow[a]) A.sb_dense[pr.second] = a * ns + A.loc_of[pr.first];
}

}  // namespace

// epilogue partial runs (Analysis::RunRecs): per block, its runs packed onto
// the k_blk warps by LPT on their entry counts (+ a per-run latency)
struct PRun {
  int g;
  std::vector<std::pair<int, int>> ent;   // (coefficient source, tile byte offset)
};
void build_run_recs(Analysis::RunRecs &R, const std::vector<std::vector<PRun>> &per, int nruns) {
  constexpr int kHdr = 3;   // header slots: 12 ints, warp w's runs are run slots [wr[w], wr[w + 1])
  const int nb = (int)per.size();
  R = Analysis::RunRecs();
  R.nruns = nruns;
  R.off.assign(nb + 1, 0);
  for (int b = 0; b < nb; ++b) {
    const int base = R.off[b], nr = (int)per[b].size();
    std::vector<int> ord(nr), wof(nr);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return per[b][x].ent.size() > per[b][y].ent.size(); });
    std::vector<long long> load(UnitSweep::kWarps, 0);
    for (int i : ord) {
      const int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      load[w] += 4 + (long long)per[b][i].ent.size();
      wof[i] = w;
    }
    std::vector<const PRun *> runs;
    std::vector<int> wr(kHdr * 4, 0);
    for (int w = 0; w < UnitSweep::kWarps; ++w) {
      wr[w] = (int)runs.size();
      for (int i = 0; i < nr; ++i)
        if (wof[i] == w) runs.push_back(&per[b][i]);
    }
    wr[UnitSweep::kWarps] = (int)runs.size();
    if (nr) R.init.insert(R.init.end(), wr.begin(), wr.end());
    int k = base + (nr ? kHdr : 0) + nr;   // first entry slot
    for (const PRun *r : runs) {
      R.init.insert(R.init.end(), {r->g, k - base, (int)r->ent.size(), 0});
      for (const auto &en : r->ent) {
        R.ent_slot.push_back(k++);
        R.ent_src.push_back(en.first);
        R.ent_trow.push_back(en.second);
      }
    }
    R.init.resize(4 * (size_t)k, 0);
    R.off[b + 1] = k;
  }
}

std::string analyze(const ::rh_grid &g, Analysis &A, int rmax) {
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

  // ---------------- incidence owners; slot uniqueness (two-kernel assembly) ----------------
  {
    A.bl_bus.assign(2 * m, -1);
    for (int b = 0; b < n; ++b)
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) A.bl_bus[s] = b;
    std::vector<int32_t> seen;
    for (int v : A.slot_pos)
      if (v >= 0) seen.push_back(v);
    const size_t nf = seen.size();
    sort_unique(seen);
    bool uniq = seen.size() == nf;
    seen.clear();
    for (int v : A.gp_slot_pos)
      if (v >= 0) seen.push_back(v);
    const size_t ng = seen.size();
    sort_unique(seen);
    uniq = uniq && seen.size() == ng;
    seen.clear();
    if (A.ref >= 0) {
      for (int s = A.bl_ptr[A.ref]; s < A.bl_ptr[A.ref + 1]; ++s) seen.push_back(A.bl_other[s]);
      const size_t nr = seen.size();
      sort_unique(seen);
      uniq = uniq && seen.size() == nr;
    }
    A.asm_unique = uniq;
  }

  // ---------------- column coloring of [J | G_p] (NEXT-4) ----------------
  // Columns: x entries, then p entries (R-C1).  Structural rows (natural residual
  // rows) of a theta_o / v_o column: the P / Q rows of o and its neighbours; of a
  // Pg_o column: P_o (R-C2).  Greedy: each column takes the smallest color unused
  // by its conflicting predecessors.
  {
    const int np_ = A.n_p, ncol = nx + np_;
    std::vector<std::vector<int32_t>> nbr(n);
    for (int b = 0; b < n; ++b) {
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) nbr[b].push_back(A.bl_other[s]);
      nbr[b].push_back(b);
      sort_unique(nbr[b]);
    }
    std::vector<std::vector<int32_t>> crow(ncol);
    auto bus_rows = [&](int o, std::vector<int32_t> &out) {
      out.clear();
      for (int c : nbr[o]) {
        if (A.th_x[c] >= 0) out.push_back(A.th_x[c]);
        if (A.v_x[c] >= 0) out.push_back(A.v_x[c]);
      }
    };
    for (int j = 0; j < nx; ++j) bus_rows(A.x_bus[j], crow[j]);
    for (int k = 0; k < np_; ++k) {
      if (A.p_kind[k] == RH_KIND_PG) crow[nx + k] = {A.th_x[A.p_bus[k]]};
      else bus_rows(A.p_bus[k], crow[nx + k]);
    }
    std::vector<std::vector<int32_t>> row_cols(nx);
    std::vector<int32_t> stamp(ncol + 1, -1);
    A.colors.assign(ncol, -1);
    A.ncolors = 0;
    for (int j = 0; j < ncol; ++j) {
      for (int r : crow[j])
        for (int k : row_cols[r]) stamp[A.colors[k]] = j;
      int c = 0;
      while (stamp[c] == j) ++c;
      A.colors[j] = c;
      A.ncolors = std::max(A.ncolors, c + 1);
      for (int r : crow[j]) row_cols[r].push_back(j);
    }
    A.col_th.assign(n, -1);
    A.col_v.assign(n, -1);
    A.col_pg.assign(n, -1);
    for (int b = 0; b < n; ++b) {
      if (A.th_x[b] >= 0) A.col_th[b] = A.colors[A.th_x[b]];
      if (A.v_x[b] >= 0) A.col_v[b] = A.colors[A.v_x[b]];
      else if (A.v_p[b] >= 0) A.col_v[b] = A.colors[nx + A.v_p[b]];
      if (A.pg_p[b] >= 0) A.col_pg[b] = A.colors[nx + A.pg_p[b]];
    }
    // decompression entries: F (J) and G_p positions with their row and column color
    A.jd_pos.clear(); A.jd_row.clear(); A.jd_col.clear();
    A.gd_pos.clear(); A.gd_row.clear(); A.gd_col.clear();
    auto addj = [&](int pos, int row, int color) {
      if (pos < 0) return;
      A.jd_pos.push_back(pos); A.jd_row.push_back(row); A.jd_col.push_back(color);
    };
    auto addg = [&](int pos, int row, int color) {
      if (pos < 0) return;
      A.gd_pos.push_back(pos); A.gd_row.push_back(row); A.gd_col.push_back(color);
    };
    for (int b = 0; b < n; ++b) {
      if (b == A.ref) continue;
      const int rP = A.th_x[b], rQ = A.v_x[b];
      addj(A.diag_pos[4 * b + 0], rP, A.col_th[b]);
      if (rQ >= 0) {
        addj(A.diag_pos[4 * b + 1], rP, A.col_v[b]);
        addj(A.diag_pos[4 * b + 2], rQ, A.col_th[b]);
        addj(A.diag_pos[4 * b + 3], rQ, A.col_v[b]);
      }
      addg(A.gp_self_pos[b], rP, A.col_v[b]);
      addg(A.gp_pg_pos[b], rP, A.col_pg[b]);
      for (int s = A.bl_ptr[b]; s < A.bl_ptr[b + 1]; ++s) {
        const int o = A.bl_other[s];
        addj(A.slot_pos[4 * s + 0], rP, A.col_th[o]);
        addj(A.slot_pos[4 * s + 1], rP, A.col_v[o]);
        if (rQ >= 0) {
          addj(A.slot_pos[4 * s + 2], rQ, A.col_th[o]);
          addj(A.slot_pos[4 * s + 3], rQ, A.col_v[o]);
        }
        addg(A.gp_slot_pos[2 * s + 0], rP, A.col_v[o]);
        if (rQ >= 0) addg(A.gp_slot_pos[2 * s + 1], rQ, A.col_v[o]);
      }
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
  build_segments(A, Ls, Lrow, fpos, rmax);
  if (A.ufwd.overflow || A.ubwd.overflow) return "block sweep schedule exceeds its 16-bit offset encoding";
  {  // epilogue partial runs of the U^T and L^T sweeps (analysis.hpp RunRecs)
    const int rowb = UnitSweep::kCols * 8;
    // separator rows' external entries, runs of one block in separator-row order
    std::vector<std::vector<PRun>> per(A.nblk);
    const int qb = A.fwd.lvl_ptr[A.fwd.seg_lvl[A.nblk]], qe = A.fwd.lvl_ptr[A.fwd.seg_lvl[A.nblk + 1] - 1];
    int g = 0;
    for (int q = qb; q < qe; ++q) {
      int e = A.fwd.rptr[q];
      while (e < A.fwd.rext[q]) {
        const int b = A.seg_of[A.fwd.dep[e]];
        PRun r{g++, {}};
        for (; e < A.fwd.rext[q] && A.seg_of[A.fwd.dep[e]] == b; ++e) r.ent.push_back({e, A.loc_of[A.fwd.dep[e]] * rowb});
        per[b].push_back(std::move(r));
      }
    }
    build_run_recs(A.sr, per, g);
    // G_p columns' block entries, runs of one block per column (blocks ascending)
    per.assign(A.nblk, {});
    A.ma_run_ptr.assign(1, 0);
    A.ma_sep_ptr.assign(1, 0);
    A.ma_sep_q.clear();
    g = 0;
    for (int j = 0; j < A.n_p; ++j) {
      std::vector<std::pair<int, int>> bq;   // (block, q) of the column's block entries, CSC order within a block
      for (int q = A.gpc_ptr[j]; q < A.gpc_ptr[j + 1]; ++q) {
        const int sg = A.seg_of[A.gpc_row[q]];
        if (sg == A.nblk) A.ma_sep_q.push_back(q);
        else bq.push_back({sg, q});
      }
      std::stable_sort(bq.begin(), bq.end(), [](const std::pair<int, int> &x, const std::pair<int, int> &y) { return x.first < y.first; });
      for (size_t i = 0; i < bq.size();) {
        const int b = bq[i].first;
        PRun r{g++, {}};
        for (; i < bq.size() && bq[i].first == b; ++i) r.ent.push_back({bq[i].second, A.loc_of[A.gpc_row[bq[i].second]] * rowb});
        per[b].push_back(std::move(r));
      }
      A.ma_run_ptr.push_back(g);
      A.ma_sep_ptr.push_back((int)A.ma_sep_q.size());
    }
    build_run_recs(A.ma, per, g);
  }
  if (getenv("RH_DEBUG_SCHED")) {   // separator gather statistics
    const int qb = A.fwd.lvl_ptr[A.fwd.seg_lvl[A.nblk]], qe = A.fwd.lvl_ptr[A.fwd.seg_lvl[A.nblk + 1] - 1];
    long long ext = 0, loc = 0, runs = 0;
    std::set<int> rows;
    for (int q = qb; q < qe; ++q) {
      for (int e = A.fwd.rptr[q]; e < A.fwd.rext[q]; ++e) {
        rows.insert(A.fwd.dep[e]);
        if (e == A.fwd.rptr[q] || A.seg_of[A.fwd.dep[e]] != A.seg_of[A.fwd.dep[e - 1]]) ++runs;
      }
      ext += A.fwd.rext[q] - A.fwd.rptr[q];
      loc += A.fwd.rptr[q + 1] - A.fwd.rext[q];
    }
    {
      std::vector<long long> pb(A.nblk, 0), rb(A.nblk, 0);
      long long mxrun = 0, n32 = 0;
      for (int q = qb; q < qe; ++q) {
        int e = A.fwd.rptr[q];
        while (e < A.fwd.rext[q]) {
          int f = e;
          const int b = A.seg_of[A.fwd.dep[e]];
          while (f < A.fwd.rext[q] && A.seg_of[A.fwd.dep[f]] == b) ++f;
          pb[b] += f - e;
          rb[b]++;
          mxrun = std::max<long long>(mxrun, f - e);
          if (f - e > 32) n32 += f - e - 32;
          e = f;
        }
      }
      {
      long long runs = 0, single = 0, sepent = 0, ent = 0;
      for (int j = 0; j < A.n_p; ++j) {
        std::set<int> sg;
        for (int q = A.gpc_ptr[j]; q < A.gpc_ptr[j + 1]; ++q) {
          const int sgm = A.seg_of[A.gpc_row[q]];
          sg.insert(sgm);
          ++ent;
          if (sgm == A.nblk) ++sepent;
        }
        runs += (long long)sg.size() - (sg.count(A.nblk) ? 1 : 0);
        single += sg.size() == 1 && !sg.count(A.nblk);
      }
      fprintf(stderr, "G_p columns: %d, entries %lld (separator %lld), block runs %lld, single-block columns %lld\n", A.n_p, ent,
              sepent, runs, single);
    }
    fprintf(stderr, "separator runs: max entries per block %lld, max runs per block %lld, max run %lld, entries beyond 32 %lld\n",
              *std::max_element(pb.begin(), pb.end()), *std::max_element(rb.begin(), rb.end()), mxrun, n32);
    }
    fprintf(stderr, "separator: rows %d, external entries %lld (distinct block rows %zu, runs %lld), local entries %lld, S slots %zu\n",
            qe - qb, ext, rows.size(), runs, loc, A.sb_src.size());
  }
  build_for_groups(A);
  return "";
}

}  // namespace rh
