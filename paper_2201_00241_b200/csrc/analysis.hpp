// Host-side setup (once per grid): validation, index maps, patterns, ordering,
// symbolic LU with static diagonal pivots, level sets, sweep tables.
// SURVEY.md 8(a)-1; PAPER.md:758-767 ("LU factorization ... precomputed on the
// host, and transfers it to the device"; refactorization reuses the pattern).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/redhess.h"

namespace rh {

struct Sweep {
  // Rows in level order; entries of each row in CSR (level order).
  // col[] holds permuted row indices of the dependencies, src[] the position
  // of the coefficient in the F (= L+U) value array.
  std::vector<int32_t> lev_ptr;   // [nlev + 1] into rows
  std::vector<int32_t> rows;      // [n] permuted row ids, level order
  std::vector<int32_t> rptr;      // [n + 1] into col/src, level order
  std::vector<int32_t> col;       // [nnz]
  std::vector<int32_t> src;       // [nnz] F positions
  std::vector<int32_t> diag_src;  // [n] F position of the pivot of rows[i] (or -1: unit)
  int nlev() const { return (int)lev_ptr.size() - 1; }
};

struct Analysis {
  // ---------------- grid copy ----------------
  int n_bus = 0, n_line = 0, n_gen = 0, ref = -1;
  std::vector<int32_t> bus_type, line_f, line_t;
  std::vector<double> G_ii, B_ii, Pd, Qd, G_ft, B_ft, G_tf, B_tf;
  std::vector<double> c2b, c1b, c0b;   // per-bus cost (0 if no generator)
  std::vector<int32_t> has_gen;        // per bus
  double theta_ref = 0.0;

  // ---------------- maps (R3, R5) ----------------
  int n_x = 0, n_p = 0;
  std::vector<int32_t> x_bus, x_kind, p_bus, p_kind;
  std::vector<int32_t> th_x, v_x, v_p, pg_p;  // per bus, -1 if none

  // bus -> incident line CSR (slots); end = 0 if bus is the line's from-end
  std::vector<int32_t> bl_ptr, bl_line, bl_other, bl_end;

  // ---------------- ordering + symbolic ----------------
  std::vector<int32_t> perm, pinv;          // perm[new] = old x index
  std::vector<int32_t> F_rowptr, F_col;     // L+U pattern, permuted, sorted
  std::vector<int32_t> F_diag;              // position of the diagonal in each row
  std::vector<int32_t> lev_fwd, lev_bwd;    // per permuted row
  int nlev_fwd = 0, nlev_bwd = 0, max_level_rows = 0;
  int nnz_J = 0;
  std::vector<int32_t> J_rowptr, J_col;     // natural-order J pattern (diagnostics)

  // ---------------- assembly maps (F positions) ----------------
  // per bus: F positions of (P_b,th_b), (P_b,v_b), (Q_b,th_b), (Q_b,v_b); -1 if absent
  std::vector<int32_t> diag_pos;            // [n_bus * 4]
  // per incident slot s (bus b, other end o): (P_b,th_o), (P_b,v_o), (Q_b,th_o), (Q_b,v_o)
  std::vector<int32_t> slot_pos;            // [2 n_line * 4]
  // G_p CSR over permuted rows; values assembled per bus
  std::vector<int32_t> gp_rptr, gp_col;     // [n_x + 1], [nnz_Gp] (p column index)
  std::vector<int32_t> gp_self_pos;         // per bus: position of (P_b, v_p[b]) if b PV else -1
  std::vector<int32_t> gp_pg_pos;           // per bus: position of (P_b, Pg_b) if b PV else -1
  std::vector<int32_t> gp_slot_pos;         // [2 n_line * 2]: (P_b, v_o), (Q_b, v_o)
  // G_p CSC (by p column): positions into gp value array and permuted rows
  std::vector<int32_t> gpc_ptr, gpc_pos, gpc_row;

  // refactorization schedule: rows in forward level order
  std::vector<int32_t> fact_order;

  // the four sweeps
  Sweep sL, sU, sUt, sLt;

  // FoR delta sources: >=0 row of Z (permuted), <=-2 row -(s+2) of W, -1 zero
  std::vector<int32_t> dth_src, dv_src;     // per bus
  // outputs: >= 0 permuted row of -Y_x ; <= -2 row -(d+2) of Y_p ; -1 none
  std::vector<int32_t> yth_dst, yv_dst;     // per bus
  std::vector<int32_t> near_ref;            // buses b in {ref} u A(ref) (unique)
};

// Returns "" on success, else an error message (grid rejected).
std::string analyze(const ::rh_grid &g, Analysis &A);

}  // namespace rh
