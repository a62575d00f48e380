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

// Segment decomposition of the elimination tree:
// segments 0..nblk-1 are BLOCKS (unions of whole subtrees of <= Rmax rows);
// segment nblk is the SEPARATOR (the rows above the blocks).  A block row
// depends (forward: L, U^T) only on rows of its own block; backward (U, L^T)
// on its block and the separator.  A separator row depends forward on blocks
// and the separator, backward only on the separator.
struct SegSweep {
  std::vector<int32_t> lvl_ptr;   // per segment s: lvl_ptr[seg_lvl[s] .. seg_lvl[s+1]-1] = level bounds (into q)
  std::vector<int32_t> seg_lvl;   // [nseg + 1]
  std::vector<int32_t> order;     // [n_x] q -> local row index within the segment
  std::vector<int32_t> rptr;      // [n_x + 1] q -> entry range: [rptr[q], rext[q]) external, [rext[q], rptr[q+1]) local
  std::vector<int32_t> rext;      // [n_x]
  std::vector<int32_t> dep;       // [nnz] local: index in the same segment; external: global permuted row
  std::vector<int32_t> src_a;     // [nnz] F position, first sweep (fwd: L[i,k];  bwd: U[i,k])
  std::vector<int32_t> src_b;     // [nnz] F position, second sweep (fwd: U[k,i]; bwd: L[k,i])
  std::vector<int32_t> dsrc;      // [n_x] F position of the pivot of row (q)
  // blocks: the separator rows a block's sweep depends on are staged next to the
  // block's own rows (local indices nr .. nr + n_ext - 1), so block sweeps have
  // no external entries; the separator keeps external (global-row) entries.
  std::vector<int32_t> ext_off;   // [nseg + 1]
  std::vector<int32_t> ext_rows;  // global permuted rows
  int max_levels = 0;
};

struct BlockSplit {
  std::vector<std::vector<int32_t>> warp_rows;  // per warp: piece rows (global, ascending); unit sweeps: forward
  std::vector<std::vector<int32_t>> warp_rows_b;  // unit sweeps: the backward sweeps' packing of the same pieces
  std::vector<int32_t> tops;                    // top rows (global, ascending)
};

// Bus-unit schedule of the block sweeps.  The
// (theta_b, v_b) rows of a PQ bus are consecutive in the ordering and have the
// same L / U pattern outside their 2 x 2 diagonal block, so a sweep processes
// a bus ("unit", 1 or 2 rows) at once: every dependency value loaded from
// shared memory feeds both rows (half the shared-memory traffic per FMA).
// Per block, units are listed warp piece by warp piece (sweep order), then the
// tops.  Tile rows: the block's rows (local index), then its staged separator
// rows (backward sweeps).
struct UnitSweep {
  static constexpr int kWarps = 8;   // warps of the unit sweep kernel (k_blk: 2 CTAs per SM)
  static constexpr int kLvl = 12;    // per block: kWarps + 1 piece bounds, 2 tops bounds, 1 pad
  static constexpr int kCols = 32;   // columns of a sweep tile (one per lane)
  static constexpr int kMaxTopUnits = 16;   // one tops unit per warp
  std::vector<int32_t> unit_off;     // [nblk + 1] units of each block
  std::vector<int32_t> lvl;          // [nblk * kLvl], block-relative unit indices
  // per unit (int4): tile byte offsets of row_f and row_s (sweep order), byte
  // offset of the first record (block-relative), byte offset of the first
  // dependency offset pair (block-relative, multiple of 16) | ndeps << 16
  // (13 bits) | swapped << 29 | two_rows << 30 | forwarded << 31: a forwarded
  // unit's dependency on the unit solved just before it (same warp) is taken
  // from that unit's results in registers, its coefficient records follow the
  // header (swapped: the previous unit's first row is the pair's second).  A dependency is a
  // pair of tile-row byte offsets (o0, o1) and one (one-row unit) or two
  // (two-row unit) double2 coefficient records (c_f0, c_f1), (c_s0, c_s1);
  // lists are padded to an even count (r02: to chunks of 4, which read 2.5x
  // the real dependencies in the forward sweeps).
  bool overflow = false;              // a field of the meta encoding overflowed (grid rejected)
  std::vector<int32_t> meta;
  std::vector<int32_t> tmeta;        // (unused: the tops' dense product runs on DMMA, see top_rows)
  std::vector<int32_t> tmeta_off;    // [nblk + 1] into tmeta (units)
  static constexpr int kTopRows = 32;   // tops rows of a block (dense 32 x 32 product)
  std::vector<int32_t> top_rows;     // [nblk * kTopRows] tile rows of the tops, ascending (padded with the first)
  std::vector<int32_t> rec_off;      // [nblk + 1] double2 records
  // per record double: F position (>= 0), -1 zero, <= -2: 1 / F[-s - 2];
  // a: first sweep of the pattern (fwd L, bwd U), b: second (fwd U^T, bwd L^T)
  std::vector<int32_t> src_a, src_b;
  std::vector<int32_t> doff_off;     // [nblk + 1]
  std::vector<int32_t> doff;         // (o0, o1) byte offsets of a dependency's tile rows
  std::vector<int32_t> cost;         // [nblk] per-tile cost estimate (scheduling weight)
  int max_units = 0, max_tunits = 0, max_rec = 0, max_doff = 0, max_rows = 0;
};

// Tiles of the staged tensor projection (k_for):
// output buses grouped by the segment of their theta row (blocks; the
// separator in chunks), each group with its halo of neighbour buses, so one
// CTA stages every delta row a group needs once in shared memory.
struct ForGroups {
  static constexpr int kMaxLoc = 160;   // locals (outputs + halo) per group: 2 CTAs of k_for per SM
  std::vector<int32_t> grp_off;    // [ng + 1] locals of each group: its output buses first, then the halo
  std::vector<int32_t> grp_nout;   // [ng]
  std::vector<int32_t> grp_obase;  // [ng + 1] first output of each group in out_ptr
  std::vector<int32_t> grp_zrows;  // [ng] staged Z rows of each group
  // per local (int4): theta source, v source (permuted row >= 0, W row -(p + 2), -1 zero), bus, 0
  std::vector<int32_t> loc;
  std::vector<int32_t> grp_sbase;  // [ng + 1] first slot of each group (groups padded to 4 slots)
  std::vector<int32_t> out_bus;    // [n_out] bus of every output
  // [4 * n_out]: theta output row (permuted, -1 none), v output row (permuted >= 0, Y_p row -(p + 2)),
  // first slot (group-local), slot count
  std::vector<int32_t> out_dst;
  std::vector<int32_t> slots;      // [2 * nslots]: line (-1 padding), other end's local index * 2 + (1 if the bus is the to-end)
  std::vector<int32_t> grp_ref;    // [ng + 1] into ref_loc (groups with an output in {ref} u A(ref))
  std::vector<int32_t> ref_loc;    // local indices of the {ref} u A(ref) buses
  int max_loc = 0, max_nout = 0, max_slots = 0;
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
  std::vector<int32_t> bl_bus;   // [2 n_line] owner bus of each incidence
  bool asm_unique = false;       // no two incidences share a J / G_p / REF-gradient slot (no parallel lines)

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
  // column coloring of [J | G_p] (NEXT-4, DESIGN.md R-C1..R-C3): colors of the
  // n_x + n_p columns, per-bus seed colors, decompression entries (F / G_p
  // position, natural residual row, color)
  std::vector<int32_t> colors;
  int ncolors = 0;
  std::vector<int32_t> col_th, col_v, col_pg;
  std::vector<int32_t> jd_pos, jd_row, jd_col, gd_pos, gd_row, gd_col;
  // G_p CSC (by p column): positions into gp value array and permuted rows
  std::vector<int32_t> gpc_ptr, gpc_pos, gpc_row;

  // refactorization schedule: per segment, rows in forward local level order (local indices)
  std::vector<int32_t> fact_seg_lvl, fact_lvl_ptr, fact_order;

  // the four sweeps
  Sweep sL, sU, sUt, sLt;

  // FoR delta sources: >=0 row of Z (permuted), <=-2 row -(s+2) of W, -1 zero
  std::vector<int32_t> dth_src, dv_src;     // per bus
  // outputs: >= 0 permuted row of -Y_x ; <= -2 row -(d+2) of Y_p ; -1 none
  std::vector<int32_t> yth_dst, yv_dst;     // per bus
  std::vector<int32_t> near_ref;            // buses b in {ref} u A(ref) (unique)

  // ---------------- etree segments ----------------
  int rmax = 0;                             // max rows per block
  int nblk = 0;                             // number of blocks; segment nblk = separator
  std::vector<int32_t> seg_row_off;         // [nblk + 2]
  std::vector<int32_t> row_global;          // [n_x] local -> permuted global row, per segment (ascending)
  std::vector<int32_t> seg_of, loc_of;      // [n_x] segment / local index of every permuted row
  int max_seg_rows = 0, sep_rows = 0;
  SegSweep fwd, bwd;                        // fwd: L and U^T ; bwd: U and L^T
  std::vector<int32_t> blk_gp_ptr, blk_gp_loc;  // per block: local rows carrying G_p entries
  // per block, the G_p entries of its rows in tile order (row ascending, CSR order within a
  // row): tile-row byte offset, p column, G_p value position; and 8 warp ranges split at rows
  std::vector<int32_t> gpe_off;                 // [nblk + 1]
  std::vector<int32_t> gpe_row, gpe_col, gpe_src;
  std::vector<int32_t> gpe_split;               // [nblk * 12]: 9 block-relative bounds, pad
  int max_gpe = 0;
  std::vector<BlockSplit> split;            // per block (16 warps: refactorization R_A)
  std::vector<BlockSplit> usplit;           // per block (UnitSweep::kWarps: unit sweeps, tops)
  std::vector<int32_t> unit_lo;             // [n_x] lowest permuted row of the row's bus unit
  UnitSweep ufwd, ubwd;                     // bus-unit block sweeps (fwd: L, U^T; bwd: U, L^T)
  ForGroups fg;                             // staged tensor projection tiles
  // tops of every block (densely inverted per state): rows, F positions of T x T,
  // and the first dense entry of every top row in the fwd / bwd entry arrays
  std::vector<int32_t> top_ptr, top_rows, top_fpos_ptr, top_fpos, top_fwd_base, top_bwd_base;
  int max_tops = 0;

  // ---------------- refactorization schedule ----------------
  // R_A (per block, shared memory): F rows of the block staged at fo (block-local offsets)
  std::vector<int32_t> blk_fo_off;          // [nblk + 1] offset into fo (rows of the block, local order)
  std::vector<int32_t> fo;                  // [n_block_rows + nblk] smem offsets of each block row (+ end)
  int max_blk_fnnz = 0;
  // k-steps of the up-looking elimination, by SEGMENT position q (row_global order)
  std::vector<int32_t> ks_ptr;              // [n_x + 1]
  std::vector<int32_t> ks4;                 // per k-step: (offset of column k in row i, pivot of row k
                                            //  (R_A: smem offset / R_B1: F position), U length of row k, tgt start)
  std::vector<int32_t> ks_k;                // k: block-local index (R_A) or global row (R_B1)
  std::vector<uint16_t> tgt16;              // offsets inside row i of the U columns of row k
  int max_blk_ks = 0, max_blk_tgt = 0;
  // separator block S (Schur complement after R_B1), densified for its inversion
  std::vector<int32_t> sb_src;              // [nslots] F positions of separator-column entries of separator rows
  std::vector<int32_t> sb_dense;            // [nslots] row-major position in the dense ns x ns block
  // Epilogue partials of the block sweeps (k_blk): runs = (output row, block)
  // pairs, each a list of entries (coefficient, block row); per block a record
  // region of 16-byte slots [3 header slots: warp w's runs are run slots
  // [wr[w], wr[w + 1]) (LPT on entries) | run table (g, first entry slot,
  // entries, 0) | entries (coefficient, tile byte offset of the block row)],
  // staged behind the tile's rows; entry coefficients are filled per state.
  struct RunRecs {
    int nruns = 0;
    std::vector<int32_t> off;                         // [nblk + 1] record slots
    std::vector<int32_t> init;                        // [4 * slots] run slots' ints, entry slots 0
    std::vector<int32_t> ent_slot, ent_src, ent_trow; // per entry: slot, coefficient source, tile byte offset
  };
  // U^T sweep (MODE_UT): the separator rows' external entries in runs of one
  // block (runs numbered in separator-row order, as k_sep_gather reads them);
  // coefficient source = fwd entry e (U^T value)
  RunRecs sr;
  // L^T sweep (MODE_LT): G_p^T Psi of SpMulAdd, G_p column entries in runs of
  // one block (runs numbered by p column, blocks ascending); coefficient source
  // = CSC position q (G_p value).  Separator entries of each column are added
  // by k_muladd from Psi itself.
  RunRecs ma;
  std::vector<int32_t> ma_run_ptr;   // [n_p + 1] runs of each p column
  std::vector<int32_t> ma_sep_ptr;   // [n_p + 1] into ma_sep_q
  std::vector<int32_t> ma_sep_q;     // CSC positions of separator-row entries
};

// Returns "" on success, else an error message (grid rejected).
std::string analyze(const ::rh_grid &g, Analysis &A, int rmax = 512);

}  // namespace rh
