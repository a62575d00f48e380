// Device-side parameter blocks of the batched adjoint-adjoint reduced Hessian
// (sm_100a, fp64).  See redhess.cu for the kernels and DESIGN.md for the design.
//
// Batched blocks in HBM: Z and Psi are [n_x][ld]
// row-major in the PERMUTED row numbering of the factorization, batch index
// fastest (SoA across the batch), ld = N rounded up to a multiple of 32.
// W and HW are the caller's [n_p][ldw] / [n_p][ldhw] blocks.
#pragma once

#include <cstdint>

namespace rh {

constexpr int kThreads = 256;
constexpr int kSegThreads = 512;   // block kernels: 16 warps (must match the host schedule's kSchedWarps)

// One dependency pattern (forward: L / U^T, backward: U / L^T) split into
// elimination-tree segments (blocks + separator), each with its own levels.
struct DSeg {
  const int *__restrict__ seg_lvl;   // [nseg + 1] into lvl_ptr
  const int *__restrict__ lvl_ptr;   // level bounds into q
  const int *__restrict__ order;     // [n_x] q -> local row
  const int *__restrict__ rptr;      // [n_x + 1]
  const int *__restrict__ rext;      // [n_x]: [rptr, rext) external entries, [rext, rptr+1) local
  const int *__restrict__ dep;       // local row index (local entries) / global permuted row (external)
  const int *__restrict__ ext_off;   // [nseg + 1] blocks: staged separator rows
  const int *__restrict__ ext_rows;
  // fwd only: per separator row q (index q - first separator q), its external entries
  // in runs of one block each: runs [grp_ptr[i], grp_ptr[i + 1]), run g = block grp_blk[g]
  // over entries [.., grp_end[g])
  const int *__restrict__ grp_ptr, *__restrict__ grp_blk, *__restrict__ grp_end;
};

// Bus-unit schedule of one pattern direction (analysis.hpp UnitSweep).
struct DUnit {
  const int4 *__restrict__ meta;     // per unit
  const int *__restrict__ top_rows;  // [nblk][32] tile rows of the tops (ascending, padded)
  const int *__restrict__ unit_off, *__restrict__ tmeta_off, *__restrict__ lvl, *__restrict__ rec_off;
  const int *__restrict__ doff_off, *__restrict__ doff;
  const int *__restrict__ blk_order;  // blocks by decreasing cost (tile tickets are block-major in this order)
  const int *__restrict__ ext_off, *__restrict__ ext_rows;   // staged separator rows (Z rows)
};

struct SegParams {
  int n_x, n_p, n_bus, N, ld;
  int nblk;                          // segment nblk = separator
  DUnit uf, ub;                      // bus-unit block sweeps: fwd (L, U^T), bwd (U, L^T)
  DUnit ubp;                         // bwd pruned to the rows G_p^T Psi needs (L^T of Cartesian batches)
  const double2 *uL, *uUt, *uU, *uLt;  // their record values (per state)
  const double *tL, *tUt, *tU, *tLt;   // [nblk][32][36] dense tops inverses per sweep (k_tops_inverse)
  const int *gpe_off, *gpe_split;      // L sweep: per block G_p entry records and 8 warp ranges
  const double2 *gpe_rec;
  int maxrx;                         // max tile rows (block rows + staged separator rows)
  int smem_stride;                   // bytes per buffer (two buffers: current tile, prefetched tile)
  int smem_x_off, smem_meta_off, smem_tmeta_off, smem_rec_off, smem_doff_off, smem_lvl_off;  // bytes (tmeta: tops M + rows)
  int *blk_ctr;                      // [2 per mode] tile ticket counter, CTAs done (self-resetting)
  // 2D TMA tensor maps (CUtensorMap, device memory) of Z and P for this ld: pairs
  // [box 32 x 64 rows, box 32 x 8 rows]; null = per-row copies (k_blk)
  const void *tmZ, *tmP;
  int kblk_group;                    // k_blk: column chunks per ticket (one block's structure staged once)
  // split U sweep of Cartesian batches: k_blk MODE_U with
  // spike = 1 sweeps the live tiles with the staged separator rows taken as zero (Z^0,
  // dead tiles skipped), spike = 2 computes the blocks' spikes (block rows zero,
  // staged separator rows = identity columns) into Msp; k_spike then forms
  // Z_b = Z_b^0 + Msp_b z_ext
  int spike;
  const int *ma_gptr;                // k_muladd: per group of 4 p rows, its items (static)
  const int2 *ma_items;              // (target j << 30 | kind << 28 | row, CSC position)
  int ma_ngrp;
  const int *tlist;                  // Cartesian batch: live tiles (count, then block << 16 | chunk)
  const double *Msp;                 // [n_x][kSpLd] per block row: -(U_bb^-1 U_bs) over the block's staged separator rows
  const int *seg_row_off, *row_global;
  DSeg fwd, bwd;
  const double *vL, *vUt;             // separator rows' L / U^T values (fwd entry order)
  int ns, sep_off;                     // separator rows, first separator slot in row_global
  const double *Sinv, *SinvT;          // dense [ns][ns] inverse of the separator block L_ss U_ss (+ transpose)
  double *Tsep;                        // [ns][ld] separator right-hand sides, then the run partials:
  // U^T sweep epilogue (k_blk MODE_UT): Part[g] = sum over run g's entries (one block's
  // rows) of U^T value x P row, [nruns][ld] behind Tsep; k_sep_gather (UTLT) sums the runs
  unsigned char *nzf;                  // Cartesian LU: [chunk][ns] separator rows of T that are nonzero (k_sep_spmm)
  int nruns;
  const int *sr_off;                   // per block: its record slots (analysis.hpp sr_*)
  const double2 *sr_rec;               // [run table (g, first entry slot, entries) | entries (value, tile offset)]
  // L^T sweep epilogue (k_blk MODE_LT): Mp[g] = sum over G_p run g's entries (one
  // p column's rows in one block) of G_p value x Psi row; k_muladd adds the runs
  const int *ma_off;
  const double2 *ma_rec;
  double *Mp;                          // [ma runs][ld], null: no partials (gradient sweeps)
  const int *ma_run_ptr, *ma_sep_ptr, *ma_sep_q;   // per p column: its runs; its separator entries (CSC q)
  const int *blk_gp_ptr, *blk_gp_loc;  // per block: local rows with G_p entries
  const double *W;                   // [n_p][ldw]; null for a Cartesian block (icol)
  long long ldw;
  // Cartesian batch (full Hessian): column k of the batch is e_{icol[k]} (k < N);
  // its output goes to position icol[k] - icol_base of the caller's block.
  // tmask[s * tmask_words + c / 32] bit c % 32: chunk c of block s has a nonzero
  // right-hand side -G_p W (null: every chunk).  k_batch_plan writes both.
  const int *icol;
  int icol_base;
  const unsigned *tmask;
  int tmask_words;
  double *HW;
  long long ldhw;
  int transposed;
  double *Z, *P;                     // [n_x][ld] work blocks (Z, then -Y_x -> Psi)
  double *Yp;                        // [n_p][ld] Y_p of the voltage parameters (k_for -> k_muladd)
  const int *gp_rptr, *gp_col;       // G_p CSR over permuted rows
  const double *gp_val;
  const int *gpc_ptr, *gpc_row;      // G_p CSC (p columns), rows permuted
  const double *gpc_val;
  // forward-over-reverse tape
  const int *bl_ptr, *bl_line, *bl_end, *o_dth_src, *o_dv_src;
  const int *dth_src, *dv_src, *yth_dst, *yv_dst, *pg_p;
  const double4 *coef;
  const double *dcoef, *refg_th, *refg_v, *c2b;
  const int *near_ref;
  int n_near_ref;
  double f2ref;
  // staged tensor projection tiles (analysis.hpp ForGroups; sources / outputs in Z rows).
  // Staging rows (32 doubles each): rows [0, zn) are Z rows [zlo, zlo + zn) (the
  // outputs' range, 2D TMA boxes), then one row per remaining Z source (per-row
  // bulk copies, fg_cp: staging row, Z row) and per W / zero source (fg_fill:
  // staging row, p row or -1).  A local's (theta, v) staging rows are packed
  // theta | v << 16 in fg_loc .w; fg_soe holds the other end's rows of a slot as byte offsets.
  const int *fg_off, *fg_nout, *fg_obase, *fg_sbase, *fg_ref, *fg_ref_loc;
  const int *fg_zlo, *fg_zn, *fg_cp_off, *fg_fill_off;
  const int2 *fg_cp, *fg_fill;
  int fg_maxrows, fg_maxout, fg_maxslots;
  const int4 *fg_loc, *fg_odst;        // per local: sources, bus, packed staging rows; per output: theta row, v row, first slot, slots
  const int2 *fg_soe;                  // per slot: byte offsets (theta, v) of the other end's staging rows
  const double4 *fg_scoef, *fg_ometa;  // per state and lambda (k_for_tape): slot coefficients; dcoef, grad P_ref
  const int *p_kind;                   // Pg diagonal of Y_p in k_muladd
  const double *pdiag;                 // [n_p] 2 c2 (Pg parameters) else 0
  int debug;                         // experiment bits (0 in production)
  long long *dbg;
};

struct FactParams {
  int nblk, ns;
  const int *seg_row_off, *row_global;
  const int *fwd_seg_lvl, *fwd_lvl_ptr, *fwd_order;
  const int *blk_fo_off, *fo;
  const int *F_rowptr, *F_diag;
  double *F_val;
  const int *ks_ptr, *ks4, *ks_k;
  const unsigned short *tgt16;
  double *dinv, *rowmax;             // per permuted row
  int *status;
  double pivtol;
  int sep_maxlen;                    // R_B1: longest separator row of F (shared-memory staging)
  int sep_maxu;                      // R_B1: most U entries one separator row's k-steps read
  long long *dbg;                    // timing experiment (RH_DEBUG & 128): per-block phase stamps, else null
  int df;                            // R_A: one dataflow pass over the block's rows (else pieces + tops phases)
};

}  // namespace rh
