// ffm_plan.cuh -- device-side views of a system plan (built on the host by
// ffm_capi.cu, resident in HBM for the lifetime of an ffm_system).
#pragma once
#include "ffm_common.cuh"

namespace ffm {

// Nonbonded all-pairs plan.  Atoms are padded to np = nb * S; the upper
// triangle of S x S super-units (r <= c) is enumerated in unit_rc, heavy
// off-diagonal units first.  Pairs whose scale is not 1 ("special" pairs:
// excluded 1-2/1-3 and scaled 1-4, ffmin/model.py:290-295) are masked out of
// the dense sweep through per-tile bitmasks; the scaled ones are evaluated
// by the sparse term kernel instead.
struct NbPlanDev {
  int n;        // real atoms
  int np;       // padded atoms
  int S;        // super-unit edge (multiple of 128)
  int nb;       // np / S
  int nunits;   // nb * (nb + 1) / 2
  const int2* unit_rc;       // [nunits] (row block, column block)
  const int2* unit_ks;       // [nunits] sub-block rows [ks0, ks1) a unit covers (the last
                             // wave's units come in halves), or null = all
  const int* unit_list;      // units this launch evaluates (row sharding), or null = all
  int nlaunch;               // number of CTAs along x (= nunits without sharding)
  const int* spt_ptr;        // [np/128 + 1] special tiles per i-sub-block
  const int* spt_m;          // [nspt] global j-block index of the tile
  const uint32_t* spt_mask;  // [nspt][128] bit jj set: pair (i, jb+jj) special
  int has_cutoff;
  double cut2;
  double cull2;  // (cutoff + margin)^2: boxes farther apart than this never interact
  // small systems (ntiles > 0): the sweep runs one warp per 128 x 32 tile
  // instead of per super-unit (nb_tiles_kernel); nlaunch then counts tiles
  int ntiles;
  const int4* tiles;         // [ntiles] (i-sub-block, global j-block, special-pair
                             // mask entry or -1, 0), row-major
  const int* tile_list;      // tiles this launch evaluates (row sharding), or null = all
};

// Bonded terms + scaled (1-4) pairs, all evaluated in FP64.
struct TermPlanDev {
  int n;
  int nbond, nangle, ndih, nscaled;
  const int* bond_idx;     // [nbond][2]
  const double* bond_K;
  const double* bond_r0;
  const int* ang_idx;      // [nangle][3]
  const double* ang_K;
  const double* ang_t0;
  const int* dih_idx;      // [ndih][4]
  const double* dih_V;     // [ndih][4]
  const int* sc_idx;       // [nscaled][2]
  const double* sc_s;      // [nscaled]
  const double* q;         // [n] charges
  const double* sigma;     // [n]
  const double* eps;       // [n]
  int has_cutoff;
  double cutoff;
  // slot layout: bonds 2/term, angles 3/term, dihedrals 4/term, scaled 2/term
  int slot_angle0, slot_dih0, slot_sc0, nslots;
  // energy layout: [bonds | angles | dihedrals | scaled coulomb | scaled vdw]
  int e_angle0, e_dih0, e_scc0, e_scv0, nterm_e;
};

}  // namespace ffm
