// ffm_capi.cu -- the extern "C" boundary (include/ffmin_b200.h): system
// plans resident in HBM, workspace management and launch sequencing.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/ffmin_b200.h"
#include "ffm_kernels.h"
#include "ffm_min.cuh"

// ncclAllReduce from the libnccl.so.2 the process has loaded (torch's), or
// any the loader finds; resolved once
using AllReduceFn = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                     ncclComm_t, cudaStream_t);
static AllReduceFn nccl_allreduce() {
  static AllReduceFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) fn = reinterpret_cast<AllReduceFn>(dlsym(h, "ncclAllReduce"));
    if (!fn) fn = reinterpret_cast<AllReduceFn>(dlsym(RTLD_DEFAULT, "ncclAllReduce"));
  }
  return fn;
}


using namespace ffm;

std::atomic<long long> ffm::g_launch_count{0};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define FFM_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(FFM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));  \
  } while (0)

#define FFM_TRYR(x)    \
  do {                 \
    int rc_ = (x);     \
    if (rc_) return rc_; \
  } while (0)

template <typename T>
int upload(T** dst, const std::vector<T>& src) {
  *dst = nullptr;
  if (src.empty()) return FFM_OK;
  if (cudaMalloc(dst, src.size() * sizeof(T)) != cudaSuccess)
    return fail(FFM_ENOMEM, "cudaMalloc failed for a system table");
  FFM_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return FFM_OK;
}

struct Work {
  void* pos = nullptr;     // [batch][np] Vec4 (j side)
  void* ipos = nullptr;    // [batch][4][np/2] pairs (i side)
  void* bbox = nullptr;    // [batch][np/32][6] block boxes (cutoff culling)
  int pos_batch = 0;
  void* ipart = nullptr;   // [nunits][3][S]
  void* jpart = nullptr;
  double* epart = nullptr; // [batch][nunits][3]
  int e_batch = 0;
  double* term_e = nullptr;  // [batch][nterm_e]
  int64_t* term_st = nullptr;  // [term blocks * 4 warps][4]: tiny systems' term status slots
  int te_batch = 0;
  double* term_f = nullptr;  // [nslots][3]
  double* escratch = nullptr;  // split energy reduction: [kMaxEnergyParts][3] + counter
};

// the split energy reduction's counter sits after its [kMaxEnergyParts][3] partials
inline unsigned* ecount(Work& w) {
  return reinterpret_cast<unsigned*>(w.escratch + (size_t)kMaxEnergyParts * 3);
}

}  // namespace

struct ffm_system {
  int device = 0;
  NbPlanDev plan{};
  int S0 = 0;  // the super-unit edge chosen at creation (single-rank plan)
  // sharded evaluations completed on the device (ffm_system_set_comm)
  void* comm = nullptr;
  double* d_comb = nullptr;  // [3n + 13]
  // batched (multi-candidate, energy-only) sweeps: super-units as large as
  // divide np -- with B geometries per launch the grid is large whatever the
  // unit size, so larger units amortise their overheads (configs[3])
  NbPlanDev bplan{};
  int2* d_unit_rc_b = nullptr;
  TermPlanDev tp{};
  int nspt = 0;
  // device tables
  int2* d_unit_rc = nullptr;
  int* d_unit_index = nullptr;  // the gather's unit lists (build_units)
  int2* d_unit_ks = nullptr;
  int* d_spt_ptr = nullptr;
  int* d_spt_m = nullptr;
  uint32_t* d_spt_mask = nullptr;
  int* d_sp_ptr = nullptr;   // upper special rows (finder)
  int* d_sp_j = nullptr;
  double* d_sp_s = nullptr;
  int* d_fsp_ptr = nullptr;  // full special rows (atom delta)
  int* d_fsp_j = nullptr;
  double* d_fsp_s = nullptr;
  double* d_qt = nullptr;    // q sqrt(C), [np]
  float2* d_lj32 = nullptr;  // [np]
  double2* d_lj64 = nullptr;
  float* d_ilj32 = nullptr;  // LJ in the i-side pair layout, [2][np/2] pairs
  double* d_ilj64 = nullptr;
  double* d_q = nullptr;
  double* d_sigma = nullptr;
  double* d_eps = nullptr;
  int* d_sc_idx = nullptr;
  double* d_sc_s = nullptr;
  // bonded
  int* d_bond_idx = nullptr;
  double* d_bond_K = nullptr;
  double* d_bond_r0 = nullptr;
  int* d_ang_idx = nullptr;
  double* d_ang_K = nullptr;
  double* d_ang_t0 = nullptr;
  int* d_dih_idx = nullptr;
  double* d_dih_V = nullptr;
  int* d_slot_ptr = nullptr;
  int* d_slot_idx = nullptr;
  int* d_aterm_ptr = nullptr;
  int* d_aterm_idx = nullptr;
  // row sharding (ffm_system_set_shard): units u with u % nranks == rank
  int rank = 0, nranks = 1;
  // fused small-system evaluation: cooperative grid per [precision][grad], 0 = not sized yet
  int small_grid[2][2][2] = {};  // [precision][grad][kernel variant (small_fromx)]
  unsigned long long* phase_clock = nullptr;  // ffm_debug_phase_clock (tuning aid)
  int* d_unit_list = nullptr;
  std::vector<char> unit_live;  // host: slot holds a real unit (build_units)
  // small-system tile mode (NbPlanDev::ntiles > 0)
  int4* d_tiles = nullptr;
  // atom-delta scratch (launch_atom_delta's multi-block candidates)
  double* dl_part = nullptr;
  long long* dl_bad = nullptr;
  unsigned* dl_cnt = nullptr;
  int64_t dl_cap = 0;
  int* d_tile_list = nullptr;
  int* d_trow_ptr = nullptr;  // [np/128 + 1] tiles of each i-sub-block (contiguous)
  int* d_tcol_ptr = nullptr;  // [np/32 + 1] tiles of each j-block ...
  int* d_tcol_idx = nullptr;  // ... listed here, by i-sub-block
  // host copies needed to rebuild the term plan
  std::vector<std::pair<int, int>> scaled;  // (i, j)
  std::vector<double> scaled_s;
  Work w[2];  // [precision]
  // captured evaluation sequences (CUDA graphs), keyed by the call's
  // arguments; invalidated whenever a workspace buffer moves
  struct GraphEntry {
    int prec, flags;
    const void *coords, *grad, *energies, *status;
    long long gen;
    long long kernels;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  long long gen = 0;
  cudaStream_t cap_stream = nullptr;
  // the O(N) term kernel runs on a forked branch beside the pair sweep
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // FFM_TIME_NB: events around the pair sweep of the last evaluation
  cudaEvent_t ev_nb0 = nullptr, ev_nb1 = nullptr;
  bool timed = false;
  // host-path staging
  double* h_coords_d = nullptr;
  double* h_grad_d = nullptr;
  double* h_en_d = nullptr;
  int64_t* h_st_d = nullptr;
};

namespace {

void free_all(ffm_system* s) {
  void* ptrs[] = {s->d_comb, s->d_unit_rc, s->d_unit_rc_b, s->d_unit_index, s->d_unit_ks,
                  s->d_spt_ptr, s->d_spt_m,
                  s->d_spt_mask,
                  s->d_sp_ptr, s->d_sp_j, s->d_sp_s, s->d_fsp_ptr, s->d_fsp_j, s->d_fsp_s,
                  s->d_qt, s->d_lj32, s->d_lj64, s->d_ilj32, s->d_ilj64, s->d_q, s->d_sigma, s->d_eps, s->d_sc_idx,
                  s->d_sc_s, s->d_bond_idx, s->d_bond_K, s->d_bond_r0, s->d_ang_idx,
                  s->d_ang_K, s->d_ang_t0, s->d_dih_idx, s->d_dih_V, s->d_slot_ptr,
                  s->d_slot_idx, s->d_aterm_ptr, s->d_aterm_idx, s->h_coords_d, s->h_grad_d,
                  s->h_en_d, s->h_st_d, s->d_unit_list, s->d_tiles, s->d_tile_list,
                  s->d_trow_ptr, s->d_tcol_ptr, s->d_tcol_idx};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& g : s->graphs) cudaGraphExecDestroy(g.exec);
  s->graphs.clear();
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  if (s->side) cudaStreamDestroy(s->side);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  if (s->ev_nb0) cudaEventDestroy(s->ev_nb0);
  if (s->ev_nb1) cudaEventDestroy(s->ev_nb1);
  for (void* p : {(void*)s->dl_part, (void*)s->dl_bad, (void*)s->dl_cnt})
    if (p) cudaFree(p);
  for (auto& w : s->w) {
    void* wp[] = {w.pos, w.ipos, w.bbox, w.ipart, w.jpart, w.epart, w.term_e, w.term_f,
                  w.escratch, w.term_st};
    for (void* p : wp)
      if (p) cudaFree(p);
  }
}

void drop_graphs(ffm_system* s) {
  for (auto& g : s->graphs) cudaGraphExecDestroy(g.exec);
  s->graphs.clear();
  s->gen++;
}

// Super-unit edge: the largest S that still gives >= 2048 units (about 3.5
// CTAs per SM slot at 4 CTAs/SM), so the hardware block scheduler balances
// the triangle; never below 256.
int choose_S(int64_t n) {
  if (const char* f = getenv("FFM_FORCE_S")) {  // tuning aid; njb = S / 32 must fit 32 bits
    const int v = atoi(f);
    if (v >= 128 && v <= 1024 && v % 128 == 0) return v;
  }
  // largest super-unit that still gives ~6 waves of units on 148 SMs x 2
  // CTAs: bigger units amortise the per-sub-block reductions, more units
  // shorten the tail (measured on B200, 5k..100k atoms, tools/time_nb.py)
  for (int S : {1024, 768, 512, 256}) {
    const int64_t nb = (n + S - 1) / S;
    if (nb * (nb + 1) / 2 >= 1700) return S;
  }
  return 256;
}

// (Re)build the super-unit tables of edge S (a divisor of np): units in
// evaluation order -- off-diagonal first (full work), then the last `nsplit`
// off-diagonal units as two halves each (rows [0, nsub/2) and [nsub/2, nsub):
// the final wave runs in half-size pieces, so its tail is half as long),
// then the diagonal units (half work) -- and the gather's unit lists
// (gather_group: the units holding each super-block half's rows, then the
// units holding each super-block's columns).
//
// Row-sharded plans (nranks > 1) deal the units in that order to the rank
// with the least work so far (counted in 128 x 32 tiles; ties go to the
// lowest rank), rank 0 starting at the tile-equivalent of the O(N) bonded
// and 1-4 work only it evaluates; unit slot u then belongs to rank
// u % nranks (the gather's ownership test), each rank's units keep their
// order, and slots a shorter rank leaves over hold null units (never
// launched: zero partials, energy slot (0, 0, 1e30)).  s->unit_live marks
// the real ones.
#ifndef FFM_TERM_PAIRS_PER_ATOM
#define FFM_TERM_PAIRS_PER_ATOM 400  // measured: rank 0 ran 31-45 us longer at 100k
#endif
int build_units(ffm_system* s, int S, int nsplit, int nranks) {
  NbPlanDev& p = s->plan;
  p.S = S;
  p.nb = p.np / S;
  const int nb = p.nb, nsub = S / kIB, hs = nsub / 2, njb = S / kJB;
  const int noff = nb * (nb - 1) / 2;
  if (nsplit > noff) nsplit = noff;
  if (nsub < 2) nsplit = 0;
  std::vector<int2> lrc, lks;  // logical order
  for (int r = 0, k = 0; r < nb; ++r)
    for (int c = r + 1; c < nb; ++c, ++k) {
      if (k < noff - nsplit) {
        lrc.push_back(make_int2(r, c));
        lks.push_back(make_int2(0, nsub));
      } else {
        lrc.push_back(make_int2(r, c));
        lks.push_back(make_int2(0, hs));
        lrc.push_back(make_int2(r, c));
        lks.push_back(make_int2(hs, nsub));
      }
    }
  for (int r = 0; r < nb; ++r) {
    lrc.push_back(make_int2(r, r));
    lks.push_back(make_int2(0, nsub));
  }
  // slot of each logical unit (identity for one rank)
  std::vector<int> slot(lrc.size());
  int nslot = (int)lrc.size();
  if (nranks > 1) {
    int term_pairs = FFM_TERM_PAIRS_PER_ATOM;
    if (const char* f = getenv("FFM_TERM_PAIRS_PER_ATOM")) term_pairs = atoi(f);  // tuning aid
    std::vector<double> load(nranks, 0.0);
    std::vector<int> count(nranks, 0);
    load[0] = (double)term_pairs * p.n / (kIB * kJB);
    for (size_t k = 0; k < lrc.size(); ++k) {
      int tiles = 0;
      for (int ks = lks[k].x; ks < lks[k].y; ++ks)
        tiles += lrc[k].x == lrc[k].y ? njb - (kIB / kJB) * ks : njb;
      int r = 0;
      for (int q = 1; q < nranks; ++q)
        if (load[q] < load[r]) r = q;
      load[r] += tiles;
      slot[k] = count[r]++ * nranks + r;
    }
    nslot = *std::max_element(count.begin(), count.end()) * nranks;
  } else {
    for (size_t k = 0; k < slot.size(); ++k) slot[k] = (int)k;
  }
  std::vector<int2> urc(nslot, make_int2(0, 0)), uks(nslot, make_int2(0, 0));
  s->unit_live.assign(nslot, 0);
  std::vector<int> half0((size_t)nb * nb, -1), half1((size_t)nb * nb, -1);
  for (size_t k = 0; k < lrc.size(); ++k) {
    const int u = slot[k];
    urc[u] = lrc[k];
    uks[u] = lks[k];
    s->unit_live[u] = 1;
    const size_t key = (size_t)lrc[k].x * nb + lrc[k].y;
    if (lks[k].x == 0 && lks[k].y == nsub) half0[key] = half1[key] = u;
    else (lks[k].x == 0 ? half0 : half1)[key] = u;
  }
  p.nunits = (int)urc.size();
  // gather lists: [row ptr (2 nb + 1) | column ptr (nb + 1) | rows | columns]
  std::vector<int> rptr(2 * nb + 1, 0), cptr(nb + 1, 0), rows, cols;
  for (int b = 0; b < nb; ++b)
    for (int h = 0; h < 2; ++h) {
      for (int cc = b; cc < nb; ++cc) rows.push_back((h ? half1 : half0)[(size_t)b * nb + cc]);
      rptr[2 * b + h + 1] = (int)rows.size();
    }
  for (int b = 0; b < nb; ++b) {
    for (int r = 0; r <= b; ++r) {
      const size_t key = (size_t)r * nb + b;
      cols.push_back(half0[key]);
      if (half1[key] != half0[key]) cols.push_back(half1[key]);
    }
    cptr[b + 1] = (int)cols.size();
  }
  std::vector<int> lists;
  lists.insert(lists.end(), rptr.begin(), rptr.end());
  lists.insert(lists.end(), cptr.begin(), cptr.end());
  lists.insert(lists.end(), rows.begin(), rows.end());
  lists.insert(lists.end(), cols.begin(), cols.end());
  for (int2** d : {&s->d_unit_rc, &s->d_unit_ks})
    if (*d) cudaFree(*d), *d = nullptr;
  if (s->d_unit_index) cudaFree(s->d_unit_index);
  s->d_unit_index = nullptr;
  FFM_TRYR(upload(&s->d_unit_rc, urc));
  FFM_TRYR(upload(&s->d_unit_ks, uks));
  FFM_TRYR(upload(&s->d_unit_index, lists));
  p.unit_rc = s->d_unit_rc;
  p.unit_ks = s->d_unit_ks;
  p.unit_list = nullptr;
  if (p.ntiles == 0) p.nlaunch = p.n > 0 ? p.nunits : 0;
  return FFM_OK;
}

// units of the last wave split in halves: one wave of CTA slots (2 per SM)
// per rank, since every rank gets an equal share of them -- for S = 1024 only: a
// half unit of S <= 512 pays the whole per-unit overhead for one or two
// tiles per warp (measured, tools/mid_sweep.py A/B: 100k atoms, S = 1024
// 4.41 -> 4.37 ms; 10k, S = 256 70.0 -> 71.8 us; 30k, S = 512 426 -> 433 us)
int split_count(const ffm_system* s, int S, int nranks) {
  if (const char* f = getenv("FFM_SPLIT_UNITS")) return atoi(f);  // tuning / tests
  if (S < 1024) return 0;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
  return 2 * sms * nranks;
}

// Super-unit edge of a row-sharded plan: every rank should still see about
// six waves of units (the single-GPU rule of choose_S, per rank), so the
// edge shrinks with the shard count -- 100k atoms: 1024 up to 2 ranks, 512
// at 4 and 8 (at S = 1024 eight ranks would get 606 units each, 2.05 waves
// of ~265 us units: a third wave almost empty).  Only edges dividing np.
#ifndef FFM_SHARD_UNITS
#define FFM_SHARD_UNITS 1700  // units per rank wanted (~6 waves of 296 CTA slots)
#endif
int choose_S_sharded(const NbPlanDev& p, int S0, int nranks) {
  for (int S : {1024, 768, 512, 256}) {
    if (S > S0 || p.np % S) continue;
    const int64_t nb = p.np / S;
    if (nb * (nb + 1) / 2 >= (int64_t)FFM_SHARD_UNITS * nranks) return S;
  }
  return p.np % 256 == 0 ? std::min(256, S0) : S0;  // never above the single-rank edge
}

// rebuild the term plan device view (after set_terms or creation)
int build_terms(ffm_system* s, int64_t nbond, const int64_t* bidx, const double* bK,
                const double* br0, int64_t nang, const int64_t* aidx, const double* aK,
                const double* at0, int64_t ndih, const int64_t* didx, const double* dV) {
  const int n = s->plan.n;
  TermPlanDev& tp = s->tp;
  auto chk = [&](int64_t v) { return v >= 0 && v < n; };
  std::vector<int> bi(2 * nbond), ai(3 * nang), di(4 * ndih);
  for (int64_t k = 0; k < 2 * nbond; ++k) {
    if (!chk(bidx[k])) return fail(FFM_EINVAL, "bond index out of range");
    bi[k] = (int)bidx[k];
  }
  for (int64_t k = 0; k < 3 * nang; ++k) {
    if (!chk(aidx[k])) return fail(FFM_EINVAL, "angle index out of range");
    ai[k] = (int)aidx[k];
  }
  for (int64_t k = 0; k < 4 * ndih; ++k) {
    if (!chk(didx[k])) return fail(FFM_EINVAL, "dihedral index out of range");
    di[k] = (int)didx[k];
  }
  for (void* p : {(void*)s->d_bond_idx, (void*)s->d_bond_K, (void*)s->d_bond_r0,
                  (void*)s->d_ang_idx, (void*)s->d_ang_K, (void*)s->d_ang_t0,
                  (void*)s->d_dih_idx, (void*)s->d_dih_V, (void*)s->d_slot_ptr,
                  (void*)s->d_slot_idx, (void*)s->d_aterm_ptr, (void*)s->d_aterm_idx})
    if (p) cudaFree(p);
  int rc;
  if ((rc = upload(&s->d_bond_idx, bi))) return rc;
  if ((rc = upload(&s->d_bond_K, std::vector<double>(bK, bK + nbond)))) return rc;
  if ((rc = upload(&s->d_bond_r0, std::vector<double>(br0, br0 + nbond)))) return rc;
  if ((rc = upload(&s->d_ang_idx, ai))) return rc;
  if ((rc = upload(&s->d_ang_K, std::vector<double>(aK, aK + nang)))) return rc;
  if ((rc = upload(&s->d_ang_t0, std::vector<double>(at0, at0 + nang)))) return rc;
  if ((rc = upload(&s->d_dih_idx, di))) return rc;
  if ((rc = upload(&s->d_dih_V, std::vector<double>(dV, dV + 4 * ndih)))) return rc;

  const int nsc = (int)s->scaled.size();
  tp.n = n;
  tp.nbond = (int)nbond;
  tp.nangle = (int)nang;
  tp.ndih = (int)ndih;
  tp.nscaled = nsc;
  tp.bond_idx = s->d_bond_idx;
  tp.bond_K = s->d_bond_K;
  tp.bond_r0 = s->d_bond_r0;
  tp.ang_idx = s->d_ang_idx;
  tp.ang_K = s->d_ang_K;
  tp.ang_t0 = s->d_ang_t0;
  tp.dih_idx = s->d_dih_idx;
  tp.dih_V = s->d_dih_V;
  tp.sc_idx = s->d_sc_idx;
  tp.sc_s = s->d_sc_s;
  tp.q = s->d_q;
  tp.sigma = s->d_sigma;
  tp.eps = s->d_eps;
  tp.slot_angle0 = 2 * (int)nbond;
  tp.slot_dih0 = tp.slot_angle0 + 3 * (int)nang;
  tp.slot_sc0 = tp.slot_dih0 + 4 * (int)ndih;
  tp.nslots = tp.slot_sc0 + 2 * nsc;
  tp.e_angle0 = (int)nbond;
  tp.e_dih0 = tp.e_angle0 + (int)nang;
  tp.e_scc0 = tp.e_dih0 + (int)ndih;
  tp.e_scv0 = tp.e_scc0 + nsc;
  tp.nterm_e = tp.e_scv0 + nsc;

  // atom -> slot CSR in slot order (fixed summation order of the gather)
  std::vector<std::vector<int>> slots(n);
  for (int t = 0; t < nbond; ++t)
    for (int q = 0; q < 2; ++q) slots[bi[2 * t + q]].push_back(2 * t + q);
  for (int t = 0; t < nang; ++t)
    for (int q = 0; q < 3; ++q) slots[ai[3 * t + q]].push_back(tp.slot_angle0 + 3 * t + q);
  for (int t = 0; t < ndih; ++t)
    for (int q = 0; q < 4; ++q) slots[di[4 * t + q]].push_back(tp.slot_dih0 + 4 * t + q);
  for (int t = 0; t < nsc; ++t) {
    slots[s->scaled[t].first].push_back(tp.slot_sc0 + 2 * t);
    slots[s->scaled[t].second].push_back(tp.slot_sc0 + 2 * t + 1);
  }
  std::vector<int> sptr(n + 1, 0), sidx;
  for (int a = 0; a < n; ++a) {
    std::sort(slots[a].begin(), slots[a].end());
    sptr[a + 1] = sptr[a] + (int)slots[a].size();
    sidx.insert(sidx.end(), slots[a].begin(), slots[a].end());
  }
  if ((rc = upload(&s->d_slot_ptr, sptr))) return rc;
  if ((rc = upload(&s->d_slot_idx, sidx))) return rc;
  // atom -> bonded term ids (ffmin/model.py:321-347 atom_terms)
  std::vector<std::vector<int>> at(n);
  for (int t = 0; t < nbond; ++t)
    for (int q = 0; q < 2; ++q) at[bi[2 * t + q]].push_back(t);
  for (int t = 0; t < nang; ++t)
    for (int q = 0; q < 3; ++q) at[ai[3 * t + q]].push_back((int)nbond + t);
  for (int t = 0; t < ndih; ++t)
    for (int q = 0; q < 4; ++q) at[di[4 * t + q]].push_back((int)(nbond + nang) + t);
  std::vector<int> aptr(n + 1, 0), aidx2;
  for (int a = 0; a < n; ++a) {
    aptr[a + 1] = aptr[a] + (int)at[a].size();
    aidx2.insert(aidx2.end(), at[a].begin(), at[a].end());
  }
  if ((rc = upload(&s->d_aterm_ptr, aptr))) return rc;
  if ((rc = upload(&s->d_aterm_idx, aidx2))) return rc;
  // term workspaces are sized by the term plan: drop them
  for (auto& w : s->w) {
    if (w.term_e) cudaFree(w.term_e);
    if (w.term_f) cudaFree(w.term_f);
    if (w.term_st) cudaFree(w.term_st);
    w.term_e = nullptr;
    w.term_f = nullptr;
    w.term_st = nullptr;
    w.te_batch = 0;
  }
  return FFM_OK;
}

// energy-partial slots of the pair sweep: one per tile or per super-unit
int nb_slots(const NbPlanDev& p) { return p.ntiles ? p.ntiles : p.nunits; }

// small systems sweep tiles (one CTA per 128 x 32 tile, ffm_tile.cuh)
// instead of super-units: below ~150 units (about 4300 atoms at S = 256)
// the units leave SMs idle and the one-launch tile evaluation is faster;
// above it the tile gather (a row of up to np/32 tile partials per atom)
// costs more than it saves.  Measured (tools/mid_sweep.py, tiles vs units,
// FP32 / FP64 energy+gradient, us): 2000 atoms 21.2 / 24.8 vs 28.9 / 43.2;
// 4000 atoms 37.1 / 55.0 vs 37.3 / 69.8; 5000 atoms 47.4 / 74.2 vs 37.7 / 70.0
bool use_tiles(const NbPlanDev& p, int device) {
  if (const char* f = getenv("FFM_FORCE_TILES")) return atoi(f) != 0;  // tuning / tests
  (void)device;
  return p.nb * (p.nb + 1) / 2 < 150;  // whole units (before the last wave's split)
}

int build_tiles(ffm_system* s, const std::vector<int>& spt_ptr, const std::vector<int>& spt_m) {
  NbPlanDev& p = s->plan;
  const int nkk = p.np / kIB, nmg = p.np / kJB;
  std::vector<int4> tiles;
  std::vector<int> rptr(nkk + 1, 0);
  std::vector<std::vector<int>> col(nmg);
  for (int kk = 0; kk < nkk; ++kk) {
    for (int mg = 4 * kk; mg < nmg; ++mg) {
      if (kk * kIB >= p.n || mg * kJB >= p.n) continue;  // padding only
      col[mg].push_back((int)tiles.size());
      int spe = -1;  // the tile's special-pair mask entry (ffm_plan.cuh)
      for (int e = spt_ptr[kk]; e < spt_ptr[kk + 1]; ++e)
        if (spt_m[e] == mg) spe = e;
      tiles.push_back(make_int4(kk, mg, spe, 0));
    }
    rptr[kk + 1] = (int)tiles.size();
  }
  std::vector<int> cptr(nmg + 1, 0), cidx;
  for (int mg = 0; mg < nmg; ++mg) {
    cptr[mg + 1] = cptr[mg] + (int)col[mg].size();
    cidx.insert(cidx.end(), col[mg].begin(), col[mg].end());
  }
  if (cidx.empty()) cidx.push_back(0);
  if (tiles.empty()) tiles.push_back(make_int4(0, 0, -1, 0));  // n = 0: never launched
  FFM_TRYR(upload(&s->d_tiles, tiles));
  FFM_TRYR(upload(&s->d_trow_ptr, rptr));
  FFM_TRYR(upload(&s->d_tcol_ptr, cptr));
  FFM_TRYR(upload(&s->d_tcol_idx, cidx));
  p.tiles = s->d_tiles;
  p.tile_list = nullptr;
  p.ntiles = (int)tiles.size();
  p.nlaunch = p.n > 0 ? p.ntiles : 0;
  return FFM_OK;
}

// allocate / grow the workspace of one precision
int ensure_work(ffm_system* s, int prec, int batch, bool grad) {
  Work& w = s->w[prec];
  struct Bump {
    ffm_system* s;
    Work* w;
    void* p[9];
    Bump(ffm_system* s_, Work* w_) : s(s_), w(w_) {
      void* q[9] = {w->pos, w->ipos, w->ipart, w->jpart, w->epart, w->term_e, w->term_f, w->bbox,
                    w->term_st};
      for (int i = 0; i < 9; ++i) p[i] = q[i];
    }
    ~Bump() {
      void* q[9] = {w->pos, w->ipos, w->ipart, w->jpart, w->epart, w->term_e, w->term_f, w->bbox,
                    w->term_st};
      for (int i = 0; i < 9; ++i)
        if (q[i] != p[i]) {
          drop_graphs(s);
          break;
        }
    }
  } bump(s, &w);
  const bool f64 = prec == FFM_F64;
  const NbPlanDev& p = s->plan;
  const size_t tsz = f64 ? 8 : 4;
  if (w.pos_batch < batch) {
    if (w.pos) cudaFree(w.pos);
    if (w.ipos) cudaFree(w.ipos);
    if (w.bbox) cudaFree(w.bbox);
    w.pos = w.ipos = w.bbox = nullptr;
    const size_t bytes = (size_t)batch * p.np * 4 * tsz;
    if (cudaMalloc(&w.pos, bytes) != cudaSuccess || cudaMalloc(&w.ipos, bytes) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for packed coordinates");
    if (p.has_cutoff &&
        cudaMalloc(&w.bbox, (size_t)batch * (p.np / kJB) * 6 * tsz) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for block boxes");
    w.pos_batch = batch;
    FFM_CUDA(launch_pad(p.n, p.np, batch, f64, w.pos, w.ipos, 0));
    FFM_CUDA(cudaDeviceSynchronize());
  }
  // partial slots of units another rank owns are never written: they must
  // read as zero in the gather and the energy reduction
  if (grad && !w.ipart) {
    const size_t ib = p.ntiles ? (size_t)p.ntiles * 3 * kIB * tsz : (size_t)p.nunits * 3 * p.S * tsz;
    const size_t jb = p.ntiles ? (size_t)p.ntiles * 3 * kJB * tsz : ib;
    if (cudaMalloc(&w.ipart, ib) != cudaSuccess || cudaMalloc(&w.jpart, jb) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for gradient partials");
    FFM_CUDA(cudaMemset(w.ipart, 0, ib));
    FFM_CUDA(cudaMemset(w.jpart, 0, jb));
    // the caller's stream may not be ordered after the legacy stream
    FFM_CUDA(cudaDeviceSynchronize());
  }
  if (w.e_batch < batch) {
    if (w.epart) cudaFree(w.epart);
    w.epart = nullptr;
    // (the batch plan's units, too: batch > 1 sweeps use s->bplan)
    const size_t slots = std::max<size_t>(nb_slots(p), (size_t)s->bplan.nunits);
    const size_t bytes = (size_t)batch * slots * 3 * sizeof(double);
    if (cudaMalloc(&w.epart, bytes) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for energy partials");
    // units another rank owns: no energy, no close contact (min r^2 = 1e30)
    std::vector<double> init((size_t)batch * slots * 3, 0.0);
    for (size_t k = 2; k < init.size(); k += 3) init[k] = 1e30;
    FFM_CUDA(cudaMemcpy(w.epart, init.data(), bytes, cudaMemcpyHostToDevice));
    w.e_batch = batch;
  }
  if (!w.escratch) {
    const size_t bytes = (size_t)kMaxEnergyParts * 3 * sizeof(double) + 64;
    if (cudaMalloc(&w.escratch, bytes) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for the energy reduction scratch");
    FFM_CUDA(cudaMemset(w.escratch, 0, bytes));
    FFM_CUDA(cudaDeviceSynchronize());
  }
  if (w.te_batch < batch) {
    if (w.term_e) cudaFree(w.term_e);
    w.term_e = nullptr;
    const size_t ne = (size_t)std::max(1, term_blocks(s->tp)) * 5;
    if (cudaMalloc(&w.term_e, (size_t)batch * ne * sizeof(double)) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for term energies");
    w.te_batch = batch;
  }
  if (!w.term_st) {
    const size_t nw = (size_t)std::max(1, term_blocks(s->tp)) * kTermSlotsPerBlock;
    if (cudaMalloc(&w.term_st, nw * 4 * sizeof(int64_t)) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for term status slots");
  }
  if (grad && !w.term_f) {
    const size_t nsl = std::max(1, s->tp.nslots);
    if (cudaMalloc(&w.term_f, nsl * 3 * sizeof(double)) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for term forces");
  }
  return FFM_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

const char* ffm_version(void) { return "ffmin_b200 0.1.0 (sm_100a)"; }
const char* ffm_last_error(void) { return g_err.c_str(); }

int ffm_system_create(ffm_system_t** out, int device, int64_t n, const double* q_h,
                      const double* sigma_h, const double* eps_h, int64_t nspecial,
                      const int64_t* special_i_h, const int64_t* special_j_h,
                      const double* special_s_h, double cutoff) {
  if (!out) return fail(FFM_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 0 || n > (1LL << 26)) return fail(FFM_EINVAL, "atom count out of range");
  if (n > 0 && (!q_h || !sigma_h || !eps_h)) return fail(FFM_EINVAL, "parameter array is NULL");
  if (nspecial < 0 || (nspecial > 0 && (!special_i_h || !special_j_h || !special_s_h)))
    return fail(FFM_EINVAL, "special pair arrays are NULL");
  FFM_CUDA(cudaSetDevice(device));
  DeviceGuard guard(device);
  auto* s = new ffm_system();
  s->device = device;
  NbPlanDev& p = s->plan;
  p.n = (int)n;
  p.S = s->S0 = choose_S(n);
  p.nb = (int)std::max<int64_t>(1, (n + p.S - 1) / p.S);
  p.np = p.nb * p.S;
  p.nunits = p.nb * (p.nb + 1) / 2;
  p.has_cutoff = cutoff > 0.0 ? 1 : 0;
  p.unit_list = nullptr;
  p.nlaunch = p.nunits;
  p.cut2 = cutoff > 0.0 ? cutoff * cutoff : 0.0;
  {  // culling margin: the boxes are built in the kernel precision, so pad
     // the cutoff by a relative and an absolute slack before comparing
    const double cm = cutoff > 0.0 ? cutoff * (1.0 + 1e-5) + 1e-4 : 0.0;
    p.cull2 = cm * cm;
  }
  int rc;
#define FFM_TRY(x)     \
  do {                 \
    rc = (x);          \
    if (rc) {          \
      free_all(s);     \
      delete s;        \
      return rc;       \
    }                  \
  } while (0)

  // ---- per-atom records (padding atoms keep zero charge / LJ)
  std::vector<double> qt(p.np, 0.0), qv(q_h, q_h + n), sg(sigma_h, sigma_h + n),
      ep(eps_h, eps_h + n);
  std::vector<float2> lj32(p.np, make_float2(0.f, 0.f));
  std::vector<double2> lj64(p.np, make_double2(0.0, 0.0));
  const double sqc = std::sqrt(kCoulomb);
  for (int64_t a = 0; a < n; ++a) {
    if (!(sigma_h[a] > 0.0) || !(eps_h[a] >= 0.0) || !std::isfinite(q_h[a]))
      FFM_TRY(fail(FFM_EINVAL, "atom parameters invalid (sigma > 0, eps >= 0, finite q)"));
    qt[a] = q_h[a] * sqc;
    const double se = 2.0 * std::sqrt(eps_h[a]);
    const double s3 = sigma_h[a] * sigma_h[a] * sigma_h[a];
    lj64[a] = make_double2(se * s3 * s3, se * s3);
    lj32[a] = make_float2((float)lj64[a].x, (float)lj64[a].y);
  }
  FFM_TRY(upload(&s->d_qt, qt));
  FFM_TRY(upload(&s->d_lj32, lj32));
  FFM_TRY(upload(&s->d_lj64, lj64));
  if (cudaMalloc(&s->d_ilj32, (size_t)p.np * 2 * sizeof(float)) != cudaSuccess ||
      cudaMalloc(&s->d_ilj64, (size_t)p.np * 2 * sizeof(double)) != cudaSuccess)
    FFM_TRY(fail(FFM_ENOMEM, "cudaMalloc failed for LJ records"));
  {
    cudaError_t e = launch_ilj(p.np, false, s->d_lj64, s->d_ilj32, 0);
    if (e == cudaSuccess) e = launch_ilj(p.np, true, s->d_lj64, s->d_ilj64, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess)
      FFM_TRY(fail(FFM_ECUDA, std::string("building the LJ pair records failed: ") +
                                  cudaGetErrorString(e)));
  }
  FFM_TRY(upload(&s->d_q, qv));
  FFM_TRY(upload(&s->d_sigma, sg));
  FFM_TRY(upload(&s->d_eps, ep));

  // ---- special pairs: canonical (i < j), sorted, unique
  std::vector<std::tuple<int, int, double>> sp;
  sp.reserve(nspecial);
  for (int64_t k = 0; k < nspecial; ++k) {
    int64_t i = special_i_h[k], j = special_j_h[k];
    if (i == j || i < 0 || j < 0 || i >= n || j >= n)
      FFM_TRY(fail(FFM_EINVAL, "special pair index out of range or i == j"));
    if (i > j) std::swap(i, j);
    if (!std::isfinite(special_s_h[k]))
      FFM_TRY(fail(FFM_EINVAL, "special pair scale not finite"));
    if (special_s_h[k] == 1.0) continue;  // same as the default
    sp.emplace_back((int)i, (int)j, special_s_h[k]);
  }
  std::sort(sp.begin(), sp.end());
  for (size_t k = 1; k < sp.size(); ++k)
    if (std::get<0>(sp[k]) == std::get<0>(sp[k - 1]) && std::get<1>(sp[k]) == std::get<1>(sp[k - 1]))
      FFM_TRY(fail(FFM_EINVAL, "duplicate special pair"));

  // upper rows (finder) and full rows (atom delta)
  std::vector<int> sp_ptr(n + 1, 0), sp_j;
  std::vector<double> sp_s;
  std::vector<std::vector<std::pair<int, double>>> full(n);
  for (auto& e : sp) {
    sp_ptr[std::get<0>(e) + 1]++;
    full[std::get<0>(e)].emplace_back(std::get<1>(e), std::get<2>(e));
    full[std::get<1>(e)].emplace_back(std::get<0>(e), std::get<2>(e));
  }
  for (int64_t a = 0; a < n; ++a) sp_ptr[a + 1] += sp_ptr[a];
  for (auto& e : sp) {
    sp_j.push_back(std::get<1>(e));
    sp_s.push_back(std::get<2>(e));
  }
  std::vector<int> fptr(n + 1, 0), fj;
  std::vector<double> fs;
  for (int64_t a = 0; a < n; ++a) {
    std::sort(full[a].begin(), full[a].end());
    fptr[a + 1] = fptr[a] + (int)full[a].size();
    for (auto& e : full[a]) {
      fj.push_back(e.first);
      fs.push_back(e.second);
    }
  }
  if (n == 0) sp_ptr.assign(1, 0), fptr.assign(1, 0);
  FFM_TRY(upload(&s->d_sp_ptr, sp_ptr));
  FFM_TRY(upload(&s->d_sp_j, sp_j));
  FFM_TRY(upload(&s->d_sp_s, sp_s));
  FFM_TRY(upload(&s->d_fsp_ptr, fptr));
  FFM_TRY(upload(&s->d_fsp_j, fj));
  FFM_TRY(upload(&s->d_fsp_s, fs));

  // ---- tile masks for the dense sweep, and the scaled list
  const int nsub = p.np / kIB, njbt = p.np / kJB;
  std::map<int64_t, std::vector<uint32_t>> tiles;
  for (auto& e : sp) {
    const int i = std::get<0>(e), j = std::get<1>(e);
    const int64_t key = (int64_t)(i / kIB) * njbt + j / kJB;
    auto& m = tiles[key];
    if (m.empty()) m.assign(kIB, 0u);
    m[i % kIB] |= 1u << (j % kJB);
    if (std::get<2>(e) != 0.0) {
      s->scaled.emplace_back(i, j);
      s->scaled_s.push_back(std::get<2>(e));
    }
  }
  std::vector<int> spt_ptr(nsub + 1, 0), spt_m;
  std::vector<uint32_t> spt_mask;
  for (auto& kv : tiles) {
    const int k = (int)(kv.first / njbt), m = (int)(kv.first % njbt);
    spt_ptr[k + 1]++;
    spt_m.push_back(m);
    spt_mask.insert(spt_mask.end(), kv.second.begin(), kv.second.end());
  }
  for (int k = 0; k < nsub; ++k) spt_ptr[k + 1] += spt_ptr[k];
  s->nspt = (int)spt_m.size();
  FFM_TRY(upload(&s->d_spt_ptr, spt_ptr));
  FFM_TRY(upload(&s->d_spt_m, spt_m));
  FFM_TRY(upload(&s->d_spt_mask, spt_mask));
  std::vector<int> scidx;
  for (auto& e : s->scaled) {
    scidx.push_back(e.first);
    scidx.push_back(e.second);
  }
  FFM_TRY(upload(&s->d_sc_idx, scidx));
  FFM_TRY(upload(&s->d_sc_s, s->scaled_s));

  // ---- units: off-diagonal first (full work), diagonal last (half work)
  FFM_TRY(build_units(s, p.S, split_count(s, p.S, 1), 1));
  {  // the batch plan: the largest unit edge that divides np (units mode)
    NbPlanDev& b = s->bplan;
    b = p;
    for (int Sb : {1024, 512, 256})
      if (Sb >= p.S && p.np % Sb == 0) {
        b.S = Sb;
        break;
      }
    b.nb = p.np / b.S;
    b.nunits = b.nb * (b.nb + 1) / 2;
    b.nlaunch = n > 0 ? b.nunits : 0;
    std::vector<int2> brc;
    for (int r = 0; r < b.nb; ++r)
      for (int c = r + 1; c < b.nb; ++c) brc.push_back(make_int2(r, c));
    for (int r = 0; r < b.nb; ++r) brc.push_back(make_int2(r, r));
    FFM_TRY(upload(&s->d_unit_rc_b, brc));
    b.unit_rc = s->d_unit_rc_b;
    b.unit_ks = nullptr;  // whole units
    b.unit_list = nullptr;
    b.ntiles = 0;
    b.tiles = nullptr;
    b.tile_list = nullptr;
  }
  if (n > 0 && use_tiles(p, device)) FFM_TRY(build_tiles(s, spt_ptr, spt_m));
  p.spt_ptr = s->bplan.spt_ptr = s->d_spt_ptr;
  p.spt_m = s->bplan.spt_m = s->d_spt_m;
  p.spt_mask = s->bplan.spt_mask = s->d_spt_mask;

  s->tp.has_cutoff = p.has_cutoff;
  s->tp.cutoff = cutoff > 0.0 ? cutoff : 0.0;
  FFM_TRY(build_terms(s, 0, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0,
                      nullptr, nullptr));
#undef FFM_TRY
  *out = s;
  return FFM_OK;
}

int ffm_system_set_terms(ffm_system_t* s, int64_t nbond, const int64_t* bond_idx_h,
                         const double* bond_K_h, const double* bond_r0_h, int64_t nangle,
                         const int64_t* ang_idx_h, const double* ang_K_h,
                         const double* ang_t0_h, int64_t ndih, const int64_t* dih_idx_h,
                         const double* dih_V_h) {
  if (!s) return fail(FFM_EINVAL, "system is NULL");
  if (nbond < 0 || nangle < 0 || ndih < 0) return fail(FFM_EINVAL, "negative term count");
  if ((nbond && (!bond_idx_h || !bond_K_h || !bond_r0_h)) ||
      (nangle && (!ang_idx_h || !ang_K_h || !ang_t0_h)) || (ndih && (!dih_idx_h || !dih_V_h)))
    return fail(FFM_EINVAL, "term array is NULL");
  DeviceGuard guard(s->device);
  cudaDeviceSynchronize();
  drop_graphs(s);
  return build_terms(s, nbond, bond_idx_h, bond_K_h, bond_r0_h, nangle, ang_idx_h, ang_K_h,
                     ang_t0_h, ndih, dih_idx_h, dih_V_h);
}

int ffm_system_destroy(ffm_system_t* s) {
  if (!s) return FFM_OK;
  DeviceGuard guard(s->device);
  cudaDeviceSynchronize();
  free_all(s);
  delete s;
  return FFM_OK;
}

int ffm_system_set_shard(ffm_system_t* s, int rank, int nranks) {
  if (!s || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FFM_EINVAL, "bad shard (rank, nranks)");
  DeviceGuard guard(s->device);
  FFM_CUDA(cudaDeviceSynchronize());
  drop_graphs(s);
  if (s->d_unit_list) cudaFree(s->d_unit_list);
  s->d_unit_list = nullptr;
  s->rank = rank;
  s->nranks = nranks;
  if (s->d_tile_list) cudaFree(s->d_tile_list);
  s->d_tile_list = nullptr;
  if (s->plan.ntiles > 0) {  // tile mode: tiles dealt round-robin
    s->plan.tile_list = nullptr;
    s->plan.nlaunch = s->plan.n > 0 ? s->plan.ntiles : 0;
    if (nranks > 1) {
      std::vector<int> mine;
      for (int t = rank; t < s->plan.ntiles; t += nranks) mine.push_back(t);
      if (mine.empty()) mine.push_back(0), s->plan.nlaunch = 0;
      else s->plan.nlaunch = (int)mine.size();
      int rc = upload(&s->d_tile_list, mine);
      if (rc) return rc;
      s->plan.tile_list = s->d_tile_list;
    }
  } else {
    // re-plan the super-unit edge for this shard count (the single-rank
    // edge is kept from creation: s->S0)
    const int S = nranks == 1 ? s->S0 : choose_S_sharded(s->plan, s->S0, nranks);
    int rc = build_units(s, S, split_count(s, S, nranks), nranks);
    if (rc) return rc;
  }
  if (s->plan.ntiles > 0) {
  } else if (nranks == 1) {
    s->plan.unit_list = nullptr;
    s->plan.nlaunch = s->plan.nunits;
  } else {
    // this rank's slots (u % nranks == rank, build_units), null units skipped
    std::vector<int> mine;
    for (int u = rank; u < s->plan.nunits; u += nranks)
      if (s->unit_live[u]) mine.push_back(u);
    if (mine.empty()) {
      mine.push_back(0);
      s->plan.nlaunch = 0;
    }
    int rc = upload(&s->d_unit_list, mine);
    if (rc) return rc;
    s->plan.unit_list = s->d_unit_list;
    if (s->plan.nlaunch != 0) s->plan.nlaunch = (int)mine.size();
  }
  // drop the partial buffers so stale slots of other ranks read as zero
  for (auto& w : s->w) {
    for (void** p : {&w.ipart, &w.jpart})
      if (*p) {
        cudaFree(*p);
        *p = nullptr;
      }
    if (w.epart) cudaFree(w.epart);
    w.epart = nullptr;
    w.e_batch = 0;
  }
  return FFM_OK;
}

// FP64 sweeps of mid-size systems run faster on 128-atom super-units than on
// the 256 choose_S picks for both precisions (tools/mid_sweep.py, one B200,
// FP64 S = 256 vs 128, us per evaluation: energy+gradient 4500 atoms 66.9 ->
// 49.4, 5000 67.0 -> 56.4, 6000 82.8 -> 68.6, 8000 114.3 -> 102.3, 10000
// 155.0 -> 147.4, 12000 198.1 -> 198.2; energy only 4500 49.4 -> 31.0, 6000
// 50.0 -> 41.2, 8000 63.9 -> 60.9, 10000 86.5 -> 86.4, 12000 109.3 -> 113.2;
// graph-resident L-BFGS per iteration 5000 0.576 -> 0.451 ms, 8000 0.729 ->
// 0.720, 10000 0.930 -> 0.937); FP32 is not (5000 atoms 37.5 -> 41.2 us)
#ifndef FFM_F64_EDGE128_UNITS
#define FFM_F64_EDGE128_UNITS 800  // S = 256 plans with fewer units switch to 128
#endif
int ffm_preferred_edge(int64_t n, int precision, int* edge) {
  if (!edge || n < 0) return fail(FFM_EINVAL, "bad argument");
  const int S = choose_S(n);
  const int64_t nb = std::max<int64_t>(1, (n + S - 1) / S);
  const int64_t units = nb * (nb + 1) / 2;
  if (units < 150) *edge = 0;  // tile mode (use_tiles)
  else if (precision == FFM_F64 && S == 256 && units < FFM_F64_EDGE128_UNITS) *edge = 128;
  else *edge = S;
  return FFM_OK;
}

int ffm_system_set_edge(ffm_system_t* s, int S) {
  if (!s) return fail(FFM_EINVAL, "system is NULL");
  if (s->plan.ntiles > 0) return fail(FFM_EINVAL, "a tile-mode plan has no super-unit edge");
  if (S < 128 || S > 1024 || S % 128 || s->plan.np % S)
    return fail(FFM_EINVAL, "edge must be a multiple of 128 in [128, 1024] dividing the padded atom count");
  s->S0 = S;
  return ffm_system_set_shard(s, s->rank, s->nranks);  // rebuilds the units with edge S0
}

int ffm_system_set_comm(ffm_system_t* s, void* comm) {
  if (!s) return fail(FFM_EINVAL, "NULL argument");
  DeviceGuard guard(s->device);
  FFM_CUDA(cudaDeviceSynchronize());
  drop_graphs(s);
  s->comm = nullptr;
  if (!comm) return FFM_OK;
  if (!nccl_allreduce()) return fail(FFM_EINVAL, "ncclAllReduce not found (libnccl.so.2 not loaded)");
  if (!s->d_comb) {
    const size_t bytes = ((size_t)3 * s->plan.n + FFM_NTERMS + 8) * sizeof(double);
    if (cudaMalloc(&s->d_comb, bytes) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for the all-reduce buffer");
  }
  s->comm = comm;
  return FFM_OK;
}

int ffm_debug_phase_clock(ffm_system_t* s, void* clock_d, int* grids) {
  if (!s || !grids) return fail(FFM_EINVAL, "NULL argument");
  s->phase_clock = static_cast<unsigned long long*>(clock_d);
  for (int p = 0; p < 2; ++p)
    for (int g = 0; g < 2; ++g) grids[2 * p + g] = s->small_grid[p][g][0] ? s->small_grid[p][g][0] : s->small_grid[p][g][1];
  return FFM_OK;
}

int ffm_system_nb_ms(ffm_system_t* s, float* ms) {
  if (!s || !ms) return fail(FFM_EINVAL, "NULL argument");
  if (!s->timed) return fail(FFM_EINVAL, "last evaluation was not timed (FFM_TIME_NB)");
  DeviceGuard guard(s->device);
  FFM_CUDA(cudaEventSynchronize(s->ev_nb1));
  FFM_CUDA(cudaEventElapsedTime(ms, s->ev_nb0, s->ev_nb1));
  return FFM_OK;
}

long long ffm_launch_count(void) { return g_launch_count.load(); }

int ffm_system_info(const ffm_system_t* s, int64_t* info) {
  if (!s || !info) return fail(FFM_EINVAL, "NULL argument");
  info[0] = s->plan.n;
  info[1] = s->plan.np;
  info[2] = s->plan.S;
  info[3] = s->plan.nb;
  info[4] = s->plan.nunits;
  info[5] = s->nspt;
  info[6] = (int64_t)s->scaled.size();
  info[7] = s->device;
  return FFM_OK;
}

// The launch sequence of one evaluation (no host synchronisation).
// The one-launch small-system evaluation (ffm_small.cu) of a tile-mode,
// unsharded system with every term; false when it does not apply.
// trial_*: a line-search trial of a graph-resident driver (see
// SmallEvalArgs), else all null.
static bool small_fused_applies(const ffm_system* s) {
  return s->plan.ntiles > 0 && s->plan.n > 0 && s->nranks == 1;
}

static int issue_small(ffm_system* s, int precision, bool grad, const double* coords_d,
                       double* grad_d, double* energies_d, int64_t* status_d, cudaStream_t st,
                       bool* launched, double* trial_out = nullptr,
                       const double* trial_x = nullptr, const double* trial_r = nullptr,
                       const double* trial_h = nullptr, MinState* ls_state = nullptr,
                       cudaGraphConditionalHandle ls_loop = 0) {
  *launched = false;
  Work& w = s->w[precision];
  const bool f64 = precision == FFM_F64;
  int* grid_slot = s->small_grid[precision][grad ? 1 : 0];  // [variant], picked once a is filled
  SmallEvalArgs a;
  a.plan = s->plan;
  a.tp = s->tp;
  a.nterm_blocks = term_blocks(s->tp);
  a.coords = coords_d;
  a.qt = s->d_qt;
  a.pos = w.pos;
  a.ipos = w.ipos;
  a.lj = f64 ? (const void*)s->d_lj64 : (const void*)s->d_lj32;
  a.ilj = f64 ? (const void*)s->d_ilj64 : (const void*)s->d_ilj32;
  a.ipart = w.ipart;
  a.jpart = w.jpart;
  a.epart = w.epart;
  a.term_part = w.term_e;
  a.term_f = w.term_f;
  a.term_st = w.term_st;
  a.trow_ptr = s->d_trow_ptr;
  a.tcol_ptr = s->d_tcol_ptr;
  a.tcol_idx = s->d_tcol_idx;
  a.slot_ptr = s->d_slot_ptr;
  a.slot_idx = s->d_slot_idx;
  a.sp_ptr = s->d_sp_ptr;
  a.sp_j = s->d_sp_j;
  a.sp_s = s->d_sp_s;
  a.grad = grad_d;
  a.energies = energies_d;
  a.status = status_d;
  a.phase_clock = s->phase_clock;
  a.trial_out = trial_out;
  a.trial_x = trial_x;
  a.trial_r = trial_r;
  a.trial_h = trial_h;
  a.ls_state = ls_state;
  a.ls_loop = ls_loop;
  int& grid = grid_slot[small_fromx(a, f64) ? 1 : 0];
  if (grid == 0) grid = small_eval_grid(a, f64, grad, s->device);
  if (grid <= 0) return FFM_OK;
  FFM_CUDA(launch_small_eval(a, f64, grad, grid, st));
  *launched = true;
  return FFM_OK;
}

static int issue_eval_local(ffm_system* s, int precision, int flags, const double* coords_d,
                            double* grad_d, double* energies_d, int64_t* status_d,
                            cudaStream_t st);

// One evaluation; a sharded system with a communicator completes it on the
// device: encode, one NCCL all-reduce, decode (parallel.py's ShardCombiner)
static int issue_eval(ffm_system* s, int precision, int flags, const double* coords_d,
                      double* grad_d, double* energies_d, int64_t* status_d, cudaStream_t st) {
  FFM_TRYR(issue_eval_local(s, precision, flags, coords_d, grad_d, energies_d, status_d, st));
  if (s->nranks <= 1 || !s->comm) return FFM_OK;
  const bool grad = (flags & FFM_GRAD) != 0;
  const int64_t n = s->plan.n, n3 = 3 * n;
  double* buf = grad ? s->d_comb : s->d_comb + n3;
  const size_t count = (size_t)(grad ? n3 : 0) + FFM_NTERMS + 8;
  FFM_CUDA(launch_combine_encode(n, grad ? grad_d : nullptr, energies_d, status_d, s->d_comb, st));
  const ncclResult_t r = nccl_allreduce()(buf, buf, count, ncclFloat64, ncclSum,
                                          static_cast<ncclComm_t>(s->comm), st);
  if (r != ncclSuccess) return fail(FFM_ECUDA, "ncclAllReduce failed (" + std::to_string((int)r) + ")");
  FFM_CUDA(launch_combine_decode(n, s->d_comb, grad ? grad_d : nullptr, energies_d, status_d, st));
  return FFM_OK;
}

static int issue_eval_local(ffm_system* s, int precision, int flags, const double* coords_d,
                            double* grad_d, double* energies_d, int64_t* status_d,
                            cudaStream_t st) {
  const bool grad = (flags & FFM_GRAD) != 0;
  Work& w = s->w[precision];
  const bool f64 = precision == FFM_F64;
  const bool do_nb = !(flags & FFM_NO_NB), do_terms = !(flags & FFM_NO_TERMS);
  const void* lj = f64 ? (const void*)s->d_lj64 : (const void*)s->d_lj32;
  const void* ilj = f64 ? (const void*)s->d_ilj64 : (const void*)s->d_ilj32;
  TermPlanDev tp = s->tp;  // the term types this call evaluates
  if (!do_terms || s->rank != 0) tp.nbond = tp.nangle = tp.ndih = 0;  // O(N) terms: rank 0
  if (!do_nb || s->rank != 0) tp.nscaled = 0;
  const bool time_nb = (flags & FFM_TIME_NB) != 0 && do_nb;
  // small system evaluated whole: one cooperative launch (ffm_small.cu)
  if (small_fused_applies(s) && do_nb && do_terms && !time_nb && !(flags & FFM_NO_FUSE)) {
    bool launched = false;
    FFM_TRYR(issue_small(s, precision, grad, coords_d, grad_d, energies_d, status_d, st,
                         &launched));
    if (launched) return FFM_OK;
  }
  FFM_CUDA(launch_pack(s->plan.n, s->plan.np, 1, f64, coords_d, s->d_qt, w.pos, w.ipos,
                       status_d, st));
  // fork: the term kernel (bonded terms, scaled pairs) beside the sweep; it
  // fills the sweep's last partial wave instead of running after it
  const bool fork = term_blocks(tp) > 0 && do_nb && s->plan.n > 0;
  if (fork) {
    if (!s->side) {
      FFM_CUDA(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking));
      FFM_CUDA(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
      FFM_CUDA(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    }
    FFM_CUDA(cudaEventRecord(s->ev_fork, st));
    FFM_CUDA(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
    FFM_CUDA(launch_terms(tp, grad, 1, coords_d, w.term_e, w.term_f, status_d, s->side));
    FFM_CUDA(cudaEventRecord(s->ev_join, s->side));
  }
  if (time_nb) FFM_CUDA(cudaEventRecord(s->ev_nb0, st));
  if (do_nb && s->plan.has_cutoff)
    FFM_CUDA(launch_bbox(s->plan.n, s->plan.np, 1, f64, w.pos, w.bbox, st));
  if (do_nb)
    FFM_CUDA(launch_nb(s->plan, f64, grad, w.pos, lj, w.ipos, ilj, w.bbox, w.ipart, w.jpart,
                       w.epart, 1, st));
  if (time_nb) FFM_CUDA(cudaEventRecord(s->ev_nb1, st));
  if (fork)
    FFM_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
  else
    FFM_CUDA(launch_terms(tp, grad, 1, coords_d, w.term_e, w.term_f, status_d, st));
  if (grad && s->plan.n > 0) {
    // gather + energy reduction in one launch
    FFM_CUDA(launch_gather_reduce(
        s->plan.n, s->plan.S, s->plan.nb, f64, s->d_unit_index,
        s->plan.ntiles ? s->d_trow_ptr : nullptr, s->d_tcol_ptr, s->d_tcol_idx, w.ipart,
        w.jpart, s->d_slot_ptr, s->d_slot_idx, w.term_f, s->tp.slot_sc0, do_nb,
        do_terms && s->rank == 0, do_nb && s->rank == 0, grad_d,
        do_nb ? nb_slots(s->plan) : 0, tp, w.epart, w.term_e, energies_d, status_d, s->rank,
        s->nranks, w.escratch, ecount(w), st));
    FFM_CUDA(launch_finder(s->plan.n, s->plan.np, 1, f64, w.pos, s->d_sp_ptr, s->d_sp_j,
                           s->d_sp_s, status_d, st));
    return FFM_OK;
  }
  FFM_CUDA(launch_reduce(do_nb ? nb_slots(s->plan) : 0, tp, 1, w.epart, w.term_e, energies_d,
                         status_d, s->plan.n, w.escratch, ecount(w), st));
  FFM_CUDA(launch_finder(do_nb ? s->plan.n : 0, s->plan.np, 1, f64, w.pos, s->d_sp_ptr,
                         s->d_sp_j, s->d_sp_s, status_d, st));
  return FFM_OK;
}

int ffm_eval(ffm_system_t* s, int precision, int flags, const double* coords_d,
             double* grad_d, double* energies_d, int64_t* status_d, void* stream) {
  if (!s || !energies_d || !status_d) return fail(FFM_EINVAL, "NULL argument");
  if (precision != FFM_F64 && precision != FFM_F32) return fail(FFM_EINVAL, "bad precision");
  const bool grad = (flags & FFM_GRAD) != 0;
  if (grad && !grad_d) return fail(FFM_EINVAL, "grad_d is NULL with FFM_GRAD");
  if (s->plan.n > 0 && !coords_d) return fail(FFM_EINVAL, "coords_d is NULL");
  DeviceGuard guard(s->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = ensure_work(s, precision, 1, grad);
  if (rc) return rc;
  const bool time_nb = (flags & FFM_TIME_NB) != 0 && !(flags & FFM_NO_NB);
  s->timed = time_nb;
  if (time_nb) {
    if (!s->ev_nb0) {
      FFM_CUDA(cudaEventCreate(&s->ev_nb0));
      FFM_CUDA(cudaEventCreate(&s->ev_nb1));
    }
    return issue_eval(s, precision, flags, coords_d, grad_d, energies_d, status_d, st);
  }
  if (flags & FFM_NO_GRAPH)
    return issue_eval(s, precision, flags, coords_d, grad_d, energies_d, status_d, st);
  // replay a captured graph of this exact call when there is one: one
  // launch instead of seven (small systems are launch-bound)
  for (size_t k = 0; k < s->graphs.size(); ++k) {
    auto& g = s->graphs[k];
    if (g.prec == precision && g.flags == flags && g.coords == coords_d && g.grad == grad_d &&
        g.energies == energies_d && g.status == status_d && g.gen == s->gen) {
      FFM_CUDA(cudaGraphLaunch(g.exec, st));
      count_launch(g.kernels);
      if (k + 1 != s->graphs.size()) std::rotate(s->graphs.begin() + k,
                                                 s->graphs.begin() + k + 1, s->graphs.end());
      return FFM_OK;
    }
  }
  if (!s->cap_stream) FFM_CUDA(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
  const long long before = g_launch_count.load();
  FFM_CUDA(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeRelaxed));
  rc = issue_eval(s, precision, flags, coords_d, grad_d, energies_d, status_d, s->cap_stream);
  cudaGraph_t graph = nullptr;
  cudaError_t ec = cudaStreamEndCapture(s->cap_stream, &graph);
  const long long kernels = g_launch_count.load() - before;
  g_launch_count.fetch_sub(kernels);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ec != cudaSuccess) return fail(FFM_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
  cudaGraphExec_t exec = nullptr;
  ec = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ec != cudaSuccess) return fail(FFM_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ec));
  if (s->graphs.size() >= 16) {
    cudaGraphExecDestroy(s->graphs.front().exec);
    s->graphs.erase(s->graphs.begin());
  }
  s->graphs.push_back({precision, flags, coords_d, grad_d, energies_d, status_d, s->gen, kernels, exec});
  FFM_CUDA(cudaGraphLaunch(exec, st));
  count_launch(kernels);
  return FFM_OK;
}

int ffm_eval_host(ffm_system_t* s, int precision, int flags, const double* coords_h,
                  double* grad_h, double* energies_h, int64_t* status_h) {
  if (!s || !energies_h || !status_h) return fail(FFM_EINVAL, "NULL argument");
  const bool grad = (flags & FFM_GRAD) != 0;
  if (grad && !grad_h) return fail(FFM_EINVAL, "grad_h is NULL with FFM_GRAD");
  DeviceGuard guard(s->device);
  const size_t cb = (size_t)std::max(1, s->plan.n) * 3 * sizeof(double);
  if (!s->h_coords_d) {
    if (cudaMalloc(&s->h_coords_d, cb) != cudaSuccess || cudaMalloc(&s->h_grad_d, cb) != cudaSuccess ||
        cudaMalloc(&s->h_en_d, FFM_NTERMS * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s->h_st_d, FFM_STATUS_WORDS * sizeof(int64_t)) != cudaSuccess)
      return fail(FFM_ENOMEM, "cudaMalloc failed for host-path staging");
  }
  const size_t nb = (size_t)s->plan.n * 3 * sizeof(double);
  if (nb) FFM_CUDA(cudaMemcpyAsync(s->h_coords_d, coords_h, nb, cudaMemcpyHostToDevice, 0));
  int rc = ffm_eval(s, precision, flags, s->h_coords_d, grad ? s->h_grad_d : nullptr,
                    s->h_en_d, s->h_st_d, nullptr);
  if (rc) return rc;
  if (grad && nb) FFM_CUDA(cudaMemcpyAsync(grad_h, s->h_grad_d, nb, cudaMemcpyDeviceToHost, 0));
  FFM_CUDA(cudaMemcpyAsync(energies_h, s->h_en_d, FFM_NTERMS * sizeof(double),
                           cudaMemcpyDeviceToHost, 0));
  FFM_CUDA(cudaMemcpyAsync(status_h, s->h_st_d, FFM_STATUS_WORDS * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, 0));
  FFM_CUDA(cudaStreamSynchronize(0));
  return FFM_OK;
}

int ffm_eval_batch(ffm_system_t* s, int precision, int64_t batch, const double* coords_d,
                   double* energies_d, int64_t* status_d, void* stream) {
  if (!s || !energies_d || !status_d) return fail(FFM_EINVAL, "NULL argument");
  if (precision != FFM_F64 && precision != FFM_F32) return fail(FFM_EINVAL, "bad precision");
  if (batch < 1 || batch > 65535) return fail(FFM_EINVAL, "batch must be in [1, 65535]");
  if (s->plan.n > 0 && !coords_d) return fail(FFM_EINVAL, "coords_d is NULL");
  DeviceGuard guard(s->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = ensure_work(s, precision, (int)batch, false);
  if (rc) return rc;
  Work& w = s->w[precision];
  const bool f64 = precision == FFM_F64;
  const void* lj = f64 ? (const void*)s->d_lj64 : (const void*)s->d_lj32;
  const int B = (int)batch;
  const void* ilj = f64 ? (const void*)s->d_ilj64 : (const void*)s->d_ilj32;
  FFM_CUDA(launch_pack(s->plan.n, s->plan.np, B, f64, coords_d, s->d_qt, w.pos, w.ipos,
                       status_d, st));
  if (s->plan.has_cutoff) FFM_CUDA(launch_bbox(s->plan.n, s->plan.np, B, f64, w.pos, w.bbox, st));
  // unsharded systems sweep the batch with the batch plan (large units);
  // sharded ones keep their rank's share of the main plan
  const NbPlanDev& bp = s->nranks == 1 ? s->bplan : s->plan;
  FFM_CUDA(launch_nb(bp, f64, false, w.pos, lj, w.ipos, ilj, w.bbox, nullptr, nullptr,
                     w.epart, B, st));
  TermPlanDev tp = s->tp;
  if (s->rank != 0) tp.nbond = tp.nangle = tp.ndih = tp.nscaled = 0;
  FFM_CUDA(launch_terms(tp, false, B, coords_d, w.term_e, nullptr, status_d, st));
  FFM_CUDA(launch_reduce(nb_slots(bp), tp, B, w.epart, w.term_e, energies_d, status_d,
                         s->plan.n, w.escratch, ecount(w), st));
  FFM_CUDA(launch_finder(s->plan.n, s->plan.np, B, f64, w.pos, s->d_sp_ptr, s->d_sp_j,
                         s->d_sp_s, status_d, st));
  return FFM_OK;
}

int ffm_atom_delta(ffm_system_t* s, const double* coords_d, int64_t ncand,
                   const int32_t* atoms_d, const double* newpos_d, double* out_d,
                   int64_t* status_d, void* stream) {
  return ffm_atom_delta_lin(s, coords_d, ncand, atoms_d, newpos_d, 0.0, out_d, status_d,
                            stream);
}

}  // extern "C"

// candidates below this count are split over delta_blocks(n) blocks each
// (a few probes of a large system would otherwise run on a few SMs); larger
// batches fill the GPU with one block per candidate
constexpr int64_t kDeltaSplitMax = 148;

// atom-delta scratch for up to ncand split candidates (outside graph capture)
static int ensure_delta_scratch(ffm_system* s, int64_t ncand) {
  if (ncand >= kDeltaSplitMax || ncand <= s->dl_cap) return FFM_OK;
  FFM_CUDA(cudaDeviceSynchronize());
  for (void* p : {(void*)s->dl_part, (void*)s->dl_bad, (void*)s->dl_cnt})
    if (p) cudaFree(p);
  s->dl_part = nullptr;
  s->dl_bad = nullptr;
  s->dl_cnt = nullptr;
  s->dl_cap = 0;
  const int64_t cap = kDeltaSplitMax;
  const size_t nb = (size_t)delta_blocks(s->plan.n);
  if (cudaMalloc(&s->dl_part, cap * nb * 6 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&s->dl_bad, cap * nb * 3 * sizeof(long long)) != cudaSuccess ||
      cudaMalloc(&s->dl_cnt, cap * sizeof(unsigned)) != cudaSuccess)
    return fail(FFM_ENOMEM, "cudaMalloc failed for the atom-delta scratch");
  FFM_CUDA(cudaMemset(s->dl_cnt, 0, cap * sizeof(unsigned)));
  FFM_CUDA(cudaDeviceSynchronize());
  s->dl_cap = cap;
  return FFM_OK;
}

static cudaError_t issue_atom_delta(ffm_system* s, const double* coords, int ncand,
                                    const int* atoms, const double* newpos, double lin,
                                    double* out, int64_t* status, cudaStream_t st) {
  const bool split = ncand < kDeltaSplitMax && ncand <= s->dl_cap;
  return launch_atom_delta(s->tp, coords, s->d_fsp_ptr, s->d_fsp_j, s->d_fsp_s, s->d_aterm_ptr,
                           s->d_aterm_idx, ncand, atoms, newpos, lin, out, status,
                           split ? s->dl_part : nullptr, split ? s->dl_bad : nullptr,
                           split ? s->dl_cnt : nullptr, st);
}

extern "C" {

int ffm_atom_delta_lin(ffm_system_t* s, const double* coords_d, int64_t ncand,
                       const int32_t* atoms_d, const double* newpos_d, double lin_cutoff,
                       double* out_d, int64_t* status_d, void* stream) {
  if (!s) return fail(FFM_EINVAL, "system is NULL");
  if (ncand < 0 || ncand > (1LL << 30)) return fail(FFM_EINVAL, "bad candidate count");
  if (lin_cutoff > 0.0 && s->plan.has_cutoff)
    return fail(FFM_EINVAL, "incremental delta requires a system nonbonded cutoff of none");
  if (ncand == 0) return FFM_OK;
  if (!coords_d || !atoms_d || !newpos_d || !out_d || !status_d)
    return fail(FFM_EINVAL, "NULL argument");
  DeviceGuard guard(s->device);
  FFM_TRYR(ensure_delta_scratch(s, ncand));
  FFM_CUDA(issue_atom_delta(s, coords_d, (int)ncand, atoms_d, newpos_d,
                            lin_cutoff > 0.0 ? lin_cutoff : 0.0, out_d, status_d,
                            static_cast<cudaStream_t>(stream)));
  return FFM_OK;
}

int ffm_farfield_build(ffm_system_t* s, const double* coords_d, int64_t atom, double cutoff,
                       double* e0_coef_d, uint8_t* near_mask_d, int64_t* bad_d,
                       void* stream) {
  if (!s || !coords_d || !e0_coef_d || !near_mask_d || !bad_d)
    return fail(FFM_EINVAL, "NULL argument");
  if (atom < 0 || atom >= s->plan.n) return fail(FFM_EINVAL, "atom index out of range");
  if (!(cutoff > 0.0)) return fail(FFM_EINVAL, "cutoff must be > 0");
  DeviceGuard guard(s->device);
  FFM_CUDA(launch_farfield(s->tp, coords_d, s->d_fsp_ptr, s->d_fsp_j, s->d_fsp_s, (int)atom,
                           cutoff, e0_coef_d, near_mask_d, bad_d,
                           static_cast<cudaStream_t>(stream)));
  return FFM_OK;
}

int64_t ffm_vec_scratch_doubles(void) {
  return (int64_t)std::max<size_t>(two_loop_scratch_doubles(), (size_t)vec_reduce_blocks());
}

int ffm_dot(int64_t n, const double* x_d, const double* y_d, double* out_d, double* scratch_d,
            void* stream) {
  if (n < 0 || !out_d || !scratch_d || (n > 0 && (!x_d || !y_d)))
    return fail(FFM_EINVAL, "bad dot arguments");
  FFM_CUDA(launch_dot(n, x_d, y_d, scratch_d, out_d, static_cast<cudaStream_t>(stream)));
  return FFM_OK;
}

int ffm_dots(int64_t n, int k, const double* const* xs_h, const double* const* ys_h,
             double* out_d, double* scratch_d, void* stream) {
  if (n < 0 || k < 1 || k > 8 || !xs_h || !ys_h || !out_d || !scratch_d)
    return fail(FFM_EINVAL, "bad dots arguments");
  FFM_CUDA(launch_dots(n, k, xs_h, ys_h, scratch_d, out_d, static_cast<cudaStream_t>(stream)));
  return FFM_OK;
}

int ffm_axpby(int64_t n, const double* a_d, double a_h, double sa, const double* x_d,
              const double* b_d, double b_h, const double* y_d, double* z_d, void* stream) {
  if (n < 0 || (n > 0 && (!x_d || !z_d))) return fail(FFM_EINVAL, "bad axpby arguments");
  if (n == 0) return FFM_OK;
  FFM_CUDA(launch_axpby(n, a_d, a_h, sa, x_d, b_d, b_h, y_d, z_d,
                        static_cast<cudaStream_t>(stream)));
  return FFM_OK;
}

int ffm_lbfgs_two_loop(int64_t n, int count, const int32_t* order_h, const double* rho_h,
                       const double* S_d, const double* Y_d, const double* g_d, double* d_d,
                       double* scratch_d, void* stream) {
  if (n < 1 || count < 1 || count > kMaxLbfgsPairs || !order_h || !rho_h || !S_d || !Y_d ||
      !g_d || !d_d || !scratch_d)
    return fail(FFM_EINVAL, "bad two-loop arguments");
  FFM_CUDA(launch_lbfgs_two_loop(n, count, order_h, rho_h, S_d, Y_d, g_d, d_d, scratch_d,
                                 static_cast<cudaStream_t>(stream)));
  return FFM_OK;
}


// ------------------------------------------------- graph-resident L-BFGS
}  // extern "C"

struct ffm_lbfgs {
  ffm_system* sys = nullptr;
  int device = 0;  // kept apart from sys: destroy must not touch a freed system
  int prec = 0;
  MinConfig cfg{};
  int64_t n = 0;  // 3 * atoms
  MinState* S = nullptr;
  double* rec = nullptr;
  double* buf = nullptr;  // x, g, x_new, g_new, x_trial, d, r, s_tmp, y_tmp, best, ring S, ring Y
  // (FGM: xn = w, st = x_prev, yt = x - x_prev, xt = x+ after the search;
  //  OFGM: xn = y, gnew = grad f(y), d = the aggregated direction)
  double *x, *g, *xn, *gnew, *xt, *d, *r, *st, *yt, *best, *ring_s, *ring_y;
  double* scratch = nullptr;
  double* en = nullptr;      // energies of the last evaluation
  int64_t* stw = nullptr;    // its status words
  cudaStream_t cap[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  // wiggle: probe scratch (atoms6, newpos6, out6, st6, atoms1, newpos1,
  // out1, st1) and the atoms of a launch
  void* wbuf = nullptr;
  int* wig_atoms = nullptr;
  double* gsum = nullptr;    // OFGM: running weighted gradient sum
  double* anchor = nullptr;  // OFGM: x0
  double* sched = nullptr;   // OFGM: t[0..N] (device)
  cudaGraphExec_t exec = nullptr;
  long long gen = -1;
  std::vector<double> rec_h;
};

namespace {

// append a conditional node to the capture running on `st`; its body graph
// is filled by a nested capture on another stream
int add_conditional(cudaStream_t st, cudaGraphConditionalHandle h,
                    cudaGraphConditionalNodeType type, cudaGraph_t* body) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  FFM_CUDA(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  FFM_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
  FFM_CUDA(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  *body = p.conditional.phGraph_out[0];
  return FFM_OK;
}


// bodies of the iteration graph (see ffm_min.cuh); each runs inside a
// capture on stream st
int cap_direction(ffm_lbfgs* L, cudaStream_t st, cudaGraphConditionalHandle hls) {
  MinState* S = L->S;
  const int method = L->cfg.method;
  if (method == kMethodLbfgs && lbfgs_dir_small_applies(L->n, L->cfg.m)) {
    // short vectors: the direction, its norm and the search's r and slope
    // in one launch (the line search below then skips its axpby and dot)
    FFM_CUDA(launch_lbfgs_dir_small(S, L->n, L->cfg.m, L->d, L->r, L->ring_s, L->ring_y, L->g, hls,
                                    st));
    return FFM_OK;
  }
  if (method == kMethodLbfgs)
    FFM_CUDA(launch_lbfgs_two_loop_dev(L->n, L->cfg.m, &S->count, S->idx_nf, S->rho_nf, &S->gn,
                                       L->ring_s, L->ring_y, L->g, L->d, L->scratch, st));
  if (method != kMethodSd) {  // L-BFGS: d = two-loop direction; CG: d = p
    const double* xs[1] = {L->d};
    FFM_CUDA(launch_dots(L->n, 1, xs, xs, L->scratch, &S->dd, st));
  }
  FFM_CUDA(launch_min_dir(S, hls, st));
  if (method == kMethodCg) FFM_CUDA(launch_select_neg(S, L->n, L->g, L->d, st));
  return FFM_OK;
}

int cap_trial(ffm_lbfgs* L, cudaStream_t st, cudaGraphConditionalHandle hloop) {
  MinState* S = L->S;
  // phi(h) = f(x + h r): lincomb(1.0, x, h, r)  (FGM: from w, OFGM: from y)
  const double* base = (L->cfg.method == kMethodFgm || L->cfg.method == kMethodOfgm) ? L->xn : L->x;
  if (small_fused_applies(L->sys)) {
    // small systems: the trial point, its evaluation and the probe
    // controller in one cooperative launch (was axpby + evaluation + ls_step)
    bool launched = false;
    FFM_TRYR(issue_small(L->sys, L->prec, false, L->xt, nullptr, L->en, L->stw, st, &launched,
                         L->xt, base, L->r, &S->h_trial, S, hloop));
    if (launched) return FFM_OK;
  }
  FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, base, &S->h_trial, 0.0, L->r, L->xt, st));
  FFM_TRYR(issue_eval(L->sys, L->prec, FFM_ENERGY, L->xt, nullptr, L->en, L->stw, st));
  FFM_CUDA(launch_min_ls_step(S, L->en, L->stw, hloop, st));
  return FFM_OK;
}

// FGM head of an iteration (ffmin/optimizers/fgm.py): theta / beta, the
// extrapolated point w, f and grad f at w (skipped at k = 0, where w = x),
// <g_w, g_w> and the checks; c3 captures the conditional evaluation
int cap_fgm_head(ffm_lbfgs* L, cudaStream_t st, cudaStream_t c3, cudaGraph_t bdir,
                 cudaGraphConditionalHandle hls) {
  MinState* S = L->S;
  cudaGraphConditionalHandle heval;
  FFM_CUDA(cudaGraphConditionalHandleCreate(&heval, bdir, 0, 0));
  FFM_CUDA(launch_fgm_pre(S, heval, st));
  // w = lincomb(1, x, beta, lincomb(1, x, -1, x_prev))
  FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->x, nullptr, -1.0, L->st, L->yt, st));
  FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->x, &S->beta, 0.0, L->yt, L->xn, st));
  cudaGraph_t beval = nullptr, tmp = nullptr;
  FFM_TRYR(add_conditional(st, heval, cudaGraphCondTypeIf, &beval));
  FFM_CUDA(cudaStreamBeginCaptureToGraph(c3, beval, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeRelaxed));
  int rc = issue_eval(L->sys, L->prec, FFM_ENERGY | FFM_GRAD, L->xn, L->g, L->en, L->stw, c3);
  cudaError_t e = cudaStreamEndCapture(c3, &tmp);
  if (rc) return rc;
  FFM_CUDA(e);
  const double* gs[1] = {L->g};
  FFM_CUDA(launch_dots(L->n, 1, gs, gs, L->scratch, &S->gg, st));
  FFM_CUDA(launch_fgm_post_eval(S, L->en, L->stw, hls, st));
  return FFM_OK;
}

// fixed-step family (ffmin/optimizers/gradient.py): the whole iteration,
// no line search; c3 captures the conditional gradient at w (Nesterov)
int cap_fixed(ffm_lbfgs* L, cudaStream_t st, cudaStream_t c3, cudaGraph_t bdir) {
  MinState* S = L->S;
  const int kind = L->cfg.momentum_kind;
  const double step = L->cfg.fixed_step;
  // the conditional gradient at w exists only for the Nesterov schemes (a
  // handle without its conditional node fails graph instantiation)
  cudaGraphConditionalHandle heval{};
  if (kind >= 2) FFM_CUDA(cudaGraphConditionalHandleCreate(&heval, bdir, 0, 0));
  FFM_CUDA(launch_mom_pre(S, heval, kind >= 2 ? 1 : 0, st));
  double* x_new = L->xn;
  if (kind == 0) {  // x - step g
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->x, nullptr, -step, L->g, L->xn, st));
  } else if (kind == 1) {  // lincomb(1, lincomb(1, x, -step, g), m, lincomb(1, x, -1, x_prev))
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->x, nullptr, -step, L->g, L->yt, st));
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->x, nullptr, -1.0, L->st, L->d, st));
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->yt, &S->beta, 0.0, L->d, L->xn, st));
  } else {  // w = lincomb(1, x, m, x - x_prev); g_w (k > 0); x+ = lincomb(1, w, -step, g_w)
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->x, nullptr, -1.0, L->st, L->d, st));
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->x, &S->beta, 0.0, L->d, L->xn, st));
    cudaGraph_t beval = nullptr, tmp = nullptr;
    FFM_TRYR(add_conditional(st, heval, cudaGraphCondTypeIf, &beval));
    FFM_CUDA(cudaStreamBeginCaptureToGraph(c3, beval, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed));
    int rc = issue_eval(L->sys, L->prec, FFM_ENERGY | FFM_GRAD, L->xn, L->g, L->en, L->stw, c3);
    if (!rc && launch_mom_wcheck(S, L->stw, c3) != cudaSuccess) rc = fail(FFM_ECUDA, "mom_wcheck");
    cudaError_t e = cudaStreamEndCapture(c3, &tmp);
    if (rc) return rc;
    FFM_CUDA(e);
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->xn, nullptr, -step, L->g, L->xt, st));
    x_new = L->xt;
  }
  FFM_CUDA(launch_fgm_shift(S, L->n, L->x, L->st, L->xn, x_new, L->best, st));
  const bool wform = kind >= 2;
  FFM_TRYR(issue_eval(L->sys, L->prec, wform ? FFM_ENERGY : (FFM_ENERGY | FFM_GRAD), L->x,
                      wform ? nullptr : L->g, L->en, L->stw, st));
  const double* gs[1] = {L->g};
  FFM_CUDA(launch_dots(L->n, 1, gs, gs, L->scratch, &S->gg, st));
  FFM_CUDA(launch_mom_post(S, L->en, L->stw, L->rec, st));
  return FFM_OK;
}

// OFGM (ffmin/optimizers/fgm.py, Eq. (12)): the whole iteration inside the
// IF(go) body; c3 / c4 capture the nested bodies (x = y, or the search)
int cap_ofgm(ffm_lbfgs* L, cudaStream_t st, cudaStream_t c3, cudaStream_t c4, cudaGraph_t bdir) {
  MinState* S = L->S;
  const int64_t n = L->n;
  FFM_CUDA(launch_ofgm_pre(S, st));
  // grad_sum = lincomb(1, grad_sum, t_k, g); d = lincomb(1 - 1/t, g, 2/t, grad_sum);
  // y = lincomb(1 - 1/t, x, 1/t, anchor)
  FFM_CUDA(launch_axpby(n, nullptr, 1.0, 1.0, L->gsum, &S->oc[0], 0.0, L->g, L->gsum, st));
  FFM_CUDA(launch_axpby(n, &S->oc[1], 0.0, 1.0, L->g, &S->oc[2], 0.0, L->gsum, L->d, st));
  FFM_CUDA(launch_axpby(n, &S->oc[1], 0.0, 1.0, L->x, &S->oc[3], 0.0, L->anchor, L->xn, st));
  const double* gs[1] = {L->g};
  if (L->cfg.fixed_step > 0.0) {  // x = lincomb(1, y, -(1/L), d); f, g = value_and_gradient(x)
    FFM_CUDA(launch_axpby(n, nullptr, 1.0, 1.0, L->xn, nullptr, -L->cfg.fixed_step, L->d, L->x,
                          st));
    FFM_TRYR(issue_eval(L->sys, L->prec, FFM_ENERGY | FFM_GRAD, L->x, L->g, L->en, L->stw, st));
    FFM_CUDA(launch_dots(n, 1, gs, gs, L->scratch, &S->gg, st));
    FFM_CUDA(launch_ofgm_post(S, L->en, L->stw, L->rec, 1, st));
    return FFM_OK;
  }
  const double* ds[1] = {L->d};
  FFM_CUDA(launch_dots(n, 1, ds, ds, L->scratch, &S->dd, st));
  cudaGraphConditionalHandle hz, hnz, hloop;
  FFM_CUDA(cudaGraphConditionalHandleCreate(&hz, bdir, 0, 0));
  FFM_CUDA(cudaGraphConditionalHandleCreate(&hnz, bdir, 0, 0));
  FFM_CUDA(launch_ofgm_dir(S, hz, hnz, st));
  cudaGraph_t bz = nullptr, bnz = nullptr, bloop = nullptr, tmp = nullptr;
  int rc = FFM_OK;
  cudaError_t e;
  // dn == 0: x = y, f = value(x)
  FFM_TRYR(add_conditional(st, hz, cudaGraphCondTypeIf, &bz));
  FFM_CUDA(cudaStreamBeginCaptureToGraph(c3, bz, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  if (launch_ofgm_x(S, n, L->xn, L->r, L->x, 0, c3) != cudaSuccess) rc = fail(FFM_ECUDA, "ofgm_x");
  if (!rc) rc = issue_eval(L->sys, L->prec, FFM_ENERGY, L->x, nullptr, L->en, L->stw, c3);
  if (!rc && launch_ofgm_value(S, L->en, L->stw, 1, c3) != cudaSuccess) rc = fail(FFM_ECUDA, "ofgm_value");
  e = cudaStreamEndCapture(c3, &tmp);
  if (rc) return rc;
  FFM_CUDA(e);
  // dn > 0: r = div(lincomb(-1, d), dn); f_y = value(y); [g_y = gradient(y)];
  // search from y; x = lincomb(1, y, h, r) or y
  FFM_TRYR(add_conditional(st, hnz, cudaGraphCondTypeIf, &bnz));
  FFM_CUDA(cudaGraphConditionalHandleCreate(&hloop, bnz, 0, 0));
  FFM_CUDA(cudaStreamBeginCaptureToGraph(c3, bnz, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  do {
    if (launch_axpby(n, &S->inv_dn, 0.0, -1.0, L->d, nullptr, 0.0, nullptr, L->r, c3) != cudaSuccess) {
      rc = fail(FFM_ECUDA, "axpby");
      break;
    }
    if ((rc = issue_eval(L->sys, L->prec, FFM_ENERGY, L->xn, nullptr, L->en, L->stw, c3))) break;
    if (launch_ofgm_value(S, L->en, L->stw, 0, c3) != cudaSuccess) {
      rc = fail(FFM_ECUDA, "ofgm_value");
      break;
    }
    if (L->cfg.ls_needs_grad) {
      if ((rc = issue_eval(L->sys, L->prec, FFM_ENERGY | FFM_GRAD, L->xn, L->gnew, L->en, L->stw,
                           c3)))
        break;
      const double* gy[1] = {L->gnew};
      const double* rs[1] = {L->r};
      if (launch_ofgm_gcheck(S, L->stw, c3) != cudaSuccess ||
          launch_dots(n, 1, gy, rs, L->scratch, &S->slope, c3) != cudaSuccess) {
        rc = fail(FFM_ECUDA, "ofgm slope");
        break;
      }
    }
    if (launch_min_ls_init(S, hloop, c3) != cudaSuccess) {
      rc = fail(FFM_ECUDA, "ls_init");
      break;
    }
    if ((rc = add_conditional(c3, hloop, cudaGraphCondTypeWhile, &bloop))) break;
    if (cudaStreamBeginCaptureToGraph(c4, bloop, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      rc = fail(FFM_ECUDA, "capture");
      break;
    }
    rc = cap_trial(L, c4, hloop);
    e = cudaStreamEndCapture(c4, &tmp);
    if (!rc && e != cudaSuccess) rc = fail(FFM_ECUDA, "capture end");
    if (rc) break;
    if (launch_ofgm_ls_post(S, c3) != cudaSuccess ||
        launch_ofgm_x(S, n, L->xn, L->r, L->x, 1, c3) != cudaSuccess)
      rc = fail(FFM_ECUDA, "ofgm_ls_post");
  } while (false);
  e = cudaStreamEndCapture(c3, &tmp);
  if (rc) return rc;
  FFM_CUDA(e);
  // g = gradient(x)
  FFM_TRYR(issue_eval(L->sys, L->prec, FFM_ENERGY | FFM_GRAD, L->x, L->g, L->en, L->stw, st));
  FFM_CUDA(launch_ofgm_gcheck(S, L->stw, st));
  FFM_CUDA(launch_dots(n, 1, gs, gs, L->scratch, &S->gg, st));
  FFM_CUDA(launch_ofgm_post(S, L->en, L->stw, L->rec, 0, st));
  return FFM_OK;
}

// wiggle scratch layout inside L->wbuf (8-byte slots)
struct WigBufs {
  int* atoms6;
  double* newpos6;
  double* out6;
  int64_t* st6;
  int* atoms1;
  double* newpos1;
  double* out1;
  int64_t* st1;
};
constexpr size_t kWigBufBytes = 8 * (8 + 18 + 36 + 18 + 8 + 3 + 6 + 3);
WigBufs wig_bufs(void* base) {
  double* p = static_cast<double*>(base);
  WigBufs b;
  b.atoms6 = reinterpret_cast<int*>(p);
  b.newpos6 = p + 8;
  b.out6 = p + 26;
  b.st6 = reinterpret_cast<int64_t*>(p + 62);
  b.atoms1 = reinterpret_cast<int*>(p + 80);
  b.newpos1 = p + 88;
  b.out1 = p + 91;
  b.st1 = reinterpret_cast<int64_t*>(p + 97);
  return b;
}

// gradient-free wiggle (ffmin/optimizers/wiggle.py): six axis probes, the
// parabola-vertex probe (IF), the exact check of the best candidate (IF),
// the epoch re-evaluation (IF) and the record -- one iteration inside the
// IF(go) body; c3 captures the nested bodies
int cap_wiggle(ffm_lbfgs* L, cudaStream_t st, cudaStream_t c3, cudaGraph_t bdir) {
  MinState* S = L->S;
  ffm_system* s = L->sys;
  const WigBufs b = wig_bufs(L->wbuf);
  const double lin = L->cfg.wig_cutoff;
  auto delta = [&](int k, const int* atoms, const double* newpos, double lc, double* out,
                   int64_t* stw, cudaStream_t q) {
    return issue_atom_delta(s, L->x, k, atoms, newpos, lc, out, stw, q);
  };
  FFM_CUDA(launch_wig_prep(S, L->x, b.atoms6, b.newpos6, st));
  FFM_CUDA(delta(6, b.atoms6, b.newpos6, lin, b.out6, b.st6, st));
  cudaGraphConditionalHandle hv, hx, he;
  FFM_CUDA(cudaGraphConditionalHandleCreate(&hv, bdir, 0, 0));
  FFM_CUDA(cudaGraphConditionalHandleCreate(&hx, bdir, 0, 0));
  FFM_CUDA(cudaGraphConditionalHandleCreate(&he, bdir, 0, 0));
  FFM_CUDA(launch_wig_ctrl1(S, b.out6, b.st6, b.atoms1, hv, st));
  cudaGraph_t body = nullptr, tmp = nullptr;
  cudaError_t e;
  int rc = FFM_OK;
  // the vertex probe
  FFM_TRYR(add_conditional(st, hv, cudaGraphCondTypeIf, &body));
  FFM_CUDA(cudaStreamBeginCaptureToGraph(c3, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  if (launch_wig_pos(S, L->x, b.newpos1, 0, c3) != cudaSuccess ||
      delta(1, b.atoms1, b.newpos1, lin, b.out1, b.st1, c3) != cudaSuccess ||
      launch_wig_ctrl_v(S, b.out1, b.st1, c3) != cudaSuccess)
    rc = fail(FFM_ECUDA, "wiggle vertex probe");
  e = cudaStreamEndCapture(c3, &tmp);
  if (rc) return rc;
  FFM_CUDA(e);
  FFM_CUDA(launch_wig_ctrl2(S, hx, st));
  // the exact check of the chosen move
  FFM_TRYR(add_conditional(st, hx, cudaGraphCondTypeIf, &body));
  FFM_CUDA(cudaStreamBeginCaptureToGraph(c3, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  if (launch_wig_pos(S, L->x, b.newpos1, 1, c3) != cudaSuccess ||
      delta(1, b.atoms1, b.newpos1, 0.0, b.out1, b.st1, c3) != cudaSuccess ||
      launch_wig_ctrl3(S, b.out1, b.st1, L->x, c3) != cudaSuccess)
    rc = fail(FFM_ECUDA, "wiggle exact probe");
  e = cudaStreamEndCapture(c3, &tmp);
  if (rc) return rc;
  FFM_CUDA(e);
  FFM_CUDA(launch_wig_end(S, he, st));
  // the epoch re-evaluation (incremental probes)
  FFM_TRYR(add_conditional(st, he, cudaGraphCondTypeIf, &body));
  FFM_CUDA(cudaStreamBeginCaptureToGraph(c3, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  rc = issue_eval(s, L->prec, FFM_ENERGY, L->x, nullptr, L->en, L->stw, c3);
  if (!rc && launch_wig_epoch(S, L->en, L->stw, c3) != cudaSuccess) rc = fail(FFM_ECUDA, "wig_epoch");
  e = cudaStreamEndCapture(c3, &tmp);
  if (rc) return rc;
  FFM_CUDA(e);
  FFM_CUDA(launch_wig_record(S, L->rec, st));
  return FFM_OK;
}

int cap_accept(ffm_lbfgs* L, cudaStream_t st) {
  MinState* S = L->S;
  if (L->cfg.method == kMethodFgm) {  // x+ = lincomb(1, w, h, r); no gradient at x+
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->xn, &S->res_h, 0.0, L->r, L->xt, st));
    FFM_CUDA(launch_fgm_accept(S, L->rec, st));
    return FFM_OK;
  }
  FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->x, &S->res_h, 0.0, L->r, L->xn, st));
  FFM_TRYR(issue_eval(L->sys, L->prec, FFM_ENERGY | FFM_GRAD, L->xn, L->gnew, L->en, L->stw,
                      st));
  if (L->cfg.method == kMethodLbfgs && L->n <= kAcceptSmallN) {
    // short vectors: the whole tail below in one launch (same bits)
    FFM_CUDA(launch_lbfgs_accept_small(S, L->n, L->stw, L->xn, L->gnew, L->x, L->g, L->st, L->yt,
                                       L->ring_s, L->ring_y, L->rec, st));
    return FFM_OK;
  }
  const double* gs[1] = {L->gnew};
  FFM_CUDA(launch_dots(L->n, 1, gs, gs, L->scratch, &S->gg, st));
  FFM_CUDA(launch_min_acc_check(S, L->stw, st));
  if (L->cfg.method == kMethodCg) {
    // y = g+ - g; beta from five dot products; p+ in place; descent test
    FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->gnew, nullptr, -1.0, L->g, L->yt, st));
    const double* xa[5] = {L->gnew, L->gnew, L->g, L->d, L->d};
    const double* ya[5] = {L->gnew, L->yt, L->g, L->yt, L->g};
    FFM_CUDA(launch_dots(L->n, 5, xa, ya, L->scratch, S->cgd, st));
    FFM_CUDA(launch_min_cg_beta(S, st));
    FFM_CUDA(launch_cg_update(S, L->n, L->gnew, L->d, st));
    const double* pa[1] = {L->d};
    FFM_CUDA(launch_dots(L->n, 1, pa, gs, L->scratch, &S->pg, st));
    FFM_CUDA(launch_min_cg_check(S, st));
    FFM_CUDA(launch_select_neg(S, L->n, L->gnew, L->d, st));
  }
  if (L->cfg.method != kMethodLbfgs) {  // no memory: x <- x+, g <- g+ (store_slot -1)
    FFM_CUDA(launch_min_store(S, L->n, L->st, L->yt, L->ring_s, L->ring_y, L->xn, L->gnew,
                              L->x, L->g, st));
    FFM_CUDA(launch_min_iter_end(S, L->rec, st));
    return FFM_OK;
  }
  // s = x_new - x, y = g_new - g (LbfgsMemory._axpy_into)
  FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->xn, nullptr, -1.0, L->x, L->st, st));
  FFM_CUDA(launch_axpby(L->n, nullptr, 1.0, 1.0, L->gnew, nullptr, -1.0, L->g, L->yt, st));
  const double* xa[3] = {L->st, L->st, L->yt};
  const double* ya[3] = {L->yt, L->st, L->yt};
  FFM_CUDA(launch_dots(L->n, 3, xa, ya, L->scratch, &S->sy, st));
  FFM_CUDA(launch_min_commit(S, st));
  FFM_CUDA(launch_min_store(S, L->n, L->st, L->yt, L->ring_s, L->ring_y, L->xn, L->gnew, L->x,
                            L->g, st));
  FFM_CUDA(launch_min_iter_end(S, L->rec, st));
  return FFM_OK;
}

int lbfgs_build(ffm_lbfgs* L) {
  ffm_system* s = L->sys;
  if (L->exec) {
    cudaGraphExecDestroy(L->exec);
    L->exec = nullptr;
  }
  FFM_TRYR(ensure_work(s, L->prec, 1, true));
  // first use of each kernel variant outside any capture (function
  // attributes are set on first launch)
  FFM_TRYR(issue_eval(s, L->prec, FFM_ENERGY, L->x, nullptr, L->en, L->stw, L->cap[0]));
  FFM_TRYR(issue_eval(s, L->prec, FFM_ENERGY | FFM_GRAD, L->x, L->gnew, L->en, L->stw, L->cap[0]));
  FFM_CUDA(two_loop_small_prepare());
  if (L->cfg.method == kMethodWiggle) FFM_TRYR(ensure_delta_scratch(s, 6));
  FFM_CUDA(lbfgs_dir_small_prepare());
  FFM_CUDA(cudaStreamSynchronize(L->cap[0]));
  MinState* S = L->S;
  const long long before = g_launch_count.load();
  cudaGraph_t top = nullptr;
  FFM_CUDA(cudaGraphCreate(&top, 0));
  auto fail_graph = [&](int rc) {
    g_launch_count.fetch_sub(g_launch_count.load() - before);
    for (cudaStream_t c : L->cap) {
      cudaStreamCaptureStatus cs;
      if (cudaStreamIsCapturing(c, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        cudaGraph_t t = nullptr;
        cudaStreamEndCapture(c, &t);
        if (t && t != top) cudaGraphDestroy(t);
      }
    }
    cudaGraphDestroy(top);
    return rc;
  };
#define FFM_G(x)                     \
  do {                               \
    int rc_ = (x);                   \
    if (rc_) return fail_graph(rc_); \
  } while (0)
#define FFM_GC(x)                                                                        \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      return fail_graph(fail(FFM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_))); \
  } while (0)
  cudaGraphConditionalHandle hout, hdir, hls, hacc, hloop;
  FFM_GC(cudaGraphConditionalHandleCreate(&hout, top, 1, cudaGraphCondAssignDefault));
  cudaStream_t c0 = L->cap[0], c1 = L->cap[1], c2 = L->cap[2], c3 = L->cap[3], c4 = L->cap[4];
  cudaGraph_t tmp = nullptr;
  // top: launch_begin -> WHILE(hout) { iteration }
  FFM_GC(cudaStreamBeginCaptureToGraph(c0, top, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  FFM_GC(launch_min_launch_begin(S, c0));
  cudaGraph_t body = nullptr;
  FFM_G(add_conditional(c0, hout, cudaGraphCondTypeWhile, &body));
  FFM_GC(cudaGraphConditionalHandleCreate(&hdir, body, 0, 0));
  FFM_GC(cudaGraphConditionalHandleCreate(&hls, body, 0, 0));
  FFM_GC(cudaGraphConditionalHandleCreate(&hacc, body, 0, 0));
  {  // iteration
    FFM_GC(cudaStreamBeginCaptureToGraph(c1, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    FFM_GC(launch_min_it_begin(S, hdir, hls, hacc, c1));
    cudaGraph_t bdir = nullptr, bls = nullptr, bacc = nullptr, bloop = nullptr;
    FFM_G(add_conditional(c1, hdir, cudaGraphCondTypeIf, &bdir));
    FFM_GC(cudaStreamBeginCaptureToGraph(c2, bdir, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    if (L->cfg.method == kMethodFgm)
      FFM_G(cap_fgm_head(L, c2, c3, bdir, hls));
    else if (L->cfg.method == kMethodFixed)
      FFM_G(cap_fixed(L, c2, c3, bdir));
    else if (L->cfg.method == kMethodOfgm)
      FFM_G(cap_ofgm(L, c2, c3, c4, bdir));
    else if (L->cfg.method == kMethodWiggle)
      FFM_G(cap_wiggle(L, c2, c3, bdir));
    else
      FFM_G(cap_direction(L, c2, hls));
    FFM_GC(cudaStreamEndCapture(c2, &tmp));
    FFM_G(add_conditional(c1, hls, cudaGraphCondTypeIf, &bls));
    {  // line search
      FFM_GC(cudaGraphConditionalHandleCreate(&hloop, bls, 0, 0));
      FFM_GC(cudaStreamBeginCaptureToGraph(c2, bls, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      const bool dir_fused = L->cfg.method == kMethodLbfgs && lbfgs_dir_small_applies(L->n, L->cfg.m);
      if (dir_fused) {
        // r and the slope came with the direction (lbfgs_dir_small_kernel)
      } else {
        if (L->cfg.method == kMethodSd || L->cfg.method == kMethodFgm)  // r = (1 / |g|) (-g)
          FFM_GC(launch_axpby(L->n, &S->inv_dn, 0.0, -1.0, L->g, nullptr, 0.0, nullptr, L->r, c2));
        else
          FFM_GC(launch_axpby(L->n, &S->inv_dn, 0.0, 1.0, L->d, nullptr, 0.0, nullptr, L->r, c2));
        const double* gs[1] = {L->g};
        const double* rs[1] = {L->r};
        FFM_GC(launch_dots(L->n, 1, gs, rs, L->scratch, &S->slope, c2));
      }
      FFM_GC(launch_min_ls_init(S, hloop, c2));
      FFM_G(add_conditional(c2, hloop, cudaGraphCondTypeWhile, &bloop));
      FFM_GC(cudaStreamBeginCaptureToGraph(c3, bloop, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
      FFM_G(cap_trial(L, c3, hloop));
      FFM_GC(cudaStreamEndCapture(c3, &tmp));
      FFM_GC(launch_min_ls_post(S, L->rec, hacc, c2));
      if (L->cfg.method == kMethodCg) FFM_GC(launch_select_neg(S, L->n, L->g, L->d, c2));
      FFM_GC(cudaStreamEndCapture(c2, &tmp));
    }
    FFM_G(add_conditional(c1, hacc, cudaGraphCondTypeIf, &bacc));
    FFM_GC(cudaStreamBeginCaptureToGraph(c2, bacc, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    FFM_G(cap_accept(L, c2));
    FFM_GC(cudaStreamEndCapture(c2, &tmp));
    if (L->cfg.method == kMethodFgm)
      FFM_GC(launch_fgm_shift(S, L->n, L->x, L->st, L->xn, L->xt, L->best, c1));
    FFM_GC(launch_min_it_end(S, hout, c1));
    FFM_GC(cudaStreamEndCapture(c1, &tmp));
  }
  FFM_GC(cudaStreamEndCapture(c0, &tmp));
#undef FFM_G
#undef FFM_GC
  g_launch_count.fetch_sub(g_launch_count.load() - before);
  cudaError_t e = cudaGraphInstantiate(&L->exec, top, 0);
  cudaGraphDestroy(top);
  if (e != cudaSuccess) {
    L->exec = nullptr;
    return fail(FFM_ECUDA, std::string("lbfgs graph instantiate: ") + cudaGetErrorString(e));
  }
  L->gen = s->gen;
  return FFM_OK;
}

void lbfgs_free(ffm_lbfgs* L) {
  if (L->exec) cudaGraphExecDestroy(L->exec);
  for (void* p : {(void*)L->S, (void*)L->rec, (void*)L->buf, (void*)L->scratch, (void*)L->en,
                  (void*)L->stw, (void*)L->sched, L->wbuf, (void*)L->wig_atoms})
    if (p) cudaFree(p);
  for (cudaStream_t c : L->cap)
    if (c) cudaStreamDestroy(c);
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

int check_config(const ffm_lbfgs_config* cfg) {
  if (cfg->m < 1 || cfg->m > kMaxLbfgsPairs) return fail(FFM_EINVAL, "memory depth m out of range");
  if (cfg->ls_kind != 0 && cfg->ls_kind != 1) return fail(FFM_EINVAL, "bad line-search kind");
  if (cfg->ls_kind == 1 && (cfg->K < 2 || cfg->K > kLsMaxPoints - 2))
    return fail(FFM_EINVAL, "ls_par K out of range");
  if (cfg->chunk < 1) return fail(FFM_EINVAL, "chunk must be >= 1");
  if (cfg->method < kMethodLbfgs || cfg->method > kMethodWiggle) return fail(FFM_EINVAL, "bad method");
  if (cfg->method == kMethodWiggle && (!(cfg->wiggle_h > 0.0) || cfg->wiggle_epoch < 1 ||
                                       cfg->wiggle_cutoff < 0.0))
    return fail(FFM_EINVAL, "bad wiggle configuration");
  if (cfg->method == kMethodFixed &&
      (cfg->momentum_kind < 0 || cfg->momentum_kind > 3 || !(cfg->fixed_step > 0.0)))
    return fail(FFM_EINVAL, "bad fixed-step configuration");
  if (cfg->method == kMethodCg && (cfg->cg_kind < 0 || cfg->cg_kind > 6 || cfg->restart_period < 1))
    return fail(FFM_EINVAL, "bad CG variant");
  return FFM_OK;
}

// fields that shape the captured graph (buffer sizes, which kernels are
// captured, host constants baked into launches); the rest is read from the
// device state at run time and may change between runs (ffm_lbfgs_configure)
bool same_structure(const MinConfig& c, const ffm_lbfgs_config* cfg) {
  return c.m == cfg->m && c.chunk == cfg->chunk && c.method == cfg->method &&
         c.momentum_kind == cfg->momentum_kind && c.fixed_step == cfg->fixed_step &&
         c.ls_needs_grad == (cfg->ls_kind == 1 && cfg->use_gradient_start) &&
         (c.wig_cutoff > 0.0) == (cfg->wiggle_cutoff > 0.0);
}

void set_config(MinConfig& c, const ffm_lbfgs_config* cfg) {
  c.m = cfg->m;
  c.ls_kind = cfg->ls_kind;
  c.K = cfg->K;
  c.use_gs = cfg->use_gradient_start;
  c.stop_on_ls_failure = cfg->stop_on_linesearch_failure;
  c.chunk = cfg->chunk;
  c.max_iter = cfg->max_iterations;
  c.max_calls = cfg->max_oracle_calls;
  c.thr = cfg->threshold;
  c.h0 = cfg->h0;
  c.eps_h = cfg->eps_h;
  c.k_plus = cfg->k_plus;
  c.k_minus = cfg->k_minus;
  c.trust = cfg->trust;
  c.method = cfg->method;
  c.cg_kind = cfg->cg_kind;
  c.restart_period = cfg->restart_period;
  c.momentum_kind = cfg->momentum_kind;
  c.fixed_step = cfg->fixed_step;
  c.momentum = cfg->momentum;
  c.ls_needs_grad = cfg->ls_kind == 1 && cfg->use_gradient_start;
  c.wig_h = cfg->wiggle_h;
  c.wig_cutoff = cfg->wiggle_cutoff;
  c.wig_epoch = cfg->wiggle_epoch;
}

}  // namespace

extern "C" {

int ffm_lbfgs_create(ffm_system_t* s, int precision, const ffm_lbfgs_config* cfg,
                     ffm_lbfgs_t** out) {
  if (!s || !cfg || !out) return fail(FFM_EINVAL, "NULL argument");
  *out = nullptr;
  if (precision != FFM_F64 && precision != FFM_F32) return fail(FFM_EINVAL, "bad precision");
  if (s->nranks != 1 && !s->comm)
    return fail(FFM_EINVAL, "graph-resident drivers need an unsharded system or a communicator "
                            "(ffm_system_set_comm)");
  FFM_TRYR(check_config(cfg));
  DeviceGuard guard(s->device);
  auto* L = new ffm_lbfgs();
  L->sys = s;
  L->device = s->device;
  L->prec = precision;
  MinConfig& c = L->cfg;
  set_config(c, cfg);
  c.horizon = 0;
  c.sched = nullptr;
  c.wig_atoms = nullptr;
  if (c.method == kMethodWiggle) {
    if (cudaMalloc(&L->wbuf, kWigBufBytes) != cudaSuccess ||
        cudaMalloc(&L->wig_atoms, (size_t)c.chunk * sizeof(int)) != cudaSuccess ||
        cudaMemset(L->wig_atoms, 0, (size_t)c.chunk * sizeof(int)) != cudaSuccess) {
      lbfgs_free(L);
      delete L;
      return fail(FFM_ENOMEM, "cudaMalloc failed for the wiggle run");
    }
    c.wig_atoms = L->wig_atoms;
  }
  L->n = 3 * (int64_t)std::max(1, s->plan.n);
  const int64_t n = L->n;
  const size_t nbuf = (size_t)n * (12 + 2 * (c.m + 1));
  bool ok = cudaMalloc(&L->S, sizeof(MinState)) == cudaSuccess &&
            cudaMalloc(&L->rec, (size_t)(c.chunk + 1) * kMinRecWidth * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&L->buf, nbuf * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&L->scratch, two_loop_scratch_doubles() * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&L->en, FFM_NTERMS * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&L->stw, FFM_STATUS_WORDS * sizeof(int64_t)) == cudaSuccess;
  if (!ok) {
    lbfgs_free(L);
    delete L;
    return fail(FFM_ENOMEM, "cudaMalloc failed for the L-BFGS run");
  }
  double* p = L->buf;
  for (double** v : {&L->x, &L->g, &L->xn, &L->gnew, &L->xt, &L->d, &L->r, &L->st, &L->yt,
                     &L->best, &L->gsum, &L->anchor}) {
    *v = p;
    p += n;
  }
  L->ring_s = p;
  L->ring_y = p + (size_t)n * (c.m + 1);
  cudaMemset(L->buf, 0, nbuf * sizeof(double));
  cudaDeviceSynchronize();  // before any use on the caller's (maybe non-blocking) stream
  for (cudaStream_t& cs : L->cap)
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
      lbfgs_free(L);
      delete L;
      return fail(FFM_ECUDA, "stream creation failed");
    }
  L->rec_h.resize((size_t)(c.chunk + 1) * kMinRecWidth);
  *out = L;
  return FFM_OK;
}

int ffm_lbfgs_configure(ffm_lbfgs_t* L, const ffm_lbfgs_config* cfg) {
  if (!L || !cfg) return fail(FFM_EINVAL, "NULL argument");
  FFM_TRYR(check_config(cfg));
  if (!same_structure(L->cfg, cfg))
    return fail(FFM_EINVAL, "configuration changes the graph structure: create a new run");
  const long long horizon = L->cfg.horizon;
  const double* sched = L->cfg.sched;
  const int* atoms = L->cfg.wig_atoms;
  set_config(L->cfg, cfg);
  L->cfg.horizon = horizon;
  L->cfg.sched = sched;
  L->cfg.wig_atoms = atoms;
  return FFM_OK;
}

int ffm_lbfgs_start(ffm_lbfgs_t* L, const double* x_d, const double* g_d, double f, double gnorm,
                    double warm_h, void* stream) {
  if (!L || !x_d || !g_d) return fail(FFM_EINVAL, "NULL argument");
  DeviceGuard guard(L->sys->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t nb = (size_t)3 * L->sys->plan.n * sizeof(double);
  FFM_CUDA(cudaMemcpyAsync(L->x, x_d, nb, cudaMemcpyDeviceToDevice, st));
  FFM_CUDA(cudaMemcpyAsync(L->g, g_d, nb, cudaMemcpyDeviceToDevice, st));
  MinState h;
  std::memset(&h, 0, sizeof(h));
  h.c = L->cfg;
  h.f = f;
  h.gn = gnorm;
  h.warm = warm_h;
  h.count = 0;
  h.nfree = L->cfg.m + 1;
  for (int q = 0; q <= L->cfg.m; ++q) h.freel[q] = q;
  h.store_slot = -1;
  h.best_f = f;  // OptimizationRun.update_best(x0, f0)
  h.f_init = f;
  h.theta_prev = h.theta = 1.0;
  FFM_CUDA(cudaMemcpyAsync(L->best, x_d, nb, cudaMemcpyDeviceToDevice, st));
  if (L->cfg.method == kMethodOfgm) {
    if (!L->sched) return fail(FFM_EINVAL, "OFGM needs ffm_lbfgs_set_schedule before start");
    FFM_CUDA(cudaMemcpyAsync(L->anchor, x_d, nb, cudaMemcpyDeviceToDevice, st));  // anchor = x0
    FFM_CUDA(cudaMemsetAsync(L->gsum, 0, nb, st));                                // zeros_like
  }
  if (L->cfg.method == kMethodFgm || L->cfg.method == kMethodFixed)  // x_prev = copy(x0)
    FFM_CUDA(cudaMemcpyAsync(L->st, x_d, nb, cudaMemcpyDeviceToDevice, st));
  if (L->cfg.method == kMethodCg)  // p = lincomb(-1, g) (ffmin/optimizers/cg.py:101)
    FFM_CUDA(launch_axpby(L->n, nullptr, -1.0, 1.0, L->g, nullptr,
                          0.0, nullptr, L->d, st));
  FFM_CUDA(cudaMemcpyAsync(L->S, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  FFM_CUDA(cudaStreamSynchronize(st));  // h lives on this stack frame
  return FFM_OK;
}

int ffm_lbfgs_run(ffm_lbfgs_t* L, void* stream) {
  if (!L) return fail(FFM_EINVAL, "NULL argument");
  DeviceGuard guard(L->sys->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!L->exec || L->gen != L->sys->gen) {
    // (re)build after the system's workspace moved; x/g already hold the
    // iterate, the warm-up evaluations only touch scratch outputs
    FFM_CUDA(cudaStreamSynchronize(st));
    FFM_TRYR(lbfgs_build(L));
  }
  FFM_CUDA(cudaGraphLaunch(L->exec, st));
  count_launch();
  return FFM_OK;
}

int ffm_lbfgs_poll(ffm_lbfgs_t* L, int64_t* ints, double* dbls, double* rec_h, int64_t cap,
                   int64_t* nrec, int64_t* err_status_h) {
  if (!L || !ints || !dbls || !nrec) return fail(FFM_EINVAL, "NULL argument");
  DeviceGuard guard(L->sys->device);
  MinState h;
  FFM_CUDA(cudaDeviceSynchronize());
  FFM_CUDA(cudaMemcpy(&h, L->S, sizeof(h), cudaMemcpyDeviceToHost));
  ints[0] = h.k;
  ints[1] = h.status;
  ints[2] = h.done;
  ints[3] = h.err;
  ints[4] = h.err_grad;
  ints[5] = h.vcalls;
  ints[6] = h.gcalls;
  ints[7] = h.count;
  dbls[0] = h.f;
  dbls[1] = h.gn;
  dbls[2] = h.warm;
  dbls[3] = h.best_f;
  const int64_t k = std::min<int64_t>(h.nrec, cap);
  if (k > 0 && rec_h)
    FFM_CUDA(cudaMemcpy(rec_h, L->rec, (size_t)k * kMinRecWidth * sizeof(double),
                        cudaMemcpyDeviceToHost));
  *nrec = h.nrec;
  if (err_status_h)
    for (int q = 0; q < 8; ++q) err_status_h[q] = h.err_st[q];
  return FFM_OK;
}

int ffm_lbfgs_result(ffm_lbfgs_t* L, double* x_d, double* g_d, void* stream) {
  if (!L) return fail(FFM_EINVAL, "NULL argument");
  DeviceGuard guard(L->sys->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t nb = (size_t)3 * L->sys->plan.n * sizeof(double);
  if (x_d) FFM_CUDA(cudaMemcpyAsync(x_d, L->x, nb, cudaMemcpyDeviceToDevice, st));
  if (g_d) FFM_CUDA(cudaMemcpyAsync(g_d, L->g, nb, cudaMemcpyDeviceToDevice, st));
  return FFM_OK;
}

int ffm_lbfgs_set_schedule(ffm_lbfgs_t* L, const double* t_h, int64_t len) {
  if (!L || !t_h || len < 2) return fail(FFM_EINVAL, "bad OFGM schedule");
  DeviceGuard guard(L->device);
  if (L->sched) cudaFree(L->sched);
  L->sched = nullptr;
  FFM_CUDA(cudaMalloc(&L->sched, (size_t)len * sizeof(double)));
  FFM_CUDA(cudaMemcpy(L->sched, t_h, (size_t)len * sizeof(double), cudaMemcpyHostToDevice));
  L->cfg.horizon = len - 1;
  L->cfg.sched = L->sched;
  return FFM_OK;
}

int ffm_lbfgs_set_atoms(ffm_lbfgs_t* L, const int32_t* atoms_h, int64_t count) {
  if (!L || !atoms_h) return fail(FFM_EINVAL, "NULL argument");
  if (L->cfg.method != kMethodWiggle) return fail(FFM_EINVAL, "not a wiggle run");
  if (count < L->cfg.chunk) return fail(FFM_EINVAL, "need one atom per iteration of a launch");
  for (int64_t k = 0; k < L->cfg.chunk; ++k)
    if (atoms_h[k] < 0 || atoms_h[k] >= L->sys->plan.n) return fail(FFM_EINVAL, "atom out of range");
  DeviceGuard guard(L->device);
  FFM_CUDA(cudaMemcpy(L->wig_atoms, atoms_h, (size_t)L->cfg.chunk * sizeof(int),
                      cudaMemcpyHostToDevice));
  return FFM_OK;
}

int ffm_lbfgs_best(ffm_lbfgs_t* L, double* x_d, void* stream) {
  if (!L || !x_d) return fail(FFM_EINVAL, "NULL argument");
  DeviceGuard guard(L->sys->device);
  const size_t nb = (size_t)3 * L->sys->plan.n * sizeof(double);
  FFM_CUDA(cudaMemcpyAsync(x_d, L->best, nb, cudaMemcpyDeviceToDevice,
                           static_cast<cudaStream_t>(stream)));
  return FFM_OK;
}

int ffm_lbfgs_destroy(ffm_lbfgs_t* L) {
  if (!L) return FFM_OK;
  // (its system may already be gone: garbage collection of a reference
  // cycle finalises in any order; L->sys is not dereferenced here)
  DeviceGuard guard(L->device);
  cudaDeviceSynchronize();
  lbfgs_free(L);
  delete L;
  return FFM_OK;
}

}  // extern "C"
