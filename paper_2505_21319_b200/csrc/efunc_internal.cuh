// efunc_internal.cuh — shared device/host definitions of libefunc (not part of the ABI).
//
// Data layout in HBM:
//   theta / m / v / grad : float [R^3][13]  (ABI layout, node-major)
//   gpad                 : float [R^3][16]  padded gradient accumulator (red.v4 targets)
//   key record (32 B)    : float4 a = {x, y, z, bl}, float4 b = {c, gx, gy, gz},
//                          bl = beta * log2(e)  (exponents are evaluated in base 2)
//                          key id i < R^3: grid bank node i; i >= R^3: offset bank node i-R^3
//   key_raw              : [2R^3] records in key-id order (grid bank = lattice order)
//   key_sorted           : [2R^3] records sorted by lattice cell (x fastest), stable by key id
//   cell_start           : [(R-1)^3 + 1] exclusive prefix of keys per cell
//   brick lists          : per brick (B^3 lattice cells, Morton-coded) the sorted-key positions
//                          of every key that can reach a query inside the brick (pool + off/n)
//   queries (per forward): qs float4 {x,y,z,o} sorted by brick (Morton), stable by index;
//                          perm[sorted] = user index; rec float4 {-lambda_j log2e, dL/dO_j, O_j, 0}
//   work item            : <= QW consecutive sorted queries of one brick (one warp)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/efunc.h"

#define EF_NCH 13
#define EF_LOG2E 1.4426950408889634f
#define EF_LN2 0.6931471805599453f

namespace ef {

constexpr int QW = 32;              // max queries per work item (one warp)
#ifndef ITEM_Q
#define ITEM_Q 32
#endif
constexpr int IQ = ITEM_Q;          // queries per work item the binning produces (<= QW)
constexpr int NTHREADS = 32;        // one warp per CTA: items retire independently
constexpr int NWARP = NTHREADS / 32;
constexpr int BL_CAP = 16384;       // max list length per brick (longer: enumerate fallback)
constexpr uint32_t BL_OVERFLOW = 0xffffffffu;
constexpr int POOL_PER_KEY = 640;   // brick-list pool capacity per key
// per-warp id scratch of the persistent list builders (k_fit, k_brick_lists): SCRATCH_WARPS slots
// of BL_CAP ids, padded so the slots do not alias in L1
constexpr int SCRATCH_WARPS = 148 * 16;
constexpr int ENUM_CAP = 32768;     // k_fit: candidate ids per enumeration chunk (overflowed bricks)
// a slot also holds two k_brick_lists warps' staging (BL_CAP ids each), so the list build runs
// 2 x SCRATCH_WARPS warps
constexpr size_t SCRATCH_HALF = BL_CAP + 32;
constexpr size_t SCRATCH_STRIDE = (2 * SCRATCH_HALF > (size_t)ENUM_CAP + 32 ? 2 * SCRATCH_HALF : (size_t)ENUM_CAP + 32);

constexpr int WL_PER_QUERY = 64;    // forward->backward candidate pool capacity per query
#ifndef EF_SKIN_H
#define EF_SKIN_H 0.25f
#endif
#ifndef EF_SKIN_MU
#define EF_SKIN_MU 0.05f
#endif
constexpr float SKIN_H = EF_SKIN_H;    // Verlet skin of the brick lists, in lattice spacings
constexpr float SKIN_MU = EF_SKIN_MU;  // allowed relative drift of beta between list builds

struct KeysView {
  const float4* ks;        // sorted records, 2 float4 per key (a at 2k, b at 2k+1)
  const int* kid;          // sorted -> key id
  const uint32_t* cell_start;
  const float4* grid_raw;  // raw records of the grid bank in lattice order (2 float4 per node)
  const float* bl_min;     // device scalar: min bl over all keys
  int R, NC;               // NC = R-1 cells per axis
  float inv_h;             // 1/h, h = 2/(R-1)
  float h;
  int n_nodes;
  // brick lists
  const uint32_t* bl_pool;
  const uint32_t* bl_off;
  const uint32_t* bl_n;    // BL_OVERFLOW: enumerate instead
};

struct DevScalars {
  float bl_min;            // as float; written via atomicMin on its bits (bl > 0)
  uint32_t nonfinite;
  uint32_t pool_top;       // brick-list pool allocation cursor
  uint32_t lists_invalid;  // 1: the brick lists must be rebuilt (skin exceeded / new theta)
  uint32_t list_builds;    // number of brick-list builds (diagnostics)
  uint32_t ovf_count;      // bricks overflowed in the running build
  uint32_t pool_used;      // entries of the last completed build
  uint32_t ovf_last;       // overflowed bricks of the last completed build
  float umax;              // deterministic backward: max_j (|dL/dO_j| + |dL/dG_j|_1) of the call
  uint32_t fix_overflow;   // deterministic backward: a partial left the fixed-point range
  uint32_t adam_done;      // k_adamw blocks finished (the last one advances adam_t and resets this)
  uint32_t keys_resort;    // an offset key changed lattice cell: re-sort the keys (else only regather)
  unsigned long long adam_t;  // AdamW step counter (device-side so CUDA graphs replay it correctly)
  // ---- reset by every forward (one memset from overflow_items to the end)
  uint32_t overflow_items;
  uint32_t wl_top;         // per-item candidate-list pool cursor
  uint32_t slow_n;         // items left to the exact-shift / no-list split kernels
  uint32_t fwd_next;       // persistent fetch cursors
  uint32_t bwd_next;
  uint32_t fit_next;
  unsigned long long cand_pairs;
  unsigned long long kept_pairs;
  unsigned long long kept_pairs_offset;
};



struct FwdArgs {
  KeysView kv;
  const float4* qs;       // sorted queries {x,y,z,o}
  const int* perm;        // sorted -> user index
  int64_t J;
  const int4* items;      // work items {first sorted query, count, brick (-1: outside), 0}
  const uint32_t* n_items;  // device count (grid is launched with an upper bound)
  float T_l;              // cutoff in log2 units (inf = dense)
  // loss
  int loss_kind;
  float inv_J;            // 1/J_global
  float eik_lambda;
  // outputs
  float* O;               // user order (may be null)
  float* G;               // user order [J*3] (may be null)
  float4* rec;            // sorted {-lam_l, r, O, 0}
  float4* gs;             // sorted G (if WANT_G)
  float4* us;             // sorted ubar (if WANT_G)
  float4* hs;             // sorted fused Eikonal upstream h (if loss eikonal)
  float* loss_part;       // per item partial loss
  float* qmh;             // sorted shift bound mh_j (k_item_lists -> k_forward_keys)
  float* qf0;             // sorted f_j of the shift key (k_fit_eik), or null
  DevScalars* ds;
  int count_kept;
  // per-item candidate key ids handed to the backward (reserved: the brick list length)
  uint32_t* wl_pool;
  uint32_t wl_cap;
  uint32_t* wl_off;
  uint32_t* wl_n;         // BL_OVERFLOW: the backward streams the brick list itself
  uint32_t* slow_items;   // items whose shift bound overflowed (ds->slow_n of them)
};

struct BwdArgs {
  KeysView kv;
  const float4* qs;
  const int* perm;
  int64_t J;
  const int4* items;
  const uint32_t* n_items;
  float T_l;              // cutoff in log2 units (inf = dense)
  const float4* rec;
  const float4* gs;
  const float4* us;
  const float4* hs;       // fused h (sorted) or null
  const float* dL_dO;     // user order or null (use rec.y)
  const float* dL_dG;     // user order [J*3] or null
  float* grad;            // [R^3][13] +=
  int eik;                // 1: add the dL/dG terms
  float* gpad;            // [R^3][16] padded accumulation buffer (zero on entry, zeroed by k_fold)
  const uint32_t* wl_pool;  // the forward's per-item candidate lists
  const uint32_t* wl_off;
  const uint32_t* wl_n;
  // deterministic mode: 64-bit fixed point, value = int * umax * 2^-FIX_BITS (integer adds are
  // associative, so the sum is independent of the order the atomics land in)
  unsigned long long* gfix;  // [R^3][16]
  const float* umax;
  uint32_t* fix_overflow;
  uint32_t* next;            // persistent fetch cursor (zeroed before the launch)
  const uint32_t* list;      // null: every item; else the items list[0 .. *list_n)
  const uint32_t* list_n;
};

// Fused fit item kernel (k_fit.cu): value-only forward + MSE upstream + backward per work item.
struct FitArgs {
  FwdArgs f;
  float* gpad;            // [R^3][16] padded gradient accumulator
  uint32_t* scratch;      // per-warp candidate-id scratch: SCRATCH_WARPS slots of SCRATCH_STRIDE ids
  const uint32_t* iota;   // dense mode (cutoff_T = inf): the enabled key ids, every key a candidate; else null
  uint32_t iota_n;        // their count (2R^3 with both banks)
  int pre;                // 1: k_fit_lists built the items' candidate ids (f.wl_*) and box centres
  float4* item_o;         // [items] box centre of each item (k_fit_lists -> k_fit)
  const uint32_t* n_heavy;  // items of cost class 0 (the first n_heavy items)
  // deterministic mode: 64-bit fixed-point accumulation (BwdArgs::gfix) with the unit umax * 2^-FIX_BITS,
  // umax an a-priori bound of max_j |r_j| (k_det_bound); null gfix: float reds into gpad
  unsigned long long* gfix;
  const float* umax;
  uint32_t* fix_overflow;
};

constexpr int FIX_BITS = 36;  // resolution umax * 2^-36; range |partial| < umax * 2^26

struct BrickGeom {
  int B;          // lattice cells per brick edge
  int nb;         // bricks per axis
  int bits;       // Morton bits per axis (2^bits >= nb)
  uint32_t n_codes;  // 2^(3 bits)
  int sdiv;       // query sub-bins per lattice cell edge (2: half-cells, 4: quarter-cells)
  int sub_bits;   // query sub-bins per brick edge = 2^sub_bits = sdiv B
  uint32_t qsub;  // query sub-bins per brick = (sdiv B)^3, Morton ordered inside the brick
};

// Parameter layout of a Table 3 variant (k_var.cu; include/efunc.h efunc_channels): channel
// offsets of the grid bank's s, the offset bank's s and Delta (-1: the bank is absent), the
// polynomial degree, channels per node.
struct VarLayout {
  int nch;
  int grid;   // [s, c, g(3) if deg >= 1, H(6) if deg >= 2] or -1
  int off;    // same for the offset bank, or -1
  int delta;  // offset bank's Delta(3), or -1
  int deg;
};

// ---------------------------------------------------------------- launchers (host)
int launch_prep_keys(const float* theta, int R, int banks, float4* key_raw, uint32_t* key_cell, uint32_t* key_rank,
                     uint32_t* cell_count,
                     const float4* key_ref, float skin2, float mu, DevScalars* ds, cudaStream_t s);
int launch_list_snapshot(const float4* key_raw, float4* key_ref, int n_keys, DevScalars* ds,
                         cudaStream_t s);
int launch_scan_u32(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* block_tmp,
                    cudaStream_t s, const uint32_t* gate = nullptr);
size_t radix_hist_elems(uint32_t n);
int launch_stable_sort(const uint32_t* bin, uint32_t n, int bits, uint32_t* rk, uint32_t* hist, uint32_t* scan_tmp,
                       uint32_t* tmp_idx, uint32_t* out_idx, cudaStream_t s, const uint32_t* gate = nullptr);
int launch_gather_keys(const uint32_t* order, const float4* key_raw, float4* key_sorted,
                       int* kid, uint32_t n, cudaStream_t s);
int launch_brick_lists(const KeysView& kv, const BrickGeom& bg, float T_l, uint32_t* pool,
                       uint32_t pool_cap, uint32_t* off, uint32_t* n, DevScalars* ds, uint32_t* scratch,
                       cudaStream_t s);
int launch_query_bins(const float* q, const float* o, int64_t J, const BrickGeom& bg, int NC,
                      float inv_h, uint32_t* bins, uint32_t* count, uint32_t* rank, DevScalars* ds,
                      cudaStream_t s);
int launch_scatter_ranked(const uint32_t* bin, const uint32_t* rank, uint32_t n, const uint32_t* bin_start,
                          uint32_t* out_idx, cudaStream_t s, const uint32_t* gate = nullptr);
int launch_gather_queries(const uint32_t* order, const float* q, const float* o, int64_t J,
                          float4* qs, int* perm, cudaStream_t s);
int launch_gather_queries_mh(const KeysView& kv, const uint32_t* order, const float* q, const float* o, int64_t J,
                             float4* qs, int* perm, float* qmh, float* qf0, cudaStream_t s);
int launch_scatter_only(const uint32_t* bin, uint32_t n, const uint32_t* bin_start, uint32_t* fill,
                        uint32_t* out_idx, cudaStream_t s, const uint32_t* gate = nullptr);
int launch_items_count(const uint32_t* bin_start, uint32_t nb, uint32_t qsub, const uint32_t* bl_n,
                       const DevScalars* ds, uint32_t* cnt, cudaStream_t s);
int launch_items_write(const uint32_t* bin_start, uint32_t nb, uint32_t qsub, const uint32_t* bl_n,
                       const DevScalars* ds, const uint32_t* off, int4* items, cudaStream_t s);
int launch_items_fused(const uint32_t* bin_start, uint32_t nb, uint32_t qsub, uint32_t* item_off, int4* items,
                       cudaStream_t s);
// work items in cost classes (k_items_count): item_off[ITEMS_N_AT(nb)] = the number of items
#ifndef EF_ITEM_CLASSES
#define EF_ITEM_CLASSES 3
#endif
#define ITEMS_N_AT(nb) (EF_ITEM_CLASSES * ((nb) + 1))
int launch_forward(const FwdArgs& a, int want_g, int64_t n_items, cudaStream_t s);
int launch_forward_slow(const FwdArgs& a, int want_g, cudaStream_t s);
int launch_backward(const BwdArgs& a, int64_t n_items, cudaStream_t s);
int launch_fit(const FitArgs& a, int64_t n_items, cudaStream_t s);
int launch_fit_tc(const FitArgs& a, int64_t n_items, cudaStream_t s);  // tensor-core pair loops
int launch_fit_lists(const FitArgs& a, int64_t n_items, cudaStream_t s);
int launch_det_bound(const float* theta, int n_nodes, const float4* qs, int64_t J, float inv_J, float* umax,
                     cudaStream_t s);
int launch_backward_list_det(const BwdArgs& a, cudaStream_t s);
// dense mode (cutoff_T = inf, MSE): key-sliced forward, combine, key-stationary backward (k_fit.cu)
int64_t dense_zm_elems(int64_t n_items, uint32_t iota_n);
void dense_split_dims(int64_t n_items, uint32_t iota_n, int& S, uint32_t& ks, int& G);
int64_t dense_eik_part_elems(int64_t n_items, uint32_t iota_n);
int launch_dense_fit_eik(const FitArgs& a, int64_t n_items, float* part, float4* dq, cudaStream_t s);
int launch_dense_fit(const FitArgs& a, int64_t n_items, float2* zm, float4* dq, cudaStream_t s, int* fwd_launches);
int launch_fit_eik(const FitArgs& a, int64_t n_items, cudaStream_t s);
int launch_sum_partials(const float* part, const uint32_t* n, int mult, float* out, cudaStream_t s);
int launch_fold(float* gpad, float* grad, int n_nodes, cudaStream_t s);
// the fold fused with the ranks' gradient reduction (efunc_set_grad_peers)
int launch_fold_peers(float* gpad, int n_nodes, float* const* peers, int n_peers, float* mc, cudaStream_t s);
int launch_backward_det(const BwdArgs& a, int64_t n_items, cudaStream_t s);
int launch_fold_fix(unsigned long long* gfix, const float* umax, float* grad, int n_nodes, cudaStream_t s);
struct AdamWConst {  // the efunc_adamw hyper-parameters (doubles, like torch's python floats)
  double lr, beta1, beta2, eps, weight_decay;
  uint32_t decay_mask;
  uint32_t frozen_mask;  // channels AdamW leaves untouched (degree 0: the g channels, held at 0)
  int nch;               // channels per node of the parameter array (13, or the variant's)
};
int launch_adamw(float* theta, const float* grad, float* m, float* v, int64_t n, const AdamWConst& hc,
                 DevScalars* ds, cudaStream_t s);
// S6 + S0 in one pass (13-channel layout): AdamW of each node's channels, then its two key records
// from the updated theta (k_bin.cu k_adamw_keys; the same arithmetic as k_adamw + k_prep_keys)
int launch_adamw_keys(float* theta, const float* grad, float* m, float* v, const AdamWConst& hc, int R, int banks,
                      float4* key_raw, uint32_t* key_cell, uint32_t* key_rank, uint32_t* cell_count,
                      const float4* key_ref, float skin2, float mu, DevScalars* ds, cudaStream_t s);

// AdamW scalars for step t (torch's single-tensor AdamW; derived in double, rounded to fp32 once)
struct AdamWScal {
  float decay, omb1, b2, omb2, eps, step_size, sqrt_bc2;
};
__device__ __forceinline__ AdamWScal adamw_scal(const AdamWConst& hc, const unsigned long long t) {
  const double bc1 = 1.0 - pow(hc.beta1, (double)t);
  const double bc2 = 1.0 - pow(hc.beta2, (double)t);
  AdamWScal c;
  c.decay = (float)(1.0 - hc.lr * hc.weight_decay);
  c.omb1 = (float)(1.0 - hc.beta1);
  c.b2 = (float)hc.beta2;
  c.omb2 = (float)(1.0 - hc.beta2);
  c.eps = (float)hc.eps;
  c.step_size = (float)(hc.lr / bc1);
  c.sqrt_bc2 = (float)sqrt(bc2);
  return c;
}
// one element: p *= decay (masked); m += (1-b1)(g-m); v = v b2 + (1-b2) g^2;
// p += -step_size m / (sqrt(v)/sqrt(bc2) + eps)
__device__ __forceinline__ float adamw_elem(float p, const float g, float& mi, float& vi, const bool dec,
                                            const AdamWScal& c) {
  if (dec) p *= c.decay;
  mi = fmaf(c.omb1, g - mi, mi);
  vi = fmaf(c.omb2, g * g, vi * c.b2);
  const float denom = __fdiv_rn(__fsqrt_rn(vi), c.sqrt_bc2) + c.eps;
  return fmaf(-c.step_size, __fdiv_rn(mi, denom), p);
}
int launch_mean_shift(float* theta, int R, const float* surf, int64_t N, float bw,
                      cudaStream_t s);
int launch_fill_zero_f32(float* p, int64_t n, cudaStream_t s);
struct FillSeg {
  uint32_t* p;
  uint32_t n;  // u32 words
  uint32_t v;
};
struct FillSegs {
  static constexpr int MAX = 4;
  FillSeg s[MAX];
  int k = 0;
  void add(void* p, size_t bytes, uint32_t v) {  // callers add at most MAX segments of whole u32 words
    if (k < MAX) s[k++] = FillSeg{static_cast<uint32_t*>(p), (uint32_t)(bytes / 4), v};
  }
};
int launch_fill_segs(const FillSegs& f, cudaStream_t s);
int launch_zero_channels(float* theta, int n_nodes, uint32_t mask, cudaStream_t s);
// NEXT-4 (k_var.cu): variant layouts and the degree-2 forward / backward
int launch_var_unpack(const float* tv, int n, const VarLayout& L, float* t13, float* tH, cudaStream_t s);
int launch_var_pack_grad(const float* g13, const float* gH, int n, const VarLayout& L, float* gv, cudaStream_t s);
int launch_var_delta_out(const float* t13, int n, const VarLayout& L, float* tv, cudaStream_t s);
int launch_var_keyH(const float* tH, int n, float4* keyH, cudaStream_t s);
int launch_var_forward(const FwdArgs& a, const float4* keyH, const uint32_t* iota, uint32_t iota_n, int want_g,
                       int64_t n_items, cudaStream_t s);
int launch_var_backward(const FwdArgs& a, const float4* keyH, const uint32_t* iota, uint32_t iota_n,
                        const float* dL_dO, float* g13, float* gH, int64_t n_items, cudaStream_t s);
int launch_item_lists(const FwdArgs& a, int64_t n_items, cudaStream_t s);
// NEXT-4 cosine-series stacks (k_cosine.cu)
int launch_cos_replicate(const float* q, int64_t J, int B, float* qr, cudaStream_t s);
int launch_cos_combine(const float* q, int64_t J, int B, const float* O, const float* G, const float* o, float inv_J,
                       float* S, float* GS, float* dL_dO, float* loss, cudaStream_t s);
// NEXT-3 (k_mesh.cu): lattice queries, Marching Cubes, vertex normals
cudaError_t mc_upload_table();
int launch_lattice_q(int N, const float* lo, const float* step, int k0, int nk, float* q, cudaStream_t s);
int launch_mc_count(const float* O, int N, float iso, uint8_t* mask, uint32_t* vcnt, uint32_t* tcnt, cudaStream_t s);
int launch_mc_emit(const float* O, int N, float iso, const float* lo, const float* step, const uint8_t* mask,
                   const uint32_t* voff, const uint32_t* toff, float* verts, int32_t* tris, cudaStream_t s);
int launch_normalize3(float* v, int64_t n, cudaStream_t s);

}  // namespace ef

// ---------------------------------------------------------------- the handle
struct efunc {
  efunc_config cfg;
  int R = 0, n_nodes = 0, n_keys = 0, NC = 0, n_cells = 0;
  float h = 0.f, inv_h = 0.f;
  ef::BrickGeom bg{};
  // parameters + optimizer state
  float* theta = nullptr;
  float* m = nullptr;
  float* v = nullptr;
  // Table 3 variants other than the 13-channel default (NEXT-4): parameters and AdamW moments in
  // the user's layout; theta above (+ thetaH) is derived from them before every key rebuild
  int vmode = 0;                    // 1: the user layout differs from the internal 13 channels
  int vk = 0;                       // 1: degree 2 or O^Delta only: forward/backward in k_var.cu
  int banks = 3;                    // 1 grid, 2 offset, 3 both
  int pnch = EF_NCH;                // channels per node of the user's parameter arrays
  ef::VarLayout vlay{};
  float* theta_v = nullptr;
  float* m_v = nullptr;
  float* v_v = nullptr;
  float* thetaH = nullptr;          // [R^3][12] degree-2 squares (grid, offset)
  float4* keyH = nullptr;           // [2R^3][2] per key id
  float* gint = nullptr;            // [R^3][13] internal gradient scratch (vmode)
  float* gH = nullptr;              // [R^3][12] degree-2 gradient scratch
  uint32_t iota_n = 0;
  float2* dn_zm = nullptr;          // dense mode: per (item, key slice) partial Z, M
  int64_t dn_zm_cap = 0;
  float4* dn_dq = nullptr;          // dense mode: per item packed query table for the backward
  int64_t dn_dq_cap = 0;
  // keys
  float4* key_raw = nullptr;
  float4* key_sorted = nullptr;
  int* kid = nullptr;
  uint32_t* key_cell = nullptr;
  uint32_t* cell_count = nullptr;   // n_cells + 1
  uint32_t* cell_start = nullptr;   // n_cells + 1
  uint32_t* cell_fill = nullptr;
  uint32_t* key_tmp = nullptr;
  uint32_t* key_rank = nullptr;     // each key's position in its cell (ranked scatter)
  uint32_t* key_order = nullptr;
  uint32_t* scan_tmp = nullptr;     // block sums for scans
  size_t scan_tmp_cap = 0;
  uint32_t* rk = nullptr;           // stable radix sort: 2 x rk_cap u32 key ping-pong
  uint32_t* rh = nullptr;           // its digit histograms (radix_hist_elems(rk_cap))
  size_t rk_cap = 0;
  ef::DevScalars* ds = nullptr;
  float* fit_grad = nullptr;
  float* gpad = nullptr;            // [R^3][16] padded gradient accumulator (kept zero between calls)
  float** peer_grad = nullptr;      // efunc_set_grad_peers: device array of every rank's gradient copy
  int n_peers = 0;
  float* mc_grad = nullptr;         // and its NVLS multicast address (or null)
  unsigned long long* gfix = nullptr;  // [R^3][16] fixed-point accumulator (deterministic mode)
  // brick lists
  uint32_t* bl_pool = nullptr;
  uint32_t bl_pool_cap = 0;
  uint32_t* bl_off = nullptr;
  uint32_t* bl_n = nullptr;
  float4* key_ref = nullptr;        // [2R^3] key {x,y,z,bl} at the last list build
  // queries
  int64_t J_cap = 0;
  uint32_t* q_bin = nullptr;
  uint32_t* bin_count = nullptr;    // nbins + 1
  uint32_t* bin_start = nullptr;
  uint32_t* bin_fill = nullptr;
  uint32_t* item_cnt = nullptr;
  uint32_t* item_off = nullptr;     // item_off[nbins] = item count
  uint32_t* q_tmp = nullptr;
  uint32_t* q_order = nullptr;
  float4* qs = nullptr;
  int* perm = nullptr;
  float4* rec = nullptr;
  float4* gs = nullptr;
  float4* us = nullptr;
  float4* hs = nullptr;
  float* loss_part = nullptr;
  float* qmh = nullptr;
  float* qf0 = nullptr;
  int64_t items_cap = 0;
  int4* items = nullptr;            // [items bound]
  uint32_t* wl_pool = nullptr;      // forward -> backward candidate ids
  uint32_t wl_cap = 0;
  uint32_t* wl_off = nullptr;       // [items bound]
  uint32_t* wl_n = nullptr;         // [items bound]
  uint32_t* slow_items = nullptr;   // [items bound]
  float4* item_o = nullptr;         // [items bound] item box centres (k_fit_lists -> k_fit)
  uint32_t* iota = nullptr;         // dense mode: key ids 0 .. 2R^3-1 (k_fit candidate list)
  uint32_t* scratch = nullptr;      // per-warp id scratch (k_fit, k_brick_lists): SCRATCH_WARPS x SCRATCH_STRIDE
  int64_t fwd_items_bound = 0;
  float* io_q = nullptr;  // device staging for host_io fit_step
  float* io_o = nullptr;
  float* io_loss = nullptr;
  int64_t io_cap = 0;
  // saved forward state
  int have_fwd = 0;
  int64_t fwd_J = 0;
  int fwd_has_g = 0;
  int fwd_loss_kind = 0;
  int count_kept = 0;
  int64_t launches = 0;
  // efunc_fit_step CUDA graph (cfg.fit_graph): the key of the last call, the captured executable
  struct FitKey {
    const float* q; const float* o; float* g; float* lossd;
    int64_t J, J_global;
    int kind;
    float eik;
    double lr, b1, b2, eps, wd;
    uint32_t mask;
    int count_kept;
  } fit_key[2]{};
  int fit_seen[2] = {0, 0};          // fit_key[slot] holds the last (eager) call of that slot
  cudaGraphExec_t fit_exec[2] = {nullptr, nullptr};  // slot 0: host_io 0/1; slots 0/1: host_io 2
  int64_t fit_launches[2] = {0, 0};  // kernels inside the captured graphs
  // host_io 2 (pipelined host I/O): double-buffered device staging, a copy stream, events
  float* aio_q[2] = {nullptr, nullptr};
  float* aio_o[2] = {nullptr, nullptr};
  float* aio_loss[2] = {nullptr, nullptr};
  float* aio_pin = nullptr;          // pinned host float[2]: the losses read back
  struct LossCopy { const float* src; float* dst; } aio_pay[2]{};
  int64_t aio_cap = 0;
  int64_t aio_seq = 0;
  cudaStream_t aio_stream = nullptr;
  cudaEvent_t aio_copied[2] = {nullptr, nullptr};
  cudaEvent_t aio_done[2] = {nullptr, nullptr};
  cudaStream_t cap_stream = nullptr;
  // kernel timing (efunc_set_timing): event pairs, slot = call index mod slots
  std::vector<efunc*> kids;          // n_shapes > 1: one single-shape handle per shape
  std::vector<cudaStream_t> kid_streams;  // batched calls fork the shapes onto these and join
  std::vector<cudaEvent_t> kid_events;
  cudaEvent_t fork_event = nullptr;
  std::vector<cudaEvent_t> tev;
  std::vector<int> tev_used;
  int64_t tseq = 0;
  std::string err;
};
