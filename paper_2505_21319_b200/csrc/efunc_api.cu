// efunc_api.cu — the C ABI (include/efunc.h): handle lifetime, workspaces, call sequencing.
// Every step of the path runs in the kernels of k_bin.cu / k_lists.cu / k_forward.cu / k_backward.cu / k_adamw.cu; this
// file only validates arguments, sizes workspaces and enqueues launches on the caller's stream.
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "efunc_internal.cuh"

using namespace ef;

static thread_local std::string g_err;

static efunc_status fail(efunc_t* h, efunc_status s, const std::string& m) {
  if (h) h->err = m;
  g_err = m;
  return s;
}

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) {                                                                  \
      return fail(h, e_ == cudaErrorMemoryAllocation ? EFUNC_ENOMEM : EFUNC_ECUDA,            \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                           \
    }                                                                                         \
  } while (0)

#define RET(x)                                    \
  do {                                            \
    efunc_status st_ = (x);                       \
    if (st_ != EFUNC_OK) return st_;              \
  } while (0)

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
cudaError_t dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
}

template <class T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

float cutoff_log2(const efunc_config& c) {
  if (!(c.cutoff_T > 0.0f) || std::isinf(c.cutoff_T)) return INFINITY;
  return c.cutoff_T * EF_LOG2E;
}

// Brick edge (in lattice cells) ~ half the search radius at the paper's init (beta = e^7,
// PAPER.md:L908): rho^2 = 3h^2/4 + T/beta. Dense mode (T = inf): one brick for everything.
BrickGeom brick_geom(const efunc_config& cfg, int NC, float h) {
  BrickGeom g;
  if (!(cfg.cutoff_T > 0.0f) || std::isinf(cfg.cutoff_T)) {
    g.B = NC;
  } else {
    const double rho = std::sqrt(0.75 * h * h + cfg.cutoff_T / std::exp(7.0));
    int B = 1;
    while (2 * B * h <= 0.5 * rho && 2 * B <= NC) B *= 2;  // largest power of 2 with B h <= rho / 2
#ifdef EF_BRICK_B
    B = EF_BRICK_B < NC ? EF_BRICK_B : NC;
#endif
    g.B = B;
  }
  g.nb = (NC + g.B - 1) / g.B;
  g.bits = 0;
  while ((1 << g.bits) < g.nb) ++g.bits;
  g.n_codes = 1u << (3 * g.bits);
  // work items are balanced runs of the Morton-sorted queries of one brick: sorting them by
  // quarter-cell (rather than half-cell) sub-bins makes the items' boxes tighter (fewer candidate
  // keys) while the bin arrays stay small (<= 8M bins); EF_SUBDIV overrides for experiments
  g.sdiv = 4;
#ifdef EF_SUBDIV
  g.sdiv = EF_SUBDIV;
#endif
  auto set_sub = [&]() {
    g.sub_bits = 0;
    while ((1 << g.sub_bits) < g.sdiv * g.B) ++g.sub_bits;
    g.qsub = 1u << (3 * g.sub_bits);
  };
  set_sub();
#ifndef EF_BIN_CAP
#define EF_BIN_CAP (8u << 20)
#endif
  while ((uint64_t)g.n_codes * g.qsub > EF_BIN_CAP && g.sdiv > 2) {
    g.sdiv /= 2;
    set_sub();
  }
  return g;
}

KeysView keys_view(efunc_t* h) {
  KeysView kv;
  kv.ks = h->key_sorted;
  kv.kid = h->kid;
  kv.cell_start = h->cell_start;
  kv.grid_raw = h->key_raw;
  kv.bl_min = &h->ds->bl_min;
  kv.R = h->R;
  kv.NC = h->NC;
  kv.inv_h = h->inv_h;
  kv.h = h->h;
  kv.n_nodes = h->n_nodes;
  kv.bl_pool = h->bl_pool;
  kv.bl_off = h->bl_off;
  kv.bl_n = h->bl_n;
  return kv;
}

void drop_fit_graph(efunc_t* h) {
  for (int k = 0; k < 2; ++k) {
    if (h->fit_exec[k]) cudaGraphExecDestroy(h->fit_exec[k]);
    h->fit_exec[k] = nullptr;
    h->fit_seen[k] = 0;
  }
}

efunc_status ensure_scan_tmp(efunc_t* h, size_t n_elems) {
  size_t tiles = (n_elems + 4095) / 4096 + 1;
  if (tiles <= h->scan_tmp_cap) return EFUNC_OK;
  drop_fit_graph(h);
  dfree(h->scan_tmp);
  CK(dalloc(&h->scan_tmp, tiles));
  h->scan_tmp_cap = tiles;
  return EFUNC_OK;
}

// scratch of the stable radix sort for up to n elements
efunc_status ensure_radix(efunc_t* h, size_t n) {
  if (n <= h->rk_cap) return EFUNC_OK;
  drop_fit_graph(h);
  dfree(h->rk);
  dfree(h->rh);
  CK(dalloc(&h->rk, 2 * n));
  CK(dalloc(&h->rh, radix_hist_elems((uint32_t)n)));
  h->rk_cap = n;
  return ensure_scan_tmp(h, radix_hist_elems((uint32_t)n));
}

int bits_for(size_t nvals) {  // bits of the largest value nvals - 1
  int b = 1;
  while (b < 32 && ((size_t)1 << b) < nvals) ++b;
  return b;
}

#ifndef EF_ITEMS_FUSED_MAX
#define EF_ITEMS_FUSED_MAX 0u  // the single-CTA item pass measured slower at C2 (32k bricks): off
#endif

// S0 + key binning + brick lists. force = 1: theta was replaced wholesale, rebuild the lists
// regardless of the Verlet skin.
// degree 0 (Table 3 G-0: f = c): the g channels of both banks held at 0
uint32_t g_channels(const efunc_t* h) {
  return (!h->vmode && h->cfg.degree == 0) ? ((7u << 2) | (7u << 10)) : 0u;
}

// Variants (NEXT-4): the internal 13-channel theta (+ the degree-2 squares and their per-key
// records) derived from the user's parameters; call before rebuild_keys
void sync_internal_theta(efunc_t* h, cudaStream_t s) {
  if (!h->vmode) return;
  h->launches += launch_var_unpack(h->theta_v, h->n_nodes, h->vlay, h->theta, h->thetaH, s);
  if (h->keyH) h->launches += launch_var_keyH(h->thetaH, h->n_nodes, h->keyH, s);
}

// channels of the user's parameter layout for a (variant, degree), or -1 (include/efunc.h)
int variant_channels(int variant, int degree, ef::VarLayout* L) {
  if (degree < 0 || degree > 2 || variant < 0 || variant > 2) return -1;
  const int coef = degree == 0 ? 1 : (degree == 1 ? 4 : 10);
  ef::VarLayout v{};
  v.deg = degree;
  v.grid = v.off = v.delta = -1;
  if (variant == EFUNC_VARIANT_COMBINED && degree <= 1) {  // the 13-channel layout (Table 3 Full-4)
    v.nch = EF_NCH;
    v.grid = 0;
    v.delta = 5;
    v.off = 8;
  } else {
    int o = 0;
    if (variant != EFUNC_VARIANT_OFFSET) {
      v.grid = o;
      o += 1 + coef;
    }
    if (variant != EFUNC_VARIANT_GRID) {
      v.delta = o;
      v.off = o + 3;
      o += 4 + coef;
    }
    v.nch = o;
  }
  if (L) *L = v;
  return v.nch;
}

// the per-rebuild counters k_prep_keys / k_adamw_keys accumulate into
// (one fill launch; lists_invalid starts every rebuild at force, so no reset is needed after it)
efunc_status reset_key_counters(efunc_t* h, cudaStream_t s, int force) {
  FillSegs f;
  f.add(h->cell_count, sizeof(uint32_t) * (h->n_cells + 1), 0u);
  f.add(&h->ds->bl_min, sizeof(float), 0x7f7f7f7fu);  // 3.39e38
  f.add(&h->ds->lists_invalid, sizeof(uint32_t), force ? 1u : 0u);
  f.add(&h->ds->keys_resort, sizeof(uint32_t), force ? 1u : 0u);
  h->launches += launch_fill_segs(f, s);
  return EFUNC_OK;
}

// prepped: the key records were written by k_adamw_keys (AdamW and S0 in one pass)
efunc_status rebuild_keys(efunc_t* h, cudaStream_t s, int force = 0, int prepped = 0) {
  if (!prepped) {
    if (force) h->launches += launch_zero_channels(h->theta, h->n_nodes, g_channels(h), s);
    RET(reset_key_counters(h, s, force));
    const float skin = SKIN_H * h->h;
    h->launches += launch_prep_keys(h->theta, h->R, h->banks, h->key_raw, h->key_cell,
                                    h->cfg.deterministic ? nullptr : h->key_rank, h->cell_count, h->key_ref,
                                    skin * skin, SKIN_MU, h->ds, s);
  }
  // the cell sort only when some offset key changed cell (k_prep_keys sets keys_resort)
  const uint32_t* gate = &h->ds->keys_resort;
  h->launches += launch_scan_u32(h->cell_count, h->cell_start, h->n_cells + 1, h->scan_tmp, s, gate);
  // deterministic mode: stable (LSD radix) so the per-cell key order, and with it every list and
  // summation order, repeats run to run; otherwise the atomic scatter (any in-cell order is valid)
  if (h->cfg.deterministic)
    h->launches += launch_stable_sort(h->key_cell, h->n_keys, bits_for((size_t)h->n_cells + 1), h->rk, h->rh,
                                      h->scan_tmp, h->key_tmp, h->key_order, s, gate);
  else
    h->launches += launch_scatter_ranked(h->key_cell, h->key_rank, h->n_keys, h->cell_start, h->key_order, s, gate);
  h->launches += launch_gather_keys(h->key_order, h->key_raw, h->key_sorted, h->kid, h->n_keys, s);
  // per-brick candidate lists for the next forward/backward (query independent)
  h->launches += launch_brick_lists(keys_view(h), h->bg, cutoff_log2(h->cfg), h->bl_pool, h->bl_pool_cap,
                                    h->bl_off, h->bl_n, h->ds, h->scratch, s);
  h->launches += launch_list_snapshot(h->key_raw, h->key_ref, h->n_keys, h->ds, s);
  CK(cudaGetLastError());
  h->have_fwd = 0;
  return EFUNC_OK;
}

efunc_status ensure_queries(efunc_t* h, int64_t J) {
  const int64_t bound = (J + IQ - 1) / IQ + h->bg.n_codes + 1;
  if (bound > h->items_cap || J > h->J_cap) drop_fit_graph(h);
  if (bound > h->items_cap) {
    dfree(h->loss_part); dfree(h->items); dfree(h->wl_off); dfree(h->wl_n); dfree(h->slow_items);
    dfree(h->item_o);
    CK(dalloc(&h->item_o, bound));
    CK(dalloc(&h->loss_part, bound));
    CK(dalloc(&h->slow_items, bound));
    CK(dalloc(&h->items, bound));
    CK(dalloc(&h->wl_off, bound));
    CK(dalloc(&h->wl_n, bound));
    h->items_cap = bound;
  }
  // forward -> backward candidate-id pool: reserved per item = its brick list length
  const double want = std::fmin((double)J * WL_PER_QUERY, 3.9e9);
  if (want > (double)h->wl_cap) {
    drop_fit_graph(h);
    dfree(h->wl_pool);
    CK(dalloc(&h->wl_pool, (size_t)want));
    h->wl_cap = (uint32_t)want;
  }
  RET(ensure_radix(h, (size_t)J));
  if (J > h->J_cap) {
    dfree(h->q_bin); dfree(h->q_tmp); dfree(h->q_order); dfree(h->qs); dfree(h->perm);
    dfree(h->rec); dfree(h->gs); dfree(h->us); dfree(h->hs); dfree(h->qmh); dfree(h->qf0);
    CK(dalloc(&h->q_bin, J));
    CK(dalloc(&h->qmh, J));
    CK(dalloc(&h->qf0, J));
    CK(dalloc(&h->q_tmp, J));
    CK(dalloc(&h->q_order, J));
    CK(dalloc(&h->qs, J));
    CK(dalloc(&h->perm, J));
    CK(dalloc(&h->rec, J));
    CK(dalloc(&h->gs, J));
    CK(dalloc(&h->us, J));
    CK(dalloc(&h->hs, J));
    h->J_cap = J;
  }
  return EFUNC_OK;
}

// Kernel timing: record an event pair around the call's dominant kernel (capture-safe).
void record_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else cudaEventRecord(e, s);
}

int timing_begin(efunc_t* h, cudaStream_t s) {
  if (h->tev.empty()) return -1;
  const int slot = (int)(h->tseq++ % (int64_t)(h->tev.size() / 2));
  record_event(h->tev[2 * slot], s);
  return slot;
}

void timing_end(efunc_t* h, int slot, cudaStream_t s) {
  if (slot < 0) return;
  record_event(h->tev[2 * slot + 1], s);
  h->tev_used[slot] = 1;
}

void free_timing(efunc_t* h) {
  for (cudaEvent_t e : h->tev) cudaEventDestroy(e);
  h->tev.clear();
  h->tev_used.clear();
  h->tseq = 0;
}

void free_all(efunc_t* h) {
  dfree(h->theta); dfree(h->m); dfree(h->v);
  dfree(h->theta_v); dfree(h->m_v); dfree(h->v_v); dfree(h->thetaH); dfree(h->keyH); dfree(h->gint); dfree(h->gH);
  dfree(h->key_raw); dfree(h->key_sorted); dfree(h->kid); dfree(h->key_cell);
  dfree(h->cell_count); dfree(h->cell_start); dfree(h->cell_fill); dfree(h->key_tmp); dfree(h->key_rank); dfree(h->key_order);
  dfree(h->scan_tmp); dfree(h->ds); dfree(h->fit_grad); dfree(h->rk); dfree(h->rh);
  dfree(h->q_bin); dfree(h->bin_count); dfree(h->bin_start); dfree(h->bin_fill); dfree(h->q_tmp);
  dfree(h->q_order); dfree(h->qs); dfree(h->perm); dfree(h->rec); dfree(h->gs); dfree(h->us); dfree(h->hs);
  dfree(h->qmh); dfree(h->qf0); dfree(h->loss_part); dfree(h->io_q); dfree(h->io_o); dfree(h->io_loss);
  dfree(h->items); dfree(h->item_cnt); dfree(h->item_off); dfree(h->gpad); dfree(h->peer_grad);
  dfree(h->bl_pool); dfree(h->bl_off); dfree(h->bl_n); dfree(h->key_ref); dfree(h->gfix);
  dfree(h->wl_pool); dfree(h->wl_off); dfree(h->wl_n); dfree(h->slow_items); dfree(h->item_o);
  dfree(h->scratch); dfree(h->iota); dfree(h->dn_zm); dfree(h->dn_dq);
  drop_fit_graph(h);
  free_timing(h);
  for (int k = 0; k < 2; ++k) {
    if (h->aio_done[k]) cudaEventSynchronize(h->aio_done[k]);
    dfree(h->aio_q[k]); dfree(h->aio_o[k]); dfree(h->aio_loss[k]);
    if (h->aio_copied[k]) cudaEventDestroy(h->aio_copied[k]);
    if (h->aio_done[k]) cudaEventDestroy(h->aio_done[k]);
    h->aio_copied[k] = h->aio_done[k] = nullptr;
  }
  if (h->aio_pin) cudaFreeHost(h->aio_pin);
  h->aio_pin = nullptr;
  if (h->aio_stream) cudaStreamDestroy(h->aio_stream);
  h->aio_stream = nullptr;
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  h->cap_stream = nullptr;
}

// S1 for one forward: query bins, stable counting sort, gather, work items; then the forward
// arguments (everything but the outputs).
efunc_status prep_queries(efunc_t* h, const float* q, const float* o_used, int64_t J, const efunc_loss* loss,
                          FwdArgs& a, cudaStream_t s, int with_mh = 0) {
  const int kind = loss ? loss->kind : EFUNC_LOSS_NONE;
  RET(ensure_queries(h, J));
  const uint32_t nb = h->bg.n_codes;             // bricks
  const uint32_t nbins = nb * h->bg.qsub + 1;    // sub-cell bins + the out-of-domain bin
  FillSegs fz;  // the bin histogram and the per-forward counters, one fill launch
  fz.add(h->bin_count, sizeof(uint32_t) * (nbins + 1), 0u);
  // fused path: each query's rank inside its bin comes from the histogram's atomic (no fill
  // counters, no second atomic pass); the other paths sort stably instead
  const bool ranked = with_mh && !h->cfg.deterministic;
  static_assert(offsetof(DevScalars, kept_pairs_offset) + sizeof(unsigned long long) == sizeof(DevScalars),
                "the per-forward counters end DevScalars");
  static_assert(offsetof(DevScalars, overflow_items) % 4 == 0 && sizeof(DevScalars) % 4 == 0, "u32 fill");
  fz.add(&h->ds->overflow_items, sizeof(DevScalars) - offsetof(DevScalars, overflow_items), 0u);
  h->launches += launch_fill_segs(fz, s);
  h->launches += launch_query_bins(q, o_used, J, h->bg, h->NC, h->inv_h, h->q_bin, h->bin_count,
                                   ranked ? h->q_tmp : nullptr, h->ds, s);
  h->launches += launch_scan_u32(h->bin_count, h->bin_start, nbins + 1, h->scan_tmp, s);
  if (with_mh && !h->cfg.deterministic) {
    // fused path: the atomic scatter order inside a bin is kept (only deterministic mode needs the
    // stable rank); the gather then runs in sorted order, so the shift bounds' key loads of
    // neighbouring threads hit the same cells
    h->launches += launch_scatter_ranked(h->q_bin, h->q_tmp, (uint32_t)J, h->bin_start, h->q_order, s);
    h->launches += launch_gather_queries_mh(keys_view(h), h->q_order, q, o_used, J, h->qs, h->perm, h->qmh,
                                            with_mh == 2 ? h->qf0 : nullptr, s);
  } else {
    h->launches += launch_stable_sort(h->q_bin, (uint32_t)J, bits_for(nbins), h->rk, h->rh, h->scan_tmp, h->q_tmp,
                                      h->q_order, s);
    if (with_mh)  // + the per-query shift bound
      h->launches += launch_gather_queries_mh(keys_view(h), h->q_order, q, o_used, J, h->qs, h->perm, h->qmh,
                                              with_mh == 2 ? h->qf0 : nullptr, s);
    else
      h->launches += launch_gather_queries(h->q_order, q, o_used, J, h->qs, h->perm, s);
  }
  // work items: balanced runs of <= QW sorted queries of one brick
  if (nb + 2 <= EF_ITEMS_FUSED_MAX) {  // one single-CTA pass
    h->launches += launch_items_fused(h->bin_start, nb, h->bg.qsub, h->item_off, h->items, s);
  } else {
    // cost classes need the brick lists (cutoff mode): heavy items first, the lightest last
    const uint32_t* bl_n = std::isinf(cutoff_log2(h->cfg)) ? nullptr : h->bl_n;
    h->launches += launch_items_count(h->bin_start, nb, h->bg.qsub, bl_n, h->ds, h->item_cnt, s);
    h->launches += launch_scan_u32(h->item_cnt, h->item_off, ITEMS_N_AT(nb) + 1, h->scan_tmp, s);
    h->launches += launch_items_write(h->bin_start, nb, h->bg.qsub, bl_n, h->ds, h->item_off, h->items, s);
  }
  const int64_t items = (J + IQ - 1) / IQ + nb + 1;  // launch bound; kernels read the count
  h->fwd_items_bound = items;
  a = FwdArgs{};
  a.kv = keys_view(h);
  a.qs = h->qs;
  a.perm = h->perm;
  a.J = J;
  a.items = h->items;
  a.n_items = h->item_off + ITEMS_N_AT(nb);
  a.T_l = cutoff_log2(h->cfg);
  a.loss_kind = kind;
  const int64_t Jg = (loss && loss->J_global > 0) ? loss->J_global : J;
  a.inv_J = (float)(1.0 / (double)Jg);
  a.eik_lambda = loss ? loss->eikonal_lambda : 0.0f;
  a.rec = h->rec;
  a.gs = h->gs;
  a.us = h->us;
  a.hs = h->hs;
  a.loss_part = h->loss_part;
  a.qmh = h->qmh;
  a.qf0 = h->qf0;
  a.wl_pool = h->wl_pool;
  a.wl_cap = h->wl_cap;
  a.wl_off = h->wl_off;
  a.wl_n = h->wl_n;
  a.slow_items = h->slow_items;
  a.ds = h->ds;
  a.count_kept = h->count_kept;
  return EFUNC_OK;
}

efunc_status do_forward(efunc_t* h, const float* q, const float* o, int64_t J, const efunc_loss* loss,
                        float* O, float* G, float* loss_out, int keep_state, cudaStream_t s) {
  const int kind = loss ? loss->kind : EFUNC_LOSS_NONE;
  if (J < 0) return fail(h, EFUNC_EINVAL, "J < 0");
  if (kind < EFUNC_LOSS_NONE || kind > EFUNC_LOSS_MSE_EIKONAL) return fail(h, EFUNC_EINVAL, "bad loss kind");
  if (J > 0 && !q) return fail(h, EFUNC_EINVAL, "q is NULL");
  if (J > 0 && kind != EFUNC_LOSS_NONE && !o) return fail(h, EFUNC_EINVAL, "loss requires targets o");
  if (J > (int64_t)0x7fffffff) return fail(h, EFUNC_EINVAL, "J > 2^31-1 per call");
  const int want_g = (G != nullptr) || kind == EFUNC_LOSS_MSE_EIKONAL;
  h->have_fwd = 0;
  if (J == 0) {
    if (loss_out) CK(cudaMemsetAsync(loss_out, 0, sizeof(float), s));
    h->have_fwd = keep_state;
    h->fwd_J = 0;
    h->fwd_has_g = want_g;
    h->fwd_loss_kind = kind;
    return EFUNC_OK;
  }
  const float* o_used = (kind != EFUNC_LOSS_NONE) ? o : nullptr;
  if (h->vk && kind == EFUNC_LOSS_MSE_EIKONAL)
    return fail(h, EFUNC_EINVAL, "degree 2 / O^Delta only: the Eikonal loss is not supported (MSE or no loss)");
  FwdArgs a;
  RET(prep_queries(h, q, o_used, J, loss, a, s));
  const int64_t items = h->fwd_items_bound;
  const uint32_t* n_items = a.n_items;
  a.O = O;
  a.G = G;
  if (h->vk) {  // NEXT-4 (k_var.cu): certified item lists (or every key), exact shift, O (+G)
    if (!std::isinf(a.T_l)) h->launches += launch_item_lists(a, items, s);
    h->launches += launch_var_forward(a, h->keyH, h->iota, h->iota_n, G != nullptr, items, s);
  } else {
    h->launches += launch_forward(a, want_g, items, s);
  }
  if (kind != EFUNC_LOSS_NONE && loss_out) h->launches += launch_sum_partials(h->loss_part, n_items, 1, loss_out, s);
  else if (loss_out) CK(cudaMemsetAsync(loss_out, 0, sizeof(float), s));
  CK(cudaGetLastError());
  if (h->cfg.sync_checks) {
    CK(cudaStreamSynchronize(s));
    DevScalars d;
    CK(cudaMemcpy(&d, h->ds, sizeof(d), cudaMemcpyDeviceToHost));
    if (d.nonfinite) {
      CK(cudaMemset(&h->ds->nonfinite, 0, sizeof(uint32_t)));
      return fail(h, EFUNC_ENONFINITE, "non-finite query or target");
    }
  }
  h->have_fwd = keep_state;
  h->fwd_J = J;
  h->fwd_has_g = want_g;
  h->fwd_loss_kind = kind;
  return EFUNC_OK;
}

BwdArgs bwd_args(efunc_t* h, const float* dL_dO, const float* dL_dG, float* grad, int eik) {
  BwdArgs b{};
  b.kv = keys_view(h);
  b.qs = h->qs;
  b.perm = h->perm;
  b.J = h->fwd_J;
  b.items = h->items;
  b.n_items = h->item_off + ITEMS_N_AT(h->bg.n_codes);
  b.T_l = cutoff_log2(h->cfg);
  b.gpad = h->gpad;
  b.gfix = h->gfix;
  b.wl_pool = h->wl_pool;
  b.wl_off = h->wl_off;
  b.wl_n = h->wl_n;
  b.umax = &h->ds->umax;
  b.fix_overflow = &h->ds->fix_overflow;
  b.rec = h->rec;
  b.gs = h->gs;
  b.us = h->us;
  b.hs = h->hs;
  b.dL_dO = dL_dO;
  b.dL_dG = dL_dG;
  b.grad = grad;
  b.eik = eik;
  b.next = &h->ds->bwd_next;
  b.list = nullptr;
  b.list_n = nullptr;
  return b;
}

efunc_status do_backward(efunc_t* h, const float* dL_dO, const float* dL_dG, float* grad, cudaStream_t s) {
  if (!grad) return fail(h, EFUNC_EINVAL, "grad is NULL");
  if (!h->have_fwd) return fail(h, EFUNC_ESTATE, "backward without a valid forward (saved e_j missing)");
  if (h->fwd_J == 0) return EFUNC_OK;
  if (!dL_dO && h->fwd_loss_kind == EFUNC_LOSS_NONE)
    return fail(h, EFUNC_EINVAL, "dL_dO is NULL and the forward had no fused loss");
  const int eik = (dL_dG != nullptr) || (!dL_dO && h->fwd_loss_kind == EFUNC_LOSS_MSE_EIKONAL);
  if (eik && !h->fwd_has_g) return fail(h, EFUNC_ESTATE, "dL_dG needs a forward that computed G");
  BwdArgs b = bwd_args(h, dL_dO, dL_dG, grad, eik);
  CK(cudaMemsetAsync(&h->ds->bwd_next, 0, sizeof(uint32_t), s));
  if (h->cfg.deterministic) {
    CK(cudaMemsetAsync(&h->ds->umax, 0, sizeof(float), s));
    const int slot = timing_begin(h, s);
    h->launches += launch_backward_det(b, h->fwd_items_bound, s);
    timing_end(h, slot, s);
    h->launches += launch_fold_fix(h->gfix, &h->ds->umax, grad, h->n_nodes, s);
  } else {
    const int slot = timing_begin(h, s);
    h->launches += launch_backward(b, h->fwd_items_bound, s);
    timing_end(h, slot, s);
    h->launches += (h->n_peers > 0 || h->mc_grad)
                       ? launch_fold_peers(h->gpad, h->n_nodes, h->peer_grad, h->n_peers, h->mc_grad, s)
                       : launch_fold(h->gpad, grad, h->n_nodes, s);
  }
  CK(cudaGetLastError());
  return EFUNC_OK;
}

// the FwdArgs of the last forward (its sorted queries, items, records and candidate lists)
FwdArgs saved_fwd_args(efunc_t* h) {
  FwdArgs a{};
  a.kv = keys_view(h);
  a.qs = h->qs;
  a.perm = h->perm;
  a.J = h->fwd_J;
  a.items = h->items;
  a.n_items = h->item_off + ITEMS_N_AT(h->bg.n_codes);
  a.T_l = cutoff_log2(h->cfg);
  a.rec = h->rec;
  a.wl_pool = h->wl_pool;
  a.wl_cap = h->wl_cap;
  a.wl_off = h->wl_off;
  a.wl_n = h->wl_n;
  a.ds = h->ds;
  return a;
}

// degree-2 backward (k_var.cu) into the internal gradient scratch (g13 += ..., gH += ...)
efunc_status do_backward_var2(efunc_t* h, const float* dL_dO, const float* dL_dG, float* g13, float* gH,
                              cudaStream_t s) {
  if (!h->have_fwd) return fail(h, EFUNC_ESTATE, "backward without a valid forward (saved e_j missing)");
  if (dL_dG) return fail(h, EFUNC_EINVAL, "degree 2: dL_dG (Eikonal terms) is not supported");
  if (h->fwd_J == 0) return EFUNC_OK;
  if (!dL_dO && h->fwd_loss_kind == EFUNC_LOSS_NONE)
    return fail(h, EFUNC_EINVAL, "dL_dO is NULL and the forward had no fused loss");
  const FwdArgs a = saved_fwd_args(h);
  const int slot = timing_begin(h, s);
  h->launches += launch_var_backward(a, h->keyH, h->iota, h->iota_n, dL_dO, g13, gH, h->fwd_items_bound, s);
  timing_end(h, slot, s);
  CK(cudaGetLastError());
  return EFUNC_OK;
}

efunc_status zero_internal_grad(efunc_t* h, cudaStream_t s) {
  CK(cudaMemsetAsync(h->gint, 0, sizeof(float) * (size_t)h->n_nodes * EF_NCH, s));
  if (h->gH) CK(cudaMemsetAsync(h->gH, 0, sizeof(float) * (size_t)h->n_nodes * 12, s));
  return EFUNC_OK;
}

// backward in the user's layout (grad += dL/dtheta)
efunc_status any_backward(efunc_t* h, const float* dL_dO, const float* dL_dG, float* grad, cudaStream_t s) {
  if (!h->vmode) return do_backward(h, dL_dO, dL_dG, grad, s);
  if (!grad) return fail(h, EFUNC_EINVAL, "grad is NULL");
  RET(zero_internal_grad(h, s));
  if (h->vk) RET(do_backward_var2(h, dL_dO, dL_dG, h->gint, h->gH, s));
  else RET(do_backward(h, dL_dO, dL_dG, h->gint, s));
  h->launches += launch_var_pack_grad(h->gint, h->gH, h->n_nodes, h->vlay, grad, s);
  return EFUNC_OK;
}

efunc_status do_forward_backward(efunc_t* h, const float* q, const float* o, int64_t J, const efunc_loss* loss,
                                 float* O, float* grad, float* loss_out, cudaStream_t s);

efunc_status any_forward_backward(efunc_t* h, const float* q, const float* o, int64_t J, const efunc_loss* loss,
                                  float* O, float* grad, float* loss_out, cudaStream_t s) {
  if (!h->vmode) return do_forward_backward(h, q, o, J, loss, O, grad, loss_out, s);
  if (!grad) return fail(h, EFUNC_EINVAL, "grad is NULL");
  if (!loss || loss->kind == EFUNC_LOSS_NONE) return fail(h, EFUNC_EINVAL, "forward_backward needs a loss");
  RET(zero_internal_grad(h, s));
  if (h->vk) {
    RET(do_forward(h, q, o, J, loss, O, nullptr, loss_out, 1, s));
    const efunc_status st = do_backward_var2(h, nullptr, nullptr, h->gint, h->gH, s);
    h->have_fwd = 0;  // like the fused call: no saved state afterwards
    RET(st);
  } else {
    RET(do_forward_backward(h, q, o, J, loss, O, h->gint, loss_out, s));
  }
  h->launches += launch_var_pack_grad(h->gint, h->gH, h->n_nodes, h->vlay, grad, s);
  return EFUNC_OK;
}

// EFUNC_FIT_PRE=1: the items' candidate lists are built by k_fit_lists before k_fit (measured
// slower than k_fit building them itself; kept for A/B runs)
int fit_pre_off() {
  static const int off = [] {
    const char* e = std::getenv("EFUNC_FIT_PRE");
    return (e && e[0] == '1') ? 0 : 1;
  }();
  return off;
}

// EFUNC_FIT_TC=0/1: the MSE fused fit step on k_fit (FP32 pair loops) or k_fit_tc (tensor-core
// pair loops, 3xTF32)
int fit_tc_on() {
  static const int on = [] {
    const char* e = std::getenv("EFUNC_FIT_TC");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return on;
}

// efunc_forward_backward: the fused fit kernel for the MSE loss (k_fit.cu), the split kernels for
// its leftover items; forward + backward otherwise.
efunc_status do_forward_backward(efunc_t* h, const float* q, const float* o, int64_t J, const efunc_loss* loss,
                                 float* O, float* grad, float* loss_out, cudaStream_t s) {
  if (!grad) return fail(h, EFUNC_EINVAL, "grad is NULL");
  if (!loss || loss->kind == EFUNC_LOSS_NONE) return fail(h, EFUNC_EINVAL, "forward_backward needs a loss");
  const int eik = loss->kind == EFUNC_LOSS_MSE_EIKONAL;
  const bool dense = std::isinf(cutoff_log2(h->cfg));
  // deterministic mode: the fused MSE kernel with 64-bit fixed-point sums (cutoff mode); otherwise split
  const int det = h->cfg.deterministic;
  const int fused = !h->count_kept && !(det && (eik || dense));
  if (!fused || J == 0) {
    RET(do_forward(h, q, o, J, loss, O, nullptr, loss_out, 1, s));
    RET(do_backward(h, nullptr, nullptr, grad, s));
    h->have_fwd = 0;
    return EFUNC_OK;
  }
  if (J < 0) return fail(h, EFUNC_EINVAL, "J < 0");
  if (loss->kind < EFUNC_LOSS_NONE || loss->kind > EFUNC_LOSS_MSE_EIKONAL) return fail(h, EFUNC_EINVAL, "bad loss kind");
  if (!q || !o) return fail(h, EFUNC_EINVAL, "q or o is NULL");
  if (J > (int64_t)0x7fffffff) return fail(h, EFUNC_EINVAL, "J > 2^31-1 per call");
  h->have_fwd = 0;
  FwdArgs a;
  RET(prep_queries(h, q, o, J, loss, a, s, eik ? 2 : 1));  // + the shift keys' f0 for k_fit_eik
  a.O = O;
  a.G = nullptr;
  FitArgs f;
  f.f = a;
  f.gpad = h->gpad;
  f.scratch = h->scratch;
  f.iota = dense ? h->iota : nullptr;
  f.iota_n = h->iota_n;
  f.item_o = h->item_o;
  f.n_heavy = h->item_off + (h->bg.n_codes + 1);  // the exclusive scan at the first class-1 slot
  f.gfix = det ? h->gfix : nullptr;
  f.umax = &h->ds->umax;
  f.fix_overflow = &h->ds->fix_overflow;
  if (det) {  // the fixed-point unit: an a-priori bound of max_j |r_j| (k_det_bound)
    CK(cudaMemsetAsync(&h->ds->umax, 0, sizeof(float), s));
    h->launches += launch_det_bound(h->theta, h->n_nodes, h->qs, J, a.inv_J, &h->ds->umax, s);
  }
  // MSE, cutoff mode: the items' candidate lists are built first by k_fit_lists (latency-bound list
  // stream at full occupancy), then k_fit computes; the timed "dominant kernel" spans both
  f.pre = (!eik && !dense && !det && !fit_pre_off()) ? 1 : 0;
  if (dense) {  // NEXT-2: key-sliced dense kernels (all warp slots busy at small J)
    const int64_t nz = eik ? dense_eik_part_elems(h->fwd_items_bound, h->iota_n)
                           : dense_zm_elems(h->fwd_items_bound, h->iota_n);
    // dn_zm holds float2 (MSE: Z, M per query and slice) or the Eikonal path's 11 floats per query
    // and slice (half as many float2); dn_dq a packed query table per item (48 / 80 float4)
    const int64_t nz2 = eik ? (nz + 1) / 2 : nz;
    if (nz2 > h->dn_zm_cap) {
      drop_fit_graph(h);
      dfree(h->dn_zm);
      CK(dalloc(&h->dn_zm, (size_t)nz2));
      h->dn_zm_cap = nz2;
    }
    const int64_t ndq = h->fwd_items_bound * (eik ? 80 : 48);
    if (ndq > h->dn_dq_cap) {
      drop_fit_graph(h);
      dfree(h->dn_dq);
      CK(dalloc(&h->dn_dq, (size_t)ndq));
      h->dn_dq_cap = ndq;
    }
    const int slot = timing_begin(h, s);
    if (eik)
      h->launches += launch_dense_fit_eik(f, h->fwd_items_bound, reinterpret_cast<float*>(h->dn_zm), h->dn_dq, s);
    else
      h->launches += launch_dense_fit(f, h->fwd_items_bound, h->dn_zm, h->dn_dq, s, nullptr);
    timing_end(h, slot, s);
  } else {
    const int slot = timing_begin(h, s);
    if (f.pre) h->launches += launch_fit_lists(f, h->fwd_items_bound, s);
    h->launches += eik ? launch_fit_eik(f, h->fwd_items_bound, s)
                       : (fit_tc_on() && !f.pre) ? launch_fit_tc(f, h->fwd_items_bound, s)
                                                 : launch_fit(f, h->fwd_items_bound, s);
    timing_end(h, slot, s);
  }
  // items the fused kernel left (no brick list / shift-bound overflow): the split kernels
  h->fwd_J = J;
  h->launches += launch_forward_slow(a, eik, s);
  BwdArgs b = bwd_args(h, nullptr, nullptr, grad, eik);
  b.list = h->slow_items;
  b.list_n = &h->ds->slow_n;  // (bwd_next is still 0 from prep_queries: k_fit and k_forward use other cursors)
  if (det) {  // fixed point with the unit k_det_bound set, then folded into grad
    h->launches += launch_backward_list_det(b, s);
    h->launches += launch_fold_fix(h->gfix, &h->ds->umax, grad, h->n_nodes, s);
  } else {
    h->launches += launch_backward(b, h->fwd_items_bound, s);
    h->launches += (h->n_peers > 0 || h->mc_grad)
                       ? launch_fold_peers(h->gpad, h->n_nodes, h->peer_grad, h->n_peers, h->mc_grad, s)
                       : launch_fold(h->gpad, grad, h->n_nodes, s);
  }
  if (loss_out) h->launches += launch_sum_partials(h->loss_part, a.n_items, 1, loss_out, s);
  CK(cudaGetLastError());
  if (h->cfg.sync_checks) {
    CK(cudaStreamSynchronize(s));
    uint32_t nf = 0;
    CK(cudaMemcpy(&nf, &h->ds->nonfinite, sizeof(nf), cudaMemcpyDeviceToHost));
    if (nf) {
      CK(cudaMemset(&h->ds->nonfinite, 0, sizeof(uint32_t)));
      return fail(h, EFUNC_ENONFINITE, "non-finite query or target");
    }
  }
  return EFUNC_OK;
}

efunc_status do_adamw(efunc_t* h, const float* grad, const efunc_adamw* hp, cudaStream_t s) {
  if (!grad || !hp) return fail(h, EFUNC_EINVAL, "NULL argument");
  // the step counter and the bias corrections live on the device (k_adamw)
  AdamWConst hc;
  hc.lr = hp->lr;
  hc.beta1 = hp->beta1;
  hc.beta2 = hp->beta2;
  hc.eps = hp->eps;
  hc.weight_decay = hp->weight_decay;
  hc.decay_mask = hp->decay_mask;
  hc.frozen_mask = g_channels(h);
  hc.nch = h->pnch;
  if (h->vmode) {  // NEXT-4: the update runs on the user's layout, then the internal theta follows
    h->launches += launch_adamw(h->theta_v, grad, h->m_v, h->v_v, (int64_t)h->n_nodes * h->pnch, hc, h->ds, s);
    sync_internal_theta(h, s);
  } else {  // AdamW and the key records of the updated theta in one pass (S6 + S0)
    RET(reset_key_counters(h, s, 0));
    const float skin = SKIN_H * h->h;
    h->launches += launch_adamw_keys(h->theta, grad, h->m, h->v, hc, h->R, h->banks, h->key_raw, h->key_cell,
                                     h->cfg.deterministic ? nullptr : h->key_rank, h->cell_count, h->key_ref,
                                     skin * skin, SKIN_MU, h->ds, s);
    CK(cudaGetLastError());
    return rebuild_keys(h, s, 0, 1);
  }
  CK(cudaGetLastError());
  return rebuild_keys(h, s);
}

// The device work of one fit step (grad zero, forward_backward, AdamW) on stream s, replayed from
// a CUDA graph once the same call repeats (graph slot `slot`: one per staging buffer).
efunc_status fit_device_step(efunc_t* h, int slot, const float* qd, const float* od, int64_t J,
                             const efunc_loss* loss, const efunc_adamw* hp, float* grad_ws, float* lossd,
                             cudaStream_t s) {
  float* g = grad_ws ? grad_ws : h->fit_grad;
  auto device_work = [&](cudaStream_t st) -> efunc_status {
    CK(cudaMemsetAsync(g, 0, sizeof(float) * (size_t)h->n_nodes * h->pnch, st));
    RET(any_forward_backward(h, qd, od, J, loss, nullptr, g, lossd, st));
    return do_adamw(h, g, hp, st);
  };
  efunc_t::FitKey key{};
  key.q = qd; key.o = od; key.g = g; key.lossd = lossd;
  key.J = J; key.J_global = loss->J_global; key.kind = loss->kind; key.eik = loss->eikonal_lambda;
  key.lr = hp->lr; key.b1 = hp->beta1; key.b2 = hp->beta2; key.eps = hp->eps; key.wd = hp->weight_decay;
  key.mask = hp->decay_mask; key.count_kept = h->count_kept;
  const bool same = h->fit_seen[slot] && std::memcmp(&key, &h->fit_key[slot], sizeof(key)) == 0;
  if (h->cfg.fit_graph && !h->cfg.sync_checks && same) {
    if (!h->fit_exec[slot]) {
      // second identical call: capture the device work once (nothing reallocates: the first,
      // eager call sized every workspace) and replay it from now on
      if (!h->cap_stream) CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
      const int64_t l0 = h->launches;
      CK(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
      const efunc_status st = device_work(h->cap_stream);
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(h->cap_stream, &graph);
      if (st != EFUNC_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      CK(ce);
      const cudaError_t ie = cudaGraphInstantiate(&h->fit_exec[slot], graph, 0);
      cudaGraphDestroy(graph);
      CK(ie);
      h->fit_launches[slot] = h->launches - l0;
      h->launches = l0;
    }
    CK(cudaGraphLaunch(h->fit_exec[slot], s));
    h->launches += h->fit_launches[slot];
  } else {
    if (h->fit_exec[slot]) cudaGraphExecDestroy(h->fit_exec[slot]);
    h->fit_exec[slot] = nullptr;
    RET(device_work(s));
    h->fit_key[slot] = key;
    h->fit_seen[slot] = 1;
  }
  return EFUNC_OK;
}

// host_io 2: store a finished step's loss (read back into pinned memory) to the caller's float
void flush_loss(efunc_t* h, int slot) {
  efunc_t::LossCopy& c = h->aio_pay[slot];
  if (c.dst) *c.dst = *c.src;
  c.dst = nullptr;
}

// host_io 2: H2D into staging slot k % 2 on the handle's copy stream (after step k-2 released
// that slot), the step on the caller's stream after the copy, the loss D2H into pinned memory;
// the host stores it to *loss_out when it next waits on that slot (call k+2 or efunc_sync). The
// host blocks only for step k-2, so the copy of step k+1 overlaps the compute of step k. (A
// cudaLaunchHostFunc callback instead serialises the copy stream with the compute: measured.)
efunc_status fit_step_async(efunc_t* h, const float* q, const float* o, int64_t J, const efunc_loss* loss,
                            const efunc_adamw* hp, float* grad_ws, float* loss_out, cudaStream_t s) {
  if (J > 0 && (!q || !o)) return fail(h, EFUNC_EINVAL, "q or o is NULL");
  if (!h->aio_stream) {
    CK(cudaStreamCreateWithFlags(&h->aio_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventCreateWithFlags(&h->aio_copied[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->aio_done[k], cudaEventDisableTiming));
      CK(dalloc(&h->aio_loss[k], 1));
    }
    CK(cudaHostAlloc((void**)&h->aio_pin, 2 * sizeof(float), cudaHostAllocDefault));
  }
  const int slot = (int)(h->aio_seq & 1);
  CK(cudaEventSynchronize(h->aio_done[slot]));  // step k-2 finished: its loss is in aio_pin
  flush_loss(h, slot);
  if (J > h->aio_cap) {
    CK(cudaEventSynchronize(h->aio_done[slot ^ 1]));
    drop_fit_graph(h);
    for (int k = 0; k < 2; ++k) {
      dfree(h->aio_q[k]);
      dfree(h->aio_o[k]);
      CK(dalloc(&h->aio_q[k], 3 * (size_t)J));
      CK(dalloc(&h->aio_o[k], (size_t)J));
    }
    h->aio_cap = J;
  }
  ++h->aio_seq;
  if (J > 0) {
    CK(cudaMemcpyAsync(h->aio_q[slot], q, sizeof(float) * 3 * (size_t)J, cudaMemcpyHostToDevice, h->aio_stream));
    CK(cudaMemcpyAsync(h->aio_o[slot], o, sizeof(float) * (size_t)J, cudaMemcpyHostToDevice, h->aio_stream));
  }
  CK(cudaEventRecord(h->aio_copied[slot], h->aio_stream));
  CK(cudaStreamWaitEvent(s, h->aio_copied[slot], 0));
  RET(fit_device_step(h, slot, h->aio_q[slot], h->aio_o[slot], J, loss, hp, grad_ws, h->aio_loss[slot], s));
  if (loss_out) {
    CK(cudaMemcpyAsync(h->aio_pin + slot, h->aio_loss[slot], sizeof(float), cudaMemcpyDeviceToHost, s));
    h->aio_pay[slot].src = h->aio_pin + slot;
    h->aio_pay[slot].dst = loss_out;
  }
  CK(cudaEventRecord(h->aio_done[slot], s));  // the host waits for it before reusing the slot
  return EFUNC_OK;
}

// batched handles (n_shapes > 1): the k-th shape's slice of a per-shape array, and error relay
template <class T>
T* off(T* p, int64_t per_shape, size_t k) {
  return p ? p + per_shape * (int64_t)k : nullptr;
}

// Batched handles: fork the shapes onto per-shape streams (after the caller's prior work) and
// join them back, so the shapes' kernels overlap (each shape is a full-GPU persistent launch
// plus small kernels; overlapping fills one shape's tail and small launches with another's).
// Capture-safe (event fork/join).
efunc_status kids_fork(efunc_t* h, cudaStream_t s) {
  if (h->kid_streams.empty()) {
    h->kid_streams.resize(h->kids.size());
    h->kid_events.resize(h->kids.size());
    for (size_t k = 0; k < h->kids.size(); ++k) {
      CK(cudaStreamCreateWithFlags(&h->kid_streams[k], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h->kid_events[k], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&h->fork_event, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(h->fork_event, s));
  for (cudaStream_t ks : h->kid_streams) CK(cudaStreamWaitEvent(ks, h->fork_event, 0));
  return EFUNC_OK;
}

efunc_status kids_join(efunc_t* h, cudaStream_t s) {
  for (size_t k = 0; k < h->kids.size(); ++k) {
    CK(cudaEventRecord(h->kid_events[k], h->kid_streams[k]));
    CK(cudaStreamWaitEvent(s, h->kid_events[k], 0));
  }
  return EFUNC_OK;
}

efunc_status kid_ok(efunc_t* h, size_t k, efunc_status st) {
  if (st != EFUNC_OK) h->err = "shape " + std::to_string(k) + ": " + h->kids[k]->err;
  return st;
}

}  // namespace

extern "C" {

int32_t efunc_abi_version(void) { return EFUNC_ABI_VERSION; }

int32_t efunc_channels(int32_t variant, int32_t degree) { return variant_channels(variant, degree, nullptr); }

efunc_status efunc_cosine_replicate(const float* q, int64_t J, int32_t B, float* qr, void* stream) {
  if (B < 1 || J < 0) return fail(nullptr, EFUNC_EINVAL, "cosine: B >= 1 and J >= 0 required");
  if (J > 0 && (!q || !qr)) return fail(nullptr, EFUNC_EINVAL, "cosine: NULL q or qr");
  if (J == 0) return EFUNC_OK;
  launch_cos_replicate(q, J, B, qr, (cudaStream_t)stream);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EFUNC_OK : fail(nullptr, EFUNC_ECUDA, cudaGetErrorString(e));
}

efunc_status efunc_cosine_combine(const float* q, int64_t J, int32_t B, const float* O, const float* G, const float* o,
                                  int64_t J_global, float* S, float* GS, float* dL_dO, float* loss, void* stream) {
  if (B < 1 || J < 0) return fail(nullptr, EFUNC_EINVAL, "cosine: B >= 1 and J >= 0 required");
  if (J > 0 && (!q || !O)) return fail(nullptr, EFUNC_EINVAL, "cosine: NULL q or O");
  if (GS && !G) return fail(nullptr, EFUNC_EINVAL, "cosine: GS needs the band gradients G");
  if ((dL_dO || loss) && !o) return fail(nullptr, EFUNC_EINVAL, "cosine: the loss needs targets o");
  if (loss && !S) return fail(nullptr, EFUNC_EINVAL, "cosine: the loss needs S");
  if (J == 0) return EFUNC_OK;
  const float inv_J = (float)(1.0 / (double)(J_global > 0 ? J_global : J));
  launch_cos_combine(q, J, B, O, G, o, inv_J, S, GS, dL_dO, loss, (cudaStream_t)stream);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EFUNC_OK : fail(nullptr, EFUNC_ECUDA, cudaGetErrorString(e));
}

const char* efunc_last_error(const efunc_t* h) {
  if (h && !h->err.empty()) return h->err.c_str();
  return g_err.c_str();
}

efunc_status efunc_create(const efunc_config* cfg, const float* theta_host, efunc_t** out) {
  efunc_t* h = nullptr;
  if (!cfg || !out) return fail(nullptr, EFUNC_EINVAL, "NULL argument");
  *out = nullptr;
  if (cfg->R < 2 || cfg->R > 256) return fail(nullptr, EFUNC_EINVAL, "R must be in [2, 256]");
  if (cfg->n_shapes < 0 || cfg->n_shapes > 4096) return fail(nullptr, EFUNC_EINVAL, "n_shapes must be in [0, 4096]");
  ef::VarLayout vlay{};
  const int pnch = variant_channels(cfg->variant, cfg->degree, &vlay);
  if (pnch < 0) return fail(nullptr, EFUNC_EINVAL, "variant must be COMBINED, GRID or OFFSET and degree 0, 1 or 2");
  if ((cfg->degree == 2 || cfg->variant == EFUNC_VARIANT_OFFSET) && cfg->deterministic)
    return fail(nullptr, EFUNC_EINVAL, "degree 2 and O^Delta-only have no deterministic mode");
  if (cfg->n_shapes > 1) {  // C5: one single-shape handle per shape behind this one
    efunc_t* p = new (std::nothrow) efunc();
    if (!p) return fail(nullptr, EFUNC_ENOMEM, "host allocation failed");
    p->cfg = *cfg;
    p->R = cfg->R;
    p->n_nodes = cfg->R * cfg->R * cfg->R;
    p->pnch = pnch;
    efunc_config c1 = *cfg;
    c1.n_shapes = 1;
    for (int k = 0; k < cfg->n_shapes; ++k) {
      efunc_t* kid = nullptr;
      const efunc_status st = efunc_create(&c1, off(theta_host, p->n_nodes * (int64_t)p->pnch, k), &kid);
      if (st != EFUNC_OK) {
        for (efunc_t* q : p->kids) efunc_destroy(q);
        delete p;
        return st;
      }
      p->kids.push_back(kid);
    }
    *out = p;
    return EFUNC_OK;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(nullptr, EFUNC_ECUDA, "no CUDA device");
  if (cfg->device < 0 || cfg->device >= ndev) return fail(nullptr, EFUNC_EINVAL, "bad device ordinal");
  h = new (std::nothrow) efunc();
  if (!h) return fail(nullptr, EFUNC_ENOMEM, "host allocation failed");
  h->cfg = *cfg;
  // NEXT-4 variants: O^Delta alone has no fixed grid keys bounding each query's exponent minimum
  // (reading R-1), so it evaluates every key (dense, cutoff_T = inf)
  if (cfg->variant == EFUNC_VARIANT_OFFSET) h->cfg.cutoff_T = INFINITY;
  h->vlay = vlay;
  h->pnch = pnch;
  h->vmode = !(cfg->variant == EFUNC_VARIANT_COMBINED && cfg->degree <= 1);
  // degree 2 and O^Delta alone run the generic kernels of k_var.cu (exact per-query shift)
  h->vk = cfg->degree == 2 || cfg->variant == EFUNC_VARIANT_OFFSET;
  h->banks = cfg->variant == EFUNC_VARIANT_GRID ? 1 : (cfg->variant == EFUNC_VARIANT_OFFSET ? 2 : 3);
  DeviceGuard dg(cfg->device);
  h->R = cfg->R;
  h->n_nodes = h->R * h->R * h->R;
  h->n_keys = 2 * h->n_nodes;
  h->NC = h->R - 1;
  h->n_cells = h->NC * h->NC * h->NC;
  h->h = 2.0f / (float)(h->R - 1);
  h->inv_h = (float)((h->R - 1) / 2.0);
  const size_t np = (size_t)h->n_nodes * EF_NCH;
  auto st = [&]() -> efunc_status {
    CK(dalloc(&h->theta, np));
    CK(dalloc(&h->m, np));
    CK(dalloc(&h->v, np));
    CK(dalloc(&h->fit_grad, (size_t)h->n_nodes * std::max(h->pnch, EF_NCH)));
    if (h->vmode) {
      const size_t nv = (size_t)h->n_nodes * h->pnch;
      CK(dalloc(&h->theta_v, nv));
      CK(dalloc(&h->m_v, nv));
      CK(dalloc(&h->v_v, nv));
      CK(cudaMemset(h->m_v, 0, nv * sizeof(float)));
      CK(cudaMemset(h->v_v, 0, nv * sizeof(float)));
      CK(dalloc(&h->gint, np));
      if (h->vk) {
        CK(dalloc(&h->thetaH, (size_t)h->n_nodes * 12));
        CK(dalloc(&h->gH, (size_t)h->n_nodes * 12));
        CK(dalloc(&h->keyH, 2 * (size_t)h->n_keys));
      }
    }
    CK(dalloc(&h->key_raw, 2 * (size_t)h->n_keys));
    CK(dalloc(&h->key_sorted, 2 * (size_t)h->n_keys));
    CK(dalloc(&h->kid, h->n_keys));
    CK(dalloc(&h->key_cell, h->n_keys));
    CK(dalloc(&h->key_tmp, h->n_keys));
    CK(dalloc(&h->key_rank, h->n_keys));
    CK(dalloc(&h->key_order, h->n_keys));
    CK(dalloc(&h->cell_count, h->n_cells + 1));
    CK(dalloc(&h->cell_start, h->n_cells + 1));
    CK(dalloc(&h->cell_fill, h->n_cells + 1));
    CK(dalloc(&h->ds, 1));
    CK(dalloc(&h->scratch, (size_t)SCRATCH_WARPS * SCRATCH_STRIDE));
    if (std::isinf(cutoff_log2(h->cfg)) || h->vk) {
      // every enabled key id: the dense fused kernel's candidate list; degree 2's list for items
      // without a certified one
      std::vector<uint32_t> ids;
      for (int i = 0; i < h->n_keys; ++i)
        if ((h->banks >> (i < h->n_nodes ? 0 : 1)) & 1) ids.push_back((uint32_t)i);
      h->iota_n = (uint32_t)ids.size();
      CK(dalloc(&h->iota, ids.size()));
      CK(cudaMemcpy(h->iota, ids.data(), ids.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    h->bg = brick_geom(h->cfg, h->NC, h->h);
    const size_t nbins = (size_t)h->bg.n_codes * h->bg.qsub + 1;
    CK(dalloc(&h->bl_off, h->bg.n_codes));
    CK(dalloc(&h->bl_n, h->bg.n_codes));
    const double pool = (double)h->n_keys * POOL_PER_KEY;
    h->bl_pool_cap = (uint32_t)std::fmin(pool, 4.0e9);
    CK(dalloc(&h->bl_pool, h->bl_pool_cap));
    CK(dalloc(&h->bin_count, nbins + 1));
    CK(dalloc(&h->bin_start, nbins + 1));
    CK(dalloc(&h->bin_fill, nbins + 1));
    // the work-item scan runs over ITEMS_N_AT(nb) + 1 slots (cost classes); qsub >= 8 makes that fit
    const size_t nitem_slots = std::max(nbins + 1, (size_t)ITEMS_N_AT((size_t)h->bg.n_codes) + 1);
    CK(dalloc(&h->item_cnt, nitem_slots));
    CK(dalloc(&h->item_off, nitem_slots));
    RET(ensure_scan_tmp(h, nbins + 1));
    CK(dalloc(&h->gpad, (size_t)h->n_nodes * 16));
    CK(cudaMemset(h->gpad, 0, sizeof(float) * (size_t)h->n_nodes * 16));
    if (h->cfg.deterministic) {
      CK(dalloc(&h->gfix, (size_t)h->n_nodes * 16));
      CK(cudaMemset(h->gfix, 0, sizeof(unsigned long long) * (size_t)h->n_nodes * 16));
    }
    CK(cudaMemset(h->ds, 0, sizeof(DevScalars)));
    RET(ensure_scan_tmp(h, h->n_cells + 1));
    RET(ensure_radix(h, (size_t)h->n_keys));
    float* pdst = h->vmode ? h->theta_v : h->theta;
    const size_t pn = (size_t)h->n_nodes * h->pnch;
    if (theta_host) CK(cudaMemcpy(pdst, theta_host, pn * sizeof(float), cudaMemcpyHostToDevice));
    else CK(cudaMemset(pdst, 0, pn * sizeof(float)));
    if (h->vmode) CK(cudaMemset(h->theta, 0, np * sizeof(float)));
    sync_internal_theta(h, 0);
    CK(cudaMemset(h->m, 0, np * sizeof(float)));
    CK(cudaMemset(h->v, 0, np * sizeof(float)));
    CK(dalloc(&h->key_ref, h->n_keys));
    CK(cudaMemset(h->key_ref, 0, sizeof(float4) * (size_t)h->n_keys));
    RET(rebuild_keys(h, 0, 1));
    CK(cudaDeviceSynchronize());
    return EFUNC_OK;
  }();
  if (st != EFUNC_OK) {
    g_err = h->err;
    free_all(h);
    delete h;
    return st;
  }
  *out = h;
  return EFUNC_OK;
}

efunc_status efunc_destroy(efunc_t* h) {
  if (h && !h->kids.empty()) {
    for (efunc_t* k : h->kids) efunc_destroy(k);
    for (cudaStream_t ks : h->kid_streams) cudaStreamDestroy(ks);
    for (cudaEvent_t e : h->kid_events) cudaEventDestroy(e);
    if (h->fork_event) cudaEventDestroy(h->fork_event);
    delete h;
    return EFUNC_OK;
  }
  if (!h) return EFUNC_OK;
  {
    DeviceGuard dg(h->cfg.device);
    cudaDeviceSynchronize();
    free_all(h);
  }
  delete h;
  return EFUNC_OK;
}

efunc_status efunc_forward(efunc_t* h, const float* q, const float* o, int64_t J, const efunc_loss* loss,
                           float* O, float* G, float* loss_out, void* stream) {
  if (h && !h->kids.empty()) {
    const size_t S = h->kids.size();
    for (size_t k = 0; k < S; ++k)
      RET(kid_ok(h, k, efunc_forward(h->kids[k], off(q, 3 * J, k), off(o, J, k), J, loss, off(O, J, k),
                                     off(G, 3 * J, k), off(loss_out, 1, k), stream)));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  DeviceGuard dg(h->cfg.device);
  return do_forward(h, q, o, J, loss, O, G, loss_out, 1, (cudaStream_t)stream);
}

efunc_status efunc_backward(efunc_t* h, const float* dL_dO, const float* dL_dG, float* grad, void* stream) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k) {
      const int64_t J = h->kids[k]->fwd_J;
      RET(kid_ok(h, k, efunc_backward(h->kids[k], off(dL_dO, J, k), off(dL_dG, 3 * J, k),
                                      off(grad, h->kids[k]->n_nodes * (int64_t)h->pnch, k), stream)));
    }
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  DeviceGuard dg(h->cfg.device);
  return any_backward(h, dL_dO, dL_dG, grad, (cudaStream_t)stream);
}

efunc_status efunc_forward_backward(efunc_t* h, const float* q, const float* o, int64_t J, const efunc_loss* loss,
                                    float* O, float* grad, float* loss_out, void* stream) {
  if (h && !h->kids.empty()) {
    DeviceGuard dg(h->cfg.device);
    RET(kids_fork(h, (cudaStream_t)stream));
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_forward_backward(h->kids[k], off(q, 3 * J, k), off(o, J, k), J, loss, off(O, J, k),
                                              off(grad, h->n_nodes * (int64_t)h->pnch, k), off(loss_out, 1, k),
                                              h->kid_streams[k])));
    return kids_join(h, (cudaStream_t)stream);
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  DeviceGuard dg(h->cfg.device);
  return any_forward_backward(h, q, o, J, loss, O, grad, loss_out, (cudaStream_t)stream);
}

efunc_status efunc_adamw_step(efunc_t* h, const float* grad, const efunc_adamw* hp, void* stream) {
  if (h && !h->kids.empty()) {
    DeviceGuard dg(h->cfg.device);
    RET(kids_fork(h, (cudaStream_t)stream));
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_adamw_step(h->kids[k], off(grad, h->n_nodes * (int64_t)h->pnch, k), hp,
                                        h->kid_streams[k])));
    return kids_join(h, (cudaStream_t)stream);
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  DeviceGuard dg(h->cfg.device);
  return do_adamw(h, grad, hp, (cudaStream_t)stream);
}

efunc_status efunc_eval_grad(efunc_t* h, const float* q, int64_t J, float* O, float* G, void* stream) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_eval_grad(h->kids[k], off(q, 3 * J, k), J, off(O, J, k), off(G, 3 * J, k), stream)));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  DeviceGuard dg(h->cfg.device);
  return do_forward(h, q, nullptr, J, nullptr, O, G, nullptr, 0, (cudaStream_t)stream);
}

// NEXT-3: lattice O (forward path in z-slabs) -> Marching Cubes (k_mesh.cu) -> vertex normals
// (one eval_grad pass). Scratch is allocated per call: the call synchronises anyway.
efunc_status efunc_mesh(efunc_t* h, int32_t N, const float* lo3, const float* hi3, float iso, float* lattice_O,
                        float* verts, float* normals, int32_t* tris, int64_t max_verts, int64_t max_tris,
                        int64_t* n_verts, int64_t* n_tris, void* stream) {
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  if (!h->kids.empty()) return fail(h, EFUNC_EINVAL, "efunc_mesh: batched handle (n_shapes > 1)");
  if (N < 2 || N > 1024) return fail(h, EFUNC_EINVAL, "efunc_mesh: N must be in [2, 1024]");
  if (!lo3 || !hi3 || !n_verts || !n_tris) return fail(h, EFUNC_EINVAL, "efunc_mesh: NULL lo/hi/count pointer");
  for (int a = 0; a < 3; ++a)
    if (!(hi3[a] > lo3[a]) || !std::isfinite(lo3[a]) || !std::isfinite(hi3[a]))
      return fail(h, EFUNC_EINVAL, "efunc_mesh: need finite hi > lo on every axis");
  if (!std::isfinite(iso)) return fail(h, EFUNC_EINVAL, "efunc_mesh: iso must be finite");
  DeviceGuard dg(h->cfg.device);
  cudaStream_t s = (cudaStream_t)stream;
  CK(mc_upload_table());
  const int64_t NN = (int64_t)N * N, N3 = NN * N;
  const float step[3] = {(hi3[0] - lo3[0]) / (float)(N - 1), (hi3[1] - lo3[1]) / (float)(N - 1),
                         (hi3[2] - lo3[2]) / (float)(N - 1)};
  float* O = lattice_O;
  float* Own = nullptr;
  float* q = nullptr;
  uint8_t* mask = nullptr;
  uint32_t *vcnt = nullptr, *voff = nullptr, *tcnt = nullptr, *toff = nullptr;
  efunc_status st = EFUNC_OK;
  auto cleanup = [&]() {
    dfree(Own); dfree(q); dfree(mask); dfree(vcnt); dfree(voff); dfree(tcnt); dfree(toff);
  };
#define MCK(x)                                                                                    \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess) {                                                                      \
      cleanup();                                                                                  \
      return fail(h, e_ == cudaErrorMemoryAllocation ? EFUNC_ENOMEM : EFUNC_ECUDA,                \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                               \
    }                                                                                             \
  } while (0)
  if (!O) {
    MCK(dalloc(&Own, (size_t)N3));
    O = Own;
  }
  // 1. node values, 2^23 lattice points per slab
  const int nk = (int)std::max<int64_t>(1, std::min<int64_t>(N, ((int64_t)1 << 23) / NN));
  MCK(dalloc(&q, (size_t)(3 * NN * nk)));
  for (int k0 = 0; k0 < N; k0 += nk) {
    const int nz = std::min(nk, N - k0);
    h->launches += launch_lattice_q(N, lo3, step, k0, nz, q, s);
    st = do_forward(h, q, nullptr, NN * nz, nullptr, O + k0 * NN, nullptr, nullptr, 0, s);
    if (st != EFUNC_OK) {
      cleanup();
      return st;
    }
  }
  // 2. Marching Cubes: per-node edge masks and vertex counts, per-cube triangle counts, scans
  MCK(dalloc(&mask, (size_t)N3));
  MCK(dalloc(&vcnt, (size_t)N3 + 1));
  MCK(dalloc(&voff, (size_t)N3 + 1));
  MCK(dalloc(&tcnt, (size_t)N3 + 1));
  MCK(dalloc(&toff, (size_t)N3 + 1));
  st = ensure_scan_tmp(h, (size_t)N3 + 1);
  if (st != EFUNC_OK) {
    cleanup();
    return st;
  }
  MCK(cudaMemsetAsync(vcnt + N3, 0, sizeof(uint32_t), s));
  MCK(cudaMemsetAsync(tcnt + N3, 0, sizeof(uint32_t), s));
  h->launches += launch_mc_count(O, N, iso, mask, vcnt, tcnt, s);
  h->launches += launch_scan_u32(vcnt, voff, (uint32_t)(N3 + 1), h->scan_tmp, s);
  h->launches += launch_scan_u32(tcnt, toff, (uint32_t)(N3 + 1), h->scan_tmp, s);
  uint32_t tot[2] = {0, 0};
  MCK(cudaMemcpyAsync(&tot[0], voff + N3, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  MCK(cudaMemcpyAsync(&tot[1], toff + N3, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  MCK(cudaStreamSynchronize(s));
  *n_verts = tot[0];
  *n_tris = tot[1];
  if (verts && tris && (int64_t)tot[0] <= max_verts && (int64_t)tot[1] <= max_tris) {
    h->launches += launch_mc_emit(O, N, iso, lo3, step, mask, voff, toff, verts, tris, s);
    // 3. normals: G at the vertices (Eq. func-normal), normalised
    if (normals && tot[0] > 0) {
      st = do_forward(h, verts, nullptr, (int64_t)tot[0], nullptr, nullptr, normals, nullptr, 0, s);
      if (st != EFUNC_OK) {
        cleanup();
        return st;
      }
      h->launches += launch_normalize3(normals, (int64_t)tot[0], s);
    }
  }
  MCK(cudaStreamSynchronize(s));
#undef MCK
  cleanup();
  return EFUNC_OK;
}

efunc_status efunc_fit_step(efunc_t* h, const float* q, const float* o, int64_t J, const efunc_loss* loss,
                            const efunc_adamw* hp, float* grad_ws, float* loss_out, int32_t host_io,
                            void* stream) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_fit_step(h->kids[k], off(q, 3 * J, k), off(o, J, k), J, loss, hp,
                                      off(grad_ws, h->n_nodes * (int64_t)h->pnch, k), off(loss_out, 1, k), host_io,
                                      stream)));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  if (!loss || loss->kind == EFUNC_LOSS_NONE) return fail(h, EFUNC_EINVAL, "fit_step needs a loss");
  if (!hp) return fail(h, EFUNC_EINVAL, "NULL AdamW parameters");
  if (host_io < 0 || host_io > 2) return fail(h, EFUNC_EINVAL, "host_io must be 0, 1 or 2");
  if (J < 0) return fail(h, EFUNC_EINVAL, "J < 0");
  DeviceGuard dg(h->cfg.device);
  cudaStream_t s = (cudaStream_t)stream;
  if (host_io == 2) return fit_step_async(h, q, o, J, loss, hp, grad_ws, loss_out, s);
  const float* qd = q;
  const float* od = o;
  float* lossd = loss_out;
  if (host_io) {
    if (J > h->io_cap || !h->io_q) {
      drop_fit_graph(h);
      dfree(h->io_q);
      dfree(h->io_o);
      CK(dalloc(&h->io_q, 3 * (size_t)J));
      CK(dalloc(&h->io_o, (size_t)J));
      h->io_cap = J;
    }
    if (!h->io_loss) CK(dalloc(&h->io_loss, 1));
    if (J > 0) {
      CK(cudaMemcpyAsync(h->io_q, q, sizeof(float) * 3 * (size_t)J, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(h->io_o, o, sizeof(float) * (size_t)J, cudaMemcpyHostToDevice, s));
    }
    qd = h->io_q;
    od = h->io_o;
    lossd = h->io_loss;
  }
  RET(fit_device_step(h, 0, qd, od, J, loss, hp, grad_ws, lossd, s));
  if (host_io) {
    if (loss_out) CK(cudaMemcpyAsync(loss_out, lossd, sizeof(float), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return EFUNC_OK;
}

efunc_status efunc_sync(efunc_t* h) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k) RET(kid_ok(h, k, efunc_sync(h->kids[k])));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  DeviceGuard dg(h->cfg.device);
  for (int k = 0; k < 2; ++k) {
    if (h->aio_done[k]) CK(cudaEventSynchronize(h->aio_done[k]));
    flush_loss(h, k);
  }
  return EFUNC_OK;
}

efunc_status efunc_mean_shift_init(efunc_t* h, const float* surf, int64_t N, float bandwidth, void* stream) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_mean_shift_init(h->kids[k], off(surf, 3 * N, k), N, bandwidth, stream)));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  if (!surf || N < 1) return fail(h, EFUNC_EINVAL, "mean shift needs N >= 1 surface points");
  if (!(bandwidth > 0.0f)) return fail(h, EFUNC_EINVAL, "bandwidth must be > 0");
  DeviceGuard dg(h->cfg.device);
  cudaStream_t s = (cudaStream_t)stream;
  if (!(h->banks & 2)) return fail(h, EFUNC_EINVAL, "mean shift initialises the offset bank; this variant has none");
  h->launches += launch_mean_shift(h->theta, h->R, surf, N, bandwidth, s);
  if (h->vmode) {  // the offsets into the user's layout, then the internal theta from it
    h->launches += launch_var_delta_out(h->theta, h->n_nodes, h->vlay, h->theta_v, s);
    sync_internal_theta(h, s);
  }
  CK(cudaGetLastError());
  return rebuild_keys(h, s, 1);
}

efunc_status efunc_get_params(efunc_t* h, float* dst, int32_t on_device, void* stream) {
  if (h && !h->kids.empty() && dst) {
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_get_params(h->kids[k], off(dst, h->n_nodes * (int64_t)h->pnch, k), on_device, stream)));
    return EFUNC_OK;
  }
  if (!h || !dst) return fail(h, EFUNC_EINVAL, "NULL argument");
  DeviceGuard dg(h->cfg.device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = sizeof(float) * (size_t)h->n_nodes * h->pnch;
  CK(cudaMemcpyAsync(dst, h->vmode ? h->theta_v : h->theta, bytes,
                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return EFUNC_OK;
}

efunc_status efunc_set_params(efunc_t* h, const float* src, int32_t on_device, void* stream) {
  if (h && !h->kids.empty() && src) {
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_set_params(h->kids[k], off(src, h->n_nodes * (int64_t)h->pnch, k), on_device, stream)));
    return EFUNC_OK;
  }
  if (!h || !src) return fail(h, EFUNC_EINVAL, "NULL argument");
  DeviceGuard dg(h->cfg.device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = sizeof(float) * (size_t)h->n_nodes * h->pnch;
  CK(cudaMemcpyAsync(h->vmode ? h->theta_v : h->theta, src, bytes,
                     on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  sync_internal_theta(h, s);
  RET(rebuild_keys(h, s, 1));
  CK(cudaStreamSynchronize(s));
  return EFUNC_OK;
}

efunc_status efunc_get_adam_state(efunc_t* h, float* m_host, float* v_host, int64_t* step) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_get_adam_state(h->kids[k], off(m_host, h->n_nodes * (int64_t)h->pnch, k),
                                            off(v_host, h->n_nodes * (int64_t)h->pnch, k), k == 0 ? step : nullptr)));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  DeviceGuard dg(h->cfg.device);
  const size_t bytes = sizeof(float) * (size_t)h->n_nodes * h->pnch;
  CK(cudaDeviceSynchronize());
  if (m_host) CK(cudaMemcpy(m_host, h->vmode ? h->m_v : h->m, bytes, cudaMemcpyDeviceToHost));
  if (v_host) CK(cudaMemcpy(v_host, h->vmode ? h->v_v : h->v, bytes, cudaMemcpyDeviceToHost));
  if (step) {
    unsigned long long t = 0;
    CK(cudaMemcpy(&t, &h->ds->adam_t, sizeof(t), cudaMemcpyDeviceToHost));
    *step = (int64_t)t;
  }
  return EFUNC_OK;
}

efunc_status efunc_set_adam_state(efunc_t* h, const float* m_host, const float* v_host, int64_t step) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k)
      RET(kid_ok(h, k, efunc_set_adam_state(h->kids[k], off(m_host, h->n_nodes * (int64_t)h->pnch, k),
                                            off(v_host, h->n_nodes * (int64_t)h->pnch, k), step)));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  if (step < 0) return fail(h, EFUNC_EINVAL, "step < 0");
  DeviceGuard dg(h->cfg.device);
  const size_t bytes = sizeof(float) * (size_t)h->n_nodes * h->pnch;
  float* mm = h->vmode ? h->m_v : h->m;
  float* vv = h->vmode ? h->v_v : h->v;
  CK(cudaDeviceSynchronize());
  if (m_host) CK(cudaMemcpy(mm, m_host, bytes, cudaMemcpyHostToDevice));
  else CK(cudaMemset(mm, 0, bytes));
  if (v_host) CK(cudaMemcpy(vv, v_host, bytes, cudaMemcpyHostToDevice));
  else CK(cudaMemset(vv, 0, bytes));
  const unsigned long long t = (unsigned long long)step;
  CK(cudaMemcpy(&h->ds->adam_t, &t, sizeof(t), cudaMemcpyHostToDevice));
  return EFUNC_OK;
}

efunc_status efunc_set_counting(efunc_t* h, int32_t on) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k) RET(kid_ok(h, k, efunc_set_counting(h->kids[k], on)));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  h->count_kept = on ? 1 : 0;
  return EFUNC_OK;
}

efunc_status efunc_set_grad_peers(efunc_t* h, void* const* peers, int32_t n_peers, void* mc) {
  if (h && !h->kids.empty()) return fail(h, EFUNC_EINVAL, "batched handles (n_shapes > 1) are replicas: no reduction");
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  if (n_peers < 0 || n_peers > 1024 || (n_peers > 0 && !peers)) return fail(h, EFUNC_EINVAL, "bad peer list");
  if ((n_peers > 0 || mc) && h->cfg.deterministic)
    return fail(h, EFUNC_EINVAL, "the fused peer reduction is the float path (not deterministic mode)");
  if ((n_peers > 0 || mc) && h->vmode) return fail(h, EFUNC_EINVAL, "the 13-channel layout only");
  if (((int64_t)h->n_nodes * EF_NCH) % 4) return fail(h, EFUNC_EINVAL, "n_params must be a multiple of 4");
  DeviceGuard dg(h->cfg.device);
  CK(cudaDeviceSynchronize());
  drop_fit_graph(h);
  dfree(h->peer_grad);
  h->n_peers = 0;
  h->mc_grad = static_cast<float*>(mc);
  if (n_peers > 0) {
    CK(dalloc(&h->peer_grad, (size_t)n_peers));
    CK(cudaMemcpy(h->peer_grad, peers, sizeof(float*) * (size_t)n_peers, cudaMemcpyHostToDevice));
    h->n_peers = n_peers;
  }
  return EFUNC_OK;
}

efunc_status efunc_set_timing(efunc_t* h, int32_t slots) {
  if (h && !h->kids.empty()) {
    for (size_t k = 0; k < h->kids.size(); ++k) RET(kid_ok(h, k, efunc_set_timing(h->kids[k], slots)));
    return EFUNC_OK;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  if (slots < 0 || slots > 4096) return fail(h, EFUNC_EINVAL, "slots must be in [0, 4096]");
  DeviceGuard dg(h->cfg.device);
  CK(cudaDeviceSynchronize());
  drop_fit_graph(h);  // a captured fit step records into the events about to be destroyed
  free_timing(h);
  for (int i = 0; i < 2 * slots; ++i) {
    cudaEvent_t e = nullptr;
    CK(cudaEventCreate(&e));
    h->tev.push_back(e);
  }
  h->tev_used.assign(slots, 0);
  return EFUNC_OK;
}

efunc_status efunc_get_kernel_ms(efunc_t* h, float* ms_host, int32_t n) {
  if (h && !h->kids.empty() && ms_host && n > 0) {  // per slot: the sum over shapes
    std::vector<float> t(n);
    for (int i = 0; i < n; ++i) ms_host[i] = 0.0f;
    for (size_t k = 0; k < h->kids.size(); ++k) {
      RET(kid_ok(h, k, efunc_get_kernel_ms(h->kids[k], t.data(), n)));
      for (int i = 0; i < n; ++i) ms_host[i] += t[i];
    }
    return EFUNC_OK;
  }
  if (!h || !ms_host) return fail(h, EFUNC_EINVAL, "NULL argument");
  DeviceGuard dg(h->cfg.device);
  const int slots = (int)(h->tev.size() / 2);
  for (int i = 0; i < n; ++i) {
    ms_host[i] = NAN;
    if (i >= slots || !h->tev_used[i]) continue;
    CK(cudaEventSynchronize(h->tev[2 * i + 1]));
    float ms = NAN;
    if (cudaEventElapsedTime(&ms, h->tev[2 * i], h->tev[2 * i + 1]) == cudaSuccess) ms_host[i] = ms;
  }
  return EFUNC_OK;
}

efunc_status efunc_get_stats(efunc_t* h, efunc_stats* out, void* stream) {
  if (h && !h->kids.empty() && out) {  // counters summed over shapes, beta_min the minimum
    efunc_stats acc{};
    acc.beta_min = INFINITY;
    for (size_t k = 0; k < h->kids.size(); ++k) {
      efunc_stats t{};
      RET(kid_ok(h, k, efunc_get_stats(h->kids[k], &t, stream)));
      acc.J += t.J; acc.items += t.items; acc.candidate_pairs += t.candidate_pairs; acc.kept_pairs += t.kept_pairs;
      acc.beta_min = fminf(acc.beta_min, t.beta_min); acc.nonfinite |= t.nonfinite;
      acc.overflow_items += t.overflow_items; acc.kept_pairs_offset += t.kept_pairs_offset;
      acc.launches += t.launches; acc.list_builds += t.list_builds; acc.list_entries += t.list_entries;
      acc.list_overflow += t.list_overflow;
    }
    *out = acc;
    return EFUNC_OK;
  }
  if (!h || !out) return fail(h, EFUNC_EINVAL, "NULL argument");
  DeviceGuard dg(h->cfg.device);
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  DevScalars d;
  CK(cudaMemcpy(&d, h->ds, sizeof(d), cudaMemcpyDeviceToHost));
  out->J = h->fwd_J;
  uint32_t ni = 0;
  if (h->fwd_J > 0) CK(cudaMemcpy(&ni, h->item_off + ITEMS_N_AT(h->bg.n_codes), sizeof(ni), cudaMemcpyDeviceToHost));
  out->items = ni;
  out->candidate_pairs = (double)d.cand_pairs;
  out->kept_pairs = (double)d.kept_pairs;
  out->beta_min = d.bl_min / EF_LOG2E;
  out->nonfinite = (int32_t)d.nonfinite;
  out->overflow_items = (int32_t)d.overflow_items;
  out->kept_pairs_offset = (double)d.kept_pairs_offset;
  out->launches = h->launches;
  out->list_builds = d.list_builds;
  out->list_entries = d.pool_used;
  out->list_overflow = d.ovf_last;
  return EFUNC_OK;
}

efunc_status efunc_check(efunc_t* h, void* stream) {
  if (h && !h->kids.empty()) {
    efunc_status first = EFUNC_OK;
    for (size_t k = 0; k < h->kids.size(); ++k) {
      const efunc_status st = kid_ok(h, k, efunc_check(h->kids[k], stream));
      if (st != EFUNC_OK && first == EFUNC_OK) first = st;
    }
    return first;
  }
  if (!h) return fail(nullptr, EFUNC_EINVAL, "NULL handle");
  DeviceGuard dg(h->cfg.device);
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  uint32_t nf = 0, fo = 0;
  CK(cudaMemcpy(&nf, &h->ds->nonfinite, sizeof(nf), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&fo, &h->ds->fix_overflow, sizeof(fo), cudaMemcpyDeviceToHost));
  if (nf) {
    CK(cudaMemset(&h->ds->nonfinite, 0, sizeof(uint32_t)));
    return fail(h, EFUNC_ENONFINITE, "non-finite query or target");
  }
  if (fo) {
    CK(cudaMemset(&h->ds->fix_overflow, 0, sizeof(uint32_t)));
    return fail(h, EFUNC_ENONFINITE, "deterministic backward: a partial exceeded the fixed-point range");
  }
  return EFUNC_OK;
}

}  // extern "C"
