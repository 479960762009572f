/*
 * efunc.h — C ABI of libefunc: the B200 (sm_100a) fit-step hot path of
 * "efunc: An Efficient Function Representation without Neural Networks"
 * (arXiv 2505.21319). Citations are PAPER.md:L<line> into the paper text.
 *
 * What the library computes
 *   The O^{+Delta} representation (Eq. func-offset): one softmax
 *   over the union of a fixed lattice key bank and an offset key bank, each key
 *   carrying a degree-1 polynomial value f(x) = c + g.x (Eq. poly-func,
 *   Eq. func-interp), scale beta = exp(s) (PAPER.md:L908 init e^7).
 *   Forward = Alg. 1 (L505-518) plus the query gradient Eq. func-normal (L425-436);
 *   backward = Alg. 2 and the parameter-gradient equations (L540-601); loss = MSE
 *   (Eq. loss) optionally plus an Eikonal term (reading R-12);
 *   optimizer = AdamW (L698).
 *   The global softmax sum is evaluated with a certified cutoff: a (query j, key i)
 *   pair is skipped only if beta_i ||q_j - k_i||^2 - m_j > cutoff_T, where m_j is
 *   the smallest exponent of query j (reading R-1). cutoff_T = INFINITY
 *   (or <= 0) evaluates every pair (the paper's dense definition).
 *
 * Beyond the default model the library covers the other Table 3 families (efunc_variant and
 * degree 0/1/2, parameter layouts by efunc_channels), cosine-series stacks (efunc_cosine_*),
 * and inference to a mesh (efunc_mesh: lattice O, Marching Cubes, vertex normals).
 *
 * Parameter layout (theta, gradients, AdamW moments) of the default model: float32 [R^3][13],
 *   node n = x + R*(y + R*z), lattice k_n = float32(-1 + 2*x/(R-1), ...) on [-1,1]^3,
 *   channels (Table 3 row Full-4):
 *     0 s0 | 1 c0 | 2..4 g0 | 5..7 Delta | 8 s1 | 9 c1 | 10..12 g1
 *   grid bank key n  : position k_n,           beta = exp(s0), f = c0 + g0.(q - k_n)
 *   offset bank key n: position k_n + Delta_n, beta = exp(s1), f = c1 + g1.(q - k_n - Delta_n)
 *   This is also the payload order of the SPEC .efg file (key-major, channel-minor).
 *
 * Conventions for every call
 *   - Pointers named "dev" are device pointers on the handle's device, float32,
 *     contiguous; the caller owns them. Pointers named "host" are host memory.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream). All device work
 *     of a call is enqueued on it; calls return without synchronising unless the
 *     description says otherwise. forward/backward/adamw_step are CUDA-graph
 *     capturable (no allocation, no host sync) once the handle has seen a J at
 *     least as large (workspaces grow on the first call with a larger J).
 *   - Every call returns an efunc_status; on failure efunc_last_error() holds a
 *     message. Nothing is thrown across the ABI. A handle is not thread-safe.
 */
#ifndef EFUNC_H
#define EFUNC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EFUNC_NCH 13
#define EFUNC_ABI_VERSION 1

#if defined(__GNUC__)
#define EFUNC_API __attribute__((visibility("default")))
#else
#define EFUNC_API
#endif

typedef struct efunc efunc_t; /* opaque handle: one per (device, grid) */

typedef enum {
  EFUNC_OK = 0,
  EFUNC_EINVAL = 1,      /* bad argument: R < 2, J < 0, NULL pointer, unsupported option */
  EFUNC_ESTATE = 2,      /* backward without a matching forward (SPEC "missing e_j") */
  EFUNC_ENONFINITE = 3,  /* a NaN/Inf query or target was seen (SPEC "NaN query") */
  EFUNC_ECUDA = 4,       /* CUDA runtime error */
  EFUNC_ENOMEM = 5       /* device allocation failed */
} efunc_status;

/* Model families of Table 3:
 *   COMBINED  O^{+Delta} (Eq. func-offset): fixed grid keys + learnable
 *             offset keys k_n + Delta_n, one softmax over both banks (Table 3 Full-3/4);
 *   GRID      O (Eq. func-interp) over the fixed grid keys (Table 3 G-5..G-8);
 *   OFFSET    O^Delta (Eq. func-with-offset): learnable keys only (Full-1/2).
 *             Without fixed keys the per-query exponent minimum has no lattice bound, so this
 *             variant always evaluates every key (cutoff_T is forced to infinity, reading R-1).
 * Parameter layout per node (efunc_channels gives the count): COMBINED with degree 0/1 is the
 * 13-channel layout below; every other (variant, degree) uses, bank by bank (grid first),
 *   grid bank   [s, c, g(3) if degree >= 1, H(6) if degree == 2]
 *   offset bank [Delta(3), s, c, g(3) if degree >= 1, H(6) if degree == 2]
 * with beta = exp(s), f(x) = c + g.x + 1/2 x^T H x, x = q - key (Eq. poly-func),
 * H symmetric stored as (Hxx, Hyy, Hzz, Hxy, Hxz, Hyz): G-7 = GRID/2 = 11 channels, Full-1 =
 * OFFSET/1 = 8, G-6 = GRID/1 = 5, COMBINED/2 = 25. */
typedef enum { EFUNC_VARIANT_COMBINED = 0, EFUNC_VARIANT_GRID = 1, EFUNC_VARIANT_OFFSET = 2 } efunc_variant;

typedef struct {
  int32_t R;              /* lattice resolution per axis, 2 <= R <= 256 */
  int32_t degree;         /* polynomial degree of f: 1 (f = c + g.(q-k)), 2 (+ 1/2 (q-k)^T H (q-k)) or
                             0 (f = c). COMBINED/0 keeps the 13-channel layout (Table 3 G-0): the g
                             channels 2-4, 10-12 are held at 0 and AdamW skips them (their gradient
                             entries are the degree-1 ones at g = 0). Degree 2 supports the MSE loss
                             (no Eikonal terms) and no deterministic mode. */
  int32_t variant;        /* efunc_variant */
  float cutoff_T;         /* certified cutoff in nats (20.0f default); <=0 or inf: dense */
  int32_t deterministic;  /* 1: gradients bitwise reproducible run to run (no float atomics) */
  int32_t device;         /* CUDA device ordinal */
  int32_t sync_checks;    /* 1: forward synchronises and returns EFUNC_ENONFINITE at once */
  int32_t fit_graph;      /* 1: efunc_fit_step replays a CUDA graph of its device work, captured on
                             the second call with the same J, pointers, loss and hyper-parameters
                             (any workspace reallocation drops it); 0: plain launches */
  int32_t n_shapes;       /* 0 or 1: one grid. S > 1: S independent grids ("shapes", BASELINE config
                             C5) in one handle; every per-shape array gains a leading [S] axis
                             (theta/grad/m/v [S][R^3][13], q [S][J][3], o/O [S][J], G [S][J][3],
                             loss_out [S], surf [S][N][3]) and J, N are per shape. */
  int32_t reserved[3];    /* must be 0 */
} efunc_config;

typedef enum { EFUNC_LOSS_NONE = 0, EFUNC_LOSS_MSE = 1, EFUNC_LOSS_MSE_EIKONAL = 2 } efunc_loss_kind;

typedef struct {
  int32_t kind;           /* efunc_loss_kind */
  float eikonal_lambda;   /* lambda_E of L_E = lambda_E/J sum (||G_j|| - 1)^2 (reading R-12) */
  int64_t J_global;       /* J in the 1/J of Eq. loss; 0 = this call's J. Data-parallel ranks
                             pass the global batch size so the all-reduced gradient is exact. */
} efunc_loss;

typedef struct {
  double lr, beta1, beta2, eps, weight_decay; /* PAPER.md:L698 lr=6e-4; rest reading R-10 */
  uint32_t decay_mask;    /* bit c set = channel c is weight-decayed (default: c,g channels) */
} efunc_adamw;

typedef struct {
  int64_t J;                 /* queries in the last forward */
  int64_t items;             /* work items (fixed-size runs of the Morton-sorted queries) */
  double candidate_pairs;    /* (query, key) pairs evaluated by the last forward */
  double kept_pairs;         /* pairs with a - m <= cutoff_T (only if counting enabled) */
  float beta_min;            /* smallest beta over both banks (drives the search radius) */
  int32_t nonfinite;         /* 1 if a non-finite query/target was seen since the last check */
  int32_t overflow_items;    /* items that took the exact-shift slow path */
  double kept_pairs_offset;  /* kept pairs whose key is in the offset bank (counting mode) */
  int64_t launches;          /* kernels launched by this handle since creation */
  int64_t list_builds;       /* brick candidate-list builds since creation (Verlet skin) */
  int64_t list_entries;      /* entries of the current brick lists */
  int64_t list_overflow;     /* bricks whose list overflowed (their items enumerate directly) */
} efunc_stats;

/* efunc_create — allocate a handle on cfg->device and upload theta.
 *   theta_host: host float[R^3*13] in the layout above (NULL = all zeros); [n_shapes][R^3*13]
 *               for a batched handle.
 *   Returns EFUNC_EINVAL for R outside [2,256], an unsupported (variant, degree), or degree 2 with
 *   deterministic mode. theta_host is [R^3][efunc_channels(variant, degree)]. */
EFUNC_API efunc_status efunc_create(const efunc_config* cfg, const float* theta_host, efunc_t** out);
EFUNC_API efunc_status efunc_destroy(efunc_t* h);

/* efunc_forward — Alg. 1 for J queries, plus Eq. func-normal if G != NULL.
 *   q   dev float[J*3] query positions (any order, any location; out-of-domain allowed)
 *   o   dev float[J]   targets (required if loss->kind != NONE, else may be NULL)
 *   loss NULL or EFUNC_LOSS_NONE: no loss; MSE: Eq. loss; MSE_EIKONAL: + reading R-12
 *        (MSE_EIKONAL requires G != NULL).
 *   O   dev float[J]   output values O(q_j)          (may be NULL)
 *   G   dev float[J*3] output dO/dq_j                (may be NULL)
 *   loss_out dev float[1]: the loss of this call's queries (1/J_global scaled), or NULL.
 * Saves the per-query state (log e_j, O_j, dL/dO_j, ...) that efunc_backward consumes;
 * it is invalidated by the next forward, set_params, adamw_step or mean_shift_init.
 * A NaN/Inf query sets the non-finite flag (efunc_check); with cfg.sync_checks the call
 * synchronises and returns EFUNC_ENONFINITE. J == 0 is valid (loss_out = 0). */
EFUNC_API efunc_status efunc_forward(efunc_t* h, const float* q, const float* o, int64_t J,
                           const efunc_loss* loss, float* O, float* G, float* loss_out,
                           void* stream);

/* efunc_backward — Alg. 2 + PAPER.md:L569-598: grad += dL/dtheta over the last forward's queries.
 *   dL_dO dev float[J] upstream dL/dO_j, or NULL to use the forward's fused loss upstream
 *   dL_dG dev float[J*3] upstream dL/dG_j or NULL (non-NULL requires the forward to have
 *         computed G); with a fused MSE_EIKONAL loss and dL_dO == NULL the Eikonal
 *         upstream is used automatically.
 *   grad  dev float[R^3*13], accumulated into (+=); zero it first for a fresh gradient.
 * Returns EFUNC_ESTATE if there is no valid saved forward state. */
EFUNC_API efunc_status efunc_backward(efunc_t* h, const float* dL_dO, const float* dL_dG, float* grad,
                            void* stream);

/* efunc_forward_backward — efunc_forward followed by efunc_backward(dL_dO = NULL, dL_dG = NULL):
 * the fit step's forward, fused loss upstream and backward (Alg. 1 + Eq. loss + Alg. 2,
 * PAPER.md:L486-490, L505-568) in one call.
 *   q, o  dev float[J*3], float[J]; loss must be MSE or MSE_EIKONAL (NULL/NONE: EFUNC_EINVAL)
 *   O     dev float[J] output values or NULL
 *   grad  dev float[R^3*13], accumulated into (+=)
 *   loss_out dev float[1] or NULL
 * Outside deterministic mode (and with counting off) it runs one fused kernel per work item:
 * k_fit for MSE, k_fit_eik for MSE_EIKONAL (the MSE and Eikonal upstreams of a query depend on
 * that query alone, so each item's forward and backward share one candidate-key pass). Otherwise
 * it is exactly forward + backward. Leaves no saved forward state (a following efunc_backward
 * returns EFUNC_ESTATE). */
EFUNC_API efunc_status efunc_forward_backward(efunc_t* h, const float* q, const float* o, int64_t J,
                                    const efunc_loss* loss, float* O, float* grad, float* loss_out,
                                    void* stream);

/* efunc_adamw_step — one AdamW update of theta with torch.optim.AdamW semantics
 * (decoupled decay first, bias-corrected moments; reading R-10). grad: dev float[R^3*13],
 * already summed over data-parallel ranks. Increments the handle's step counter, then
 * rebuilds the key records and the cell binning for the next forward. */
EFUNC_API efunc_status efunc_adamw_step(efunc_t* h, const float* grad, const efunc_adamw* hp, void* stream);

/* efunc_eval_grad — O and dO/dq for J queries (normals / inference).
 * O, G dev (either may be NULL). Invalidates the saved forward state. */
EFUNC_API efunc_status efunc_eval_grad(efunc_t* h, const float* q, int64_t J, float* O, float* G,
                             void* stream);

/* efunc_fit_step — forward + loss + backward + AdamW in one call on one device.
 *   host_io == 1: q, o are HOST buffers (pinned for async copies), loss_out is a host float*;
 *                 the call copies q/o in on `stream`, reads the loss back and synchronises.
 *   host_io == 2: pipelined host I/O: q, o pinned HOST buffers, loss_out a host float*. The
 *                 call copies q/o into one of two device staging slots on the handle's copy
 *                 stream, runs the step on `stream` after the copy, reads the loss back into
 *                 pinned memory, and returns without waiting (it blocks only until the step
 *                 two calls back is done, then stores that step's loss to its *loss_out).
 *                 So the copy of step k+1 overlaps the compute of step k. q, o and *loss_out
 *                 must stay valid until efunc_sync() (or two calls later).
 *   host_io == 0: all pointers are device pointers; no synchronisation.
 * grad_ws: dev float[R^3*13] scratch for the gradient (zeroed by the call). */
EFUNC_API efunc_status efunc_fit_step(efunc_t* h, const float* q, const float* o, int64_t J,
                            const efunc_loss* loss, const efunc_adamw* hp, float* grad_ws,
                            float* loss_out, int32_t host_io, void* stream);

/* efunc_sync — waits for every step issued with host_io == 2 (their losses are then stored). */
EFUNC_API efunc_status efunc_sync(efunc_t* h);

/* efunc_mean_shift_init — Delta_n = sum_s e^{-bw||k_n - s||^2} s / sum_s e^{-bw||k_n-s||^2} - k_n
 * (bw = 100, N = 16384 in the paper) written into channels 5..7.
 *   surf dev float[N*3] surface points, N >= 1. */
EFUNC_API efunc_status efunc_mean_shift_init(efunc_t* h, const float* surf, int64_t N, float bandwidth,
                                   void* stream);

/* efunc_mesh — inference to a mesh. PAPER.md:L680 (§4.1): "we first
 * evaluate O(q) at 512-resolution grid points. Then, we use Marching Cubes on the resulting
 * grid"; PAPER.md:L962-971 (§4.5): the normals come from "a single forward pass" of
 * Eq. func-normal (L425-436).
 *   1. O at the N^3 lattice nodes p(i,j,k) = lo + (hi - lo) * (i,j,k) / (N-1), node
 *      n = i + N (j + N k), evaluated through the forward path in z-slabs;
 *   2. Marching Cubes at `iso`: one vertex per lattice edge whose end nodes lie on different
 *      sides (O < iso is inside), at the linear interpolation of O along the edge, shared by
 *      the cubes around that edge (indexed, closed mesh away from the lattice boundary);
 *      triangles are wound so their right-hand normal points from O < iso to O > iso;
 *   3. normals[v] = G/|G| at every vertex (one eval_grad pass; 0 where G = 0).
 *   N in [2, 1024]; lo3, hi3 host float[3] with hi3 > lo3 per axis.
 *   lattice_O: dev float[N^3] or NULL (receives the node values).
 *   verts, normals: dev float[max_verts*3]; tris: dev int32[max_tris*3] (vertex indices).
 *   n_verts, n_tris: host int64 outputs, required.
 * If verts/tris are NULL or too small, only the counts (and lattice_O) are produced and the
 * call returns EFUNC_OK: allocate and call again. normals may be NULL (skipped).
 * Synchronises `stream`; invalidates the saved forward state; not for batched handles.
 * Errors: EINVAL (N, box, NULL counts, n_shapes > 1), ENOMEM, ECUDA. */
EFUNC_API efunc_status efunc_mesh(efunc_t* h, int32_t N, const float* lo3, const float* hi3, float iso,
                                  float* lattice_O, float* verts, float* normals, int32_t* tris,
                                  int64_t max_verts, int64_t max_tris, int64_t* n_verts, int64_t* n_tris,
                                  void* stream);

/* Cosine-series stacks (§4.4, Eq. cosine-series):
 *   S(q) = sum_{b=0}^{B-1} w_b(q) O_b(q),  w_b(q) = cos(b pi x) cos(b pi y) cos(b pi z)
 * (reading R-C: the 3-D cosine of "cos(b pi q)" is the separable product; B terms, so B = 1 is
 * Table 3 Config G-6). The bands O_b are an n_shapes = B handle (variant GRID,
 * degree 1) evaluated on the same queries:
 *   efunc_cosine_replicate: qr[b][j][:] = q[j][:] (dev float[B*J*3]) for that handle;
 *   efunc_cosine_combine: from the band values O dev [B][J] (and G dev [B][J][3] or NULL) the
 *     stack value S dev [J], its gradient GS dev [J][3] (needs G) = sum_b (dw_b O_b + w_b G_b), and
 *     with targets o dev [J]: the MSE loss of S (loss dev [1], needs S) and the band upstreams
 *     dL_dO dev [B][J] = w_b(q_j) 2 (S_j - o_j) / J_global for efunc_backward (chain rule).
 *   q dev [J*3]. J_global <= 0 means J. Any output may be NULL. Stream-ordered; no handle.
 *   Errors: EINVAL (B < 1, J < 0, NULL q/O, GS without G, dL_dO/loss without o, loss without S). */
EFUNC_API efunc_status efunc_cosine_replicate(const float* q, int64_t J, int32_t B, float* qr, void* stream);
EFUNC_API efunc_status efunc_cosine_combine(const float* q, int64_t J, int32_t B, const float* O, const float* G,
                                            const float* o, int64_t J_global, float* S, float* GS, float* dL_dO,
                                            float* loss, void* stream);

/* Parameter / optimizer-state access. on_device=1: ptr is a device pointer, else host.
 * These synchronise the stream. set_params rebuilds keys and clears the saved state. */
EFUNC_API efunc_status efunc_get_params(efunc_t* h, float* dst, int32_t on_device, void* stream);
EFUNC_API efunc_status efunc_set_params(efunc_t* h, const float* src, int32_t on_device, void* stream);
EFUNC_API efunc_status efunc_get_adam_state(efunc_t* h, float* m_host, float* v_host, int64_t* step);
EFUNC_API efunc_status efunc_set_adam_state(efunc_t* h, const float* m_host, const float* v_host,
                                  int64_t step);

/* efunc_set_counting — 1: the forward also counts kept pairs (a - m <= T) for
 * efunc_get_stats (slower; diagnostics only). */
EFUNC_API efunc_status efunc_set_counting(efunc_t* h, int32_t on);
/* efunc_set_grad_peers — data-parallel gradient reduction fused into the gradient fold (SURVEY
 * §8(e); the loss is a batch mean, so the full-batch gradient is the sum of the
 * ranks' shard gradients). peers[0..n_peers) are device pointers, valid on this handle's device,
 * to every rank's copy of one symmetric gradient buffer of n_params floats (this rank's own copy
 * included: e.g. torch symmetric memory's buffer_ptrs over NVLink/NVSwitch peer mappings); mc is
 * its NVLS multicast address or NULL. When set, efunc_forward_backward / efunc_backward add their
 * gradient into every rank's copy (multimem.red.add.v4.f32 through mc if given, else one
 * red.global.add.v4.f32 per peer) instead of into `grad`; the caller zeroes its own copy and
 * synchronises the ranks before the call, and synchronises them again before reading the sum (its
 * own copy). n_params must be a multiple of 4 (R^3 x 13 channels with R even; checked). n_peers = 0
 * and mc = NULL restore the local fold. The float path only (EFUNC_EINVAL in deterministic mode).
 * Host pointer array, copied. */
EFUNC_API efunc_status efunc_set_grad_peers(efunc_t* h, void* const* peers, int32_t n_peers, void* mc);
/* efunc_set_timing — slots > 0: every efunc_backward / efunc_forward_backward call records a
 * CUDA event pair around its dominant kernel (k_backward, or k_fit when fused) on the call's
 * stream, into slot (call index mod slots); the records also work inside CUDA-graph capture
 * (external event nodes). slots = 0 turns timing off. efunc_get_kernel_ms synchronises and
 * writes the elapsed milliseconds of slots 0..n-1 (NaN for a slot never recorded). */
EFUNC_API efunc_status efunc_set_timing(efunc_t* h, int32_t slots);
EFUNC_API efunc_status efunc_get_kernel_ms(efunc_t* h, float* ms_host, int32_t n);
/* efunc_get_stats — synchronises `stream` and reports counters of the last forward. */
EFUNC_API efunc_status efunc_get_stats(efunc_t* h, efunc_stats* out, void* stream);
/* efunc_check — synchronises; EFUNC_ENONFINITE if a non-finite input was seen since the
 * last check (and clears the flag), else EFUNC_OK. */
EFUNC_API efunc_status efunc_check(efunc_t* h, void* stream);

EFUNC_API const char* efunc_last_error(const efunc_t* h); /* never NULL; h may be NULL */
EFUNC_API int32_t efunc_abi_version(void);
/* efunc_channels — parameter channels per node of a (variant, degree) (Table 3 "Ch"), or -1 if
 * the pair is not supported. Every theta/grad/m/v array of a handle is [R^3][channels]. */
EFUNC_API int32_t efunc_channels(int32_t variant, int32_t degree);

#ifdef __cplusplus
}
#endif
#endif /* EFUNC_H */
