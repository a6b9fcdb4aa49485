/* xmgn.h -- C-ABI of the B200-native X-MeshGraphNet processor hot path.
 *
 * Method: X-MeshGraphNet (arXiv 2411.17164).  The processor is L message-passing
 * layers (Sec. II-C, Eq. 4) run over halo-padded partitions of
 * a merged multi-scale kNN graph (Sec. III-A, 187-194 Sec. III-C).
 * Layer l, read per BASELINE.json north_star and SURVEY.md §8(c):
 *     e'_k = e_k + LN_e(MLP_e([e_k | h_src(k) | h_dst(k)]))        (Eq. 1)
 *     a_i  = sum_{k : dst(k) = i} e'_k      (CSR order)              (Eq. 2)
 *     h'_i = h_i + LN_n(MLP_n([h_i | a_i]))                          (Eq. 3)
 * MLP = Linear -> SiLU -> (Linear -> SiLU)^(m-1) -> Linear (SiLU per PAPER.md:234),
 * LN = per-row LayerNorm with affine gamma/beta, eps = cfg.ln_eps, biased variance.
 * Loss seam: the caller supplies dL/dh^L for OWNED rows only; halo rows are
 * dropped from the loss.  Parameter gradients of all partitions
 * are summed -- plain sum, not a mean.
 *
 * Conventions
 *  - Every call returns xmgn_status; on failure xmgn_last_error() returns a
 *    thread-local, library-owned message naming the call, array and index
 *    (valid until the next call on that thread).
 *  - Host arrays in descriptors are caller-owned and only read during the call.
 *  - Device pointers (params, features, gradients) are caller-owned CUDA
 *    allocations on the graph's device; fwd/bwd/reduce enqueue on `stream`
 *    (a cudaStream_t, NULL = legacy default stream) and return immediately;
 *    device faults surface at the next synchronising call.
 *  - One host thread per workspace at a time.
 *  - Local row order of a partition is ring-major: ring 0 (owned, ascending
 *    global id), then halo ring 1..depth (ascending global id inside a ring).
 *    Owned rows are therefore the prefix [0, n_owned).  Local in-edges of a row
 *    keep the global CSR order.  (SURVEY §2.2 D5.)
 *  - Parameters: one flat FP32 vector, per layer l = 0..L-1
 *      edge block: W1[3H,H] (row blocks e, h_src, h_dst), b1[H],
 *                  W_j[H,H], b_j[H] for j = 2..m+1, gamma[H], beta[H]
 *      node block: W1[2H,H] (row blocks h, agg), b1[H], W_j, b_j, gamma, beta
 *    with y = x W + b, W stored [in, out] row-major.
 *    Count = L*((5+2m)H^2 + (2m+6)H).
 */
#ifndef XMGN_H
#define XMGN_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  XMGN_OK = 0,
  XMGN_EINVAL = 1,     /* malformed argument / graph (message names array + index)      */
  XMGN_EHALO = 2,      /* halo_depth < layers, or an owned node's L-hop ball not local   */
  XMGN_ESTATE = 3,     /* call out of order (bwd without matching fwd, ...)               */
  XMGN_ENOMEM = 4,     /* device or host allocation failed                                 */
  XMGN_ECUDA = 5,      /* CUDA runtime error (message carries the runtime string)          */
  XMGN_ENCCL = 6,      /* NCCL error                                                       */
  XMGN_ENONFINITE = 7, /* non-finite value detected by xmgn_check_finite      */
  XMGN_EUNSUPPORTED = 8 /* configuration the kernels are not built for (e.g. H)           */
} xmgn_status;

const char* xmgn_last_error(void);
const char* xmgn_version(void);

/* ------------------------------------------------------------------ graph
 * Global graph in CSR by destination: row i lists the
 * sources j of edges (j -> i), strictly ascending; no self-loops, no duplicates;
 * the graph must be symmetric ((j->i) present iff (i->j) present).
 * owned: n_parts disjoint ascending lists covering [0, n_nodes).
 * halo:  per partition the nodes at undirected hop distance 1..halo_depth from
 *        its owned set, ordered by (ring, id), with their ring in halo_ring.
 * Validation: EINVAL for any malformed array; EHALO if halo_depth is smaller
 * than the layer count later used, or if the halo lists are not exactly the BFS
 * rings (checked by an independent BFS).  All arrays are copied; the device
 * copies are owned by the returned handle.                                      */
typedef struct {
  int64_t n_nodes, n_edges;
  const int64_t* csr_offsets;   /* [n_nodes+1]                               */
  const int64_t* csr_sources;   /* [n_edges]                                 */
  int32_t n_parts, halo_depth;
  const int64_t* owned_offsets; /* [n_parts+1] into owned                    */
  const int64_t* owned;         /* [n_nodes]                                 */
  const int64_t* halo_offsets;  /* [n_parts+1] into halo                     */
  const int64_t* halo;          /* concatenated halo lists                   */
  const int32_t* halo_ring;     /* ring (1..halo_depth) of each halo entry    */
} xmgn_graph_desc;

typedef struct xmgn_graph xmgn_graph;
typedef struct xmgn_workspace xmgn_workspace;
typedef struct xmgn_comm xmgn_comm;

typedef struct {
  int64_t n_owned, n_local, e_local;
  int32_t depth;
  int64_t ring_nodes[65]; /* ring_nodes[r] = #local nodes with ring < r (r = 0..depth+1) */
  int64_t ring_edges[65]; /* ring_edges[r] = #local edges whose dst ring < r             */
} xmgn_part_info;

xmgn_status xmgn_load_graph(const xmgn_graph_desc* desc, int cuda_device, xmgn_graph** out);
xmgn_status xmgn_part_info_get(const xmgn_graph* g, int part, xmgn_part_info* out);
/* Host copies of a partition's local arrays (caller-allocated, sizes from
 * part_info): local_node_gid[n_local], local_offsets[n_local+1],
 * local_src_lid[e_local], local_edge_gid[e_local], rev[e_local] (index of the
 * reverse local edge).  Any pointer may be NULL.  For bit-exact tests.        */
xmgn_status xmgn_export_part(const xmgn_graph* g, int part, int64_t* local_node_gid, int64_t* local_offsets,
                             int64_t* local_src_lid, int64_t* local_edge_gid, int64_t* rev);
void xmgn_free_graph(xmgn_graph* g);

/* ------------------------------------------------------------------ model
 * precision: XMGN_PREC_BF16 -- BF16 tensor-core operands, FP32 accumulate,
 *            FP32 residual streams / LN / SiLU / aggregation (PAPER.md:234 AMP);
 *            the node MLP's first GEMM and the pre-projection take 2 x BF16
 *            (hi + lo) operands in the forward, P is kept in FP16: max|dh| <=
 *            2e-2 x RMS after 15 layers (north_star).
 *            XMGN_PREC_FP32_CHECK -- every GEMM operand split hi+lo in BF16 and
 *            multiplied as hi*hi + lo*hi + hi*lo (FP32-class products) for the
 *            1e-4 check mode (north_star); H = 128 only.
 *            XMGN_PREC_FP16 -- FP16 tensor-core operands (same MMA rate, 3 more
 *            mantissa bits), 16-bit edge stream; the bench's mode (5x inside the
 *            2e-2 x RMS bound at 15 layers).
 * mlp_hidden_layers m in {1, 2}; hidden H in {128, 256, 512}.                  */
enum { XMGN_PREC_BF16 = 0, XMGN_PREC_FP32_CHECK = 1, XMGN_PREC_FP16 = 2 };
typedef struct {
  int32_t hidden, layers, mlp_hidden_layers, precision;
  float ln_eps;
} xmgn_model_cfg;

size_t xmgn_param_count(const xmgn_model_cfg* cfg);
/* Workspace for one GPU: per-layer 16-bit checkpoints (edge stream, node
 * states, aggregates, node pre-projections), scratch and gradient streams sized
 * for the graph's largest partition; reused across that GPU's sequential
 * partitions.  Requires cfg->layers <= halo depth (else EHALO).  With the
 * environment variable XMGN_Z1=1 (16-bit modes) it also keeps the first edge
 * GEMM's pre-activation per layer (+layers x E_max x H x 2 bytes), which lets
 * xmgn_processor_bwd skip that GEMM's recompute; results stay within the same
 * tolerance.  If that extra allocation fails the call returns ENOMEM (no silent
 * fall-back); XMGN_Z1=1 with the FP32 check mode is EUNSUPPORTED.
 * xmgn_workspace_bytes reports the total allocated.                          */
xmgn_status xmgn_workspace_create(const xmgn_graph* g, const xmgn_model_cfg* cfg, xmgn_workspace** out);
/* Inference workspace (Sec. III-D: "Inference is performed
 * independently on each partition. Predictions on halo nodes are discarded"):
 * xmgn_processor_fwd runs exactly the training forward (bitwise identical
 * h_out) but keeps no per-layer checkpoints -- the 16-bit edge / node operands,
 * aggregates and pre-projections are ping-ponged, about two layers of activation
 * memory instead of L+1, so far fewer (larger) partitions fit a GPU
 * ("significantly smaller" P_infer).  xmgn_processor_bwd on it returns ESTATE. */
xmgn_status xmgn_workspace_create_infer(const xmgn_graph* g, const xmgn_model_cfg* cfg, xmgn_workspace** out);
size_t xmgn_workspace_bytes(const xmgn_workspace* ws);
void xmgn_workspace_free(xmgn_workspace* ws);

/* Forward of partition `part`: params [param_count] FP32,
 * h0 [n_local,H] FP32, e0 [e_local,H] FP32 (local order) -> h_out [n_owned,H]
 * FP32 = h^L of the owned rows.  Keeps per-layer checkpoints in the workspace
 * (activation checkpointing) for xmgn_processor_bwd.           */
xmgn_status xmgn_processor_fwd(xmgn_workspace* ws, int part, const float* params, const float* h0,
                               const float* e0, float* h_out, void* stream);
/* Backward of the most recent fwd on this workspace (else ESTATE):
 * grad_h_out [n_owned,H] = dL/dh^L on owned rows; grad_params [param_count]
 * is ACCUMULATED (+=) so partitions sum in call order;
 * grad_h0 [n_local,H] / grad_e0 [e_local,H] are overwritten (may be NULL).   */
xmgn_status xmgn_processor_bwd(xmgn_workspace* ws, int part, const float* params, const float* grad_h_out,
                               float* grad_params, float* grad_h0, float* grad_e0, void* stream);
/* Synchronises `stream` and returns ENONFINITE if any of n FP32 values is not
 * finite.                                                  */
xmgn_status xmgn_check_finite(const float* dev, size_t n, void* stream);

/* ------------------------------------------------------------------ the model around the processor (NEXT-1)
 * encoders -> processor -> decoder -> owned-row MSE, the paper's full model:
 *  - node inputs, 24 per point ("24 input features, including Fourier features
 *    with 3 different frequencies (i.e., 2pi, 4pi, 8pi)"): [x(3), n(3), then for f in (2pi, 4pi,
 *    8pi), coordinate c in (x, y, z): sin(f c), cos(f c)] (SPEC.md:134-141 column order);
 *  - edge inputs, 4 per edge: (x_src - x_dst, ||x_src - x_dst||);
 *  - both z-scored with the caller's per-variable global mean / std:
 *    stats = device FP32 [56] = mean of the 24 node and 4 edge inputs, then their std (std > 0);
 *  - encoders: MLP (m SiLU hidden layers, linear output) + LayerNorm, no residual -> h^0, e^0;
 *  - decoder: MLP to 4 outputs (p, tau_x, tau_y, tau_z), no LayerNorm;
 *  - loss: sum over the OWNED rows of (y - t)^2 / (4 n_global) ("Halo nodes are
 *    filtered out before the loss computation"; PAPER.md:234 MSE): summed over all partitions it is
 *    the full graph's MSE, and so are the gradients.
 * IO parameters: one flat FP32 vector, node encoder [W_0 (24 x H), b_0, W_j (H x H), b_j for
 * j = 1..m, gamma, beta], edge encoder [W_0 (4 x H), b_0, ..., gamma, beta], decoder [W_0, b_0,
 * ..., W_{m-1}, b_{m-1} (H x H), W_m (H x 4), b_m (4)], y = x W + b, W stored [in, out].
 * 16-bit operand modes only (the FP32 check mode is EUNSUPPORTED).                         */
size_t xmgn_io_param_count(const xmgn_model_cfg* cfg);
/* Forward of partition `part`: pos, nrm = device FP32 [n_local, 3] in local order (positions,
 * unit normals); targets = device FP32 [n_owned, 4] z-scored targets of the owned rows or NULL;
 * n_global = node count of the whole graph (the MSE's normalisation).  pred (device FP32
 * [n_owned, 4]) receives the owned rows' predictions (halo predictions are discarded,
 * PAPER.md:197); with targets, *loss (device FP32) += this partition's loss.  Also valid on an
 * inference workspace.  The encoder/decoder buffers (~ (N_max + E_max) x 128 B + 13 x owned x H B)
 * are allocated on the first call.  EINVAL: NULL pointers, targets without loss or n_global <
 * n_owned.                                                                                     */
xmgn_status xmgn_model_fwd(xmgn_workspace* ws, int part, const float* params, const float* io_params,
                           const float* pos, const float* nrm, const float* stats, const float* targets,
                           int64_t n_global, float* pred, float* loss, void* stream);
/* Backward of the last xmgn_model_fwd WITH targets on this workspace (else ESTATE): grad_params
 * [param_count] and grad_io [io_param_count] are ACCUMULATED (+=), so partitions sum in call
 * order.                                                                       */
xmgn_status xmgn_model_bwd(xmgn_workspace* ws, int part, const float* params, const float* io_params,
                           float* grad_params, float* grad_io, void* stream);

/* ------------------------------------------------------------------ graph construction on the GPU (NEXT-4)
 * The step before the hot path (Sec. III-B/C): from a point cloud
 * whose levels are prefix-nested (level l = points [0, level_counts[l]), "the point
 * cloud from the previous scale is a subset of the point cloud at the next finer scale"):
 *  - per level, edges (j -> i) for the k nearest j != i (k capped at level size - 1), d^2 in FP64
 *    from the FP32 positions as ((dx dx) + (dy dy)) + dz dz, ties to the smaller index;
 *  - symmetrised, united over the levels, deduplicated: CSR by destination, sources ascending;
 *  - n_parts partitions by recursive coordinate bisection (the axis of largest extent, nodes ordered
 *    by (coordinate, id), left part round-half-even(len * floor(p/2) / p) nodes) -- the stand-in for
 *    METIS;
 *  - per partition the halo: nodes within halo_depth undirected hops of its owned set, ordered by
 *    (ring, id) ("equal to the number of message passing layers").
 * pos: device FP32 [n_nodes, 3] on cuda_device; level_counts: host, strictly increasing, last =
 * n_nodes; 1 <= k <= 16; 1 <= n_parts <= n_nodes; 0 <= halo_depth <= 63.  Runs on `stream` and
 * returns when the result (host arrays owned by the handle) is complete.  The result is bitwise
 * the construction of oracle/graphbuild.py.  EINVAL on malformed arguments.                  */
typedef struct xmgn_built_graph xmgn_built_graph;
xmgn_status xmgn_build_graph(const float* pos, int64_t n_nodes, const int64_t* level_counts, int n_levels, int k,
                             int n_parts, int halo_depth, int cuda_device, void* stream, xmgn_built_graph** out);
/* A descriptor pointing into the handle's host arrays (valid until xmgn_built_graph_free), ready
 * for xmgn_load_graph.                                                                        */
xmgn_status xmgn_built_graph_desc(const xmgn_built_graph* b, xmgn_graph_desc* desc);
/* owner[n_nodes] (host, caller-allocated): the partition of every node.                       */
xmgn_status xmgn_built_graph_owner(const xmgn_built_graph* b, int64_t* owner);
void xmgn_built_graph_free(xmgn_built_graph* b);

/* ------------------------------------------------------------------ gradient aggregation
 * One NCCL communicator per process/GPU (one process per GPU).  The unique id
 * is created on rank 0 and broadcast by the caller (e.g. torch.distributed).
 * xmgn_grad_reduce: in-place SUM all-reduce of `count` FP32 values on `stream`
 * ("gradients from all partitions are aggregated").            */
xmgn_status xmgn_comm_unique_id(uint8_t id[128]);
xmgn_status xmgn_comm_init(const uint8_t id[128], int nranks, int rank, int cuda_device, xmgn_comm** out);
xmgn_status xmgn_grad_reduce(xmgn_comm* comm, float* grad_params, size_t count, void* stream);
/* Inference gather ("the remaining predictions are aggregated on
 * the master rank to reconstruct the full-domain output"): every rank sends
 * send_rows x row_elems FP32 values (device) to rank 0 with NCCL point-to-point
 * calls on `stream`; rank 0 receives rank r's block at
 * recv + row_elems * sum_{q<r} recv_rows[q] (recv_rows: host [nranks], rank 0
 * only, recv_rows[0] == its own send_rows; other ranks may pass NULL).        */
xmgn_status xmgn_gather_rows(xmgn_comm* comm, const float* send, int64_t send_rows, int64_t row_elems, float* recv,
                             const int64_t* recv_rows, void* stream);
void xmgn_comm_destroy(xmgn_comm* comm);
/* dst[idx[i], :] = src[i, :] for i < n, rows of row_elems FP32 (device arrays;
 * idx int64 device).  Places gathered owned rows at their global ids.        */
xmgn_status xmgn_scatter_rows(const float* src, const int64_t* idx, int64_t n, int64_t row_elems, float* dst,
                              void* stream);

/* ------------------------------------------------------------------ optimiser step (NEXT-2)
 * After gradient aggregation, one update of the flat FP32
 * parameter vector as PAPER.md:234 (Sec. V-D) trains the model -- "Adam ... with a
 * cosine annealing learning rate schedule ranging from 1e-3 to 1e-6 ... Gradient
 * clipping with a threshold of 32" -- read per SPEC.md:373-381:
 *   g = grad_scale * grad (e.g. 1/(N d), the MSE normalisation);
 *   g *= min(1, clip / (||g||_2 + 1e-6)), the norm over all n values (global-norm);
 *   lr(t) = lr_min + (lr_max - lr_min) (1 + cos(pi t / total_steps)) / 2, t = step (0-based,
 *           clamped to total_steps);
 *   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
 *   p -= lr(t) (m / (1 - b1^(t+1))) / (sqrt(v / (1 - b2^(t+1))) + eps).
 * params, grad, m, v: device FP32 [n] (m, v zero before step 0, updated in place);
 * grad is not modified.  norm_out (device, may be NULL) receives ||g||_2 before clipping.
 * Deterministic (fixed-order reductions).  EINVAL on NULL pointers, step < 0,
 * betas outside [0, 1), eps <= 0, clip <= 0 or total_steps <= 0.               */
typedef struct {
  float lr_max, lr_min;   /* 1e-3, 1e-6 */
  int64_t total_steps;    /* schedule length T */
  float beta1, beta2, eps; /* 0.9, 0.999, 1e-8 */
  float clip;             /* 32 */
} xmgn_adam_cfg;
float xmgn_cosine_lr(const xmgn_adam_cfg* cfg, int64_t step);
xmgn_status xmgn_adam_step(const xmgn_adam_cfg* cfg, int64_t step, float* params, const float* grad, float* m,
                           float* v, size_t n, float grad_scale, float* norm_out, void* stream);

/* ------------------------------------------------------------------ diagnostics
 * C[M,N] FP32 = A * B^T on tcgen05 with A [M,K] (a_mn_major=0) or [K,M] (=1)
 * and B [N,K] (b_mn_major=0) or [K,N] (=1), BF16 device arrays; K % 64 == 0,
 * N in {64,128,256}.  Exercises the descriptor conventions of every kernel.  */
xmgn_status xmgn_selftest_gemm(int M, int N, int K, int a_mn_major, int b_mn_major, const void* A,
                               const void* B, float* C, void* stream);
/* Number of kernels this library has launched since load (monotone).        */
long long xmgn_launch_count(void);
/* When on, named launch scopes (chain_edge_fwd, chain_edge_bwd, aggregate,
 * wgrad, ...) are bracketed by CUDA events on their stream.  collect
 * synchronises on the recorded events and returns, per scope name (names
 * '\n'-separated in `names`), the summed milliseconds and the launch count;
 * it then clears the records.                                                */
xmgn_status xmgn_profile_enable(int on);
xmgn_status xmgn_profile_collect(char* names, size_t names_len, double* ms, long long* counts, int max,
                                 int* n_out);

#ifdef __cplusplus
}
#endif
#endif /* XMGN_H */
