/*
 * moe.h — C ABI of the B200-native dropless-MoE hot path (MegaBlocks,
 * arXiv 2211.15841). Only plain C types cross this boundary.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / figure),
 *            S:n = SPEC.md line n (interfaces only). Readings R1..R16 of points
 *            the paper leaves open are listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless stated, allocated and owned by the
 *    caller (e.g. through torch). The library never allocates, frees or
 *    synchronises on these calls; all work is enqueued on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).
 *  - Dense matrices are row-major. bf16 tensors are raw IEEE bfloat16
 *    (uint16) buffers. Indices are int32.
 *  - Sparse values (S) are [nnz, bs, bs] bf16: nonzero blocks contiguous in
 *    BCSR (row-major block) order, each block row-major (Fig. 4).
 *  - Data-dependent sizes (padded rows Tp, nonzero blocks nnz) are never read
 *    back to the host: moe_topology writes them to topo->sizes on the device and
 *    every later kernel reads them there. Buffers are sized with the worst-case
 *    queries below. Contents at or beyond the device-side sizes are unspecified.
 *  - Arguments are validated on the host before any launch; a bad argument
 *    returns MOE_EINVAL / MOE_ESHAPE / MOE_EUNSUPPORTED and launches nothing.
 *    Launch failures return MOE_ECUDA. Asynchronous device faults surface at
 *    the caller's next synchronisation. moe_last_error() gives a message.
 *  - Deterministic: identical inputs give bitwise-identical outputs (no
 *    floating-point atomics; each output element is reduced by one CTA in a
 *    fixed order).
 *  - Reentrant across streams and threads; the only global state is the
 *    thread-local error string.
 */
#ifndef MOE_H_
#define MOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOE_OK = 0,
  MOE_EINVAL = 1,       /* NULL pointer / bad enum / bad value */
  MOE_ESHAPE = 2,       /* inconsistent sizes */
  MOE_EUNSUPPORTED = 3, /* valid for the method but not on this GPU path (e.g. bs != 128) */
  MOE_ECUDA = 4,        /* CUDA launch/driver error */
  MOE_ENCCL = 5,        /* reserved (collectives are issued by the caller's process group) */
  MOE_EWORKSPACE = 6    /* workspace too small */
} moe_status;

/* Expert activation between SDD and DSD. The paper does not name it
 * ("iterate between SDD and DSD"); reading R2: gelu with the tanh
 * approximation is the default, identity and relu are also offered. */
typedef enum { MOE_ACT_IDENTITY = 0, MOE_ACT_GELU_TANH = 1, MOE_ACT_RELU = 2 } moe_act;

/* Layer hyper-parameters (Fig. 1; Table 1/2 P:124-140).
 * tokens = T, hidden = h, num_experts = E, top_k = k, ffn_hidden = f (per
 * expert; inner_dim = E*f), block_size = bs (128). */
typedef struct {
  int64_t tokens;
  int64_t hidden;
  int64_t num_experts;
  int64_t top_k;
  int64_t ffn_hidden;
  int64_t block_size;
  int32_t act;      /* moe_act */
  int32_t capacity; /* 0: dropless (the paper's method). > 0: the token-dropping
                       formulation it is compared against (§2.2): each
                       expert keeps at most `capacity` assignments, the earliest
                       by flat id t*k+j; the others are dropped (pos = -1,
                       sorted_pos = -1) and contribute nothing to y, dx or the
                       gradients (their dgates are 0). See moe_expert_capacity. */
  int32_t renormalize; /* 0: gate = softmax probability of the chosen expert (R4, the
                          paper's Fig. 5 reading). 1: each token's k gates divided by
                          their sum; the router backward follows it. */
  float aux_loss_coeff; /* 0: none. > 0: auxiliary load-balancing loss (P:118 names it, no formula;
                           S:354: coeff * E * sum_e f_e P_e, f_e = fraction of tokens whose top-1
                           expert is e, held constant; P_e = mean router probability). moe_forward
                           writes it to the workspace (moe_workspace_offset 5) and moe_backward
                           adds its gradient (d total / d aux = 1) to the router's. */
  int32_t unpadded;     /* 0: the dense expert-grouped rows (X_g, Y_g, dY_g, dX_g) are padded to a multiple of
                           bs per expert, as the paper implements it. 1: they are NOT padded (row u =
                           assignment sorted_idx[u]) and every expert's last block-row is a partial block at
                           the fringe ("We could remove this constraint by supporting partial blocks at
                           the fringe"; reading R23): the block topology is unchanged, the
                           sparse values' rows beyond brow_rows are exact zeros, the products read / write
                           dense rows at brow_start. Dropless only (capacity 0). Same outputs. */
} moe_config;

/* ---- configuration and size queries (host only, no CUDA calls) ---------- */

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* moe_last_error(void);

/* MOE_OK iff: T >= 1, h >= 1, 1 <= k <= E, f % bs == 0, act valid; and for the
 * GPU path: bs == 128, h % 256 == 0 and h <= 2048, E <= 1024. */
moe_status moe_check_config(const moe_config* cfg);

/* Worst-case padded rows: Tp = sum_e bs*ceil(c_e/bs) <= bs*floor((R + min(E,R)*(bs-1))/bs),
 * R = T*k (P:297 padding to a multiple of the block size). */
int64_t moe_max_padded_rows(const moe_config* cfg);

/* Capacity of the token-dropping formulation (§2.2):
 * ceil(tokens * capacity_factor / num_experts); 0 if capacity_factor <= 0. */
int64_t moe_expert_capacity(int64_t tokens, int64_t num_experts, double capacity_factor);

/* Worst-case nonzero blocks: max_padded_rows/bs * f/bs (Fig. 3C). */
int64_t moe_max_nnz_blocks(const moe_config* cfg);

/* Device scratch (bytes) needed by moe_router, moe_topology, moe_forward,
 * moe_backward and moe_router_bwd for this config (a single buffer can serve
 * all of them, but not concurrently). 256-byte aligned pointer required. */
size_t moe_workspace_bytes(const moe_config* cfg);

/* Byte offset inside the workspace of the scratch tensors moe_backward uses:
 * which = 0 dY_g [max_rows,h] bf16, 1 dH [max_nnz,bs,bs] bf16, 2 dX_g
 * [max_rows,h] bf16, 3 dgates [T,k] fp32, 4 dlogits [T,E] (bf16 on the
 * tensor-core router path), 5 the auxiliary loss: float [1 + E] = {loss,
 * per-expert logit-gradient coefficients coeff*E*f_e/T} (written by
 * moe_load_balance_loss / moe_forward, read by moe_backward; kept between
 * them). Returns (size_t)-1 for an unknown `which`. */
size_t moe_workspace_offset(const moe_config* cfg, int which);

/* Number of SMs the library sizes its persistent grids for (queried once). */
int moe_device_sm_count(void);

/* ---- topology (Fig. 5 make_topology; P:235-242 hybrid
 *      blocked-CSR-COO; P:287-292 transpose indices; P:299 built together) -- */
typedef struct {
  int32_t* counts;          /* [E]  assignments per expert                                  */
  int32_t* bins;            /* [E]  inclusive cumsum of counts                               */
  int32_t* padded_bins;     /* [E]  inclusive cumsum of bs*ceil(counts/bs)                   */
  int32_t* sorted_idx;      /* [R]  flat ids i = t*k + j in expert order, stable in i (R7)   */
  int32_t* pos;             /* [R]  padded row of flat id i (pad rows at group tail, R8)     */
  int32_t* sorted_pos;      /* [R]  unpadded expert-order position of flat id i              */
  int32_t* row_offsets;     /* [max_rows/bs + 1]  BCSR row offsets (block units)      */
  int32_t* col_indices;     /* [max_nnz]          BCSR column of each block                  */
  int32_t* row_indices;     /* [max_nnz]          COO row of each block              */
  int32_t* t_col_offsets;   /* [E*f/bs + 1]       transposed offsets per block-column (R9)   */
  int32_t* t_block_offsets; /* [max_nnz]          storage index of each block, in (col,row)
                                                  order: the transpose index          */
  int32_t* t_row_indices;   /* [max_nnz]          row of each block in transposed order      */
  int32_t* pair_bins;       /* [E]  inclusive cumsum of ceil(block_rows_e / 2): pairs of
                                    same-expert block-rows (2-SM tiles of the GEMMs)          */
  int32_t* row_src;         /* [max_rows] flat id i = t*k + j held by padded row p (the
                                    inverse of pos), -1 for pad rows                          */
  int32_t* sizes;           /* [3] = {Tp, nnz, row pairs}, written on the device             */
  int32_t* brow_start;      /* [max_rows/bs] unpadded layout (moe_config.unpadded, P:297 partial blocks at
                                    the fringe): first dense row of block-row r = bins[e]-counts[e]+bs*i
                                    for the i-th block-row of expert e                         */
  int32_t* brow_rows;       /* [max_rows/bs] rows of block-row r that hold assignments: min(bs,
                                    counts[e]-bs*i); the rest of its blocks is the fringe       */
} moe_topology_t;

/* Router, §2.1: logits = x . wr (fp32 accumulate of bf16 inputs),
 * then moe_topk. x [T,h] bf16, wr [h,E] bf16; logits [T,E] fp32 (kept for the
 * backward pass), expert_idx [T,k] int32, gates [T,k] fp32. */
moe_status moe_router(const moe_config* cfg, const void* x, const void* wr, float* logits,
                      int32_t* expert_idx, float* gates, void* ws, void* stream);

/* Top-k from fp32 logits ("greedily selecting the top_k scoring
 * experts"): per token the k largest logits in descending order, exact ties to
 * the lower expert index (R6); gate = softmax probability of the chosen
 * expert, no renormalisation (R4). Bit-exact selection contract. */
moe_status moe_topk(const moe_config* cfg, const float* logits, int32_t* expert_idx, float* gates,
                    void* stream);

/* Topology + permutation plan from expert_idx [T*k]. Unlike the
 * products, this call also accepts block_size 32 or 64 (the
 * bs = 64 topology for smaller tiles); every array then follows that
 * block size (max sizes from the same config).
 * Writes every array of *topo (caller-allocated, sized by the max queries)
 * and topo->sizes = {Tp, nnz}. Integer outputs are bit-exact (closed form of
 * the block-diagonal pattern). ws: moe_workspace_bytes.
 * With cfg->capacity > 0 (token-dropping formulation) counts are
 * the kept assignments per expert (at most capacity, the earliest by flat id),
 * dropped assignments get pos = sorted_pos = -1 and appear in no other array;
 * every later entry point skips them. */
/* moe_topology after moe_router ran with the same cfg and ws: on the
 * tensor-core router path (E % 64 == 0, E <= 256, top_k <= 8) the router's
 * epilogue already wrote per-128-token expert histograms into ws, so the
 * whole topology is one launch ("custom CUDA kernel"); otherwise it is
 * moe_topology. Same outputs, bit for bit. */
/* moe_router followed by the topology (Fig. 5 lines 1-2) in ONE
 * launch where possible: on the tensor-core router path with top_k <= 2 the
 * router kernel is launched cooperatively and, after a grid barrier, builds
 * the whole topology from its per-tile histograms. Otherwise
 * moe_router + moe_topology_from_router. Outputs identical to moe_router then
 * moe_topology, bit for bit. ws: moe_workspace_bytes, required. */
moe_status moe_router_topology(const moe_config* cfg, const void* x, const void* wr, float* logits,
                               int32_t* expert_idx, float* gates, const moe_topology_t* topo, void* ws, void* stream);
moe_status moe_topology_from_router(const moe_config* cfg, const int32_t* expert_idx, const moe_topology_t* topo,
                                    void* ws, void* stream);
moe_status moe_topology(const moe_config* cfg, const int32_t* expert_idx, const moe_topology_t* topo,
                        void* ws, void* stream);

/* Padded gather, Fig. 5 line 15 fused with zero padding:
 * x_g[pos[t*k+j]] = x[t]; every pad row = 0. x [T,h], x_g [max_rows,h] bf16. */
moe_status moe_gather(const moe_config* cfg, const void* x, const moe_topology_t* topo, void* x_g,
                      void* stream);

/* Padded scatter + weighting, Fig. 5 lines 26-27, §2.4:
 * y[t] = sum_{j ascending} gates[t,j] * y_g[pos[t*k+j]], fp32 accumulate, bf16
 * out. gates may be NULL (unit gates). */
moe_status moe_scatter(const moe_config* cfg, const void* y_g, const moe_topology_t* topo,
                       const float* gates, void* y, void* stream);

/* Backward of moe_scatter (chain rule of Fig. 5's weighted un-permutation):
 * dy_g[pos[t*k+j]] = gates[t,j]*dy[t] (pad rows 0);
 * dgates[t,j] = <y_g[pos[t*k+j]], dy[t]> (fp32). dgates may be NULL. */
moe_status moe_scatter_bwd(const moe_config* cfg, const void* dy, const void* y_g,
                           const moe_topology_t* topo, const float* gates, void* dy_g, float* dgates,
                           void* stream);

/* Backward of moe_gather (P:268 padded_gather): dx[t] = sum_j dx_g[pos[t*k+j]] (bf16 out). */
moe_status moe_gather_bwd(const moe_config* cfg, const void* dx_g, const moe_topology_t* topo, void* dx,
                          void* stream);

/* Unpadded expert-order permutation used by expert parallelism:
 * x_sorted[j] = x[sorted_idx[j] / k], j < T*k. */
moe_status moe_sort_rows(const moe_config* cfg, const void* x, const moe_topology_t* topo, void* x_sorted,
                         void* stream);
/* Un-permutation on the token owner under expert parallelism:
 * y[t] = sum_j gates[t,j] * y_sorted[sorted_pos[t*k+j]] (gates may be NULL). */
moe_status moe_unsort_rows(const moe_config* cfg, const void* y_sorted, const moe_topology_t* topo,
                           const float* gates, void* y, void* stream);
/* Backward of moe_unsort_rows (chain rule of P:280): dy_sorted[sorted_pos[i]] = g*dy[t];
 * dgates[t,j] = <y_sorted[sorted_pos[i]], dy[t]>. */
moe_status moe_unsort_rows_bwd(const moe_config* cfg, const void* dy, const void* y_sorted,
                               const moe_topology_t* topo, const float* gates, void* dy_sorted,
                               float* dgates, void* stream);
/* Backward of moe_sort_rows: dx[t] = sum_j dx_sorted[sorted_pos[t*k+j]]. */
moe_status moe_sort_rows_bwd(const moe_config* cfg, const void* dx_sorted, const moe_topology_t* topo,
                             void* dx, void* stream);

/* Expert-parallel forms of the fused router backward (P:98 softmax, P:355
 * expert parallelism; the token owner's side of b1 / b6 / b7). Same
 * arithmetic as moe_scatter_bwd_router / moe_router_dx, on the unpadded
 * expert-order rows (sorted_pos instead of pos, no pad rows):
 *   moe_unsort_rows_bwd_router: dy_sorted, dgates as moe_unsort_rows_bwd, and
 *     dlogits_bf16 [T,E] = p * (dp - <p,dp>) rounded to bf16.
 *   moe_sort_rows_bwd_router: dx [T,h] = sum_j dx_sorted[sorted_pos[t*k+j]]
 *     + dlogits . wr^T (tcgen05; wr [h,E] bf16).
 * Tensor-core router configs only (E % 64 == 0, E <= 256, top_k <= 8), else
 * MOE_EUNSUPPORTED. All pointers device, caller-owned; stream-ordered. */
moe_status moe_unsort_rows_bwd_router(const moe_config* cfg, const void* dy, const void* y_sorted,
                                      const moe_topology_t* topo, const float* gates, const float* logits,
                                      const int32_t* expert_idx, void* dy_sorted, float* dgates,
                                      void* dlogits_bf16, void* stream);
moe_status moe_sort_rows_bwd_router(const moe_config* cfg, const void* dx_sorted, const moe_topology_t* topo,
                                    const void* dlogits_bf16, const void* wr, void* dx, void* stream);

/* ---- expert parallelism over peer memory (NVLink 5 / NVSwitch; SURVEY §8(f)
 *      NEXT-1): device-initiated dispatch / combine, no host
 *      synchronisation. Each rank owns one window (moe_ep_window_alloc, a
 *      cudaMalloc'd region exported with moe_ipc_get_handle and mapped by every
 *      peer with moe_ipc_open_handle). Window layout (moe_ep_window_offset):
 *      cumulative arrival counters, an error word, the all-gathered [P,E]
 *      int32 histograms and four bf16 row regions: receive x / dy
 *      [cap_rows, hidden] (rows this rank's experts get, arrival order source
 *      rank, local expert, token) and return y / dx [owner_rows = T*k, hidden]
 *      (rows coming back, in this rank's expert-sorted order, moe_sort_rows).
 *      Every exchange bumps per-source arrival counters at its destinations;
 *      a wait spins with acquire loads until every source reached this rank's
 *      next epoch of the region (kept in the window: calls carry no host
 *      state, so a step can be captured in a CUDA graph; all ranks must issue
 *      the same sequence of exchanges). A wait gives up after 20 s, writing
 *      1 + region to the error word (mirrored in the plan's last int) instead
 *      of hanging. ---- */
enum { MOE_EP_ARRIVE = 0, MOE_EP_ERROR = 1, MOE_EP_COUNTS = 2, MOE_EP_RECV_X = 3, MOE_EP_RECV_DY = 4,
       MOE_EP_RET_Y = 5, MOE_EP_RET_DX = 6 };

typedef struct {
  int32_t nranks, rank, num_experts, hidden;  /* E % nranks == 0: rank r owns experts [r E/P, (r+1) E/P) */
  int64_t cap_rows;                           /* receive-region rows (>= rows any step can bring) */
  int64_t owner_rows;                         /* T_local * top_k */
  const void* peers;                          /* DEVICE uint64 [nranks]: every rank's window base as mapped here */
  int32_t* plan;                              /* DEVICE int32 [moe_ep_plan_ints]: counts_all [P,E], n_recv,
                                                 offsets (written by moe_ep_exchange_counts); the last
                                                 int mirrors the error word (0 = no timeout) */
} moe_ep_t;

size_t  moe_ep_window_bytes(int nranks, int num_experts, int64_t hidden, int64_t cap_rows, int64_t owner_rows);
int64_t moe_ep_window_offset(int nranks, int num_experts, int64_t hidden, int64_t cap_rows, int64_t owner_rows,
                             int which);   /* which = MOE_EP_*; -1 if unknown */
int     moe_ep_plan_ints(int nranks, int num_experts);
moe_status moe_ep_window_alloc(size_t bytes, void** window);   /* setup only: cudaMalloc + zero */
moe_status moe_ep_window_free(void* window);
moe_status moe_ipc_get_handle(const void* window, void* handle /* 64 bytes out */);
moe_status moe_ipc_open_handle(const void* handle /* 64 bytes */, void** window);
moe_status moe_ipc_close_handle(void* window);
/* counts_local [E] int32 device: this rank's per-global-expert histogram
 * (moe_topology counts). Stores it into every peer, waits for all P rows, and
 * writes ep->plan; plan[P*E] = rows this rank receives. One CTA. */
moe_status moe_ep_exchange_counts(const moe_ep_t* ep, const int32_t* counts_local, void* stream);
/* Padded exchange (the receiving side needs no gather): rows land directly in
 * the owner's padded expert-grouped layout (local expert, then source
 * rank, then token; pad rows at each expert's tail are NOT written — zero them
 * with moe_zero_pad_rows). x [T, hidden] in token order: assignment i =
 * t*k+j sends x[i / k] to its sorted position sorted_pos[i] (the rank's
 * moe_topology sorted_pos; input-driven, sequential reads), or, with
 * sorted_pos NULL, x holds rows already in expert order.
 * moe_ep_combine_padded sends this rank's padded rows [n_padded, hidden] back
 * to their sources' return regions (pad rows skipped). The receiving side's
 * topology comes from the per-source counts (moe_topology_counts with the
 * plan's compact counts, moe_ep_plan_offset 0); plan offset 1 holds its
 * padded row count. */
moe_status moe_ep_dispatch_padded(const moe_ep_t* ep, int region, const void* x, const int32_t* sorted_pos,
                                  int top_k, void* stream);
moe_status moe_ep_combine_padded(const moe_ep_t* ep, int region, const void* rows_padded, void* stream);
/* The combine fused into the expert side's DSD (P:399 overlap):
 * moe_ep_combine_dest writes, for each of this rank's padded rows p <
 * max_rows, the DEVICE address moe_ep_combine_padded would copy row p to (its
 * source's return region `region` at the row's sorted position, through the
 * peer mapping), 0 for pad rows and rows past the plan's padded count;
 * dest [max_rows] uint64 device. moe_dsd_rows then stores each output row
 * straight to dest[p] (over NVLink for remote sources), and moe_ep_signal
 * publishes the region's completion to every peer (one CTA: a system-scope
 * release after the stream-ordered stores), as the copy kernel's last CTA
 * does; moe_ep_wait on the receivers is unchanged. */
moe_status moe_ep_combine_dest(const moe_ep_t* ep, int region, uint64_t* dest, int64_t max_rows, void* stream);
moe_status moe_ep_signal(const moe_ep_t* ep, int region, void* stream);
int moe_ep_plan_offset(int nranks, int num_experts, int which);

/* Topology (P:235-242 hybrid blocked-CSR-COO, P:290 transpose indices, P:297
 * padding) of assignments that are already grouped by expert and, within an
 * expert, by source (expert parallelism's receiving side): counts_per_source
 * [nsources, E] int32 device. Writes counts, bins, padded_bins, pair_bins,
 * sizes and every BCSR / COO / transpose index (bit-identical to moe_topology
 * of the same grouping); the per-assignment arrays (sorted_idx, pos,
 * sorted_pos, row_src of real rows) are not written. */
moe_status moe_topology_counts(const moe_config* cfg, const int32_t* counts_per_source, int nsources,
                               const moe_topology_t* topo, void* stream);
/* Zero the pad rows (tail of each expert group) of a padded [max_rows, h] buffer. */
moe_status moe_zero_pad_rows(const moe_config* cfg, const moe_topology_t* topo, void* x_g, void* stream);

/* Stream-ordered wait until every source's next exchange of `region` landed here. */
moe_status moe_ep_wait(const moe_ep_t* ep, int region, void* stream);

/* Expert-parallel receive ids (DESIGN.md §7 ordering contract): rows
 * arrive ordered (source rank q, local expert l, token); ids[i] = l of arrival
 * row i, i < sum over q, l of counts_all[q*E + e0 + l]. counts_all [P,E] int32
 * device (the all-gathered per-rank histograms), ids int32 device with room for
 * every received row. One small kernel, no host synchronisation. */
moe_status moe_ep_recv_ids(const int32_t* counts_all, int nranks, int num_experts, int e0, int local_experts,
                           int32_t* ids, int64_t max_rows, void* stream);

/* ---- block-sparse products, Triton notation, §5.1 ----
 * The sparse operand has the MoE topology: logical shape [Tp, E*f] with
 * 128x128 blocks. bf16 in, fp32 accumulate on the tensor cores, bf16 out.
 *
 * moe_sdd: out_s = act(A . B) on the topology's nonzero blocks (SDD),
 *   A = a [max_rows, h]; B = b [h, E*f] (trans_b = 0, forward: W1) or
 *   B = b^T with b [E*f, h] (trans_b = 1, SDD^T backward: W2).
 *   out_pre (optional) receives the pre-activation A.B.
 *   act_grad_src != NULL selects the backward epilogue
 *   out_s = (A.B) * act'(act_grad_src) where act_grad_src is the saved
 *   pre-activation [nnz,bs,bs] (SDD^T fused with the activation derivative).
 * moe_dsd: trans_s = 0: out [max_rows, h] = S . B_eff (DSD; DSD^T uses
 *   trans_b = 1 with b = W1 [h, E*f]); B_eff = b [E*f, h] or b^T.
 *   trans_s = 1: out [E*f, h] = S^T . B_eff (DS^TD), walking the
 *   transpose index; B_eff = b [max_rows, h] (trans_b = 0) or
 *   b^T with b [h, max_rows] (trans_b = 1).
 * moe_dds: trans_s = 0: out [h, E*f] = A_eff . S (DD^TS with trans_a = 1 and
 *   a = X_g [max_rows, h]; trans_a = 0: a [h, max_rows]) via the
 *   transpose index. trans_s = 1: out [h, max_rows] = A_eff . S^T with
 *   A_eff = a [h, E*f] or a^T (a [E*f, h]).
 */
moe_status moe_sdd(const moe_config* cfg, const void* a, const void* b, int trans_b,
                   const moe_topology_t* topo, int32_t act, const void* act_grad_src, void* out_s,
                   void* out_pre, void* stream);
/* moe_sdd_deriv: the layer's form of moe_sdd, saving the activation
 * derivative instead of the pre-activation (reading R18 in DESIGN.md).
 *   deriv_src == NULL (forward): out_s = act(A.B) and, if out_deriv
 *     != NULL, out_deriv = act'(A.B) [nnz,bs,bs] bf16 (one tanh serves both).
 *   deriv_src != NULL (SDD^T): out_s = (A.B) * deriv_src, deriv_src
 *     being the saved act'(H).
 *   deriv_src and out_deriv are exclusive (MOE_EINVAL). Shapes, layouts and
 *   errors as moe_sdd. */
moe_status moe_sdd_deriv(const moe_config* cfg, const void* a, const void* b, int trans_b,
                         const moe_topology_t* topo, int32_t act, const void* deriv_src, void* out_s,
                         void* out_deriv, void* stream);
/* moe_sdd_act_coded: the layer's memory-saving form (reading R24 in DESIGN.md,
 * moe_saved.act_deriv = NULL): the forward saves ONLY the activation
 * A = act(H), and the SDD^T recovers act'(H) from A itself. P:206 lists SDD^T but not what it reads; the paper keeps
 * act(H) for DS^TD anyway ("second layer weight gradient").
 *   coded_src == NULL (forward SDD): out_s = coded act(A.B) [nnz,bs,bs]
 *     bf16. gelu: A >= 0 is RNE bf16 of act(h) (h >= 0); for h < 0 the sign bit
 *     is set and the mantissa LSB holds the branch of gelu's two pre-images
 *     (1: h < argmin gelu = -0.75246), the value being the nearest bf16 of that
 *     parity (<= 1 ulp). relu: RNE bf16 (act' = A > 0). identity: plain H.
 *     The coded A is a valid bf16 activation: every consumer (DSD, DS^TD) reads
 *     it as is.
 *   coded_src != NULL (SDD^T): out_s = (A.B) * act'(H), act'(H) decoded
 *     from coded_src (the forward's out_s): gelu by a table over A's 16 bits
 *     (act_code_table.h), relu as A > 0.
 *   Shapes, layouts, trans_b and errors as moe_sdd. */
moe_status moe_sdd_act_coded(const moe_config* cfg, const void* a, const void* b, int trans_b,
                             const moe_topology_t* topo, int32_t act, const void* coded_src, void* out_s,
                             void* stream);
/* Host only (no CUDA call): act'(H) as the SDD^T decodes it from n coded bf16
 * bit patterns (moe_sdd_act_coded's A) into out [n] fp32. MOE_EINVAL on a bad
 * act or NULL pointer. For tests of the decode table against the oracle. */
moe_status moe_act_code_decode_host(int32_t act, const uint16_t* a_bits, float* out, int64_t n);
moe_status moe_dsd(const moe_config* cfg, const void* s, int trans_s, const void* b, int trans_b,
                   const moe_topology_t* topo, void* out, void* stream);
/* moe_dsd_rows: the DSD / DSD^T (trans_s = 0) with output row p (of the padded
 * [max_rows, h] result) stored to the device address row_dst[p] instead of a
 * dense buffer (row_dst == 0: not stored); row_dst [max_rows] uint64 device,
 * each address 16-byte aligned (moe_ep_combine_dest writes them). Rows go
 * out with 16-byte st.global (peer addresses allowed). */
moe_status moe_dsd_rows(const moe_config* cfg, const void* s, const void* b, int trans_b,
                        const moe_topology_t* topo, const uint64_t* row_dst, void* stream);
/* The padded gather fused into the products that read X_g: the A rows
 * are fetched from x [T, h] by token (topo->row_src / k) with TMA
 * tile::gather4, pad rows read as zeros, so X_g is never materialised.
 * moe_sdd_gather: out_s = act(X_g . w1), out_deriv (optional) = act'(X_g . w1)
 *   (forward SDD, as moe_sdd_deriv with trans_b = 0).
 * moe_dds_gather: dw1 [h, E*f] = X_g^T . dh (DD^TS).
 * Both need even f/bs and h % 256 == 0 (CTA-pair column tiles); otherwise they
 * run moe_gather into x_g [max_rows, h] (caller scratch, then required) and the
 * unfused product. */
moe_status moe_sdd_gather(const moe_config* cfg, const void* x, const void* w1, const moe_topology_t* topo,
                          int32_t act, void* out_s, void* out_deriv, void* x_g, void* stream);
/* 1 if moe_forward / moe_backward use the gather-fused products for this config
 * (off unless MOE_GATHER_FUSED=1: the gather4 requests are issue-rate bound at
 * one 128 B row each, slower than a separate coalesced gather at MoE-XS). The
 * two entry points above always gather inside the product when the config allows. */
int moe_gather_is_fused(const moe_config* cfg);
moe_status moe_dds_gather(const moe_config* cfg, const void* x, const void* dh, const moe_topology_t* topo, void* dw1,
                          void* x_g, void* stream);

/* moe_dsd_scatter: the layer's DSD fused with the weighted
 * un-permutation: y_g [max_rows, h] = S . b (b = W2 [E*f, h]) and
 * y [T, h] with y[t] = sum_j gates[t,j] * y_g[pos[t*k+j]]. For top-1 the
 * DSD epilogue writes the gate-scaled rows straight to y[t] with TMA
 * tile::scatter4 (rows via topo->row_src, pad rows dropped); for k > 1 it is
 * moe_dsd followed by moe_scatter. y_g is still written (the backward needs it).
 * gates = NULL: unit weights (the un-permutation alone). */
moe_status moe_dsd_scatter(const moe_config* cfg, const void* s, const void* b, const moe_topology_t* topo,
                           const float* gates, void* y_g, void* y, void* stream);
moe_status moe_dds(const moe_config* cfg, const void* a, int trans_a, const void* s, int trans_s,
                   const moe_topology_t* topo, void* out, void* stream);

/* Router backward (softmax chain rule): dp[t,e] = dgates[t,j] where
 * e = expert_idx[t,j], else 0; dlogits = p * (dp - <p,dp>), p = softmax(logits);
 * dwr [h,E] fp32 = x^T . dlogits;  dx [T,h] bf16 += dlogits . wr^T (in place). */
moe_status moe_router_bwd(const moe_config* cfg, const void* x, const void* wr, const float* logits,
                          const int32_t* expert_idx, const float* dgates, float* dwr, void* dx,
                          void* ws, void* stream);

/* Auxiliary load-balancing loss (cfg->aux_loss_coeff): from the
 * fp32 logits [T,E] and expert_idx [T,k] (top-1 = slot 0) writes {loss,
 * coeff*E*f_e/T for every e} to the workspace's aux region (offset 5).
 * Deterministic: fixed token partition, fixed-order reductions. */
moe_status moe_load_balance_loss(const moe_config* cfg, const float* logits, const int32_t* expert_idx, void* ws,
                                 void* stream);

/* The auxiliary loss's router gradient added to an existing bf16 dlogits [T,E]
 * in place: dlogits += p * (c - <p,c>), p = softmax(logits), c = the per-expert
 * coefficients moe_load_balance_loss left in ws. A no-op when
 * cfg->aux_loss_coeff == 0. For callers that compose the router backward from
 * the pieces below (expert parallelism); moe_backward folds it in itself. */
moe_status moe_add_aux_dlogits(const moe_config* cfg, const float* logits, void* dlogits_bf16, const void* ws,
                               void* stream);

/* ---- fused backward pieces used by moe_backward when the router runs on the
 *      tensor cores (E % 64 == 0, E <= 256, top_k <= 8; else MOE_EUNSUPPORTED) --- */

/* b1 + the softmax part of b7 (P:98 softmax router, chain rule of P:280) in one pass per token: dy_g and dgates exactly as
 * moe_scatter_bwd, and dlogits_bf16 [T,E] = p * (dp - <p,dp>) rounded to bf16,
 * p = softmax(logits[t,:]), dp[e] = sum_{j: expert_idx[t,j] = e} dgates[t,j]. */
moe_status moe_scatter_bwd_router(const moe_config* cfg, const void* dy, const void* y_g, const moe_topology_t* topo,
                                  const float* gates, const float* logits, const int32_t* expert_idx, void* dy_g,
                                  float* dgates, void* dlogits_bf16, void* stream);

/* b7 (P:98 router projection, backward): dwr [h,E] fp32 = x^T . dlogits (tcgen05, token dimension split into a
 * fixed number of ranges, partials reduced in a fixed order). ws as above. */
moe_status moe_router_dwr(const moe_config* cfg, const void* x, const void* dlogits_bf16, float* dwr, void* ws,
                          void* stream);

/* b6 + b7 (P:268 gather, P:98 router, backward): dx [T,h] bf16 = sum_j dx_g[pos[t*k+j]] + dlogits . wr^T (tcgen05,
 * the padded-gather backward fused into the GEMM epilogue). */
moe_status moe_router_dx(const moe_config* cfg, const void* dlogits_bf16, const void* wr, const void* dx_g,
                         const moe_topology_t* topo, void* dx, void* stream);

/* b4 + b6 + b7 fused: dx [T,h] bf16 = sum_j (dh . w1^T)[pos[t*k+j]] + dlogits . wr^T,
 * i.e. DSD^T with the padded-gather backward and the router term of
 * dx. For top-1 one tcgen05 kernel: each DSD^T tile appends E/64 dense K-steps
 * whose A rows are the tile's tokens' dlogits (TMA tile::gather4 through
 * topo->row_src) and writes its rows straight to dx[token] (tile::scatter4;
 * pad rows dropped). For k > 1: moe_dsd into dx_g [max_rows, h] (caller
 * scratch, required), then moe_router_dx. dlogits bf16 [T,E]; wr [h,E].
 * dlogits = wr = NULL drops the router term (DSD^T + gather backward only; then
 * dx_g is required and also receives dX_g). */
moe_status moe_dsd_dx(const moe_config* cfg, const void* dh, const void* w1, const moe_topology_t* topo,
                      const void* dlogits_bf16, const void* wr, void* dx, void* dx_g, void* stream);

/* ---- the layer: Fig. 5 forward, §5.1 backward ---- */
typedef struct {
  const void* wr; /* [h, E]   bf16 */
  const void* w1; /* [h, E*f] bf16 */
  const void* w2; /* [E*f, h] bf16 (R1: P:274 is garbled) */
} moe_weights;

typedef struct {
  float* dwr; /* [h, E]   fp32 */
  void* dw1;  /* [h, E*f] bf16 (fp32 accumulate) */
  void* dw2;  /* [E*f, h] bf16 (fp32 accumulate) */
} moe_grads;

/* Tensors the forward pass keeps for the backward pass (caller-allocated). */
typedef struct {
  float* logits;      /* [T, E] fp32 */
  int32_t* expert_idx;/* [T, k] */
  float* gates;       /* [T, k] fp32 */
  moe_topology_t topo;
  void* x_g;          /* [max_rows, h] bf16 padded gather of x; written only when the config
                         cannot gather inside the products (moe_sdd_gather) */
  void* act_deriv;    /* [max_nnz, bs, bs] bf16 act'(pre-activation) (R18, the default), or NULL:
                         the branch-coded activation (R24, moe_sdd_act_coded): `a` alone is saved
                         and the SDD^T decodes act'(H) from it (one buffer less; measured slower at
                         MoE-XS). Unused for identity. */
  void* a;            /* [max_nnz, bs, bs] bf16 activation */
  void* y_g;          /* [max_rows, h] bf16 */
} moe_saved;

/* y [T,h] bf16 = dMoE(x [T,h] bf16): router, topology, padded gather,
 * SDD(+act), DSD, weighted scatter; stream-ordered, no host synchronisation. */
moe_status moe_forward(const moe_config* cfg, const moe_weights* w, const void* x, void* y, moe_saved* saved,
                       void* ws, void* stream);

/* Gradients of sum(y * dy): dx [T,h] bf16 and *grads, via scatter-bwd, SDD^T
 * (+act'), DS^TD, DSD^T, DD^TS, gather-bwd, router-bwd. */
moe_status moe_backward(const moe_config* cfg, const moe_weights* w, const moe_saved* saved, const void* x,
                        const void* dy, void* dx, moe_grads* grads, void* ws, void* stream);

/* ---- the expert-parallel layer ("data and expert model
 *      parallelism", "8-way expert model parallelism for MoE layers and
 *      data parallelism for all other layers") ----
 * One object per rank (one process per GPU). Rank r of nranks owns experts
 * [r E/P, (r+1) E/P) and their weight slices; the router weights are
 * replicated. Tokens travel over the peer-memory transport above (device-
 * initiated stores into every owner's IPC window, on-device count exchange):
 * forward and backward are stream-ordered with no host synchronisation and can
 * be captured in a CUDA graph; every rank must issue the same sequence of
 * forwards / backwards.
 *
 * Setup (collective over the caller's process group, which the library does
 * not own):  moe_ep_init on every rank -> moe_ep_get_handle (64 bytes) ->
 * the caller all-gathers the nranks handles (rank order) -> moe_ep_connect.
 * moe_ep_init is the only call that allocates (cudaMalloc of the rank's window
 * and of every buffer the layer needs, sized for max_tokens); the hot path
 * allocates nothing. max_tokens must be the same on every rank (window layouts
 * must agree); a step may pass fewer tokens.
 *
 * moe_ep_forward: y [tokens, h] bf16 = dMoE(x [tokens, h] bf16); w->wr [h, E]
 * (all experts), w->w1 [h, (E/P) f], w->w2 [(E/P) f, h] (this rank's slices).
 * moe_ep_backward: dx [tokens, h] bf16, g->dw1 / g->dw2 (this rank's slices,
 * bf16) and g->dwr [h, E] fp32 = THIS RANK'S PARTIAL of the router gradient
 * (its tokens only): the data-parallel sum over ranks is the caller's
 * all-reduce. The layer keeps the state of the last forward only (one forward
 * in flight): a backward must follow its forward, else MOE_EINVAL.
 * Routing, topology and the expert-side products are exactly the single-GPU
 * layer's on the global batch restricted to each rank's experts.
 * Errors: a peer that never arrives makes the waits give up after 20 s and
 * set the plan's last int (MOE_EP_T_PLAN) to 1 + region; a receive bound
 * (recv_rows_cap) that a step exceeds sets it to 100 and that rank's expert
 * side computes nothing (no write leaves any window). */
typedef struct moe_ep moe_ep;
typedef struct {
  int32_t nranks, rank;
  int64_t max_tokens;   /* per rank, identical on all ranks */
  int64_t hidden, num_experts /* global E, E % nranks == 0 */, top_k, ffn_hidden, block_size;
  int32_t act, renormalize;
  float aux_loss_coeff; /* > 0: the auxiliary loss of this rank's tokens (moe_config.aux_loss_coeff) */
  int64_t recv_rows_cap;/* rows one rank's experts may receive per step; 0 = nranks*max_tokens*top_k (never
                           exceeded; each of x_g, A, act', dH is then sized for it) */
} moe_ep_desc;
enum { MOE_EP_T_LOGITS = 0, MOE_EP_T_EXPERT_IDX = 1, MOE_EP_T_GATES = 2, MOE_EP_T_PLAN = 3, MOE_EP_T_AUX = 4,
       MOE_EP_T_X_G = 5, MOE_EP_T_A = 6, MOE_EP_T_ACT_DERIV = 7 };
moe_status moe_ep_init(moe_ep** ep, const moe_ep_desc* desc, int device);
moe_status moe_ep_get_handle(const moe_ep* ep, void* handle /* 64 bytes out */);
moe_status moe_ep_connect(moe_ep* ep, const void* handles /* nranks x 64 bytes, rank order */);
moe_status moe_ep_forward(moe_ep* ep, int64_t tokens, const moe_weights* w, const void* x, void* y, void* stream);
moe_status moe_ep_backward(moe_ep* ep, const moe_weights* w, const void* x, const void* dy, void* dx,
                           moe_grads* grads, void* stream);
/* Device pointer into the layer's state (MOE_EP_T_*; the forward's logits [T,E]
 * fp32, expert_idx [T,k], gates [T,k], the exchange plan, the auxiliary loss
 * {loss, coefficients}, the expert side's X_g / A / act'); NULL if unknown. */
void* moe_ep_tensor(const moe_ep* ep, int which);
/* The config and topology of side 0 (token owner, tokens of the last forward)
 * or side 1 (expert side at capacity); device-side sizes live in topo->sizes. */
moe_status moe_ep_state(const moe_ep* ep, int side, moe_config* cfg, moe_topology_t* topo);
moe_status moe_ep_exchange_desc(const moe_ep* ep, moe_ep_t* out);
moe_status moe_ep_destroy(moe_ep* ep);   /* synchronises the device, unmaps the peers, frees everything */

/* Number of kernel launches the last moe_forward / moe_backward on this
 * thread enqueued (for the bench's gpu_launches count). */
int moe_last_launch_count(void);

/* Kernel launches enqueued by this library since it was loaded (all threads). */
int64_t moe_total_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MOE_H_ */
