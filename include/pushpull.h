/*
 * pushpull.h — C ABI of the B200-native push-pull library (libpushpull.so).
 *
 * Hot path of Yang, Buluç, Owens, "Implementing Push-Pull Efficiently in
 * GraphBLAS" (ICPP'18, arXiv 1804.03327): the masked Boolean-semiring matvec
 * GrB_mxv that drives direction-optimised BFS.  Citations: P:n = PAPER.md line n
 * (Sec./Eq./Alg. given beside it); DESIGN.md Rn = the reading DESIGN.md fixes
 * where the paper is silent or ambiguous.
 *
 * Conventions (apply to every call):
 *  - Every function returns pp_status and never throws across the ABI.  On error
 *    pp_last_error() returns a thread-local message naming the offending
 *    argument / row / edge; outputs are then unspecified.
 *  - Ownership: the caller owns every buffer it passes.  pp_graph_upload COPIES
 *    the graph to device memory the returned handle owns (freed by
 *    pp_graph_free).  Output vectors/arrays are caller-allocated; a torch
 *    tensor's data_ptr() is fine.
 *  - Streams: all device work is stream-ordered on the ctx stream (a
 *    cudaStream_t, NULL = legacy default stream).  Calls that return a host
 *    value (pp_mxv's w->nnz when requested, pp_bfs with stats or with a host
 *    depth/parent pointer) synchronise that stream before returning.
 *  - Threading: one ctx per host thread; the library starts no host threads.
 *  - Vertex ids are uint32 (n < 2^32).  Graph offsets are accepted as int64.
 *  - There is no CPU fallback: without a usable CUDA device every call that needs
 *    one fails with PP_ERR_CUDA.
 */
#ifndef PUSHPULL_H
#define PUSHPULL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PP_OK = 0,
  PP_ERR_ARG = 1,          /* NULL / inconsistent argument                          */
  PP_ERR_RANGE = 2,        /* source or vertex id out of range         */
  PP_ERR_DIM = 3,          /* dimension / vector-format mismatch     */
  PP_ERR_GRAPH = 4,        /* malformed CSR/CSC under PP_GRAPH_VALIDATE     */
  PP_ERR_UNSUPPORTED = 5,  /* semiring other than Boolean, or a size limit          */
  PP_ERR_CUDA = 6,         /* CUDA runtime error (incl. no device)                  */
  PP_ERR_NCCL = 7,         /* reserved for the distributed context                  */
  PP_ERR_OOM = 8,          /* device allocation failed                              */
  PP_ERR_TIMEOUT = 9       /* device-side watchdog fired (persistent BFS barrier)   */
} pp_status;

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* pp_last_error(void);
/* Library version string. */
const char* pp_version(void);

typedef struct pp_ctx_s* pp_ctx;     /* device + stream                                  */
typedef struct pp_graph_s* pp_graph; /* device-resident CSR + CSC, owned by the library */

/* Bind a context to CUDA `device` and `cuda_stream` (a cudaStream_t or NULL).
 * The stream must outlive the context.  Fails with PP_ERR_CUDA without a GPU. */
pp_status pp_ctx_create(int device, void* cuda_stream, pp_ctx* out);
pp_status pp_ctx_destroy(pp_ctx ctx);
/* Number of kernels this library has launched on `ctx` so far (bench evidence). */
pp_status pp_ctx_launch_count(pp_ctx ctx, uint64_t* out);

/* ---- graph residency (P:358 CSR for push, P:318 A^T rows for pull) ----
 * A is n x n.  CSR row u lists the out-neighbours w, (u,w) in E: push expands
 * rows of CSR (= columns of A^T, Alg. 3).  CSC row v lists the in-neighbours u:
 * pull scans rows of A^T (Alg. 2).  Column ids must be < n; with
 * PP_GRAPH_VALIDATE offsets must be monotone with off[0]=0, off[n]=nnz, and each
 * row strictly increasing (sorted, no duplicates; PAPER.md:467 preprocessing).
 * Sorted rows are what make pull's early exit return the min-id parent.
 * PP_GRAPH_SYMMETRIC: csc_off/csc_idx may be NULL and then alias CSR (every
 * configuration here is undirected).  Host pointers unless
 * PP_GRAPH_DEVICE.  Offsets are stored on device as uint32 when nnz < 2^32,
 * else uint64.  Returns PP_ERR_GRAPH (message names the row) on a malformed
 * graph under VALIDATE, PP_ERR_OOM if it does not fit. */
#define PP_GRAPH_SYMMETRIC 1u
#define PP_GRAPH_DEVICE 2u
#define PP_GRAPH_VALIDATE 4u
/* PP_GRAPH_RELABEL: renumber vertices internally in order of decreasing degree (out + in;
 * ties by increasing id) and re-sort every row in that order (upload-time preprocessing,
 * DESIGN.md §5.3).  Every result is still reported in the caller's ids; the only visible
 * difference is which parent pp_bfs reports when several are valid: the in-neighbour at
 * depth-1 that comes FIRST in the internal order (highest degree, then lowest id) instead
 * of the lowest id.  Needs nnz, n < 2^31; single-GPU contexts only (else
 * PP_ERR_UNSUPPORTED). */
#define PP_GRAPH_RELABEL 8u
/* PP_GRAPH_OFF64: store 64-bit offsets even when nnz < 2^32 (the layout large graphs get;
 * lets tests exercise it on small graphs).  Results are identical. */
#define PP_GRAPH_OFF64 16u
/* Rows [row_lo, row_hi) are the rows this context owns:
 *  - single-GPU context: row_lo = 0, row_hi = n (else PP_ERR_ARG); offsets have n+1
 *    entries, nnz = off[n].
 *  - multi-rank context (pp_ctx_create_dist / pp_team_create, 1D row partition):
 *    [row_lo, row_hi) must be pp_partition(n, rank, nranks) (else PP_ERR_ARG); csr_off /
 *    csc_off are the block's row-local offsets (row_hi - row_lo + 1 entries starting at 0),
 *    ids are GLOBAL vertex ids, nnz = csr_off[row_hi - row_lo].  The library keeps only the
 *    block: its CSC rows (pull), the push structure (for every vertex u, u's out-neighbours
 *    inside the block, built on the device from the CSC rows) and the block's out-degrees;
 *    csr_idx is not used in a multi-rank context (may be NULL unless SYMMETRIC, where the
 *    CSR rows are the CSC rows).  With pp_ctx_create_dist the call is COLLECTIVE (the ranks
 *    exchange CUDA IPC handles of their exchange buffers over NCCL); in a team it is not.
 *    PP_GRAPH_RELABEL is rejected (PP_ERR_UNSUPPORTED). */
pp_status pp_graph_upload(pp_ctx ctx, int64_t n, int64_t row_lo, int64_t row_hi, int64_t nnz,
                          const int64_t* csr_off, const uint32_t* csr_idx, const int64_t* csc_off,
                          const uint32_t* csc_idx, uint32_t flags, pp_graph* out);
pp_status pp_graph_free(pp_graph g);
/* n, nnz, device bytes held by the handle (graph + BFS work buffers). */
pp_status pp_graph_info(pp_graph g, int64_t* n, int64_t* nnz, int64_t* device_bytes);

/* ---- vectors (P:83 sparse = sorted index list; P:435 DenseVector) ----------------------
 * LIST:   data = device uint32[capacity], ids sorted ascending and unique, nnz
 *         entries valid (outputs are produced sorted).
 * BITMAP: data = device uint32[ceil(n/32)], bit i of word i/32 = element i; bits
 *         >= n are zero on output.  nnz = popcount, or -1 = unknown on input. */
typedef enum { PP_VEC_LIST = 0, PP_VEC_BITMAP = 1 } pp_vec_format;
typedef struct {
  int32_t format;
  int64_t n;
  int64_t nnz;
  void* data;
  int64_t capacity; /* LIST: entries allocated in data; BITMAP: ignored */
} pp_vector;

/* ---- masked matvec GrB_mxv(w, mask, accum, semiring, A, u, desc) -------
 * Boolean semiring ({0,1}, AND, OR, 0) (Alg. 1 caption P:204; R3):
 *   t(i)    = OR_j  Op(i,j) AND u(j),  Op = A^T if transpose else A      Eq. 2, Eq. 3
 *   pass(i) = mask ? (mask(i) != 0) XOR complement : 1                  P:152, Alg. 2 line 3
 *   z(i)    = accum ? w_in(i) OR t(i) : t(i)                            Alg. 2 line 10 (R6)
 *   w(i)    = pass(i) ? z(i) : (replace ? 0 : w_in(i))                  Eq. 4, R5
 * direction PULL = row-based (Alg. 2, rows of Op, early exit on OR);
 * PUSH = column-based (Alg. 3, columns of Op, mask filter before the OR-merge);
 * AUTO = the Convert hysteresis of P:368/433 on nnz(u)/n vs switchpoint with
 * prev_nnz as its state (R25).  The result never depends on the
 * direction, only the time.  u / mask may be LIST or BITMAP (converted as
 * needed); w's format is the caller's choice; with accum or replace == 0, w
 * holds w_in on entry in that same format.  Errors: PP_ERR_ARG for complement
 * without a mask (R9) or a NULL vector; PP_ERR_DIM for length/format mismatch
 * or a LIST output whose capacity is too small (w->nnz then holds the needed
 * size); PP_ERR_UNSUPPORTED for a semiring other than PP_SR_LOR_LAND.
 * w->nnz is set when want_nnz (synchronises), else -1 for BITMAP output. */
typedef enum { PP_SR_LOR_LAND = 0 } pp_semiring;
typedef enum { PP_DIR_AUTO = 0, PP_DIR_PUSH = 1, PP_DIR_PULL = 2 } pp_direction;
typedef struct {
  const pp_vector* mask; /* NULL: no mask                                          */
  int32_t complement;    /* structural complement scmp                     */
  int32_t semiring;      /* PP_SR_LOR_LAND only                                    */
  int32_t accum;         /* 0: w = t ; 1: w = w_in OR t                            */
  int32_t replace;       /* 1: masked-out outputs are 0 (Eq. 4); 0: keep w_in      */
  int32_t direction;     /* pp_direction                                           */
  int32_t early_exit;    /* 1: stop a row at its first true term (only legal for OR) */
  int32_t transpose;     /* 1: w = A^T u (traversal, f' = A^T f); 0: w = A u       */
  int32_t want_nnz;      /* 1: compute w->nnz (synchronises)                       */
  double switchpoint;    /* AUTO threshold on nnz(u)/n, default 0.01       */
  int64_t prev_nnz;      /* Convert hysteresis state, -1 = none                    */
} pp_descriptor;
/* Fill *d with the defaults: no mask, replace=1, early_exit=1, transpose=1,
 * direction AUTO, switchpoint 0.01, prev_nnz -1, want_nnz 1. */
pp_status pp_descriptor_default(pp_descriptor* d);
pp_status pp_mxv(pp_graph g, pp_vector* w, const pp_descriptor* desc, const pp_vector* u);

/* ---- direction-optimised BFS, Algorithm 1 --------------------------------------
 * depth: int32[n], device or host memory (detected); 0 = unreached, source = 1,
 *   level-k vertices = k (Alg. 1 convention, R1).  Host memory means the
 *   result is copied back inside the call (end-to-end path).
 * parent: int32[n] or NULL; canonical min-id parent at depth-1 (R14; on a
 *   PP_GRAPH_RELABEL graph: first in the internal order), parent[source] = source,
 *   unreached = -1.
 * Direction per level (Opt. 1): mode DO uses `heuristic`:
 *   PP_HEUR_EDGES   Beamer edge-count rule (P:366 first sentence; R11), alpha=15, beta=18;
 *   PP_HEUR_PAPER_R the paper's r = nnz(f)/M rule (R10), alpha=beta=0.01;
 *   alpha/beta <= 0 select those defaults.  Level 1 is push (pull in PULL_ONLY).
 * Pull levels compute A^T v .* !v (operand reuse P:284, masking P:270, early
 * exit P:278); push levels compute A^T f .* !v column-wise (Alg. 3).
 * toggles (ablation) never change depths or parents.
 * stats (host, nullable): per-level direction / counters, synchronises.
 * Errors: PP_ERR_RANGE for a bad source, PP_ERR_TIMEOUT if the device watchdog
 * fired (never expected; depth is then invalid). */
typedef enum { PP_HEUR_EDGES = 0, PP_HEUR_PAPER_R = 1 } pp_heuristic;
typedef enum { PP_MODE_DO = 0, PP_MODE_PUSH_ONLY = 1, PP_MODE_PULL_ONLY = 2 } pp_mode;
#define PP_OPT_NO_MASKING 1u   /* pull scans every row, then filters by !v (Opt. 2 off) */
#define PP_OPT_NO_EARLYEXIT 2u /* pull scans whole rows (Opt. 3 off)                     */
#define PP_OPT_NO_REUSE 4u     /* pull tests the frontier f instead of v (Opt. 4 off)    */
typedef struct {
  int32_t heuristic;    /* pp_heuristic                                   */
  int32_t mode;         /* pp_mode                                        */
  double alpha, beta;   /* <= 0: defaults of the chosen heuristic          */
  int32_t want_parents; /* ignored if parent == NULL                       */
  uint32_t toggles;     /* PP_OPT_* (0 = all of the paper's optimisations) */
} pp_bfs_options;
pp_status pp_bfs_options_default(pp_bfs_options* o);

/* Per-level record of level k (1-based) at index k-1: dir (0 push, 1 pull),
 * c = |frontier discovered by level k|, m_f = sum of its out-degrees (Eq. 1),
 * m_u = sum of in-degrees still unvisited after level k, ns = device time of the
 * level (GPU %globaltimer between grid barriers, incl. a following convert).
 * Arrays are caller-owned host memory of `capacity` entries (any may be NULL).
 * levels = number of levels executed (= max depth); reached = #vertices with
 * depth > 0; init_ns = device time of the initialisation phase; cand / reached_nnz below. */
typedef struct {
  int32_t levels;
  int64_t reached;
  int32_t capacity;
  int8_t* dir;
  int64_t* c;
  int64_t* m_f;
  int64_t* m_u;
  int64_t* ns;
  int64_t init_ns;
  int64_t exchanged_bytes; /* multi-rank: bytes this rank stored into its peers' exchange
                              buffers over the BFS (frontier slices / id lists + records) */
  int64_t* cand;       /* per level: a pull's candidate rows (unvisited, not isolated: the rows
                          its masked mxv computes), a push's frontier size */
  int64_t reached_nnz; /* in-degree mass of the reached vertices = nnz of their rows of A^T
                          (undirected: the traversed component's edge entries) */
} pp_bfs_stats;

pp_status pp_bfs(pp_graph g, int64_t source, const pp_bfs_options* opts, int32_t* depth,
                 int32_t* parent, pp_bfs_stats* stats);

/* Diagnostics (load-balance evidence): the first call with levels > 0 makes every later
 * pp_bfs on g record, for each of its first `levels` levels and each persistent CTA, the
 * CTA's work time in that level's phase (ns, before the grid barrier).  A call with
 * out_ns != NULL copies the last BFS's records (levels x *nctas, level-major) to host. */
pp_status pp_bfs_debug_times(pp_graph g, int32_t levels, int64_t* out_ns, int32_t* nctas);
/* Diagnostics: after pp_bfs_debug_times(g, levels > 0, ...) enabled the records, copies three
 * planes of levels x nctas int64 (ns from each level's loop top, per CTA): [0] warp 0's work
 * done, [1] every warp of the CTA done (counters reduced), [2] the grid barrier released. */
pp_status pp_bfs_debug_phases(pp_graph g, int64_t* out_ns);
/* Diagnostics (profiling one level alone, e.g. the heaviest pull under ncu): runs levels
 * 1 .. level-1 of the BFS from `source` in one cooperative launch, hands the loop state over,
 * and runs level `level` ALONE in a second launch, then stops: depth (device int32[n]) holds
 * the depths up to level+1 (deeper vertices 0).  Single-GPU graphs; no parents. */
pp_status pp_bfs_debug_level(pp_graph g, int64_t source, int32_t level, const pp_bfs_options* opts,
                             int32_t* depth);

/* ---- multi-rank BFS: 1D row partition, exchange fused into the level kernel (SURVEY.md 8e,
 *      NEXT-1; P:516 names distributed GPUs as future work) --------------------------------
 * Rank p of P owns the vertex block [row_lo, row_hi) = pp_partition(n, p, P) and stores only
 * that block (see pp_graph_upload).  pp_bfs runs ONE cooperative kernel per rank for the whole
 * traversal: push levels expand the global frontier into owned targets, pull levels scan the
 * owned unvisited rows against the replicated visited bitmap; after every level the kernel
 * itself stores the owned words of the level's frontier bitmap and the rank's counters into
 * every peer's exchange buffer (peer memory over NVLink / NVSwitch), then one release flag per
 * peer; every rank then holds the global counters and takes the same push/pull decision
 * (R10/R11) with no host round trip and no host-issued collective.
 * One process per GPU: pp_nccl_unique_id (rank 0 creates the 128-byte NCCL id and shares it,
 * e.g. by a torch.distributed broadcast; PP_ERR_NCCL if libnccl.so.2 cannot be loaded) and
 * pp_ctx_create_dist (collective; the communicator is the bootstrap of the peer mappings).
 * pp_partition: rank's block [row_lo, row_hi): contiguous, 1024-vertex aligned, blocks of
 * ceil(ceil(n/32)/32/nranks)*1024 vertices (pure function, no GPU); pp_graph_partition
 * returns a graph's block.  pp_bfs on such a graph is collective: every rank passes the same
 * source/options; depth/parent hold the block's slice (row_hi - row_lo entries, same
 * conventions as single-GPU: min-id parents); stats are global and identical on all ranks.
 * nranks <= 8; ablation toggles and pp_mxv are single-GPU only (PP_ERR_UNSUPPORTED). */
pp_status pp_nccl_unique_id(void* out128);
pp_status pp_ctx_create_dist(int device, void* cuda_stream, const void* nccl_unique_id, int rank,
                             int nranks, pp_ctx* out);
pp_status pp_partition(int64_t n, int32_t rank, int32_t nranks, int64_t* row_lo, int64_t* row_hi);
pp_status pp_graph_partition(pp_graph g, int64_t* row_lo, int64_t* row_hi);

/* External bootstrap (one process per GPU without NCCL): pp_ctx_create_dist with
 * nccl_unique_id = NULL creates a multi-rank context without a communicator; after each rank's
 * pp_graph_upload (then not collective), every rank exports its 128-byte record
 * (pp_graph_export), the caller all-gathers them in rank order over any transport (e.g.
 * torch.distributed with gloo) and passes the nranks x 128 bytes to pp_graph_import, which
 * checks that the ranks agree and maps the peers' exchange buffers (CUDA IPC).  pp_bfs fails
 * with PP_ERR_ARG until then.  (With an NCCL communicator the upload does this itself.) */
pp_status pp_graph_export(pp_graph g, void* record128);
pp_status pp_graph_import(pp_graph g, const void* records);

/* Single-device team: nranks (<= 8) rank contexts on ONE device and stream, ctxs[r] = rank r.
 * Each rank uploads its block with pp_graph_upload (not collective); pp_bfs_team then runs
 * the P ranks as P CTA groups of ONE cooperative launch: the same kernel, the same peer stores,
 * counter records and cross-rank release/acquire flags as the multi-GPU path, with every
 * peer's exchange buffer on the same device.  It is how the multi-rank path is verified on one
 * GPU (tests/test_gpu_dist.py), and a way to run the partitioned layout on one GPU.
 * graphs[r] = rank r's graph (uploaded through ctxs[r]); depth[r] / parent[r] (parent may be
 * NULL, or entries NULL only together) = device slices of rank r's block; stats (host,
 * nullable) = the global per-level record (identical on every rank), synchronises.
 * Errors as pp_bfs; PP_ERR_ARG if the graphs are not ranks 0..nranks-1 of one team. */
pp_status pp_team_create(int device, void* cuda_stream, int32_t nranks, pp_ctx* ctxs);
pp_status pp_bfs_team(const pp_graph* graphs, int32_t nranks, int64_t source,
                      const pp_bfs_options* opts, int32_t* const* depth, int32_t* const* parent,
                      pp_bfs_stats* stats);

/* ---- SSSP over the min-plus semiring (Sec. 5.6) ------------
 * The paper's "simple 2-phase direction-optimized traversal" for SSSP: Bellman-Ford
 * d <- min(d, A^T (min.+) f) with an active-vertex frontier f; unmasked column-based (push)
 * mxv while nnz(f)/n <= alpha, then ONE switch to row-based (pull) mxv until f is empty.
 * No mask, no early exit; the pull reads all of d (operand reuse).  Jacobi
 * iteration, so the iteration count is deterministic (R28-R30).
 * Arguments (ALL pointers are DEVICE memory the caller owns; nothing is retained):
 *   csr_off[n+1] int64, csr_idx[nnz] uint32, csr_w[nnz] fp32: A by rows (out-edges, A(i,j)=w);
 *   csc_off/csc_idx/csc_w: the same matrix by columns (rows of A^T, in-edges);
 *   source in [0, n); alpha >= 0 the switch threshold on nnz(f)/n;
 *   dist[n] fp32 output: 0 at the source, +inf where unreachable.
 * Stream-ordered on the ctx stream: three prologue kernels, then the whole iteration loop in
 * ONE persistent cooperative kernel (frontier size and the push -> pull switch decided on the
 * device); synchronises twice: after reading off[0] / off[n] of both sides (argument check)
 * and at the end (error flags, stats) -- never per iteration.
 * Errors: PP_ERR_ARG (NULL / n <= 0 / alpha < 0), PP_ERR_RANGE (source), PP_ERR_GRAPH
 * (a negative or NaN weight), PP_ERR_CUDA / PP_ERR_OOM. */
typedef struct {
  int64_t iterations;        /* matvec steps run (the last one finds f empty)            */
  int64_t push_iterations;   /* column-based steps                                       */
  int64_t pull_iterations;   /* row-based steps                                          */
  int64_t switch_iteration;  /* index of the first pull step, -1 if none                 */
} pp_sssp_stats;
pp_status pp_sssp(pp_ctx ctx, int64_t n, int64_t nnz, const int64_t* csr_off, const uint32_t* csr_idx,
                  const float* csr_w, const int64_t* csc_off, const uint32_t* csc_idx,
                  const float* csc_w, int64_t source, double alpha, float* dist,
                  pp_sssp_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* PUSHPULL_H */
