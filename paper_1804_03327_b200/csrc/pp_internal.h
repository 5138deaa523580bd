// pp_internal.h — host-side internals of libpushpull (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "pushpull.h"

namespace pp {

// ---- tunables ---------------------------------------------------------------
constexpr int kBlock = 256;        // threads per CTA of every kernel
constexpr int kWarps = kBlock / 32;
#ifndef PP_HEAVY
#define PP_HEAVY 64
#endif
#ifndef PP_CHUNK
#define PP_CHUNK 64
#endif
constexpr unsigned kHeavy = PP_HEAVY;  // out-degree >= kHeavy: expanded as kChunk-edge chunks
constexpr unsigned kChunk = PP_CHUNK;  // edges per heavy chunk (whole warp iterations)
constexpr unsigned kSelfChunks = 32;  // heavy vertices with more chunks are hubs (block
                                      // descriptors, one per 32 chunks)
constexpr int kRing = 4;           // level-counter ring
#ifndef PP_SUM_WORDS
#define PP_SUM_WORDS 0
#endif
constexpr unsigned kSumWordsMax = PP_SUM_WORDS;  // visited summary words in shared memory (0 = off)
#ifndef PP_LOWLAT_EDGES
#define PP_LOWLAT_EDGES 32768
#endif
constexpr unsigned long long kLowLatEdges = PP_LOWLAT_EDGES;  // push levels expanding <= this
                                  // many edges: speculative offsets, no pre-test before atomicOr
constexpr unsigned kHubSplit = 2048;  // no-early-exit pull: longer row remainders are
                                      // processed grid-wide in chunks of this many ids
constexpr unsigned kBig = 1024;    // pull->push goes straight from the bitmap if no new
                                   // frontier vertex has out-degree >= kBig
#ifndef PP_BFS_BLOCK
#define PP_BFS_BLOCK 768  // round 2b: C4 6.6 -> 6.0 us per level, C2 equal
#endif
constexpr int kBfsBlock = PP_BFS_BLOCK;  // persistent BFS: one CTA per SM
constexpr int kBfsWarps = kBfsBlock / 32;
#ifndef PP_INIT_VEC
#define PP_INIT_VEC 1
#endif
constexpr bool kInitVec = PP_INIT_VEC != 0;  // BFS init: 16-byte depth stores
#ifndef PP_VREC
#define PP_VREC 1
#endif
constexpr bool kVrec = PP_VREC != 0;  // relabelled graphs: per-vertex {begin, deg, caller id}
#ifndef PP_DENSE
#define PP_DENSE 1
#endif
// dense pull levels (single GPU, 32-bit offsets): 32-byte row records streamed into shared
// memory by bulk copies (cp.async.bulk + mbarrier), one warp ring of kDenseR 1 KB slots
constexpr bool kDense = PP_DENSE != 0;
#ifndef PP_DENSE_R
#define PP_DENSE_R 1
#endif
#ifndef PP_DENSE_MIN8
#define PP_DENSE_MIN8 2
#endif
constexpr int kDenseR = kDense ? PP_DENSE_R : 0;  // ring slots (32 rows x 32 B) per warp
#ifndef PP_DENSE_IW
#define PP_DENSE_IW 8
#endif
constexpr int kDenseHead = 6;  // in-neighbour ids per row record (a 5-id record with the row
                               // begin instead of the sixth id measured equal)
constexpr unsigned kDenseIW = PP_DENSE_IW;  // bitmap words per dense work item
constexpr int kMaxRanks = 8;  // 1D row partition: ranks per multi-rank group (one node)
constexpr int kMaxCtas = 1024;  // persistent grid size bound (per-CTA work counters)

// Per-level counters, written with atomics during a level, read after the grid barrier.
// The three atomic populations sit on separate 128-byte L2 lines: the per-CTA counter flush
// (c, m_f, m_fin, nbig, cand), the per-warp light-list appends (nL), and the heavy-chunk
// appends / work counters — same-line atomics serialise in one L2 slice.  (Each flushed
// counter on its own line measured equal: DESIGN.md §11b.)
struct LevelCtr {
  unsigned long long c;      // vertices discovered by the level
  unsigned long long m_f;    // sum of their out-degrees (Eq. 1)
  unsigned long long m_fin;  // sum of their in-degrees (m_u update, directed graphs)
  unsigned long long nbig;   // discoveries with out-degree >= kBig (pull levels)
  unsigned long long cand;   // rows the pull computed (unvisited, non-isolated)
  unsigned int pad0[22];
  unsigned int nL;           // next frontier: light-list length
  unsigned int pad1[31];
  unsigned int nH, nB;       // next frontier: heavy-chunk count, hub block descriptors
  unsigned int work, work2;  // dynamic work counters (phase, convert phase)
  unsigned int nX;           // multi-rank push: discoveries appended to the rank's id list
  unsigned int pad2[27];
};
static_assert(sizeof(LevelCtr) == 384, "LevelCtr layout");


struct LevelStat {
  int dir;
  int pad;
  long long c, m_f, m_u;
  long long cand;  // pull: rows computed; push: frontier vertices expanded
  long long t_ns;  // %globaltimer when the level's barrier released (block 0)
};

// Narrow -> wide hand-over of the BFS loop state (bfs.cu, narrow mode).
struct BfsResume {
  int valid, done;  // valid: the wide kernel continues at level d; done: BFS finished
  int d, dir, cur, sel, from_bits, pad;
  unsigned nL, nH, nB, pad2;
  long long c_old, m_u, reached, mf_last;
};
constexpr int kNarrowCtas = 8;  // narrow mode: one thread-block cluster of this many CTAs
#ifndef PP_NARROW_MAX_EDGES
#define PP_NARROW_MAX_EDGES 131072
#endif
constexpr unsigned long long kNarrowMaxEdges = PP_NARROW_MAX_EDGES;  // hand over to the whole
                                  // grid before a push expanding more edges, or a pull
#ifndef PP_NARROW_MAX_DEG
#define PP_NARROW_MAX_DEG 64
#endif
constexpr int64_t kNarrowMaxDeg = PP_NARROW_MAX_DEG;  // auto: narrow start for graphs whose max
                                  // out-degree is at most this (mesh / road / geometric graphs)
struct GridBarrier {
  unsigned long long count;  // monotone arrival counter (bit 63: abort), zeroed per launch
  unsigned int pad0[30];
  unsigned int gen;
  unsigned int pad1[31];
  BfsResume rs;
};

// Device-side BFS status words.
struct BfsStatus {
  int error;   // 0 or pp_status
  int levels;  // levels executed
  long long reached;
  long long reached_nnz;      // in-degree mass of the reached vertices
  long long t_start, t_init;  // %globaltimer at kernel entry / after the init barrier
  long long xbytes;           // multi-rank: bytes this rank stored into its peers' buffers
};

}  // namespace pp

struct pp_team_s;  // single-device team of rank contexts (pp_team_create)

struct pp_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  uint64_t launches = 0;
  int refs = 1;  // the caller's handle + one per live graph
  int rank = 0, nranks = 0;  // nranks > 0: multi-rank context (one process per GPU, or a team)
  void* comm = nullptr;      // NCCL communicator (bootstrap of the peer mappings), or nullptr
  pp_team_s* team = nullptr;  // team member: the peers live on the same device
  void* sssp_ws = nullptr;  // pp_sssp workspace (grown on demand, freed with the context)
  size_t sssp_ws_bytes = 0;
};

struct pp_graph_s {
  pp_ctx ctx = nullptr;
  int64_t n = 0, nnz = 0;
  bool symmetric = false;
  bool off64 = false;
  uint32_t nwords = 0;  // bitmap words, padded to a multiple of 32 (one warp-chunk)
  void* off = nullptr;  // uint32 or uint64 [n+1]  (CSR, out-neighbours)
  uint32_t* idx = nullptr;
  void* coff = nullptr;  // CSC (in-neighbours); aliases off when symmetric
  uint32_t* cidx = nullptr;
  uint32_t* isolated = nullptr;  // nwords: bit = no in- and no out-edges, or padding
  uint32_t* drec = nullptr;      // PP_DENSE: per row {first 6 in-neighbours, caller id, in-degree}
                                 // (32 B; nwords*32 rows, padding rows zero)
  int64_t n_noniso = 0;          // rows not marked isolated / padding (multi-rank: all ranks')
  int64_t n_noniso_block = 0;    // multi-rank: this block's
  // PP_GRAPH_RELABEL: internal id = rank by decreasing degree (relabel.cu)
  uint32_t* perm = nullptr;  // internal -> caller id (nullptr: ids are the caller's)
  uint32_t* rank = nullptr;  // caller -> internal id
  uint32_t* pint = nullptr;  // BFS parents in internal ids (atomicMin key space)
  uint32_t* rbits[4] = {nullptr, nullptr, nullptr, nullptr};  // mxv: u, mask, w_in, w (internal)
  // BFS working set
  uint32_t* vis[2] = {nullptr, nullptr};
  uint32_t* fr = nullptr;  // frontier bitmap of the last pull level
  uint32_t* sumv = nullptr;  // visited summary (1 bit per 2^sum_shift vertices)
  int sum_shift = 3;
  uint32_t sum_words = 0;
  uint32_t* L[2] = {nullptr, nullptr};
  uint2* H[2] = {nullptr, nullptr};
  int64_t hcap = 0;
  pp::LevelCtr* ctr = nullptr;
  pp::LevelStat* stats = nullptr;
  int stats_cap = 0;
  pp::GridBarrier* bar = nullptr;
  pp::BfsStatus* status = nullptr;
  unsigned* gwork = nullptr;  // [kRing][kMaxCtas] per-CTA pull item counters
  pp::BfsStatus* status_host = nullptr;  // pinned
  // mxv scratch
  uint32_t* sbits[4] = {nullptr, nullptr, nullptr, nullptr};  // t, u, mask, w (bitmaps)
  uint32_t* sblock = nullptr;        // per-block counts for bitmap->list
  uint4* hubq = nullptr;             // row-mxv long-row chunks {row, len, start}
  unsigned long long* scount = nullptr;  // device counters (mxv)
  unsigned long long* scount_host = nullptr;
  int64_t max_out_deg = 0;
  uint4* vrec = nullptr;         // relabelled graph: {begin lo, hi, out-degree, caller id} per vertex       // max CSR row length (narrow-mode auto decision)
  int64_t* dtmp[2] = {nullptr, nullptr};  // upload staging / host-output staging
  int bfs_grid = 0;
  long long* dbg = nullptr;  // pp_bfs_debug_times: per level x CTA phase durations
  int dbg_levels = 0;
  int64_t device_bytes = 0;
  // multi-rank (1D row partition): rank `rank` of `nranks` owns vertices
  // [row_lo, row_hi) = bitmap words [rank*chunk_words, (rank+1)*chunk_words).  off/idx hold
  // the PUSH structure (for every global u, its out-neighbours inside the block), coff/cidx
  // the CSC rows of the block (local row = v - row_lo), bitmaps are global (nwords words).
  bool dist = false;
  int me = 0, nranks = 1;  // this graph's rank index, ranks
  int64_t row_lo = 0, row_hi = 0, chunk_words = 0, in_total = 0;
  uint32_t* odeg = nullptr;  // directed: global out-degree of the owned rows
  void* xbuf = nullptr;      // exchange buffer: frontier[2] bitmaps, counter records, flags
  uint32_t* xfr[2] = {nullptr, nullptr};
  unsigned long long* xcnt = nullptr;   // [2][kMaxRanks][8] counter records (by sender)
  uint32_t* xlst[2] = {nullptr, nullptr};  // id-list receive areas (sender q: words [q*cw, (q+1)*cw))
  uint32_t* xown = nullptr;  // this rank's discoveries of the current push level (<= cw ids)
  unsigned long long* xflag = nullptr;  // [kMaxRanks] arrival epochs (by sender)
  uint32_t* pfr[pp::kMaxRanks][2] = {};  // every rank's frontier buffers (own at [me])
  unsigned long long* pcnt[pp::kMaxRanks] = {};
  uint32_t* plst[pp::kMaxRanks][2] = {};
  unsigned long long* pflag[pp::kMaxRanks] = {};
  void* ipc_base[pp::kMaxRanks] = {};  // peer xbufs opened through CUDA IPC (multi-process)
  uint64_t xseq = 0;  // BFS calls so far (epoch of the cross-rank flags)
  bool attached = false;  // peers mapped (bootstrap done)
  void* dargs = nullptr;  // device copy of the kernel arguments (multi-rank launch)
  void* hargs = nullptr;  // pinned staging of the same
};

struct pp_team_s {
  int device = 0;
  int nranks = 0;
  int refs = 0;  // member contexts alive
  pp_ctx ctx[pp::kMaxRanks] = {};
  pp_graph graphs[pp::kMaxRanks] = {};  // the graph most recently uploaded by each rank
};

namespace pp {
void set_error(const char* fmt, ...);
pp_status cuda_fail(cudaError_t e, const char* what);

// launchers (bfs.cu / mxv.cu / graph.cu); each returns cudaSuccess or the launch error
cudaError_t launch_graph_prepare(pp_graph g, const int64_t* d_off64, const int64_t* d_coff64,
                                 unsigned long long* d_scratch, uint64_t* launches);
cudaError_t launch_graph_validate(pp_graph g, const int64_t* d_off64, const uint32_t* d_idx,
                                  unsigned long long* d_bad, uint64_t* launches, int64_t rows = -1);
cudaError_t launch_off_narrow(pp_graph g, const int64_t* in, void* out, int64_t m);
cudaError_t launch_drec(pp_graph g, const int64_t* coff, const uint32_t* cidx, int64_t rows);
cudaError_t launch_hcap(pp_graph g, const int64_t* off, int64_t rows, unsigned long long* d_cap,
                        unsigned long long* d_max);
int bfs_grid_size(pp_graph g, bool parents);
cudaError_t launch_bfs(pp_graph g, uint32_t source, int mode, int rule, double alpha, double beta,
                       uint32_t toggles, int32_t* depth, uint32_t* parent, int max_levels,
                       int split_level = 0);

struct MxvPlan {
  int pull;              // 1 = row-based (Alg. 2), 0 = column-based (Alg. 3)
  int transpose;         // operator A^T (1) or A (0)
  const uint32_t* u_bits;  // u as bitmap (pull) or nullptr
  const uint32_t* u_list;  // u as list (push) or nullptr
  int64_t u_nnz;
  const uint32_t* mask_bits;  // nullptr = no mask
  int complement, accum, replace, early_exit;
  const uint32_t* win_bits;  // w_in as bitmap (may alias out_bits)
  uint32_t* out_bits;        // result bitmap
};
cudaError_t launch_relabel(pp_graph g, const int64_t* d_off64, const int64_t* d_coff64,
                           int64_t* new_off64, int64_t* new_coff64, uint64_t* launches);
cudaError_t launch_permute_bits(pp_graph g, const uint32_t* in, bool to_internal, uint32_t* out);
cudaError_t launch_list_to_bitmap(pp_graph g, const uint32_t* list, int64_t m, uint32_t* bits,
                                  unsigned long long* d_bad);
cudaError_t launch_mxv(pp_graph g, const MxvPlan& p);
cudaError_t launch_popcount(pp_graph g, const uint32_t* bits, unsigned long long* d_out);
cudaError_t launch_bitmap_to_list(pp_graph g, const uint32_t* bits, uint32_t* list,
                                  int64_t capacity, unsigned long long* d_count);

// dist.cu
bool nccl_load(const char** why);
int nccl_unique_id(void* out128, const char** why);
int nccl_comm_init(void** comm, int nranks, const void* id128, int rank, const char** why);
int nccl_allgather_host(void* comm, const void* send, void* recv, size_t bytes, int nranks,
                        cudaStream_t st, const char** why);
void nccl_comm_destroy(void* comm);
void partition(int64_t n, int rank, int nranks, int64_t* lo, int64_t* hi, int64_t* chunk_words);
cudaError_t launch_push_structure(pp_graph g, const int64_t* d_coff64, int64_t rows, int64_t m,
                                  int64_t* poff64, uint32_t* pidx);
cudaError_t launch_block_prepare(pp_graph g, const int64_t* d_off64, const int64_t* d_coff64,
                                 int64_t rows);
// bfs.cu: one cooperative launch, graphs[r] = rank r's state; nranks = 1 for one process per
// GPU, nranks = P for a single-device team (P CTA groups)
cudaError_t launch_bfs_ranks(pp_graph* graphs, int nranks, uint32_t source, int mode, int rule,
                             double alpha, double beta, int32_t* const* depth,
                             uint32_t* const* parent);
size_t bfs_args_bytes();  // device buffer for kMaxRanks kernel-argument blocks
}  // namespace pp
