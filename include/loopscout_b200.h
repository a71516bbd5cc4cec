/*
 * loopscout_b200.h — C-ABI of the B200 batched schedule-cost engine.
 *
 * This is the drop-in boundary for the reference's batched cost-evaluation
 * path (Tuna / `loopscout`, /root/reference/pkg/src/loopscout).  The
 * reference evaluates one candidate schedule at a time in Python:
 *
 *   evaluate_population            ls/es.py:96-116   (batched seam)
 *     apply_schedule               ls/ir.py:454-474
 *     emit_mock_asm                ls/ir.py:557-659
 *     extract_features             ls/cost.py:132-152
 *     score                        ls/cost.py:155-161
 *   rank / cmd_rank sort           ls/cost.py:164-168, ls/cli.py:124-126
 *
 * Here a *task* (one loop-nest program + one schedule template + one
 * architecture) is created once, and candidates arrive as packed 32-byte
 * records.  Every entry point takes plain pointers and sizes; device
 * pointers are CUDA global-memory pointers owned by the caller, `stream` is a
 * cudaStream_t passed as void*.  Functions return 0 on success or a negative
 * LS_E_* code; ls_last_error() returns the thread-local message.
 *
 * Ownership: the library never frees caller buffers; an ls_task is owned by
 * the library, immutable after ls_task_create (except the unroll table, which
 * only grows), and may be used concurrently from distinct streams.
 */
#ifndef LOOPSCOUT_B200_H
#define LOOPSCOUT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LS_ABI_VERSION 1

/* ---- capacity limits of the descriptor (host-side; checked on create) ---- */
#define LS_MAX_TENSORS 8
#define LS_MAX_RANK 6
#define LS_MAX_TERMS 8     /* terms per index expression of the base program */
#define LS_MAX_NODES 64    /* nodes (loops + accesses) of the base program    */
#define LS_MAX_VARS 32     /* loop variables incl. names created by tiling    */
#define LS_MAX_XFORMS 32   /* transforms in one schedule template            */
#define LS_MAX_PARAMS 8    /* uint16 parameter slots per record               */
#define LS_MAX_ORDER 16    /* loops permuted by one Reorder (nibble-packed)   */
#define LS_MAX_CHAIN 16    /* loops in a transformed perfect chain            */
#define LS_NFEAT_CPU 5     /* CPU_FEATURES, ls/cost.py:24                     */
#define LS_NFEAT_GPU 7     /* GPU_FEATURES, ls/cost.py:25-26                  */
#define LS_MAX_AXES 16     /* axes of an attached schedule space              */

/* ---- enums ---- */
enum { LS_FAMILY_CPU = 0, LS_FAMILY_GPU = 1 };                  /* ArchSpec.family */
enum { LS_TARGET_X86 = 0, LS_TARGET_AARCH64 = 1, LS_TARGET_PTX = 2 }; /* ls/ir.py:554 */
/* reg_effects only distinguishes "x86-att" from everything else (ls/ilp.py:98-103) */
enum { LS_DIALECT_X86_ATT = 0, LS_DIALECT_DEST_FIRST = 1 };
enum { LS_NODE_LOOP = 0, LS_NODE_ACCESS = 1 };
enum {                                                          /* ls/ir.py:276-303 */
  LS_XF_TILE = 0,
  LS_XF_REORDER = 1,
  LS_XF_UNROLL = 2,
  LS_XF_VECTORIZE = 3,
  LS_XF_PARALLEL = 4
};
/* The instruction shapes the mock emitter produces (ls/ir.py:584-658). */
enum {
  LS_I_INIT = 0,   /* counter init: movq $0 / mov x,#0 / mov.u32 r,0 */
  LS_I_LOAD = 1,   /* vector load                                     */
  LS_I_FMA = 2,    /* fused multiply-add into accumulator             */
  LS_I_STORE = 3,  /* vector store                                    */
  LS_I_ADD = 4,    /* counter increment                               */
  LS_I_CMP = 5,    /* cmpq / cmp / setp                               */
  LS_I_BRANCH = 6, /* jne / b.ne / @p bra                             */
  LS_I_RET = 7,
  LS_I_COUNT = 8
};

/* ---- scoring paths (ls_task_set_path) ---- */
enum {
  LS_PATH_AUTO = 0,      /* tabulated when the task is eligible, else generic            */
  LS_PATH_GENERIC = 1,   /* per-candidate strided-interval folds (every perfect chain)   */
  LS_PATH_TABULATED = 2, /* dimension counts looked up in a per-task table */
  LS_PATH_SPACE = 3      /* points calls on tile+reorder spaces: chain order per reorder choice,
                            fused walk + closed-form terms; else as TABULATED      */
};

/* ---- error codes (return values) ---- */
enum {
  LS_E_OK = 0,
  LS_E_ARG = -1,         /* bad argument / descriptor */
  LS_E_CUDA = -2,        /* CUDA runtime error        */
  LS_E_UNSUPPORTED = -3, /* task outside the device class */
  LS_E_NOMEM = -4
};

/* ---- per-candidate status (mirrors the reference's exceptions) ---- */
enum {
  LS_OK = 0,
  LS_ST_NO_LOOP = 1,         /* ProgramError "no loop named"      ls/ir.py:151       */
  LS_ST_TILE_RANGE = 2,      /* tile factor out of range          ls/ir.py:363-364   */
  LS_ST_VEC_DIVIDE = 3,      /* vectorize width does not divide   ls/ir.py:465-468   */
  LS_ST_VEC_ZERO = 4,        /* vectorize width 0: ZeroDivisionError, ls/ir.py:465   */
  LS_ST_REORDER_MISSING = 5, /* reorder: missing loops            ls/ir.py:416-417   */
  LS_ST_REORDER_CHAIN = 6,   /* reorder: not a perfect nest chain ls/ir.py:398-399   */
  LS_ST_BAD_FEATURE = 7,     /* CostModelError non-finite/negative ls/cost.py:43-45  */
  LS_ST_UNSUPPORTED = 16,    /* transformed tree outside the device class            */
  LS_ST_UNROLL_TABLE = 17,   /* unroll product not prepared (ls_task_prepare_unroll) or
                                above 65536 (its block is scheduled on the host: outside
                                the device class; the reference has no limit)       */
  LS_ST_OVERFLOW = 18,       /* intermediate exceeded the device integer range       */
  LS_ST_POINT_RANGE = 19     /* space point outside the attached space (points API)  */
};

/* ---- task descriptor: the per-task parameter table ---- */
typedef struct {
  int32_t var;  /* variable id */
  int32_t coef; /* nonzero coefficient */
} ls_term;

typedef struct {
  int32_t n_terms;
  int32_t konst;
  ls_term terms[LS_MAX_TERMS]; /* sorted by var_rank (AffineExpr order, ls/ir.py:53) */
} ls_expr;

typedef struct {
  int32_t kind;   /* LS_NODE_LOOP / LS_NODE_ACCESS */
  int32_t parent; /* node index of the parent loop, -1 for the program body; nodes are in preorder */
  /* loop fields (ls/ir.py:108-116) */
  int32_t var, extent, step, parallel, unrolled, vector_width; /* vector_width 0 = None */
  /* access fields (ls/ir.py:101-105) */
  int32_t tensor, is_store;
  ls_expr idx[LS_MAX_RANK];
} ls_node;

typedef struct {
  int32_t rank;
  int32_t elem_bytes;
  int32_t shared; /* scope == "shared" */
  int32_t dims[LS_MAX_RANK];
} ls_tensor;

typedef struct {
  int32_t kind;       /* LS_XF_* */
  int32_t var;        /* target loop variable id (-1: name never exists -> LS_ST_NO_LOOP) */
  int32_t new_var;    /* TILE/VECTORIZE: id of the inner loop variable created */
  int32_t param;      /* TILE/VECTORIZE: record param slot of the factor/width, -1 = use value */
  int32_t value;      /* constant factor/width when param < 0 */
  int32_t enable_bit; /* -1 = always applied, else bit index of ls_record.flags */
  int32_t n_order;    /* REORDER: number of names in the order */
  int32_t perm_shift; /* REORDER: first nibble of this order in ls_record.perm */
  int32_t order[LS_MAX_ORDER]; /* REORDER: candidate var ids; nibble j picks the var at position j */
} ls_xform;

typedef struct {
  int32_t abi_version; /* LS_ABI_VERSION */
  int32_t family, target, dialect;
  int32_t n_tensors;
  ls_tensor tensors[LS_MAX_TENSORS];
  int32_t n_nodes;
  ls_node nodes[LS_MAX_NODES];
  int32_t n_vars;
  int32_t var_rank[LS_MAX_VARS]; /* rank of each var name in Python string order */
  int32_t tid_var;               /* id of the var literally named "tid", -1 if none */
  int32_t n_xforms;
  ls_xform xforms[LS_MAX_XFORMS];
  double coef[LS_NFEAT_GPU];   /* coefficients in feature order (ls/cost.py:155-161) */
  int64_t cache_capacity;      /* CacheSpec.capacity_elements (ls/cost.py:97) */
  int32_t issue_width;         /* SchedSpec.issue_width */
  int32_t lat[LS_I_COUNT];     /* SchedSpec.latency_of for each emitted shape */
  int32_t klass[LS_I_COUNT];   /* latency-class id per shape (same id <=> same class string) */
  int32_t unit_cap[LS_I_COUNT];/* per class id: SchedSpec.units cap, 0 = uncapped */
  double ptx_cost[LS_I_COUNT]; /* GpuSpec.instr_cost per shape root (default 1) */
  double sm_underuse;          /* per-task constant, ls/ptx.py:238-241 */
  double warp_slack;           /* per-task constant, ls/ptx.py:253-256 */
  int32_t banks, warp_size;    /* GpuSpec.banks / warp_size (32 / 32) */
} ls_task_desc;

/* ---- packed candidate record (32 bytes, 16-byte aligned) ---- */
typedef struct {
  uint16_t param[LS_MAX_PARAMS]; /* tile factors / vector widths by template slot */
  uint64_t perm;                 /* nibble-packed reorder permutations */
  uint32_t flags;                /* enable bits of optional transforms */
  uint32_t tag;                  /* reserved, must be 0 */
} ls_record;

/* ---- schedule space (space_axes, ls/ir.py:517-547) for the points API ---- */
enum {
  LS_AX_PARAM = 0, /* tile axis: values[c] -> ls_record.param[param]                       */
  LS_AX_PERM = 1,  /* reorder axis: values[c] OR-ed into ls_record.perm (already shifted)   */
  LS_AX_VEC = 2,   /* vectorize axis: values[c] -> param[param]; flags bit set iff != 0     */
  LS_AX_BIT = 3    /* unroll/parallel on-off axis: choice index c -> flags bit              */
};
typedef struct {
  int32_t kind;           /* LS_AX_* */
  int32_t param;          /* PARAM/VEC: record param slot */
  int32_t bit;            /* VEC/BIT: enable bit */
  int32_t n_choices;      /* >= 1 */
  const uint64_t* values; /* host array of n_choices values (unused for BIT) */
} ls_axis;

typedef struct {
  int32_t n_axes;
  ls_axis axes[LS_MAX_AXES];
} ls_space_desc;

typedef struct ls_task ls_task;

/* ---- entry points ---- */
const char* ls_last_error(void);
int ls_abi_version(void);

/* Validate and upload a task.  Replaces the per-candidate re-derivation of
 * load_arch (ls/cost.py:81-129), the emitter's fixed block shapes
 * (ls/ir.py:614-658) and schedule_block of those blocks (ls/ilp.py:158-204),
 * which are computed once here instead of once per candidate. */
int ls_task_create(const ls_task_desc* desc, int device, ls_task** out);
int ls_task_destroy(ls_task* task);
int ls_task_num_features(const ls_task* task);
/* Select the scoring path (LS_PATH_*); all give bit-identical results.
 * LS_PATH_AUTO takes the fastest eligible one.  LS_E_UNSUPPORTED if the task
 * is not eligible for LS_PATH_TABULATED / LS_PATH_SPACE.  Not thread-safe
 * against concurrent scoring calls on the same task. */
int ls_task_set_path(ls_task* task, int32_t path);
/* The path record calls (ls_score*) take: LS_PATH_GENERIC or LS_PATH_TABULATED. */
int ls_task_path(const ls_task* task);
/* The path points calls (ls_score*_points*) take: LS_PATH_GENERIC,
 * LS_PATH_TABULATED or LS_PATH_SPACE (needs ls_task_set_space first). */
int ls_task_points_path(const ls_task* task);
/* Precompute block-cycle entries for innermost-unroll products `u_values`
 * (candidates needing an unprepared product report LS_ST_UNROLL_TABLE). */
int ls_task_prepare_unroll(ls_task* task, const int64_t* u_values, int32_t n);

/* The cache model's inexact-footprint flag per record (NodeCost.inexact of CacheModel.run) and
 * the (loop, tensor) pairs of its diagnostic "inexact footprint for tensor T at loop L"
 * (ls/cache.py:198-202): d_flags[n] 0 exact, 1 inexact, 255 the record fails apply_schedule;
 * d_masks[2n] (optional) bit 8 * chain position + tensor index (position 0 = outermost loop;
 * the notes run innermost first, tensors in first-access order); d_chains[16n] (optional) the
 * loop slot (template variable id) at each chain position, 0xFF past the chain.  Device
 * arrays; stream-ordered.  Perfect chains (LS_E_UNSUPPORTED on a tree task). */
int ls_inexact_footprints(ls_task* t, const ls_record* d_records, int64_t n, uint8_t* d_flags,
                          unsigned long long* d_masks, uint8_t* d_chains, void* stream);
/* Distinct innermost-unroll products U needed by the structurally supported
 * records (device pass), sorted; feed them to ls_task_prepare_unroll before
 * scoring.  Only needed when the template or program marks loops `unroll`.
 * LS_E_UNSUPPORTED when a batch needs more than 16384 distinct products,
 * LS_E_ARG when they do not fit `cap`. */
int ls_collect_unroll(ls_task* task, const ls_record* d_records, int64_t n, int64_t* h_values,
                      int32_t cap, int32_t* h_count, void* stream);

/* Score n records.  Replaces evaluate_population + apply_schedule +
 * emit_mock_asm + extract_features + score (ls/es.py:96-116,
 * ls/cost.py:132-161).  Any output pointer may be NULL.  d_features is
 * n x ls_task_num_features row-major float64. */
int ls_score(ls_task* task, const ls_record* d_records, int64_t n, double* d_scores,
             double* d_features, int32_t* d_status, void* stream);

/* Score n records and return the k best by (score, base_index + i),
 * ascending, fused in one pass (cmd_rank sort, ls/cli.py:124-126; rank,
 * ls/cost.py:164-168).  Failed candidates are excluded.  Unfilled slots
 * carry score +inf and index -1.  *d_n_valid (nullable) receives the number
 * of successfully scored candidates. */
int ls_score_topk(ls_task* task, const ls_record* d_records, int64_t n, int64_t base_index,
                  int32_t k, double* d_top_scores, int64_t* d_top_index, int64_t* d_n_valid,
                  void* stream);

/* ---- multi-GPU top-k merge (no reference equivalent: the
 * reference is single-process, its order is cmd_rank's (score, index) sort,
 * ls/cli.py:124-126) ----
 * A top-k entry as one 16-byte key: the float64 score mapped to order-preserving
 * unsigned bits (negative scores bit-inverted, others with the sign bit set) and
 * the global index; (order, index) compare lexicographically.  An empty slot is
 * order = UINT64_MAX, index = INT64_MAX.  One all-gather of k keys per rank
 * (ncclAllGather of 16k bytes, or torch.distributed.all_gather_into_tensor)
 * followed by ls_topk_merge_keys on every rank gives the single-GPU answer. */
typedef struct ls_topk_key {
  uint64_t order;
  int64_t index;
} ls_topk_key;

/* Merge n_lists top-k lists (k_in entries each, contiguous, any order; index
 * < 0 marks an empty slot) into the k_out best by (score, index).  No
 * temporary allocation. */
int ls_topk_merge(const double* d_scores, const int64_t* d_index, int32_t n_lists, int32_t k_in,
                  int32_t k_out, double* d_out_scores, int64_t* d_out_index, void* stream);
/* Merge m gathered keys (any order, empty slots allowed) into the k_out best,
 * written as (score, index) ascending; unfilled slots +inf / -1. */
int ls_topk_merge_keys(const ls_topk_key* d_keys, int64_t m, int32_t k_out, double* d_out_scores,
                       int64_t* d_out_index, void* stream);
/* Pack m (score, index) entries into keys (index < 0 -> empty key). */
int ls_topk_to_keys(const double* d_scores, const int64_t* d_index, int64_t m, ls_topk_key* d_keys,
                    void* stream);
/* The whole multi-GPU step over NCCL: this rank's k best
 * (d_scores / d_index, from ls_score_topk*) are packed into d_scratch[rank*k ..
 * (rank+1)*k), one in-place ncclAllGather of 16k bytes per rank fills
 * d_scratch[world*k], and the merge kernel writes the global k best (identical
 * on every rank, equal to the single-GPU answer).  nccl_comm is the caller's
 * ncclComm_t (rank / world of it); the library binds ncclAllGather from the
 * libnccl.so.2 already loaded in the process (else dlopen), LS_E_UNSUPPORTED
 * when there is none.  Stream-ordered, no allocation. */
int ls_topk_allgather_merge(void* nccl_comm, int32_t rank, int32_t world, const double* d_scores,
                            const int64_t* d_index, int32_t k, ls_topk_key* d_scratch, double* d_out_scores,
                            int64_t* d_out_index, void* stream);

/* Host-buffer variant of ls_score_topk: records in host memory (pinned or
 * pageable), results written to host memory.  Mapped page-locked buffers
 * (cudaHostAlloc / torch pin_memory under UVA) are read by the scoring kernel
 * over the host link (the transfer overlaps the scoring, no staging copy);
 * other buffers are copied host->device in chunks overlapped with scoring.
 * Synchronous. */
int ls_score_topk_host(ls_task* task, const ls_record* h_records, int64_t n, int64_t base_index,
                       int32_t k, double* h_top_scores, int64_t* h_top_index, int64_t* h_n_valid,
                       void* stream);

/* ---- points API: candidates as space points ----
 * A point is the mixed-radix number of a candidate's per-axis choice indices,
 * axis 0 most significant: the flat index of the choices ThetaEncoding.decode
 * picks (ls/es.py:57-62) over space_axes (ls/ir.py:517-547).  Points are 3-,
 * 4- or 8-byte little-endian unsigned integers (point_bytes; 3 = packed, for
 * spaces below 2^24 points); a 4-byte point is an 8x smaller candidate than an
 * ls_record.  Results are identical to scoring the records the points decode to. */

/* Attach the task's schedule space (copied; replaces a previous one). */
int ls_task_set_space(ls_task* task, const ls_space_desc* space);
/* ls_score over points. */
int ls_score_points(ls_task* task, const void* d_points, int32_t point_bytes, int64_t n, double* d_scores,
                    double* d_features, int32_t* d_status, void* stream);
/* ls_score_topk over points. */
int ls_score_topk_points(ls_task* task, const void* d_points, int32_t point_bytes, int64_t n,
                         int64_t base_index, int32_t k, double* d_top_scores, int64_t* d_top_index,
                         int64_t* d_n_valid, void* stream);
/* ls_score_topk_host over host points (mapped, or H2D staged and overlapped). */
int ls_score_topk_points_host(ls_task* task, const void* h_points, int32_t point_bytes, int64_t n,
                              int64_t base_index, int32_t k, double* h_top_scores, int64_t* h_top_index,
                              int64_t* h_n_valid, void* stream);

/* ---- ES search on device (throughput mode of optimize, ls/es.py:130-204) ----
 * Every generation runs on the device with no host round trip: Gaussian noise
 * from Philox4x32-10 keyed by (seed, generation) with counter (member, pair)
 * and Box-Muller (not numpy's PCG64 stream: trajectories differ from the
 * reference's optimize; es.optimize is the exact-trajectory parity mode),
 * ThetaEncoding.decode, the memo of distinct schedules keyed by space point,
 * scoring of new points, the rank-shaped update and the incumbent trace.  The
 * task needs an attached space (ls_task_set_space); axes follow space_axes. */
typedef struct {
  double alpha, sigma;          /* EsParams (ls/es.py:26-41) */
  int32_t population, iterations;
  uint64_t seed;
  int32_t rank_normalize, pad;
} ls_es_params;

typedef struct ls_es ls_es;

/* Allocate a run (memo table sized for min(space, population*iterations+1)
 * distinct schedules, at most 2^28: LS_E_UNSUPPORTED above).  h_theta0: start
 * vector (NULL: ThetaEncoding.initial). */
int ls_es_create(ls_task* task, const ls_es_params* params, const double* h_theta0, ls_es** out);
/* Enqueue the start point and every generation (one CUDA graph per generation) on `stream`. */
int ls_es_run(ls_es* es, void* stream);

/* ---- the same search sharded over `world` ranks (one GPU each) ----
 * Rank r evaluates members [r P/world, (r+1) P/world) (population P a multiple
 * of world).  Per generation the caller enqueues, on one stream:
 *   ls_es_step(es, 0)   decode + memoised scoring of the local members, their F keys
 *   all-gather in place of the keys buffer (keys_per_rank uint64 per rank, rank
 *                       slices in rank order; ncclAllGather with sendbuff =
 *                       keys + r * keys_per_rank)
 *   ls_es_step(es, 1)   global stable ranks (sort of all P keys) and this rank's
 *                       chunk partials of sum_i w_i eps_i
 *   all-gather in place of the partials buffer (partials_per_rank float64 per rank)
 *   ls_es_step(es, 2)   theta update from every chunk in chunk order, trace, generation
 * after ls_es_begin (the start point).  Chunking and summation order do not
 * depend on world, so theta is bit-identical for any world; the distinct count
 * is the size of the union of the ranks' ls_es_evaluated lists and the trace is
 * the per-generation minimum over ranks.  world = 1 needs no exchange. */
int ls_es_create_shard(ls_task* task, const ls_es_params* params, const double* h_theta0, int32_t rank,
                       int32_t world, ls_es** out);
int ls_es_begin(ls_es* es, void* stream);
int ls_es_step(ls_es* es, int32_t stage, void* stream);
int ls_es_shard_buffers(ls_es* es, void** d_keys, int64_t* keys_per_rank, void** d_partials,
                        int64_t* partials_per_rank);
/* After ls_es_run: theta history [iterations+1][dim], trace [iterations] (best score after
 * each generation), distinct evaluations, first failure (0 none; else generation+1 (0: the
 * start point) << 40 | member << 8 | LS_ST_*) and best score.  Any pointer may be NULL.  Synchronous. */
int ls_es_result(ls_es* es, double* h_theta_hist, double* h_trace, int64_t* h_evaluations, int64_t* h_error,
                 double* h_best_score, void* stream);
/* Distinct evaluated schedules (space points, scores) in discovery order, at most `cap`;
 * *h_count = total.  Synchronous. */
int ls_es_evaluated(ls_es* es, uint64_t* h_points, double* h_scores, int64_t cap, int64_t* h_count, void* stream);
/* The Gaussian noise of a generation, [population][dim] float64 on the device (diagnostic). */
int ls_es_noise(ls_es* es, int32_t generation, double* d_out, void* stream);
/* The last generation's rank sort (diagnostic): the F order-bit keys as es_gen wrote them
 * (member order) and after the stable sort, the member at each sorted position and (d_ranks,
 * optional) each member's sorted position; device arrays of `population` entries,
 * stream-ordered copies. */
int ls_es_sort_state(ls_es* es, uint64_t* d_keys_in, uint64_t* d_keys_out, uint32_t* d_members, uint32_t* d_ranks,
                     void* stream);
int ls_es_destroy(ls_es* es);

/* ---- external code-text analysis (`analyze --code`, ls/cli.py:86) ----
 * The text-dependent features of extract_features (ls/cost.py:132-152) for a batch of
 * assembly / PTX texts, parsed on the device (one CUDA block per text): CPU family
 * n_fma, n_vload, n_vstore, ilp_cycles (parse_asm + loop_map + count_simd + the list
 * scheduler, ls/asm.py:110-337, ls/ilp.py:82-271); GPU family workload_per_thread,
 * n_fma, n_ld, n_st (loop_map_ptx + count_ptx + thread_cycles, ls/ptx.py:90-227).  The
 * IR-side features (cache movement; occupancy, warp slack, shared-memory ops) come from
 * the scoring path on the program.  Keys of the class / cost tables are ls_code_hash of
 * the reference's lowercase class names (fma, load, move, store, or a mnemonic root). */
#define LS_CODE_MAX_CLASSES 32
#define LS_CODE_MAX_LOOPS 64
#define LS_CODE_TARGET_X86 0
#define LS_CODE_TARGET_AARCH64 1
#define LS_CODE_DIALECT_ATT 0
#define LS_CODE_DIALECT_DEST_FIRST 1
/* per-text status: 0 ok; AsmError("empty assembly input") / AsmError("jump to undefined
 * label ...") (err_info = line, operand offset, length in the text); ValueError (a line
 * holding only a predicate); a device limit exceeded (operands / resources per
 * instruction, dependence predecessors, trip products beyond int64). */
#define LS_CODE_E_EMPTY 1
#define LS_CODE_E_LABEL 2
#define LS_CODE_E_VALUE 3
#define LS_CODE_E_LIMIT 4
typedef struct {
  int32_t family;           /* LS_FAMILY_CPU / LS_FAMILY_GPU */
  int32_t target;           /* CPU: LS_CODE_TARGET_* (count_simd's significant sets) */
  int32_t dialect;          /* CPU: LS_CODE_DIALECT_* (reg_effects' destination operand) */
  int32_t issue_width;      /* SchedSpec.issue_width */
  int32_t default_latency;  /* SchedSpec.default_latency */
  int32_t n_classes;        /* latency / unit classes (SchedSpec.latency / units keys) */
  uint64_t cls_hash[LS_CODE_MAX_CLASSES];
  int32_t cls_latency[LS_CODE_MAX_CLASSES];  /* 0: not in the latency table (default) */
  int32_t cls_units[LS_CODE_MAX_CLASSES];    /* 0: no unit cap */
  int32_t n_costs, pad0;    /* GPU: GpuSpec.instr_cost (root -> cycles; 1 otherwise) */
  uint64_t cost_hash[LS_CODE_MAX_CLASSES];
  double cost[LS_CODE_MAX_CLASSES];
  int32_t n_loops, pad1;    /* CPU: the program's branching loops in preorder (loop_map) */
  int64_t loop_extent[LS_CODE_MAX_LOOPS], loop_step[LS_CODE_MAX_LOOPS];
  int64_t loop_weight[LS_CODE_MAX_LOOPS];  /* product of its and its branching ancestors' extents */
} ls_code_desc;
uint64_t ls_code_hash(const char* s, int32_t n);
/* Device scratch a text of text_bytes needs (ls_code_features takes the sum over the
 * batch + a few KiB for the descriptor and offsets). */
int64_t ls_code_scratch_bytes(int64_t text_bytes);
/* d_texts: the texts back to back on the device; h_offsets[n_texts + 1] their byte
 * offsets (host).  d_features[4 * n_texts] (order above), d_status[n_texts],
 * d_err_info[3 * n_texts].  Stream-ordered. */
int ls_code_features(const ls_code_desc* desc, const char* d_texts, const int64_t* h_offsets, int32_t n_texts,
                     void* d_scratch, int64_t scratch_bytes, double* d_features, int32_t* d_status,
                     int64_t* d_err_info, void* stream);
/* The diagnostics extract_features appends to its `diagnostics` list (ls/cost.py:134-148):
 * CPU loop_map's unmatched blocks / bound mismatches / unmatched IR loops (ls/asm.py:
 * 276-293), GPU _loop_trip's failures (ls/ptx.py:112-189), as events of
 * LS_CODE_DIAG_WORDS int64 each: kind, block index, the block's label (offset, length in
 * the text; -1 none), three integers, an auxiliary text span (offset, length; -1 none):
 *   UNMATCHED_BLOCK  block
 *   BOUND_MISMATCH   block, [has bound, bound, loop index]
 *   LOOPS_MATCHED    [matched loop count] (the IR loops from there on are unmatched)
 *   NO_SETP / NON_IMM_BOUND                   loop target block
 *   NONLINEAR / NOT_DERIVABLE                 target, aux = the induction register
 *   UNSUPPORTED_CMP                           target, aux = the comparison
 *   INCONSISTENT     target, [init, delta, bound], aux = the comparison (-1: implicit "ne")
 * in the reference's order; the host renders the reference's messages (the GPU family's
 * list is produced twice by the reference: count_ptx, then thread_cycles).  Text i's
 * events start at event ls_code_diag_offset = sum over j < i of ls_code_diag_cap(len_j);
 * d_ndiag[i] = events written. */
#define LS_CODE_DIAG_WORDS 10
#define LS_CODE_D_UNMATCHED_BLOCK 1
#define LS_CODE_D_BOUND_MISMATCH 2
#define LS_CODE_D_LOOPS_MATCHED 3
#define LS_CODE_D_NO_SETP 10
#define LS_CODE_D_NON_IMM_BOUND 11
#define LS_CODE_D_NONLINEAR 12
#define LS_CODE_D_NOT_DERIVABLE 13
#define LS_CODE_D_UNSUPPORTED_CMP 14
#define LS_CODE_D_INCONSISTENT 15
int64_t ls_code_diag_cap(int64_t text_bytes);
int ls_code_features_diag(const ls_code_desc* desc, const char* d_texts, const int64_t* h_offsets, int32_t n_texts,
                          void* d_scratch, int64_t scratch_bytes, double* d_features, int32_t* d_status,
                          int64_t* d_err_info, int64_t* d_diag, int32_t* d_ndiag, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LOOPSCOUT_B200_H */
