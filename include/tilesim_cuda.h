/* tilesim_cuda.h -- C ABI of the B200 gate-application path.
 *
 * The drop-in boundary for CAST/tilesim's hot path: applying sparsity-aware
 * fused k-qubit gates to a 2^n complex statevector on B200 (sm_100a).  Every
 * entry point below replaces one operation of the reference's kernel / sim
 * contract or exports the C++ surface
 * that produces its input (circuit IR, fusion pass, cost model) for FFI
 * callers.  Plain pointers and sizes only; no C++ or torch types.
 *
 * Conventions
 *  - Return value: TSG_OK (0) or an error class mirroring the CLI exit codes
 *    of SPEC.md:587: 1 parse (ParseError), 2 config (ConfigError or
 *    std::invalid_argument), 3 sim (SimError, CUDA).  The message of the
 *    last failure on the calling thread is tsg_last_error().  C++ exceptions
 *    never cross this boundary.
 *  - Matrices: 2 * 4^k doubles, interleaved (re, im), row-major, index bit j
 *    = j-th SORTED target (complex_matrix.hpp:34-36), unless a function says
 *    "argument order".
 *  - Host state arrays are SoA fp64 (re[2^n], im[2^n]) for both precisions;
 *    they are borrowed only for the duration of the call.
 *  - Device memory and handles are owned by the library.  A state is used by
 *    one host thread at a time; calls are ordered on the state's CUDA stream
 *    and are asynchronous except those that return host data.
 *  - There is no CPU fallback: on a host without a CUDA device every tsg_*
 *    device call fails with TSG_ERR_SIM.  tsc_* calls are host-only.
 */
#ifndef TILESIM_CUDA_H
#define TILESIM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSG_OK 0
#define TSG_ERR_PARSE 1
#define TSG_ERR_CONFIG 2
#define TSG_ERR_SIM 3

typedef struct tsg_ctx tsg_ctx;
typedef struct tsg_state tsg_state;
typedef struct tsg_plan tsg_plan;
typedef struct tsg_program tsg_program;
typedef struct tsc_circuit tsc_circuit;
typedef struct tsc_cost_model tsc_cost_model;

/* ------------------------------------------------------------------ misc */
const char* tsg_last_error(void);
const char* tsg_version(void);
/* number of visible CUDA devices (0 on a CPU-only host; never fails) */
int tsg_device_count(int* out);

/* --------------------------------------------------------------- context
 * One context per GPU (one process per GPU in multi-GPU runs). */
int tsg_ctx_create(int device, tsg_ctx** out);
int tsg_ctx_destroy(tsg_ctx* ctx);
int tsg_ctx_info(const tsg_ctx* ctx, int* device, int* num_sms);

/* ----------------------------------------------------------------- state
 * Statevector / init_zero_state.  precision_bits: 64 for
 * complex128 (f64 re/im arrays), 32 for complex64.  Allocation failure is
 * TSG_ERR_SIM naming the 2^(n+4) / 2^(n+3) bytes required. */
int tsg_state_create(tsg_ctx* ctx, int n_qubits, int precision_bits, tsg_state** out);
int tsg_state_destroy(tsg_state* st);
int tsg_state_info(const tsg_state* st, int* n_qubits, int* precision_bits);
int tsg_state_init_zero(tsg_state* st);
int tsg_state_init_basis(tsg_state* st, uint64_t index);
/* deterministic pseudo-random normalized state (DESIGN.md §5 hash) */
int tsg_state_init_random(tsg_state* st, uint64_t seed);
int tsg_state_upload(tsg_state* st, const double* re, const double* im);
/* amplitudes [begin, begin + count) from host fp64 arrays (checkpoint chunks,
 * single-amplitude edits in tests) */
int tsg_state_upload_range(tsg_state* st, uint64_t begin, uint64_t count, const double* re, const double* im);
int tsg_state_download(tsg_state* st, double* re, double* im);
int tsg_state_download_range(tsg_state* st, uint64_t begin, uint64_t count, double* re, double* im);
/* amplitudes at arbitrary indices (a device gather, one copy back) */
int tsg_state_gather(tsg_state* st, const uint64_t* indices, uint64_t count, double* re, double* im);
int tsg_state_copy(tsg_state* dst, const tsg_state* src);
/* QSV1 amplitude dump / load: header "QSV1", u8 precision bits
 * (32 | 64), u8 n, 10 zero bytes; then re[2^n], im[2^n] little-endian in the
 * state's precision.  Load requires matching precision and n. */
int tsg_state_dump(tsg_state* st, const char* path);
int tsg_state_load(tsg_state* st, const char* path);
int tsg_synchronize(tsg_state* st);
/* CUDA events on the state's stream bracketing any sequence of calls;
 * tsg_timer_end synchronizes and returns the device seconds in between. */
int tsg_timer_begin(tsg_state* st);
int tsg_timer_end(tsg_state* st, double* seconds);

/* ------------------------------------------------------------------ plans
 * plan_kernel(g, n, s=0, zero_tol, one_tol, runtime_matrix).
 * targets: k strictly increasing qubit indices; matrix: sorted-target order.
 * The plan classifies every scalar, peels exact-identity control qubits,
 * selects the kernel class and uploads nothing until first use. */
int tsg_plan_create(tsg_ctx* ctx, int n_qubits, int k, const int* targets, const double* matrix, double zero_tol,
                    double one_tol, int runtime_matrix, tsg_plan** out);
int tsg_plan_destroy(tsg_plan* p);

typedef struct tsg_plan_info {
  int k;               /* gate size */
  int kernel_class;    /* 0 identity, 1 diagonal, 2 direct, 3 tile */
  int sub_k;           /* qubits the kernel actually mixes */
  int n_controls;      /* exact-identity control qubits peeled off */
  int sparse;          /* zero-skipping variant selected */
  uint64_t op_count;   /* SPEC op_count of the plan's profile */
  uint64_t entry_ops;  /* entries with a non-Zero scalar */
  uint64_t loop_count; /* 2^(n-k): groups of the s = 0 loop counter */
  double touched_fraction; /* share of the state the kernel reads+writes */
  int batched;         /* programs only: 0 own launch, 1 first gate of a
                          multi-gate step (diagonal batch or tile pass: one
                          streaming pass for the run), 2 applied by the step of
                          an earlier gate */
  int controls[12];    /* the n_controls peeled control qubits, ascending */
  int sub_targets[12]; /* the sub_k qubits the kernel mixes, ascending */
} tsg_plan_info;
int tsg_plan_info_get(const tsg_plan* p, tsg_plan_info* out);

/* apply_kernel(plan, state, matrix_override, t_begin, t_end).
 * t ranges over the s = 0 groups [0, 2^(n-k)); pass 0, UINT64_MAX for all.
 * matrix_override (NULL unless the plan is runtime_matrix) must classify to
 * the planned kinds scalar by scalar, else TSG_ERR_SIM. */
int tsg_apply(tsg_state* st, const tsg_plan* p, const double* matrix_override, uint64_t t_begin, uint64_t t_end);

/* ------------------------------------------------------------ measurement
 * norm: compensated fp64 sum; compare_states:
 * max_i |a_i - b_i| against host SoA fp64 arrays or another device state. */
int tsg_norm(tsg_state* st, double* out);
int tsg_compare(tsg_state* st, const double* re, const double* im, double* maxdiff);
int tsg_compare_states(tsg_state* a, tsg_state* b, double* maxdiff);
/* sum over i of conj(a_i) * b_i (fidelity = |overlap|^2 for pure states) */
int tsg_overlap(tsg_state* a, tsg_state* b, double* re, double* im);

/* ----------------------------------------------------------------- programs
 * run_circuit for a flattened (fused) circuit: every gate
 * is planned once, matrices uploaded once, and the launch sequence replayed
 * (as a CUDA graph when use_graph != 0).  Execution time is device time
 * between events on the state's stream and excludes planning. */
typedef struct tsg_run_report {
  double planning_s;   /* host planning + upload when the program was built */
  double execution_s;  /* device time of the last run */
  uint64_t gates;      /* gates in the program */
  uint64_t launches;   /* kernels launched per run (identity gates skip) */
  uint64_t bytes;      /* algorithmic bytes per run: sum of 2*2^n*B_amp over launched gates */
  uint64_t touched_bytes; /* bytes the kernels actually read+write (controls skip slices) */
  uint64_t total_op_count;
  uint64_t exchanged_bytes; /* sharded runs: bytes this rank sent to peers */
  double exchange_s;        /* sharded runs: device seconds spent in exchanges */
} tsg_run_report;

int tsg_program_create(tsg_ctx* ctx, const tsc_circuit* fused, double zero_tol, double one_tol, int precision_bits,
                       tsg_program** out);
int tsg_program_destroy(tsg_program* prog);
int tsg_program_run(tsg_state* st, tsg_program* prog, int use_graph, tsg_run_report* report);
/* asynchronous: enqueue one run on the state's stream and return */
int tsg_program_enqueue(tsg_state* st, tsg_program* prog, int use_graph);
/* per-gate device seconds into seconds[gates] (events around every launch) */
int tsg_program_run_profiled(tsg_state* st, tsg_program* prog, double* seconds, tsg_run_report* report);
/* gate i of the program: kernel class, sub_k, controls, op_count */
int tsg_program_gate_info(const tsg_program* prog, uint64_t i, tsg_plan_info* out);

/* Launch steps of a program, in order.  A step applies n_gates consecutive
 * (non-identity) gates of the program with ONE kernel: kind 0 a single gate,
 * 1 a diagonal batch, 2 a tile pass (tilesim/pass.hpp: one HBM sweep for the
 * run; high[] are its tile qubits above the contiguous runs), 3 a qubit
 * permutation (a run of SWAP-type gates; one in-place sweep, two when the
 * composed permutation is not an involution). */
typedef struct tsg_step_info {
  int kind;
  uint64_t first_gate;
  uint64_t n_gates;
  int n_high;
  int high[16];
  char kernel[48]; /* kernel template, e.g. "k_pass", "k_stream_dmma<ks=5>" */
} tsg_step_info;
int tsg_program_step_count(const tsg_program* prog, uint64_t* out);
int tsg_program_step_info(const tsg_program* prog, uint64_t i, tsg_step_info* out);
/* B200 addition: a tile-pass step's register layouts -- loaded through shared
 * memory, or reached from the previous one with warp shuffles (register <->
 * lane swaps); both 0 for other steps */
int tsg_program_pass_layouts(const tsg_program* prog, uint64_t i, int* smem_layouts, int* shuffle_layouts);
/* B200 addition: how many of the program's tile passes run JIT-compiled
 * kernels (NVRTC, op table compiled in) and how many standalone launches run
 * a JIT-compiled DMMA product (zero 8x4 tiles compiled out) */
int tsg_program_jit_kernels(const tsg_program* prog, int* jit_passes, int* jit_gate_launches);

/* --------------------------------------------------- circuit IR (host) ---
 * C exports of the kept C++ surface (include/tilesim/ir.hpp, fusion.hpp). */
int tsc_circuit_create(int n_qubits, tsc_circuit** out);
int tsc_circuit_destroy(tsc_circuit* c);
int tsc_circuit_copy(const tsc_circuit* c, tsc_circuit** out);
/* make_named_gate (circuit.cpp:135): qubits in argument order */
int tsc_circuit_add_named(tsc_circuit* c, const char* name, const double* params, int n_params, const int* qubits,
                          int n_qubits);
/* raw matrix in ARGUMENT order of `qubits` (make_gate_arg_order) */
int tsc_circuit_add_matrix(tsc_circuit* c, int k, const int* qubits, const double* matrix);
int tsc_circuit_n_qubits(const tsc_circuit* c, int* out);
int tsc_circuit_n_gates(const tsc_circuit* c, uint64_t* out);
/* gate i: k, sorted targets (k ints), matrix (2*4^k doubles); any out may be NULL */
int tsc_circuit_gate(const tsc_circuit* c, uint64_t i, int* k, int* targets, double* matrix);
/* name of gate i ("" for raw/fused); valid until the circuit changes */
const char* tsc_circuit_gate_name(const tsc_circuit* c, uint64_t i);
int tsc_gen_benchmark(const char* kind, int n, int depth, uint64_t seed, tsc_circuit** out);
int tsc_parse_circuit(const char* text, tsc_circuit** out);
/* serialize into buf (cap bytes incl. NUL); *needed gets the full size */
int tsc_serialize_circuit(const tsc_circuit* c, char* buf, size_t cap, size_t* needed);

/* --------------------------------------------------------------- fusion */
typedef struct tsc_fusion_config {
  int mode;              /* 0 none, 1 size-only, 2 adaptive */
  int k_max;
  int64_t max_op_count;  /* < 0: unset */
  int agglomerative;
  int multi_traversal;
  double zero_tol, one_tol;
  int max_traversals;
  int threads;           /* cost-model thread/CTA column (GPU: SMs) */
  int n_global;          /* shard-aware fusion over the top n_global qubits (0: off) */
} tsc_fusion_config;

typedef struct tsc_fusion_stats {
  uint64_t original_gate_count, fused_block_count, total_op_count;
  double compression_ratio, fusion_wall_time;
} tsc_fusion_stats;

int tsc_run_fusion(const tsc_circuit* c, const tsc_fusion_config* cfg, const tsc_cost_model* cm, tsc_circuit** out,
                   tsc_fusion_stats* stats);

int tsc_cost_model_parse(const char* text, tsc_cost_model** out);
int tsc_cost_model_destroy(tsc_cost_model* cm);
int tsc_cost_model_serialize(const tsc_cost_model* cm, char* buf, size_t cap, size_t* needed);
int tsc_estimate_cost(const tsc_cost_model* cm, int k, uint64_t op_count, int threads, int n, double* seconds);

/* ----------------------------------------------- sharding (host planner) ---
 * include/tilesim/shard.hpp: 2^n_global ranks, physical bits >= n - n_global
 * select the rank.  Op kinds: 0 local gate, 1 rank-selected sub-block
 * (no communication), 2 swaps of (global position, local position) pairs. */
/* Tile-pass grouping (tilesim/pass.hpp) of a fused circuit, as
 * tsg_program_create would do it for precision_bits.  Host only.
 * step_of_gate[n_gates]: step index of each gate (-1: identity, no launch);
 * step_is_pass[n_gates] (0 single-gate launch, 1 tile pass, 2 qubit
 * permutation step) and step_high[16 * n_gates] (-1 padded) describe
 * steps 0 .. *n_steps - 1 (there are never more steps than gates). */
int tsc_plan_passes(const tsc_circuit* fused, int precision_bits, double zero_tol, double one_tol, int* step_of_gate,
                    int* step_is_pass, int* step_high, uint64_t* n_steps);

/* Compile (NVRTC, no device needed) the JIT tile-pass kernels a program of
 * `fused` would use, into the JIT disk cache (TSG_JIT_CACHE_DIR); *n_passes =
 * how many passes the program has.  Warms the cache ahead of a run. */
int tsc_pass_jit_precompile(const tsc_circuit* fused, int precision_bits, double zero_tol, double one_tol,
                            int* n_passes);

typedef struct tsc_shard_plan tsc_shard_plan;
/* pipeline_bits: the top local positions that cut a shard into slabs for
 * exchange / compute overlap (shard.hpp; 0 disables, 2 is the default) */
int tsc_shard_plan_create(const tsc_circuit* fused, int n_global, double zero_tol, double one_tol, int pipeline_bits,
                          tsc_shard_plan** out);
int tsc_shard_plan_destroy(tsc_shard_plan* p);
int tsc_shard_plan_info(const tsc_shard_plan* p, int* n_qubits, int* n_global, uint64_t* n_ops, uint64_t* swaps,
                        uint64_t* rank_blocks);
/* exchanges (one grouped all-to-all each), how many pipeline, slab bits */
int tsc_shard_plan_stats(const tsc_shard_plan* p, uint64_t* swap_ops, uint64_t* pipelined_swaps, int* pipeline_bits);
/* op i: kind, gate (k, sorted physical targets, matrix 2*4^k; k = 0 for swaps),
 * swap pairs (2 ints each, *n_swaps of them), index of the source gate,
 * pipeline bits of a swap and how many following ops run slab by slab */
int tsc_shard_plan_op(const tsc_shard_plan* p, uint64_t i, int* kind, int* k, int* targets, double* matrix,
                      int* n_swaps, int* swap_pairs, int* source_gate, int* pipeline_bits, int* pipeline_ops);
/* local sub-gate of a rank-block op for `rank` (k may be 0: a scalar) */
int tsc_shard_rank_subgate(const tsc_shard_plan* p, uint64_t i, uint64_t rank, int* k, int* targets, double* matrix);
/* logical qubit -> physical position after the last op (n ints) */
int tsc_shard_final_pos(const tsc_shard_plan* p, int* pos);

/* --------------------------------------------- sharded execution (device) ---
 * Virtual shards: 2^n_global shard buffers on ONE device, exchanges by the
 * distributed exchange kernel itself -- the single-GPU emulation of the
 * distributed path.  Host arrays are the full state in logical order (fp64
 * SoA, 2^n entries). */
int tsg_vshard_run(tsg_ctx* ctx, const tsc_shard_plan* plan, int precision_bits, const double* re_in,
                   const double* im_in, double* re_out, double* im_out, tsg_run_report* report);

/* One process per GPU of one box, world = 2^n_global.  Rank 0 makes the id
 * (tsg_dist_unique_id: the name of a shared-memory rendezvous segment),
 * every rank passes the same 128 bytes (e.g. broadcast over
 * torch.distributed).  Shards are exported to every peer with CUDA IPC;
 * an exchange is an in-place peer-memory kernel on a comm stream, ordered
 * by interprocess events.  Several ranks may share one device (tests). */
typedef struct tsg_dist tsg_dist;
int tsg_dist_unique_id(unsigned char id[128]);
int tsg_dist_create(tsg_ctx* ctx, int n_qubits, int precision_bits, int n_global, int rank, const unsigned char id[128],
                    tsg_dist** out);
int tsg_dist_destroy(tsg_dist* d);  /* collective: every rank calls it */
int tsg_dist_init_basis(tsg_dist* d, uint64_t logical_index);  /* identity qubit map */
/* this rank's 2^(n-n_global) amplitudes, physical order (fp64 SoA) */
int tsg_dist_upload_local(tsg_dist* d, const double* re, const double* im);
/* collective.  report: execution_s = device seconds on this rank's compute
 * stream, exchange_s = device seconds of its exchange kernels,
 * exchanged_bytes = bytes it sent */
int tsg_dist_run(tsg_dist* d, const tsc_shard_plan* plan, tsg_run_report* report);
/* the plan's local segments only (no exchange, not collective): the
 * compute-only timeline exposed swap time is measured against; leaves the
 * state meaningless */
int tsg_dist_run_local_only(tsg_dist* d, const tsc_shard_plan* plan, tsg_run_report* report);
/* this rank's 2^(n-n_global) amplitudes (physical order of the last plan) */
int tsg_dist_download_local(tsg_dist* d, double* re, double* im);
int tsg_dist_local_sumsq(tsg_dist* d, double* out);
/* sharded QSV1: <path>.r<rank> = this shard as a QSV1 dump,
 * <path>.layout (rank 0) = n, n_global, precision and the qubit map pos[n]
 * (logical qubit q at physical position pos[q], e.g. ShardPlan final_pos);
 * load reads this rank's shard back and returns the map */
int tsg_dist_dump(tsg_dist* d, const char* path, const int* pos);
int tsg_dist_load(tsg_dist* d, const char* path, int* pos);
/* host-only check of the rendezvous (no device): `iters` rounds of
 * write-slot / barrier / sum-all-slots; *checksum = sum over rounds */
int tsg_rendezvous_selftest(const unsigned char id[128], int rank, int world, int iters, uint64_t* checksum);

/* bench_cost_model on the GPU: for k in [1, k_max] and
 * densities {diagonal, quarter, half, dense}, times the real kernel on a
 * 2^bench_n scratch state, median of `repetitions`.  `threads`
 * is the number of SMs the kernels' persistent grids span: the plain call
 * records the full device (threads = its SM count), the _sms form one record
 * set per entry of sm_counts (each in [1, SM count]). */
int tsg_bench_cost_model(tsg_ctx* ctx, int bench_n, int k_max, int precision_bits, int repetitions, uint64_t seed,
                         tsc_cost_model** out);
int tsg_bench_cost_model_sms(tsg_ctx* ctx, int bench_n, int k_max, int precision_bits, int repetitions, uint64_t seed,
                             const int* sm_counts, int n_sm_counts, tsc_cost_model** out);

#ifdef __cplusplus
}
#endif
#endif /* TILESIM_CUDA_H */
