/* include/pms8g.h — C ABI of the B200-native PMS8 per-S1-l-mer search.
 *
 * Drop-in boundary for the reference's solver entry points (the reference has
 * no FFI layer of its own); every function below names the
 * reference interface it replaces (paths relative to /root/reference/proj).
 *
 *   pms8g_solve          <- pms8::run_parallel   include/pms8/parallel.hpp:37-38
 *                           pms8::solve          include/pms8/solver.hpp:180
 *   pms8g_result_free    <- (ownership of MotifSet, solver.hpp:19)
 *   pms8g_ctx_*          <- SolverContext ctor   include/pms8/solver.hpp:65-85 (device-resident,
 *                           re-runnable context: inputs stay in HBM between runs)
 *   pms8g_generate       <- generate_planted_instance include/pms8/instance.hpp:38
 *   pms8g_estimate_threshold <- estimate_threshold include/pms8/solver.hpp:61
 *   pms8g_verify_motifs  <- naive_is_motif src/oracle.cpp:16-37 (`pms8 verify`, tools/pms8.cpp:193-256)
 *   pms8g_brute_force    <- brute_force_solve src/oracle.cpp:65-75
 *   pms8g_queue_*        <- the shared next-job counter of run_parallel src/parallel.cpp:54-60, across GPUs
 *   pms8g_solve_batch    <- several solve() calls of one shape (the paper's 5 seeds per (l,d))
 *   pms8g_gpu_threshold  <- estimate_threshold re-fitted for the GPU
 *   pms8g_int_peak       <- (measurement: the roofline's integer-issue denominator)
 *   pms8g_solve_multi / pms8g_multi_* <- run_parallel over N GPUs (parallel.hpp:37-38,
 *                           src/parallel.cpp:35-118: GPUs as the worker team)
 *   pms8g_report_json    <- report_to_json + `--format json` tools/pms8.cpp:31-60,171-176
 *   pms8g_merge_keys     <- canonical_motif_set  include/pms8/solver.hpp:22 (device sort+unique
 *                           of packed motif keys; used after the multi-GPU allgather)
 *
 * Plain pointers and sizes only. All calls are blocking unless stated, own
 * their CUDA streams, and never fall back to the CPU: without a usable sm_100
 * device they fail with PMS8G_ERR_CUDA. Errors mirror the reference's three
 * exception classes (invalid_argument / runtime_error / logic_error); the
 * message is written to err (NUL-terminated, truncated to errlen).
 */
#ifndef PMS8G_H
#define PMS8G_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    PMS8G_OK = 0,
    PMS8G_ERR_INVALID = 1, /* std::invalid_argument (Problem::validate src/problem.cpp:7-28, threshold src/solver.cpp:137) */
    PMS8G_ERR_RUNTIME = 2, /* std::runtime_error (motif cap src/solver.cpp:382-384, allocation) */
    PMS8G_ERR_LOGIC = 3,   /* std::logic_error (reverify failure src/solver.cpp:376) */
    PMS8G_ERR_CUDA = 4     /* device missing / launch failure (no CPU fallback exists) */
};

/* Mirrors SolverConfig (include/pms8/solver.hpp:24-31) plus the device and
 * sharding knobs that replace ParallelOptions (include/pms8/parallel.hpp:22-28). */
typedef struct pms8g_queue pms8g_queue; /* cross-GPU static task queue, see pms8g_queue_create */

typedef struct pms8g_options {
    int threshold;         /* 0: GPU-tuned default; else 1..n (SolverConfig::threshold_override) */
    int sort_rows;         /* 1: branch on the smallest row (reference default) */
    int prune_level;       /* 0 none, 1 pairs, 2 full (PruneLevel, neighborhood.hpp:16-20) */
    int reverify;          /* re-check every motif against all windows (reverify_against_originals) */
    int64_t max_motifs;    /* -1: unlimited; raw emissions above it -> PMS8G_ERR_RUNTIME */
    int device;            /* CUDA device ordinal; -1: current device */
    int shard_rank;        /* S1 offsets j with j % shard_count == shard_rank are searched */
    int shard_count;       /* 0 or 1: no sharding */
    const int32_t* anchors; /* optional explicit S1 offsets (subset runs), NULL: all */
    int nanchors;
    int warps_per_block;   /* 0: default */
    int blocks_per_sm;     /* 0: default */
    int exact_tree;        /* 1: filter every row at every push, exactly like the reference (same
                              search tree and counters); 0 (default): the rows of the final level
                              are filtered on demand by verification (same motif set, less work) */
    const int32_t* branches; /* optional explicit depth-1 branches: nbranches pairs (S1 offset, l-mer
                                id seq*(m-l+1)+offset of an l-mer in that S1 l-mer's branching row);
                                the result is the motif set under those branches only */
    int nbranches;
    int grid_blocks;       /* persistent grid of the search kernel; 0: one block per SM x blocks_per_sm */
    pms8g_queue* queue;    /* optional shared queue (multi-GPU dynamic pull over S1 l-mers, replacing the
                              reference's shared atomic job counter src/parallel.cpp:54-60 across GPUs):
                              every rank searches all S1 l-mers, claiming (S1 l-mer, depth-1 branch) tasks
                              from one counter; exclusive with shard_count > 1 */
    uint32_t jitter_max_us; /* test hook (ParallelOptions::jitter_max_us, include/pms8/parallel.hpp:24-27):
                               every claimed task first sleeps a seeded pseudo-random 0..jitter_max_us us,
                               shaking the schedule; the motif set must not change */
    uint64_t jitter_seed;
} pms8g_options;

/* Mirrors RunReport + SolveCounters (include/pms8/report.hpp:28-56). */
typedef struct pms8g_report {
    int n, m, l, d, sigma;
    int threshold;          /* the reference's switch depth for this call (SolverConfig override, else
                               estimate_threshold src/solver.cpp:104-117): RunReport::threshold */
    int gpus;               /* devices used by this call (1) */
    int64_t subproblems;    /* S1 l-mers searched by this call */
    int64_t motif_count;    /* unique motifs returned */
    double wall_seconds;    /* host wall clock of the call */
    double device_seconds;  /* CUDA-event time of the device pipeline */
    double sample_seconds;  /* row build + filter share (device clock estimate) */
    double pattern_seconds; /* enumerate + verify share (device clock estimate) */
    int64_t stacks_explored; /* l-mers pushed (counting the anchor) */
    int64_t neighborhoods;   /* tuples enumerated */
    int64_t neighbors_visited; /* candidates generated */
    int64_t motifs_emitted;  /* raw verified candidates (pre-dedup) */
    int64_t filter_slots;    /* l-mer slots tested by push filters (incl. row build) */
    int64_t verify_compares; /* candidate x l-mer Hamming compares in verification */
    int64_t enum_nodes;      /* enumeration tree nodes expanded */
    uint64_t device_bytes;   /* device memory held by the context */
    int device_threshold;    /* switch depth the device search used (GPU-tuned unless overridden;
                                the motif set does not depend on it) */
    /* MemoryBreakdown (include/pms8/report.hpp:9-25) of the device layout, in 8-byte words:
     * pair_matrix_words     level-1 rows of every S1 l-mer (the GPU's replacement of the K x K
     *                       pair matrix: each anchor's compatible l-mers, row-major)
     * row_matrix_words      per-warp level buffers (the RowMatrix storage of levels 2..t)
     * row_bookkeeping_words row tables, task bases/order, work ring, node stacks
     * packed_words          codes + the bit-plane l-mer table
     * lookup_table_words    0 (no 2^16 lookup table on the device) */
    uint64_t pair_matrix_words, row_matrix_words, row_bookkeeping_words, packed_words, lookup_table_words;
} pms8g_report;

/* Motifs as uppercase strings of length l, concatenated without separators,
 * sorted and deduplicated (canonical_motif_set order). */
typedef struct pms8g_result {
    int64_t count;
    int l;
    char* motifs;           /* count*l chars (+NUL), owned; free with pms8g_result_free */
    pms8g_report report;
} pms8g_result;

void pms8g_default_options(pms8g_options* opt);

/* Whole-instance (or shard / subset) search from HOST codes.
 * codes: n*m bytes, row-major, values in [0, sigma) (sigma <= 4; symbols come
 * from `alphabet`, e.g. "ACGT", used only to decode motifs). */
int pms8g_solve(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet, const pms8g_options* opt,
                pms8g_result* out, char* err, size_t errlen);
void pms8g_result_free(pms8g_result* r);

/* Several instances of one shape (the paper averages 5 seeds per (l,d)),
 * searched concurrently on one device: each in-flight instance gets an equal share of the
 * SMs (its own persistent grid) and stream; results are per instance, like pms8g_solve
 * (no reference counterpart: the reference solves one Problem per run_parallel call).
 * report.wall_seconds is the batch wall time. */
int pms8g_solve_batch(const uint8_t* const* codes, int count, int n, int m, int l, int d, const char* alphabet,
                      const pms8g_options* opt, pms8g_result* outs, char* err, size_t errlen);

/* Device-resident context: allocate once, load codes (host or device pointer),
 * run many times. Keys: 128-bit MSB-first 2-bit packing of each motif (symbol
 * 0 in the highest used bits), so integer order == lexicographic order; stored
 * as two uint64 {lo, hi} per key. */
typedef struct pms8g_ctx pms8g_ctx;
int pms8g_ctx_create(int n, int m, int l, int d, const char* alphabet, const pms8g_options* opt, pms8g_ctx** out,
                     char* err, size_t errlen);
int pms8g_ctx_load_codes(pms8g_ctx* ctx, const uint8_t* codes, int codes_on_device, char* err, size_t errlen);
/* Runs encode -> row build -> persistent search -> device sort/unique on the
 * context's stream and waits for it. */
int pms8g_ctx_run(pms8g_ctx* ctx, char* err, size_t errlen);
/* Device pointer to the unique sorted keys of the last run and their count. */
int pms8g_ctx_keys(pms8g_ctx* ctx, const uint64_t** dev_keys, int64_t* count);
/* Copies the motifs of the last run to the host (like pms8g_solve's result). */
int pms8g_ctx_result(pms8g_ctx* ctx, pms8g_result* out, char* err, size_t errlen);
void* pms8g_ctx_stream(pms8g_ctx* ctx); /* cudaStream_t */
/* Dedicated event pair around the main search kernel of the last launch. */
int pms8g_ctx_kernel_ms(pms8g_ctx* ctx, float* search_ms, float* rowbuild_ms);
/* Report of the last run (owned by the context, valid until the next run). */
int pms8g_ctx_report(pms8g_ctx* ctx, const pms8g_report** report);
/* Raw device counters of the last run (diagnostics: per-rule rejections, task
 * duration histogram); returns the number of counters available. */
int pms8g_ctx_counters(pms8g_ctx* ctx, uint64_t* out, int cap);
void pms8g_ctx_destroy(pms8g_ctx* ctx);

/* Device sort+unique of `count` keys (2 x uint64 each) at dev_in into dev_out
 * (capacity >= count); returns the unique count. Both device pointers. */
int pms8g_merge_keys(const uint64_t* dev_in, int64_t count, uint64_t* dev_out, int64_t* out_count, void* stream,
                     char* err, size_t errlen);
/* Host decode of keys into strings (count*l chars, caller-allocated). */
void pms8g_decode_keys(const uint64_t* host_keys, int64_t count, int l, const char* alphabet, char* out);

/* Planted instance generator (src/instance.cpp:22-73), byte-identical stream. */
int pms8g_generate(int n, int m, int l, int d, int sigma, uint64_t seed, int exactly_d, uint8_t* codes_out,
                   uint8_t* motif_out, int32_t* positions_out);
/* Threshold model (src/solver.cpp:75-117) and the GPU-tuned default. */
int pms8g_estimate_threshold(int n, int m, int l, int d, int sigma);
int pms8g_gpu_threshold(int n, int m, int l, int d, int sigma);

/* Brute-force scanner (the reference's `pms8 verify` subcommand, tools/pms8.cpp:193-256, over
 * naive_is_motif src/oracle.cpp:16-37), batched on the device: motifs = nmotifs*l codes in
 * [0, sigma). pass[i] = 1 iff every sequence has a window within Hamming distance d;
 * witness[i*n + r] = the first such offset in sequence r, -1 from the first sequence without
 * one on (the reference stops there). device = -1: current device. */
int pms8g_verify_motifs(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet, const uint8_t* motifs,
                        int64_t nmotifs, int32_t* witness, uint8_t* pass, int device, char* err, size_t errlen);
/* Exhaustive solver over Sigma^l (brute_force_solve src/oracle.cpp:65-75): every word, in
 * code order, checked against every sequence; sorted motif set out. sigma^l > guard ->
 * PMS8G_ERR_INVALID (check_guard src/oracle.cpp:41-46; the reference's default guard is 10^6,
 * include/pms8/oracle.hpp:28-29). Independent of the PMS8 tree: an exactness check. */
int pms8g_brute_force(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet, int64_t guard,
                      int device, pms8g_result* out, char* err, size_t errlen);

/* The `pms8 solve --format json` document (tools/pms8.cpp:31-60,171-176) for a result:
 * {"motifs": [...], "report": {...}} with the reference's report schema, keys in the order
 * nlohmann::json prints them (sorted), two-space indentation, doubles in shortest round-trip
 * form. alphabet_name: e.g. "dna"; command: the invocation line. Writes at most cap bytes
 * (NUL-terminated) and returns the full length (excluding the NUL), or -1 on a NULL result. */
int64_t pms8g_report_json(const pms8g_result* result, const char* alphabet_name, const char* command, char* out,
                          size_t cap);

/* run_parallel over several GPUs in one blocking call (include/pms8/parallel.hpp:37-38 with
 * GPUs as the workers): one host thread and device context per entry of `devices`; all
 * contexts search every S1 l-mer, claiming (S1 l-mer, depth-1 branch) tasks from one counter
 * in devices[0]'s HBM over NVLink peer access (static split offset % N == rank when a device
 * cannot reach it); the per-device motif sets are unioned with ncclAllGather (distinct devices,
 * NCCL loadable) or peer copies, then sorted and deduplicated on devices[0]. The result and
 * report cover the whole run (report.gpus = ndevices, counters summed). A device may be listed
 * more than once (several contexts share it: the one-GPU test hook). opt.queue, opt.shard_*
 * and opt.branches must be unset. pms8g_solve_multi caches one handle per process. */
typedef struct pms8g_multi pms8g_multi;
int pms8g_multi_create(int n, int m, int l, int d, const char* alphabet, const pms8g_options* opt,
                       const int* devices, int ndevices, pms8g_multi** out, char* err, size_t errlen);
/* codes: HOST n*m codes; blocking. */
int pms8g_multi_run(pms8g_multi* h, const uint8_t* codes, pms8g_result* out, char* err, size_t errlen);
/* "nccl-allgather" or "peer-copy": how the motif sets are exchanged. */
const char* pms8g_multi_exchange(const pms8g_multi* h);
void pms8g_multi_destroy(pms8g_multi* h);
int pms8g_solve_multi(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet, const pms8g_options* opt,
                      const int* devices, int ndevices, pms8g_result* out, char* err, size_t errlen);

/* Cross-GPU static task queue: one 64-bit claim counter in the HBM of the creating rank's
 * device, mapped into the other ranks' devices over NVLink/NVSwitch with CUDA IPC. Rank 0
 * creates it and passes `handle` (PMS8G_QUEUE_HANDLE_BYTES) to the others, which open it on
 * their own device; each rank then sets pms8g_options.queue. The counter is epoch-tagged, so
 * consecutive runs need no reset, as long as every rank issues the same sequence of runs
 * (the per-run motif allgather keeps them in step). Replaces the reference's
 * std::atomic<int> next-job counter (src/parallel.cpp:54-60) at node scale. */
#define PMS8G_QUEUE_HANDLE_BYTES 64
int pms8g_queue_create(int device, pms8g_queue** out, uint8_t* handle, char* err, size_t errlen);
int pms8g_queue_open(const uint8_t* handle, int device, pms8g_queue** out, char* err, size_t errlen);
void pms8g_queue_destroy(pms8g_queue* q);

/* Integer-pipe peak microbenchmark: LOP3/IADD3-class ops per second over all
 * SMs of `device` (measured, used as the roofline denominator), and the SM
 * clock (MHz) the device reported while it ran. */
int pms8g_int_peak(int device, double* ops_per_second, double* popc_per_second, char* err, size_t errlen);

const char* pms8g_version(void);

#ifdef __cplusplus
}
#endif
#endif
