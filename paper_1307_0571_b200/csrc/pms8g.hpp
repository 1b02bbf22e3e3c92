// pms8g.hpp — C++ host API over the C ABI (include/pms8g.h), shaped like the
// reference's library interface so callers switch by changing the namespace:
//
//   pms8::Problem          include/pms8/problem.hpp:11-22
//   pms8::SolverConfig     include/pms8/solver.hpp:24-31
//   pms8::ParallelOptions  include/pms8/parallel.hpp:22-28 (GpuOptions here)
//   pms8::RunReport        include/pms8/report.hpp:43-56
//   pms8::solve            include/pms8/solver.hpp:180
//   pms8::run_parallel     include/pms8/parallel.hpp:37-38
//   pms8::read_sequences   include/pms8/io.hpp:21 (FASTA/plain, metadata)
//   pms8::naive_is_motif   include/pms8/oracle.hpp:14-22 (batched: verify_motifs)
//   pms8::brute_force_solve include/pms8/oracle.hpp:27-29
//
// Errors are rethrown as the reference's exception classes.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "pms8g.h"

namespace pms8g {

using MotifSet = std::vector<std::string>;

struct Problem {
    std::vector<std::string> sequences;
    int motif_length = 0;
    int max_mismatches = 0;
    std::string alphabet = "ACGT";  // symbols in code order (Alphabet::symbols)
    std::string alphabet_name = "dna";
    int n() const { return static_cast<int>(sequences.size()); }
    int m() const { return sequences.empty() ? 0 : static_cast<int>(sequences[0].size()); }
    void validate() const;  // Problem::validate, src/problem.cpp:7-28
};

enum class PruneLevel { none = 0, pairs = 1, full = 2 };

struct SolverConfig {
    std::optional<int> threshold_override;
    bool sort_rows = true;
    bool use_pair_matrix = true;  // accepted for parity; the GPU path has no K x K matrix
    std::optional<int64_t> max_motifs;
    bool reverify_against_originals = false;
    PruneLevel prune_level = PruneLevel::full;
};

struct GpuOptions {
    int device = -1;
    int shard_rank = 0, shard_count = 1;
    std::vector<int32_t> anchors;  // empty: all S1 offsets
    // several GPUs of this process as the worker team (pms8g_solve_multi):
    // shared task counter over NVLink, NCCL allgather of the motif sets
    std::vector<int> devices;
    // ParallelOptions' schedule-shaking test hook (include/pms8/parallel.hpp:24-27)
    uint32_t jitter_max_us = 0;
    uint64_t jitter_seed = 0;
};

struct SolveCounters {
    int64_t stacks_explored = 0, neighborhoods = 0, neighbors_visited = 0, motifs_emitted = 0;
};

struct RunReport {
    int n = 0, m = 0, l = 0, d = 0;
    std::string alphabet;
    int threshold = 0;
    int workers = 1;
    int64_t subproblems = 0, motif_count = 0;
    double wall_seconds = 0, sample_seconds = 0, pattern_seconds = 0, device_seconds = 0;
    SolveCounters counters;
    int64_t filter_slots = 0, verify_compares = 0, enum_nodes = 0;
    uint64_t device_bytes = 0;
    int device_threshold = 0;  // switch depth the device search used
    std::string command;
    pms8g_report raw{};        // the C ABI report (memory breakdown, all counters)
};

// `pms8 solve --format json` (tools/pms8.cpp:31-60,171-176), byte-identical layout
std::string report_json(const MotifSet& motifs, const RunReport& report);

MotifSet run_parallel(const Problem& problem, const SolverConfig& config, const GpuOptions& options,
                      RunReport* report = nullptr);
MotifSet solve(const Problem& problem, const SolverConfig& config = {}, RunReport* report = nullptr);
// Instances of one shape searched concurrently on one device (pms8g_solve_batch).
std::vector<MotifSet> solve_batch(const std::vector<Problem>& problems, const SolverConfig& config = {},
                                  int device = -1);

struct SequenceFile {
    std::vector<std::string> names;
    std::vector<std::string> sequences;
    std::map<std::string, std::string> metadata;
};
SequenceFile read_sequences(const std::string& path);
SequenceFile read_plain(const std::string& path);  // src/io.cpp:99

// Brute-force scanner on the GPU (pms8g_verify_motifs / pms8g_brute_force).
struct MotifCheck {
    bool pass = false;
    std::vector<int> witness_offsets;  // first window within d per sequence, up to the first miss
};
std::vector<MotifCheck> verify_motifs(const Problem& problem, const std::vector<std::string>& motifs,
                                      int device = -1);
bool naive_is_motif(const Problem& problem, const std::string& motif, std::vector<int>* witness_offsets = nullptr);
MotifSet brute_force_solve(const Problem& problem, int64_t enumeration_guard = 1000000, int device = -1);
void write_fasta(const std::string& path, const std::vector<std::string>& names,
                 const std::vector<std::string>& sequences,
                 const std::vector<std::pair<std::string, std::string>>& metadata);

// "dna", "custom:<symbols>" -> symbols in code order; throws invalid_argument
std::string alphabet_symbols(const std::string& name);

// Problem::validate fused with the encoding the device consumes: n*m codes
// (row-major, 0..sigma-1 in alphabet order); throws invalid_argument.
std::vector<uint8_t> encode_problem(const Problem& problem);

}  // namespace pms8g
