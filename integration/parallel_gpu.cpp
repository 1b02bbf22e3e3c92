// integration/parallel_gpu.cpp — the translation unit a reference maintainer
// would add next to src/parallel.cpp to route run_parallel to the B200 path.
// It compiles against the reference's own headers (include/pms8/*.hpp) and
// include/pms8g.h, and links against paper_1307_0571_b200/lib/libpms8g.so.
// tests/test_integration.py compiles it against /root/reference/proj/include;
// oracle/Makefile (`refgpu`) links it with the reference's objects into
// oracle/_ref/pms8ref_gpu, which tests/test_gpu_integration.py runs on a B200.
//
//   pms8::run_parallel_gpu  <- pms8::run_parallel  include/pms8/parallel.hpp:37-38
//   errors                  <- src/parallel.cpp:84-86, src/problem.cpp:7-28 (same classes)
//   report fields           <- src/parallel.cpp:92-116 (RunReport, include/pms8/report.hpp:43-56)
#include <stdexcept>
#include <string>
#include <vector>

#include "pms8/parallel.hpp"
#include "pms8g.h"

namespace pms8 {

// GPUs replace the OpenMP team: options.workers > 1 runs that many GPUs
// (devices 0..workers-1) through pms8g_solve_multi, else one GPU.
MotifSet run_parallel_gpu(const Problem& problem, const SolverConfig& config, const ParallelOptions& options,
                          RunReport* report) {
    problem.validate();
    std::vector<uint8_t> codes;
    codes.reserve(static_cast<size_t>(problem.n()) * static_cast<size_t>(problem.m()));
    for (const auto& s : problem.sequences)
        for (char c : s) codes.push_back(problem.alphabet.code(c));
    pms8g_options o;
    pms8g_default_options(&o);
    if (config.threshold_override) o.threshold = *config.threshold_override > 0 ? *config.threshold_override : -1;
    o.sort_rows = config.sort_rows ? 1 : 0;
    o.prune_level = static_cast<int>(config.prune_level);
    o.reverify = config.reverify_against_originals ? 1 : 0;
    if (config.max_motifs) o.max_motifs = *config.max_motifs;
    pms8g_result r;
    char err[512] = {0};
    int rc;
    if (options.workers > 1) {
        std::vector<int> devices(static_cast<size_t>(options.workers));
        for (int i = 0; i < options.workers; ++i) devices[static_cast<size_t>(i)] = i;
        rc = pms8g_solve_multi(codes.data(), problem.n(), problem.m(), problem.motif_length, problem.max_mismatches,
                               problem.alphabet.symbols().c_str(), &o, devices.data(), options.workers, &r, err,
                               sizeof err);
    } else {
        rc = pms8g_solve(codes.data(), problem.n(), problem.m(), problem.motif_length, problem.max_mismatches,
                         problem.alphabet.symbols().c_str(), &o, &r, err, sizeof err);
    }
    if (rc == PMS8G_ERR_INVALID) throw std::invalid_argument(err);
    if (rc == PMS8G_ERR_LOGIC) throw std::logic_error(err);
    if (rc != PMS8G_OK) throw std::runtime_error(err);
    MotifSet out;
    out.reserve(static_cast<size_t>(r.count));
    for (int64_t i = 0; i < r.count; ++i) out.emplace_back(r.motifs + i * r.l, static_cast<size_t>(r.l));
    if (report) {
        const pms8g_report& g = r.report;
        report->n = g.n;
        report->m = g.m;
        report->l = g.l;
        report->d = g.d;
        report->alphabet = problem.alphabet.name();
        report->threshold = g.threshold;
        report->workers = g.gpus;
        report->subproblems = g.subproblems;
        report->motif_count = g.motif_count;
        report->wall_seconds = g.wall_seconds;
        report->sample_seconds = g.sample_seconds;
        report->pattern_seconds = g.pattern_seconds;
        report->memory.pair_matrix_words = g.pair_matrix_words;
        report->memory.row_matrix_words = g.row_matrix_words;
        report->memory.row_bookkeeping_words = g.row_bookkeeping_words;
        report->memory.packed_words = g.packed_words;
        report->memory.lookup_table_words = g.lookup_table_words;
        report->counters.stacks_explored = g.stacks_explored;
        report->counters.neighborhoods = g.neighborhoods;
        report->counters.neighbors_visited = g.neighbors_visited;
        report->counters.motifs_emitted = g.motifs_emitted;
    }
    pms8g_result_free(&r);
    return out;  // already canonical (sorted by byte value, unique)
}

}  // namespace pms8
