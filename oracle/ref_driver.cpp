// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A small driver that links the reference's own library objects, compiled
// unmodified from /root/reference/proj/src by oracle/Makefile into oracle/_ref/.
// It is the "reference" CPU arm: golden motif sets for tests/golden/, the
// CPU baseline timed by bench.py (--impl reference and the cpu_baseline leg),
// and per-depth work counters used to size the GPU design.
//
// Every entry point here calls the reference's public API:
//   generate_planted_instance  src/instance.cpp:22-73
//   run_parallel               src/parallel.cpp:35-118
//   MotifSearch::run_anchored  src/solver.cpp:427-432
//   MotifSearch::push/pop      src/solver.cpp:245-342
//   enumerate_and_collect      src/solver.cpp:387-404
//   canonical_motif_set        src/solver.cpp:16-21
//
// Sub-commands (all print to stdout; numbers are plain text or one JSON line):
//   gen    l d seed [n m mode alphabet]    -> motif, positions, sequences
//   solve  l d seed threads [t]            -> sorted motif set of run_parallel + report
//   anchors l d seed threads "o1,o2,.." [t] -> per-anchor sorted motif sets (run_anchored)
//   time   l d seed threads stride [t]     -> ctx build + strided anchors, timing JSON
//   branch l d seed anchor "i1,i2,.." [t]  -> motif set of depth-1 branches (anchor, row[i])
//   stats  l d seed "o1,.." [t]            -> per-depth work counters (mirrors recurse())
//   branchtime l d seed threads jobs cap [t] -> capped depth-1 branch sample (CPU baseline, (50,21))
//   branch2 l d seed t threads             -> planted depth-1 branch split into depth-2 branches (union)
//   anchorsplit l d seed t threads "o1,.." -> whole S1 l-mers, depth-1 branches of all in one dynamic loop
//   kat                                    -> SPEC known-answer values as JSON
//   file   path l d threads [t alphabet]   -> solve sequences read from a file (one per line)
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "pms8/instance.hpp"
#include "pms8/io.hpp"
#include "pms8/neighborhood.hpp"
#include "pms8/oracle.hpp"
#include "pms8/parallel.hpp"
#include "pms8/pruning.hpp"
#include "pms8/solver.hpp"

using namespace pms8;

namespace {

double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

std::vector<long> parse_list(const std::string& s) {
    std::vector<long> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) {
        if (tok.empty()) continue;
        // "a-b" ranges and "a:b:step" strides are accepted
        const auto dash = tok.find('-');
        const auto colon = tok.find(':');
        if (colon != std::string::npos) {
            long a = std::stol(tok.substr(0, colon));
            const auto rest = tok.substr(colon + 1);
            const auto c2 = rest.find(':');
            long b = std::stol(rest.substr(0, c2));
            long st = c2 == std::string::npos ? 1 : std::stol(rest.substr(c2 + 1));
            for (long x = a; x < b; x += st) out.push_back(x);
        } else if (dash != std::string::npos && dash > 0) {
            long a = std::stol(tok.substr(0, dash)), b = std::stol(tok.substr(dash + 1));
            for (long x = a; x <= b; ++x) out.push_back(x);
        } else {
            out.push_back(std::stol(tok));
        }
    }
    return out;
}

PlantedInstance make(int l, int d, uint64_t seed, int n = 20, int m = 600, bool exact = true,
                     const std::string& alphabet = "dna") {
    PlantedInstanceSpec spec;
    spec.alphabet = Alphabet::named(alphabet);
    spec.l = l;
    spec.d = d;
    spec.n = n;
    spec.m = m;
    spec.seed = seed;
    spec.mutation = exact ? MutationMode::exactly_d : MutationMode::at_most_d;
    return generate_planted_instance(spec);
}

SolverConfig config_with(int t) {
    SolverConfig c;
    if (t > 0) c.threshold_override = t;
    return c;
}

void print_report(const RunReport& r) {
    std::printf(
        "REPORT {\"threshold\": %d, \"workers\": %d, \"subproblems\": %lld, \"motif_count\": %lld, "
        "\"wall_seconds\": %.6f, \"sample_seconds\": %.6f, \"pattern_seconds\": %.6f, "
        "\"stacks_explored\": %lld, \"neighborhoods\": %lld, \"neighbors_visited\": %lld, "
        "\"motifs_emitted\": %lld, \"pair_matrix_words\": %llu}\n",
        r.threshold, r.workers, (long long)r.subproblems, (long long)r.motif_count, r.wall_seconds,
        r.sample_seconds, r.pattern_seconds, (long long)r.counters.stacks_explored,
        (long long)r.counters.neighborhoods, (long long)r.counters.neighbors_visited,
        (long long)r.counters.motifs_emitted, (unsigned long long)r.memory.pair_matrix_words);
}

// Mirrors MotifSearch::recurse (src/solver.cpp:406-419) through the public
// push/pop/rows API, counting per-depth work. Row sorting after push uses the
// reference's own RowMatrix::sort_rows_by_size (src/solver.cpp:205-217).
struct Stats {
    std::vector<long long> pushes, viable, slots, live_after;
    long long tuples = 0, leaves = 0, verify_cmp = 0, rows_touched = 0, emitted = 0;
    explicit Stats(int t) : pushes(t + 1), viable(t + 1), slots(t + 1), live_after(t + 1) {}
};

void stats_recurse(const SolverContext& ctx, MotifSearch& s, Stats& st, std::vector<std::string>& out) {
    const int p = s.depth();
    const auto& rows = s.rows();
    const int n = rows.rows();
    const auto live = rows.live(rows.row_at_position(p));
    std::vector<uint32_t> snap(live.begin(), live.end());
    for (uint32_t u : snap) {
        long long slots = 0;
        for (int q = p; q < n; ++q) slots += s.rows().live_count(s.rows().row_at_position(q));
        st.slots[p + 1] += slots;
        st.pushes[p + 1]++;
        if (s.push(u)) {
            st.viable[p + 1]++;
            auto& rw = const_cast<RowMatrix&>(s.rows());
            rw.sort_rows_by_size(s.depth());
            long long la = 0;
            for (int q = s.depth(); q < n; ++q) la += s.rows().live_count(s.rows().row_at_position(q));
            st.live_after[p + 1] += la;
            if (s.depth() == ctx.threshold()) {
                st.tuples++;
                std::vector<std::string> local;
                const auto before = s.counters();
                s.enumerate_and_collect(local);
                const auto after = s.counters();
                st.leaves += after.neighbors_visited - before.neighbors_visited;
                st.emitted += after.motifs_emitted - before.motifs_emitted;
                for (auto& m : local) out.push_back(m);
            } else {
                stats_recurse(ctx, s, st, out);
            }
        }
        s.pop();
    }
}

int cmd_gen(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int n = argc > 5 ? std::atoi(argv[5]) : 20;
    const int m = argc > 6 ? std::atoi(argv[6]) : 600;
    const bool exact = argc > 7 ? std::string(argv[7]) == "exact" : true;
    const std::string alphabet = argc > 8 ? argv[8] : "dna";
    const auto inst = make(l, d, seed, n, m, exact, alphabet);
    std::printf("MOTIF %s\nPOSITIONS", inst.motif.c_str());
    for (int p : inst.positions) std::printf(" %d", p);
    std::printf("\n");
    for (const auto& s : inst.problem.sequences) std::printf("%s\n", s.c_str());
    return 0;
}

int solve_and_print(const Problem& problem, int threads, int t) {
    ParallelOptions par;
    par.workers = threads;
    RunReport report;
    const auto motifs = run_parallel(problem, config_with(t), par, &report);
    for (const auto& m : motifs) std::printf("%s\n", m.c_str());
    print_report(report);
    return 0;
}

int cmd_solve(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int threads = std::atoi(argv[5]);
    const int t = argc > 6 ? std::atoi(argv[6]) : 0;
    const auto inst = make(l, d, seed);
    return solve_and_print(inst.problem, threads, t);
}

int cmd_file(int argc, char** argv) {
    const SequenceFile f = read_sequences(argv[2]);
    Problem problem;
    problem.sequences = f.sequences;
    problem.motif_length = std::atoi(argv[3]);
    problem.max_mismatches = std::atoi(argv[4]);
    const int threads = std::atoi(argv[5]);
    const int t = argc > 6 ? std::atoi(argv[6]) : 0;
    if (argc > 7) problem.alphabet = Alphabet::named(argv[7]);
    return solve_and_print(problem, threads, t);
}

int cmd_anchors(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int threads = std::atoi(argv[5]);
    const auto offsets = parse_list(argv[6]);
    const int t = argc > 7 ? std::atoi(argv[7]) : 0;
    const auto inst = make(l, d, seed);
    const double t0 = now();
    SolverContext ctx(inst.problem, config_with(t));
    const double t1 = now();
    std::vector<std::vector<std::string>> res(offsets.size());
    std::vector<double> secs(offsets.size());
    std::vector<SolveCounters> ctr(offsets.size());
    std::atomic<long> next{0};
#pragma omp parallel num_threads(threads)
    {
        MotifSearch search(ctx);
        for (;;) {
            const long j = next.fetch_add(1);
            if (j >= static_cast<long>(offsets.size())) break;
            const auto before = search.counters();
            const double a = now();
            search.run_anchored(static_cast<uint32_t>(offsets[j]), res[j]);
            secs[j] = now() - a;
            const auto after = search.counters();
            ctr[j].stacks_explored = after.stacks_explored - before.stacks_explored;
            ctr[j].neighborhoods = after.neighborhoods - before.neighborhoods;
            ctr[j].neighbors_visited = after.neighbors_visited - before.neighbors_visited;
            ctr[j].motifs_emitted = after.motifs_emitted - before.motifs_emitted;
        }
    }
    const double t2 = now();
    for (size_t j = 0; j < offsets.size(); ++j) {
        const auto set = canonical_motif_set(res[j]);
        std::printf("ANCHOR %ld %.6f %lld %lld %lld %lld", offsets[j], secs[j],
                    (long long)ctr[j].stacks_explored, (long long)ctr[j].neighborhoods,
                    (long long)ctr[j].neighbors_visited, (long long)ctr[j].motifs_emitted);
        for (const auto& m : set) std::printf(" %s", m.c_str());
        std::printf("\n");
    }
    std::printf("TIMING {\"ctx_seconds\": %.6f, \"anchors_seconds\": %.6f, \"threads\": %d, \"threshold\": %d}\n",
                t1 - t0, t2 - t1, threads, ctx.threshold());
    return 0;
}

// Bounded CPU-baseline sample: context build (serial pair matrix) plus a
// strided subset of S1 l-mers through run_anchored in an OpenMP dynamic loop —
// the body of run_parallel (src/parallel.cpp:54-78) restricted to the subset.
int cmd_time(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int threads = std::atoi(argv[5]);
    const int stride = std::atoi(argv[6]);
    const int t = argc > 7 ? std::atoi(argv[7]) : 0;
    const int first = argc > 8 ? std::atoi(argv[8]) : 0;
    const auto inst = make(l, d, seed);
    const double t0 = now();
    SolverContext ctx(inst.problem, config_with(t));
    const double t1 = now();
    const int jobs = inst.problem.m() - l + 1;
    std::vector<long> offsets;
    for (long o = first; o < jobs; o += stride) offsets.push_back(o);
    std::vector<std::vector<std::string>> res(offsets.size());
    std::atomic<long> next{0};
#pragma omp parallel num_threads(threads)
    {
        MotifSearch search(ctx);
        for (;;) {
            const long j = next.fetch_add(1);
            if (j >= static_cast<long>(offsets.size())) break;
            search.run_anchored(static_cast<uint32_t>(offsets[j]), res[j]);
        }
    }
    const double t2 = now();
    std::vector<std::string> raw;
    for (auto& r : res) raw.insert(raw.end(), r.begin(), r.end());
    const auto motifs = canonical_motif_set(raw);
    std::printf("TIMING {\"ctx_seconds\": %.6f, \"anchors_seconds\": %.6f, \"anchors\": %zu, \"jobs\": %d, "
                "\"threads\": %d, \"threshold\": %d, \"motifs\": %zu}\n",
                t1 - t0, t2 - t1, offsets.size(), jobs, threads, ctx.threshold(), motifs.size());
    return 0;
}

// Depth-1 branch: push the anchor, sort, then push row-at-position-1 entry i
// and recurse — the motif set under (anchor, u) is {M : M motif, Hd(M,anchor)
// <= d, Hd(M,u) <= d}, independent of the tree below.
int cmd_branch(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const long anchor = std::atol(argv[5]);
    const std::string which = argv[6];
    std::vector<long> idx = which == "planted" ? std::vector<long>{} : parse_list(which);
    const int t = argc > 7 ? std::atoi(argv[7]) : 0;
    const int threads = argc > 8 ? std::atoi(argv[8]) : 1;
    const auto inst = make(l, d, seed);
    SolverContext ctx(inst.problem, config_with(t));
    const auto& set = ctx.set();
    // branching row after the anchor push
    std::vector<uint32_t> brow;
    {
        MotifSearch s(ctx);
        // run_anchored's setup: restrict row 0 to the anchor, sort, push it
        auto& rw = const_cast<RowMatrix&>(s.rows());
        rw.reset_full();
        rw.restrict_row(0, set.lmer_id(0, static_cast<uint32_t>(anchor)));
        rw.sort_rows_by_size(0);
        if (!s.push(set.lmer_id(0, static_cast<uint32_t>(anchor)))) {
            std::printf("ANCHOR_NOT_VIABLE\n");
            return 0;
        }
        rw.sort_rows_by_size(1);
        const auto live = s.rows().live(s.rows().row_at_position(1));
        brow.assign(live.begin(), live.end());
        std::printf("BRANCHROW %d %zu\n", s.rows().row_at_position(1), brow.size());
    }
    if (which == "planted") {
        // the branching-row l-mer that is the planted occurrence of its sequence
        for (size_t j = 0; j < brow.size(); ++j) {
            const auto r = set.ref_of(brow[j]);
            if (static_cast<int>(r.offset) == inst.positions[r.seq]) idx.push_back(static_cast<long>(j));
        }
    }
    std::vector<std::vector<std::string>> res(idx.size());
    std::vector<double> secs(idx.size());
    std::atomic<long> next{0};
#pragma omp parallel num_threads(threads)
    {
        MotifSearch s(ctx);
        for (;;) {
            const long j = next.fetch_add(1);
            if (j >= static_cast<long>(idx.size())) break;
            if (idx[j] >= static_cast<long>(brow.size())) continue;
            const double a = now();
            auto& rw = const_cast<RowMatrix&>(s.rows());
            rw.reset_full();
            rw.restrict_row(0, set.lmer_id(0, static_cast<uint32_t>(anchor)));
            rw.sort_rows_by_size(0);
            if (s.push(set.lmer_id(0, static_cast<uint32_t>(anchor)))) {
                rw.sort_rows_by_size(1);
                if (s.push(brow[static_cast<size_t>(idx[j])])) {
                    rw.sort_rows_by_size(2);
                    Stats st(ctx.threshold());
                    if (s.depth() == ctx.threshold()) s.enumerate_and_collect(res[j]);
                    else stats_recurse(ctx, s, st, res[j]);
                }
                s.pop();
            }
            s.pop();
            secs[j] = now() - a;
        }
    }
    for (size_t j = 0; j < idx.size(); ++j) {
        const auto ref = set.ref_of(idx[j] < static_cast<long>(brow.size()) ? brow[static_cast<size_t>(idx[j])] : 0);
        const auto ms = canonical_motif_set(res[j]);
        std::printf("BRANCH %ld %u %u %.6f", idx[j], ref.seq, ref.offset, secs[j]);
        for (const auto& m : ms) std::printf(" %s", m.c_str());
        std::printf("\n");
    }
    return 0;
}

// The planted depth-1 branch of the planted S1 l-mer, split into its depth-2
// branches (anchor, u1, u2) run by an OpenMP dynamic loop: the union of the
// depth-2 motif sets is the depth-1 branch's set (every branching-row l-mer is
// branched on, src/solver.cpp:406-419). For (l,d) where one depth-1 branch
// takes hours of one core ((50,21)). Prints one DONE line per depth-2 branch
// to stderr (progress) and the union on stdout.
int cmd_branch2(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int t = std::atoi(argv[5]);
    const int threads = std::atoi(argv[6]);
    const auto inst = make(l, d, seed);
    SolverContext ctx(inst.problem, config_with(t));
    const auto& set = ctx.set();
    const uint32_t a = set.lmer_id(0, static_cast<uint32_t>(inst.positions[0]));
    auto setup = [&](MotifSearch& s) -> bool {
        auto& rw = const_cast<RowMatrix&>(s.rows());
        rw.reset_full();
        rw.restrict_row(0, a);
        rw.sort_rows_by_size(0);
        if (!s.push(a)) return false;
        rw.sort_rows_by_size(1);
        return true;
    };
    uint32_t u1 = 0;
    std::vector<uint32_t> brow2;
    {
        MotifSearch s(ctx);
        if (!setup(s)) {
            std::printf("ANCHOR_NOT_VIABLE\n");
            return 0;
        }
        bool found = false;
        for (uint32_t u : s.rows().live(s.rows().row_at_position(1))) {
            const auto r = set.ref_of(u);
            if (static_cast<int>(r.offset) == inst.positions[r.seq]) {
                u1 = u;
                found = true;
                break;
            }
        }
        if (!found || !s.push(u1)) {
            std::printf("PLANTED_BRANCH_NOT_VIABLE\n");
            return 0;
        }
        const_cast<RowMatrix&>(s.rows()).sort_rows_by_size(2);
        const auto live = s.rows().live(s.rows().row_at_position(2));
        brow2.assign(live.begin(), live.end());
        const auto r1 = set.ref_of(u1);
        std::printf("BRANCH1 anchor=%d u1_seq=%u u1_off=%u row2=%d size=%zu threshold=%d\n", inst.positions[0],
                    r1.seq, r1.offset, s.rows().row_at_position(2), brow2.size(), ctx.threshold());
        std::fflush(stdout);
    }
    std::vector<std::vector<std::string>> res(brow2.size());
    std::atomic<long> next{0};
    const double t0 = now();
#pragma omp parallel num_threads(threads)
    {
        MotifSearch s(ctx);
        for (;;) {
            const long j = next.fetch_add(1);
            if (j >= static_cast<long>(brow2.size())) break;
            const double b = now();
            if (setup(s)) {
                auto& rw = const_cast<RowMatrix&>(s.rows());
                if (s.push(u1)) {
                    rw.sort_rows_by_size(2);
                    if (s.push(brow2[static_cast<size_t>(j)])) {
                        rw.sort_rows_by_size(3);
                        Stats st(ctx.threshold());
                        if (s.depth() == ctx.threshold()) s.enumerate_and_collect(res[j]);
                        else stats_recurse(ctx, s, st, res[j]);
                    }
                    s.pop();
                }
                s.pop();
            }
            while (s.depth() > 0) s.pop();
            const auto r = set.ref_of(brow2[static_cast<size_t>(j)]);
            std::fprintf(stderr, "DONE %ld/%zu seq=%u off=%u %.3f s (elapsed %.1f s) motifs=%zu\n", j,
                         brow2.size(), r.seq, r.offset, now() - b, now() - t0, res[j].size());
        }
    }
    std::vector<std::string> all;
    for (auto& v : res) all.insert(all.end(), v.begin(), v.end());
    const auto ms = canonical_motif_set(all);
    std::printf("UNION %.3f", now() - t0);
    for (const auto& m : ms) std::printf(" %s", m.c_str());
    std::printf("\n");
    return 0;
}

// Whole S1 l-mers (run_anchored, src/solver.cpp:427-432), each split into its
// depth-1 branches, all branches of all listed S1 offsets in one OpenMP
// dynamic loop (one heavy S1 l-mer then uses every thread). Prints one
// ANCHOR line per offset: offset, thread-seconds, motif set.
int cmd_anchorsplit(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int t = std::atoi(argv[5]);
    const int threads = std::atoi(argv[6]);
    const auto offsets = parse_list(argv[7]);
    const auto inst = make(l, d, seed);
    SolverContext ctx(inst.problem, config_with(t));
    const auto& set = ctx.set();
    auto setup = [&](MotifSearch& s, uint32_t a) -> bool {
        auto& rw = const_cast<RowMatrix&>(s.rows());
        rw.reset_full();
        rw.restrict_row(0, a);
        rw.sort_rows_by_size(0);
        if (!s.push(a)) return false;
        rw.sort_rows_by_size(1);
        return true;
    };
    struct Job {
        size_t ai;
        uint32_t u;
    };
    std::vector<Job> jobs;
    {
        MotifSearch s(ctx);
        for (size_t i = 0; i < offsets.size(); ++i) {
            const uint32_t a = set.lmer_id(0, static_cast<uint32_t>(offsets[i]));
            if (setup(s, a))
                for (uint32_t u : s.rows().live(s.rows().row_at_position(1))) jobs.push_back({i, u});
            while (s.depth() > 0) s.pop();
        }
    }
    std::vector<std::vector<std::string>> res(offsets.size());
    std::vector<double> secs(offsets.size(), 0.0);
    std::atomic<long> next{0};
    const double t0 = now();
#pragma omp parallel num_threads(threads)
    {
        MotifSearch s(ctx);
        std::vector<std::string> out;
        for (;;) {
            const long j = next.fetch_add(1);
            if (j >= static_cast<long>(jobs.size())) break;
            const double b = now();
            const Job jb = jobs[static_cast<size_t>(j)];
            out.clear();
            if (setup(s, set.lmer_id(0, static_cast<uint32_t>(offsets[jb.ai])))) {
                if (s.push(jb.u)) {
                    const_cast<RowMatrix&>(s.rows()).sort_rows_by_size(2);
                    Stats st(ctx.threshold());
                    if (s.depth() == ctx.threshold()) s.enumerate_and_collect(out);
                    else stats_recurse(ctx, s, st, out);
                }
            }
            while (s.depth() > 0) s.pop();
            const double dt = now() - b;
#pragma omp critical
            {
                secs[jb.ai] += dt;
                res[jb.ai].insert(res[jb.ai].end(), out.begin(), out.end());
            }
            if (j % 500 == 0) std::fprintf(stderr, "job %ld/%zu elapsed %.1f s\n", j, jobs.size(), now() - t0);
        }
    }
    for (size_t i = 0; i < offsets.size(); ++i) {
        const auto ms = canonical_motif_set(res[i]);
        std::printf("ANCHOR %ld %.6f", offsets[i], secs[i]);
        for (const auto& m : ms) std::printf(" %s", m.c_str());
        std::printf("\n");
    }
    std::printf("TIMING {\"wall_seconds\": %.6f, \"jobs\": %zu, \"threads\": %d, \"threshold\": %d}\n", now() - t0,
                jobs.size(), threads, ctx.threshold());
    return 0;
}

// recurse (src/solver.cpp:406-419) through the public push/pop/rows API like
// stats_recurse, giving up once `deadline` passes (the subtree is then only
// partly searched: its time is a lower bound). Returns false on timeout.
bool timed_recurse(const SolverContext& ctx, MotifSearch& s, double deadline, std::vector<std::string>& out) {
    const int p = s.depth();
    const auto& rows = s.rows();
    const auto live = rows.live(rows.row_at_position(p));
    std::vector<uint32_t> snap(live.begin(), live.end());
    for (uint32_t u : snap) {
        if (now() > deadline) return false;
        bool ok = true;
        if (s.push(u)) {
            auto& rw = const_cast<RowMatrix&>(s.rows());
            rw.sort_rows_by_size(s.depth());
            if (s.depth() == ctx.threshold()) s.enumerate_and_collect(out);
            else ok = timed_recurse(ctx, s, deadline, out);
        }
        s.pop();
        if (!ok) return false;
    }
    return true;
}

// Bounded CPU sample for configs where one S1 l-mer exceeds any budget
// ((50,21)): `jobs` depth-1 branches spread over the S1
// l-mers (anchor = i * w / jobs, branch index = a fixed hash of i modulo the
// anchor's branching-row size), run in an OpenMP dynamic loop, each capped
// at cap_seconds. Also counts every S1 l-mer's depth-1 branches (the
// projection's multiplier). Output: one BTIME line per job, then SUMMARY.
int cmd_branchtime(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const int threads = std::atoi(argv[5]);
    const int jobs = std::atoi(argv[6]);
    const double cap = std::atof(argv[7]);
    const int t = argc > 8 ? std::atoi(argv[8]) : 0;
    const auto inst = make(l, d, seed);
    const double t0 = now();
    SolverContext ctx(inst.problem, config_with(t));
    const double t1 = now();
    const auto& set = ctx.set();
    const int w = inst.problem.m() - l + 1;
    // depth-1 branch rows of every S1 l-mer (run_anchored's setup, src/solver.cpp:427-432)
    std::vector<std::vector<uint32_t>> brow(static_cast<size_t>(w));
    std::atomic<long> next{0};
#pragma omp parallel num_threads(threads)
    {
        MotifSearch s(ctx);
        for (;;) {
            const long a = next.fetch_add(1);
            if (a >= w) break;
            auto& rw = const_cast<RowMatrix&>(s.rows());
            rw.reset_full();
            rw.restrict_row(0, set.lmer_id(0, static_cast<uint32_t>(a)));
            rw.sort_rows_by_size(0);
            if (s.push(set.lmer_id(0, static_cast<uint32_t>(a)))) {
                rw.sort_rows_by_size(1);
                const auto live = s.rows().live(s.rows().row_at_position(1));
                brow[static_cast<size_t>(a)].assign(live.begin(), live.end());
            }
            s.pop();
        }
    }
    long long total_branches = 0;
    for (const auto& b : brow) total_branches += static_cast<long long>(b.size());
    const double t2 = now();
    std::vector<long> ja(static_cast<size_t>(jobs)), jb(static_cast<size_t>(jobs));
    for (int i = 0; i < jobs; ++i) {
        long a = static_cast<long>(i) * w / jobs;
        while (brow[static_cast<size_t>(a)].empty()) a = (a + 1) % w;
        ja[static_cast<size_t>(i)] = a;
        const unsigned long long h = (static_cast<unsigned long long>(i) + 1) * 0x9E3779B97F4A7C15ull;
        jb[static_cast<size_t>(i)] = static_cast<long>((h >> 33) % brow[static_cast<size_t>(a)].size());
    }
    std::vector<double> secs(static_cast<size_t>(jobs));
    std::vector<int> done(static_cast<size_t>(jobs));
    std::vector<size_t> nmot(static_cast<size_t>(jobs));
    next = 0;
#pragma omp parallel num_threads(threads)
    {
        MotifSearch s(ctx);
        for (;;) {
            const long j = next.fetch_add(1);
            if (j >= jobs) break;
            const long a = ja[static_cast<size_t>(j)];
            const double b0 = now();
            std::vector<std::string> out;
            bool complete = true;
            auto& rw = const_cast<RowMatrix&>(s.rows());
            rw.reset_full();
            rw.restrict_row(0, set.lmer_id(0, static_cast<uint32_t>(a)));
            rw.sort_rows_by_size(0);
            if (s.push(set.lmer_id(0, static_cast<uint32_t>(a)))) {
                rw.sort_rows_by_size(1);
                if (s.push(brow[static_cast<size_t>(a)][static_cast<size_t>(jb[static_cast<size_t>(j)])])) {
                    rw.sort_rows_by_size(2);
                    if (s.depth() == ctx.threshold()) s.enumerate_and_collect(out);
                    else complete = timed_recurse(ctx, s, b0 + cap, out);
                }
                s.pop();
            }
            s.pop();
            secs[static_cast<size_t>(j)] = now() - b0;
            done[static_cast<size_t>(j)] = complete ? 1 : 0;
            nmot[static_cast<size_t>(j)] = canonical_motif_set(out).size();
        }
    }
    const double t3 = now();
    double sum = 0;
    int ndone = 0;
    for (int j = 0; j < jobs; ++j) {
        sum += secs[static_cast<size_t>(j)];
        ndone += done[static_cast<size_t>(j)];
        std::printf("BTIME %ld %ld %.6f %d %zu\n", ja[static_cast<size_t>(j)], jb[static_cast<size_t>(j)],
                    secs[static_cast<size_t>(j)], done[static_cast<size_t>(j)], nmot[static_cast<size_t>(j)]);
    }
    std::printf("SUMMARY {\"ctx_seconds\": %.6f, \"branchrow_seconds\": %.6f, \"sample_seconds\": %.6f, "
                "\"jobs\": %d, \"completed\": %d, \"cap_seconds\": %.3f, \"thread_seconds\": %.6f, "
                "\"total_branches\": %lld, \"s1_lmers\": %d, \"threads\": %d, \"threshold\": %d}\n",
                t1 - t0, t2 - t1, t3 - t2, jobs, ndone, cap, sum, total_branches, w, threads, ctx.threshold());
    return 0;
}

int cmd_stats(int argc, char** argv) {
    const int l = std::atoi(argv[2]), d = std::atoi(argv[3]);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const auto offsets = parse_list(argv[5]);
    const int t = argc > 6 ? std::atoi(argv[6]) : 0;
    const int threads = argc > 7 ? std::atoi(argv[7]) : 1;
    const auto inst = make(l, d, seed);
    SolverContext ctx(inst.problem, config_with(t));
    const auto& set = ctx.set();
    const int T = ctx.threshold();
    Stats total(T);
    double secs = 0;
    std::atomic<long> next{0};
#pragma omp parallel num_threads(threads)
    {
        MotifSearch s(ctx);
        Stats st(T);
        std::vector<std::string> out;
        const double a = now();
        for (;;) {
            const long j = next.fetch_add(1);
            if (j >= static_cast<long>(offsets.size())) break;
            auto& rw = const_cast<RowMatrix&>(s.rows());
            rw.reset_full();
            rw.restrict_row(0, set.lmer_id(0, static_cast<uint32_t>(offsets[j])));
            rw.sort_rows_by_size(0);
            stats_recurse(ctx, s, st, out);
        }
        const double b = now() - a;
#pragma omp critical
        {
            secs = std::max(secs, b);
            for (int k = 0; k <= T; ++k) {
                total.pushes[k] += st.pushes[k];
                total.viable[k] += st.viable[k];
                total.slots[k] += st.slots[k];
                total.live_after[k] += st.live_after[k];
            }
            total.tuples += st.tuples;
            total.leaves += st.leaves;
            total.emitted += st.emitted;
        }
    }
    std::printf("STATS threshold=%d anchors=%zu seconds=%.3f tuples=%lld leaves=%lld emitted=%lld\n", T,
                offsets.size(), secs, total.tuples, total.leaves, total.emitted);
    for (int k = 1; k <= T; ++k)
        std::printf("DEPTH %d pushes=%lld viable=%lld slots=%lld live_after=%lld avg_live_after=%.1f\n", k,
                    total.pushes[k], total.viable[k], total.slots[k], total.live_after[k],
                    total.viable[k] ? double(total.live_after[k]) / total.viable[k] : 0.0);
    return 0;
}

std::string jstr(const std::string& s) { return "\"" + s + "\""; }

// Known-answer values of SPEC.md examples, computed by the reference's own
// functions; tests/golden/spec_kat.json pins oracle/pms8_oracle.c to them.
int cmd_kat() {
    std::ostringstream o;
    o << "{";
    // N_d (src/instance.cpp:75-87)
    o << "\"neighborhood_size\": [";
    bool first = true;
    for (int l : {1, 2, 4, 6, 13, 17, 21, 23, 50})
        for (int d = 0; d <= std::min(l, 22); ++d) {
            if (!first) o << ",";
            first = false;
            o << "[" << l << "," << d << ",4," << jstr(neighborhood_size(l, d, 4).str()) << "]";
        }
    o << "],";
    // threshold (src/solver.cpp:104-117)
    o << "\"threshold\": [";
    first = true;
    for (auto [l, d] : std::vector<std::pair<int, int>>{{13, 4}, {15, 5}, {17, 6}, {19, 7}, {21, 8}, {23, 9},
                                                        {25, 10}, {50, 21}, {7, 1}, {5, 1}, {9, 2}, {11, 3}})
        for (int n : {1, 2, 3, 5, 20})
            for (int m : {600, 30, 20}) {
                if (m < l) continue;
                if (!first) o << ",";
                first = false;
                o << "[" << n << "," << m << "," << l << "," << d << ",4," << estimate_threshold(n, m, l, d, 4)
                  << "]";
            }
    o << "],";
    // Theorem 1 and Cd (src/pruning.cpp:27-75)
    const std::vector<std::string> tri{"AA", "CC", "GG"};
    o << "\"triple_AA_CC_GG_111\": "
      << (triple_common_neighbor_exists("AA", "CC", "GG", Budgets{1, 1, 1}) ? "true" : "false") << ",";
    o << "\"triple_AAAA_AAAT_AATT_111\": "
      << (triple_common_neighbor_exists("AAAA", "AAAT", "AATT", Budgets{1, 1, 1}) ? "true" : "false") << ",";
    {
        std::vector<std::string_view> t3{"ACG", "ACT", "GCT"};
        o << "\"consensus_ACG_ACT_GCT\": " << consensus_total_distance(t3) << ",";
        std::vector<std::string_view> t4{"AA", "CC", "GG", "TT"};
        o << "\"consensus_AA_CC_GG_TT\": " << consensus_total_distance(t4) << ",";
    }
    {
        int64_t c1 = generate_common_neighborhood(std::vector<std::string>{"AC"}, 1, Alphabet::dna(),
                                                  [](std::string_view) {});
        o << "\"cn_AC_d1\": " << c1 << ",";
        std::vector<std::string> got;
        generate_common_neighborhood(std::vector<std::string>{"AA", "TT"}, 1, Alphabet::dna(),
                                     [&](std::string_view s) { got.emplace_back(s); });
        o << "\"cn_AA_TT_d1\": [";
        for (size_t i = 0; i < got.size(); ++i) o << (i ? "," : "") << jstr(got[i]);
        o << "],";
    }
    // random triples: Theorem 1 decision + Cd, exercised by the C oracle
    {
        std::mt19937_64 rng(12345);
        o << "\"triples\": [";
        for (int i = 0; i < 400; ++i) {
            const int l = 1 + static_cast<int>(rng() % 8);
            std::string s[3];
            for (auto& x : s) {
                x.resize(static_cast<size_t>(l));
                for (auto& c : x) c = "ACGT"[rng() % 4];
            }
            const int b1 = static_cast<int>(rng() % 4), b2 = static_cast<int>(rng() % 4),
                      b3 = static_cast<int>(rng() % 4);
            const bool ok = triple_common_neighbor_exists(s[0], s[1], s[2], Budgets{b1, b2, b3});
            o << (i ? "," : "") << "[" << jstr(s[0]) << "," << jstr(s[1]) << "," << jstr(s[2]) << "," << b1 << ","
              << b2 << "," << b3 << "," << (ok ? 1 : 0) << "]";
        }
        o << "],";
    }
    // common neighbourhoods of random tuples (k<=5, l<=7): count + first/last
    {
        std::mt19937_64 rng(777);
        o << "\"neighborhoods\": [";
        for (int i = 0; i < 120; ++i) {
            const int k = 1 + static_cast<int>(rng() % 5);
            const int l = 2 + static_cast<int>(rng() % 6);
            const int d = static_cast<int>(rng() % 3);
            std::vector<std::string> tup(static_cast<size_t>(k));
            for (auto& x : tup) {
                x.resize(static_cast<size_t>(l));
                for (auto& c : x) c = "ACGT"[rng() % 4];
            }
            std::vector<std::string> got;
            generate_common_neighborhood(tup, d, Alphabet::dna(), [&](std::string_view s) { got.emplace_back(s); });
            o << (i ? "," : "") << "[" << d << ",[";
            for (int j = 0; j < k; ++j) o << (j ? "," : "") << jstr(tup[static_cast<size_t>(j)]);
            o << "],[";
            for (size_t j = 0; j < got.size(); ++j) o << (j ? "," : "") << jstr(got[j]);
            o << "]]";
        }
        o << "]";
    }
    o << "}";
    std::printf("%s\n", o.str().c_str());
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: pms8ref gen|solve|anchors|time|branch|stats|kat|file ...\n");
        return 2;
    }
    try {
        const std::string cmd = argv[1];
        if (cmd == "gen" && argc >= 5) return cmd_gen(argc, argv);
        if (cmd == "solve" && argc >= 6) return cmd_solve(argc, argv);
        if (cmd == "file" && argc >= 6) return cmd_file(argc, argv);
        if (cmd == "anchors" && argc >= 7) return cmd_anchors(argc, argv);
        if (cmd == "time" && argc >= 7) return cmd_time(argc, argv);
        if (cmd == "branch" && argc >= 7) return cmd_branch(argc, argv);
        if (cmd == "branch2" && argc >= 7) return cmd_branch2(argc, argv);
        if (cmd == "anchorsplit" && argc >= 8) return cmd_anchorsplit(argc, argv);
        if (cmd == "stats" && argc >= 6) return cmd_stats(argc, argv);
        if (cmd == "branchtime" && argc >= 8) return cmd_branchtime(argc, argv);
        if (cmd == "kat") return cmd_kat();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    std::fprintf(stderr, "bad arguments\n");
    return 2;
}
