// pms8g_cpp.cpp — C++ host API (pms8g.hpp) over the C ABI (sequence files and
// the problem check live in pms8g_io.cpp).
#include "pms8g.hpp"

#include <cctype>
#include <fstream>
#include <sstream>
#include <stdexcept>

namespace pms8g {

namespace {

[[noreturn]] void rethrow(int rc, const char* err) {
    switch (rc) {
        case PMS8G_ERR_INVALID: throw std::invalid_argument(err);
        case PMS8G_ERR_LOGIC: throw std::logic_error(err);
        default: throw std::runtime_error(err);
    }
}

void upcase(std::string& s) {
    for (char& c : s) c = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
}

}  // namespace

std::string alphabet_symbols(const std::string& name) {
    if (name == "dna") return "ACGT";
    if (name == "protein") return "ACDEFGHIKLMNPQRSTVWY";
    const std::string prefix = "custom:";
    if (name.rfind(prefix, 0) == 0) {
        std::string up = name.substr(prefix.size());
        upcase(up);
        // Alphabet ctor checks, src/alphabet.cpp:10-17
        if (up.size() < 2) throw std::invalid_argument("alphabet needs at least 2 symbols, got \"" + up + "\"");
        for (size_t i = 0; i < up.size(); ++i)
            if (up.find(up[i]) != i)
                throw std::invalid_argument(std::string("duplicate alphabet symbol '") + up[i] + "'");
        return up;
    }
    throw std::invalid_argument("unknown alphabet \"" + name + "\" (expected dna, protein or custom:<symbols>)");
}

MotifSet run_parallel(const Problem& problem, const SolverConfig& config, const GpuOptions& options,
                      RunReport* report) {
    const std::vector<uint8_t> codes = encode_problem(problem);  // Problem::validate + codes
    const int n = problem.n(), m = problem.m();
    pms8g_options o;
    pms8g_default_options(&o);
    if (config.threshold_override) {
        o.threshold = *config.threshold_override;
        if (o.threshold == 0) o.threshold = -1;  // rejected like the reference (t < 1)
    }
    o.sort_rows = config.sort_rows ? 1 : 0;
    o.prune_level = static_cast<int>(config.prune_level);
    o.reverify = config.reverify_against_originals ? 1 : 0;
    if (config.max_motifs) o.max_motifs = *config.max_motifs;
    o.device = options.device;
    o.shard_rank = options.shard_rank;
    o.shard_count = options.shard_count;
    o.jitter_max_us = options.jitter_max_us;
    o.jitter_seed = options.jitter_seed;
    if (!options.anchors.empty()) {
        o.anchors = options.anchors.data();
        o.nanchors = static_cast<int>(options.anchors.size());
    }
    pms8g_result res;
    char err[512] = {0};
    const int rc =
        options.devices.empty()
            ? pms8g_solve(codes.data(), n, m, problem.motif_length, problem.max_mismatches, problem.alphabet.c_str(),
                          &o, &res, err, sizeof err)
            : pms8g_solve_multi(codes.data(), n, m, problem.motif_length, problem.max_mismatches,
                                problem.alphabet.c_str(), &o, options.devices.data(),
                                static_cast<int>(options.devices.size()), &res, err, sizeof err);
    if (rc != PMS8G_OK) rethrow(rc, err);
    MotifSet out;
    out.reserve(static_cast<size_t>(res.count));
    for (int64_t i = 0; i < res.count; ++i) out.emplace_back(res.motifs + i * res.l, res.l);
    if (report) {
        const pms8g_report& r = res.report;
        report->n = r.n;
        report->m = r.m;
        report->l = r.l;
        report->d = r.d;
        report->alphabet = problem.alphabet_name;
        report->threshold = r.threshold;
        report->workers = r.gpus;
        report->subproblems = r.subproblems;
        report->motif_count = r.motif_count;
        report->wall_seconds = r.wall_seconds;
        report->sample_seconds = r.sample_seconds;
        report->pattern_seconds = r.pattern_seconds;
        report->device_seconds = r.device_seconds;
        report->counters = {r.stacks_explored, r.neighborhoods, r.neighbors_visited, r.motifs_emitted};
        report->filter_slots = r.filter_slots;
        report->verify_compares = r.verify_compares;
        report->enum_nodes = r.enum_nodes;
        report->device_bytes = r.device_bytes;
        report->device_threshold = r.device_threshold;
        report->raw = r;
    }
    pms8g_result_free(&res);
    return out;
}

std::string report_json(const MotifSet& motifs, const RunReport& report) {
    std::string flat;
    for (const auto& m : motifs) flat += m;
    pms8g_result r{};
    r.count = static_cast<int64_t>(motifs.size());
    r.l = motifs.empty() ? report.l : static_cast<int>(motifs[0].size());
    r.motifs = flat.data();
    r.report = report.raw;
    const int64_t len = pms8g_report_json(&r, report.alphabet.c_str(), report.command.c_str(), nullptr, 0);
    std::string out(static_cast<size_t>(len) + 1, '\0');
    pms8g_report_json(&r, report.alphabet.c_str(), report.command.c_str(), out.data(), out.size());
    out.resize(static_cast<size_t>(len));
    return out;
}

MotifSet solve(const Problem& problem, const SolverConfig& config, RunReport* report) {
    return run_parallel(problem, config, GpuOptions{}, report);
}

std::vector<MotifSet> solve_batch(const std::vector<Problem>& problems, const SolverConfig& config, int device) {
    std::vector<MotifSet> out(problems.size());
    if (problems.empty()) return out;
    const Problem& p0 = problems[0];
    std::vector<std::vector<uint8_t>> codes;
    std::vector<const uint8_t*> ptrs;
    for (const auto& p : problems) {
        std::vector<uint8_t> c = encode_problem(p);
        if (p.n() != p0.n() || p.m() != p0.m() || p.motif_length != p0.motif_length ||
            p.max_mismatches != p0.max_mismatches || p.alphabet != p0.alphabet)
            throw std::invalid_argument("solve_batch: every problem must have the same n, m, l, d and alphabet");
        codes.push_back(std::move(c));
    }
    for (const auto& c : codes) ptrs.push_back(c.data());
    pms8g_options o;
    pms8g_default_options(&o);
    if (config.threshold_override) o.threshold = *config.threshold_override;
    o.sort_rows = config.sort_rows ? 1 : 0;
    o.prune_level = static_cast<int>(config.prune_level);
    o.reverify = config.reverify_against_originals ? 1 : 0;
    if (config.max_motifs) o.max_motifs = *config.max_motifs;
    o.device = device;
    std::vector<pms8g_result> res(problems.size());
    char err[512] = {0};
    const int rc = pms8g_solve_batch(ptrs.data(), static_cast<int>(ptrs.size()), p0.n(), p0.m(), p0.motif_length,
                                     p0.max_mismatches, p0.alphabet.c_str(), &o, res.data(), err, sizeof err);
    if (rc != PMS8G_OK) rethrow(rc, err);
    for (size_t i = 0; i < res.size(); ++i) {
        for (int64_t k = 0; k < res[i].count; ++k) out[i].emplace_back(res[i].motifs + k * res[i].l, res[i].l);
        pms8g_result_free(&res[i]);
    }
    return out;
}

namespace {
std::vector<uint8_t> encode_codes(const std::vector<std::string>& seqs, const std::string& alphabet) {
    std::vector<uint8_t> codes;
    for (const auto& s : seqs)
        for (char ch : s) codes.push_back(static_cast<uint8_t>(alphabet.find(ch)));
    return codes;
}
}  // namespace

std::vector<MotifCheck> verify_motifs(const Problem& problem, const std::vector<std::string>& motifs, int device) {
    const std::vector<uint8_t> codes = encode_problem(problem);
    const int n = problem.n(), m = problem.m(), l = problem.motif_length;
    for (const auto& mt : motifs) {
        if (static_cast<int>(mt.size()) != l)
            throw std::invalid_argument("motif " + mt + " has length " + std::to_string(mt.size()) +
                                        ", expected l=" + std::to_string(l));
        for (char ch : mt)
            if (problem.alphabet.find(ch) == std::string::npos)
                throw std::invalid_argument("motif " + mt + " contains symbol '" + ch + "' outside alphabet " +
                                            problem.alphabet_name);
    }
    std::vector<MotifCheck> out(motifs.size());
    if (motifs.empty()) return out;
    const std::vector<uint8_t> mc = encode_codes(motifs, problem.alphabet);
    std::vector<int32_t> wit(motifs.size() * n);
    std::vector<uint8_t> pass(motifs.size());
    char err[512] = {0};
    const int rc = pms8g_verify_motifs(codes.data(), n, m, l, problem.max_mismatches, problem.alphabet.c_str(),
                                       mc.data(), static_cast<int64_t>(motifs.size()), wit.data(), pass.data(),
                                       device, err, sizeof err);
    if (rc != PMS8G_OK) rethrow(rc, err);
    for (size_t i = 0; i < motifs.size(); ++i) {
        out[i].pass = pass[i] != 0;
        for (int r = 0; r < n && wit[i * n + r] >= 0; ++r) out[i].witness_offsets.push_back(wit[i * n + r]);
    }
    return out;
}

bool naive_is_motif(const Problem& problem, const std::string& motif, std::vector<int>* witness_offsets) {
    const MotifCheck c = verify_motifs(problem, {motif})[0];
    if (witness_offsets) *witness_offsets = c.witness_offsets;
    return c.pass;
}

MotifSet brute_force_solve(const Problem& problem, int64_t enumeration_guard, int device) {
    const std::vector<uint8_t> codes = encode_problem(problem);
    pms8g_result res;
    char err[512] = {0};
    const int rc = pms8g_brute_force(codes.data(), problem.n(), problem.m(), problem.motif_length,
                                     problem.max_mismatches, problem.alphabet.c_str(), enumeration_guard, device,
                                     &res, err, sizeof err);
    if (rc != PMS8G_OK) rethrow(rc, err);
    MotifSet motifs;
    for (int64_t i = 0; i < res.count; ++i) motifs.emplace_back(res.motifs + i * res.l, res.l);
    pms8g_result_free(&res);
    return motifs;
}

}  // namespace pms8g
