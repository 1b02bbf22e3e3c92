// pms8g_cpp.cpp — C++ host API (pms8g.hpp) over the C ABI, plus FASTA/plain IO.
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

std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

std::string strip(const std::string& s) {
    const size_t b = s.find_first_not_of(" \t\r\n");
    if (b == std::string::npos) return {};
    const size_t e = s.find_last_not_of(" \t\r\n");
    return s.substr(b, e - b + 1);
}

void upcase(std::string& s) {
    for (char& c : s) c = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
}

void parse_comment(const std::string& line, SequenceFile& out) {
    const std::string body = strip(line.substr(1));
    const size_t eq = body.find('=');
    if (eq == std::string::npos || eq == 0) return;
    out.metadata[strip(body.substr(0, eq))] = strip(body.substr(eq + 1));
}

// parse_fasta / parse_plain, src/io.cpp:41-95
SequenceFile parse_fasta(const std::string& text) {
    SequenceFile out;
    std::istringstream in(text);
    std::string line, current;
    bool have = false;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        if (line[0] == ';') {
            if (!have) parse_comment(line, out);
            continue;
        }
        if (line[0] == '>') {
            if (have) out.sequences.push_back(std::move(current));
            current.clear();
            have = true;
            out.names.push_back(strip(line.substr(1)));
            continue;
        }
        if (!have)
            throw std::runtime_error("malformed FASTA: sequence data before any '>' header at line " +
                                     std::to_string(lineno));
        std::string chunk = strip(line);
        upcase(chunk);
        current += chunk;
    }
    if (have) out.sequences.push_back(std::move(current));
    if (out.sequences.empty()) throw std::runtime_error("malformed FASTA: no records found");
    for (size_t i = 0; i < out.sequences.size(); ++i)
        if (out.sequences[i].empty())
            throw std::runtime_error("malformed FASTA: record " + std::to_string(i + 1) + " (" + out.names[i] +
                                     ") is empty");
    return out;
}

SequenceFile parse_plain(const std::string& text) {
    SequenceFile out;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        std::string s = strip(line);
        if (s.empty() || s[0] == ';') {
            if (!s.empty()) parse_comment(s, out);
            continue;
        }
        upcase(s);
        out.sequences.push_back(std::move(s));
    }
    if (out.sequences.empty()) throw std::runtime_error("no sequences found");
    return out;
}

}  // namespace

std::string alphabet_symbols(const std::string& name) {
    if (name == "dna") return "ACGT";
    if (name == "protein") return "ACDEFGHIKLMNPQRSTVWY";
    const std::string prefix = "custom:";
    if (name.rfind(prefix, 0) == 0) {
        std::string up = name.substr(prefix.size());
        upcase(up);
        return up;
    }
    throw std::invalid_argument("unknown alphabet \"" + name + "\" (expected dna, protein or custom:<symbols>)");
}

void Problem::validate() const {
    if (sequences.empty()) throw std::invalid_argument("no input sequences");
    const int len = m();
    if (motif_length < 1) throw std::invalid_argument("motif length must be >= 1");
    if (motif_length > len)
        throw std::invalid_argument("motif length " + std::to_string(motif_length) + " exceeds sequence length " +
                                    std::to_string(len));
    if (max_mismatches < 0 || max_mismatches > motif_length)
        throw std::invalid_argument("mismatch budget must be in [0, l], got " + std::to_string(max_mismatches));
    for (size_t i = 0; i < sequences.size(); ++i) {
        if (static_cast<int>(sequences[i].size()) != len)
            throw std::invalid_argument("sequence " + std::to_string(i) + " has length " +
                                        std::to_string(sequences[i].size()) + ", expected " + std::to_string(len));
        for (size_t j = 0; j < sequences[i].size(); ++j)
            if (alphabet.find(sequences[i][j]) == std::string::npos)
                throw std::invalid_argument("sequence " + std::to_string(i) + ", position " + std::to_string(j) +
                                            ": symbol '" + sequences[i][j] + "' not in alphabet " + alphabet_name);
    }
}

MotifSet run_parallel(const Problem& problem, const SolverConfig& config, const GpuOptions& options,
                      RunReport* report) {
    problem.validate();
    const int n = problem.n(), m = problem.m();
    std::vector<uint8_t> codes(static_cast<size_t>(n) * m);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < m; ++j)
            codes[static_cast<size_t>(i) * m + j] = static_cast<uint8_t>(problem.alphabet.find(problem.sequences[i][j]));
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
    if (!options.anchors.empty()) {
        o.anchors = options.anchors.data();
        o.nanchors = static_cast<int>(options.anchors.size());
    }
    pms8g_result res;
    char err[512] = {0};
    const int rc = pms8g_solve(codes.data(), n, m, problem.motif_length, problem.max_mismatches,
                               problem.alphabet.c_str(), &o, &res, err, sizeof err);
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
    }
    pms8g_result_free(&res);
    return out;
}

MotifSet solve(const Problem& problem, const SolverConfig& config, RunReport* report) {
    return run_parallel(problem, config, GpuOptions{}, report);
}

SequenceFile read_plain(const std::string& path) { return parse_plain(slurp(path)); }

std::vector<MotifSet> solve_batch(const std::vector<Problem>& problems, const SolverConfig& config, int device) {
    std::vector<MotifSet> out(problems.size());
    if (problems.empty()) return out;
    const Problem& p0 = problems[0];
    std::vector<std::vector<uint8_t>> codes;
    std::vector<const uint8_t*> ptrs;
    for (const auto& p : problems) {
        p.validate();
        if (p.n() != p0.n() || p.m() != p0.m() || p.motif_length != p0.motif_length ||
            p.max_mismatches != p0.max_mismatches || p.alphabet != p0.alphabet)
            throw std::invalid_argument("solve_batch: every problem must have the same n, m, l, d and alphabet");
        codes.emplace_back();
        for (const auto& s : p.sequences)
            for (char ch : s) codes.back().push_back(static_cast<uint8_t>(p.alphabet.find(ch)));
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
    problem.validate();
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
    const std::vector<uint8_t> codes = encode_codes(problem.sequences, problem.alphabet);
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
    problem.validate();
    const std::vector<uint8_t> codes = encode_codes(problem.sequences, problem.alphabet);
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

SequenceFile read_sequences(const std::string& path) {
    // format sniff, src/io.cpp:101-111
    const std::string text = slurp(path);
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        const std::string s = strip(line);
        if (s.empty() || s[0] == ';') continue;
        return s[0] == '>' ? parse_fasta(text) : parse_plain(text);
    }
    return parse_plain(text);
}

void write_fasta(const std::string& path, const std::vector<std::string>& names,
                 const std::vector<std::string>& sequences,
                 const std::vector<std::pair<std::string, std::string>>& metadata) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot write " + path);
    for (const auto& [k, v] : metadata) out << "; " << k << "=" << v << "\n";
    constexpr size_t wrap = 70;
    for (size_t i = 0; i < sequences.size(); ++i) {
        out << ">" << (i < names.size() ? names[i] : "seq_" + std::to_string(i)) << "\n";
        for (size_t pos = 0; pos < sequences[i].size(); pos += wrap) out << sequences[i].substr(pos, wrap) << "\n";
    }
    if (!out) throw std::runtime_error("write failed for " + path);
}

}  // namespace pms8g
