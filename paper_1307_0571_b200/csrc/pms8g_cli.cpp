// pms8g — drop-in CLI for `pms8 solve` / `pms8 generate` (tools/pms8.cpp).
//
//   pms8g solve <input> [-l L] [-d D] [--alphabet A] [--workers N] [--threshold T]
//               [--max-motifs K] [--format text|json] [--prune none|pairs|full]
//               [--no-sort-rows] [--no-pair-matrix] [--reverify] [--device N]
//               [--gpus N | --devices a,b,...]   (several GPUs: pms8g_solve_multi)
//   pms8g verify <input> -M MOTIFS [-l L] [-d D] [--alphabet A] [--device N]
//   pms8g generate -l L -d D [-n N] [-m M] [--alphabet A] [--seed S]
//               [--mutation atmost|exact] [-o FILE]
//
// stdout/stderr/exit codes follow cmd_solve (tools/pms8.cpp:150-184): one motif
// per line (or JSON {motifs, report}), a one-line summary on stderr, exit 0 if
// at least one motif, 1 if none, 2 on usage/input error (:386-389). CLI11 and
// nlohmann::json are not available here: argv parsing is hand-rolled and the
// JSON document comes from pms8g_report_json (byte-identical to dump(2)).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "pms8g.hpp"

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

int to_int(const std::string& flag, const std::string& v) {
    try {
        size_t pos = 0;
        const int x = std::stoi(v, &pos);
        if (pos != v.size()) throw std::invalid_argument(v);
        return x;
    } catch (...) {
        throw Usage(flag + ": expected an integer, got '" + v + "'");
    }
}

int cmd_solve(const std::vector<std::string>& args, const std::string& command) {
    std::string input, alphabet, format = "text", prune = "full";
    std::optional<int> l, d, threshold, workers;
    std::optional<int64_t> max_motifs;
    bool no_sort = false, no_pair = false, reverify = false;
    int device = -1;
    std::vector<int> devices;  // --gpus N / --devices a,b: one process, N GPUs
    for (size_t i = 0; i < args.size(); ++i) {
        const std::string& a = args[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= args.size()) throw Usage(a + " needs a value");
            return args[++i];
        };
        if (a == "-l") l = to_int(a, val());
        else if (a == "-d") d = to_int(a, val());
        else if (a == "--alphabet") alphabet = val();
        else if (a == "--workers") workers = to_int(a, val());
        else if (a == "--threshold") threshold = to_int(a, val());
        else if (a == "--max-motifs") max_motifs = to_int(a, val());
        else if (a == "--format") {
            format = val();
            if (format != "text" && format != "json") throw Usage("--format: text or json");
        } else if (a == "--prune") {
            prune = val();
            if (prune != "none" && prune != "pairs" && prune != "full") throw Usage("--prune: none, pairs or full");
        } else if (a == "--no-sort-rows") no_sort = true;
        else if (a == "--no-pair-matrix") no_pair = true;
        else if (a == "--reverify") reverify = true;
        else if (a == "--device") device = to_int(a, val());
        else if (a == "--gpus") {
            const int g = to_int(a, val());
            if (g < 1) throw Usage("--gpus: at least 1");
            devices.clear();
            for (int i = 0; i < g; ++i) devices.push_back(i);
        } else if (a == "--devices") {
            devices.clear();
            std::string list = val(), tok;
            std::istringstream ls(list);
            while (std::getline(ls, tok, ',')) devices.push_back(to_int(a, tok));
            if (devices.empty()) throw Usage("--devices: a comma-separated list of GPU ordinals");
        } else if (!a.empty() && a[0] == '-') throw Usage("unknown option " + a);
        else if (input.empty()) input = a;
        else throw Usage("unexpected argument " + a);
    }
    if (input.empty()) throw Usage("solve: input file required");
    if (workers && *workers < 1) throw std::invalid_argument("worker count must be >= 1");
    const pms8g::SequenceFile file = pms8g::read_sequences(input);
    auto meta_int = [&](const char* key) -> std::optional<int> {
        auto it = file.metadata.find(key);
        if (it == file.metadata.end()) return std::nullopt;
        return std::stoi(it->second);
    };
    if (!l) l = meta_int("l");
    if (!d) d = meta_int("d");
    if (!l || !d) {
        std::cerr << "error: -l and -d are required (no l/d metadata in " << input << ")\n";
        return 2;
    }
    if (alphabet.empty()) {
        auto it = file.metadata.find("alphabet");
        alphabet = it != file.metadata.end() ? it->second : "dna";
    }
    pms8g::Problem problem;
    problem.sequences = file.sequences;
    problem.motif_length = *l;
    problem.max_mismatches = *d;
    problem.alphabet = pms8g::alphabet_symbols(alphabet);
    problem.alphabet_name = alphabet;
    problem.validate();

    pms8g::SolverConfig config;
    config.threshold_override = threshold;
    config.sort_rows = !no_sort;
    config.use_pair_matrix = !no_pair;
    config.max_motifs = max_motifs;
    config.reverify_against_originals = reverify;
    config.prune_level = prune == "none" ? pms8g::PruneLevel::none
                         : prune == "pairs" ? pms8g::PruneLevel::pairs
                                            : pms8g::PruneLevel::full;
    pms8g::GpuOptions gpu;
    gpu.device = device;
    if (devices.size() > 1) gpu.devices = devices;
    else if (devices.size() == 1) gpu.device = devices[0];
    pms8g::RunReport report;
    const pms8g::MotifSet motifs = pms8g::run_parallel(problem, config, gpu, &report);
    report.command = command;
    if (format == "json") {
        std::cout << pms8g::report_json(motifs, report) << "\n";
    } else {
        for (const auto& m : motifs) std::cout << m << "\n";
        std::cerr << "motifs=" << motifs.size() << " threshold=" << report.threshold << " workers=" << report.workers
                  << " wall=" << report.wall_seconds << "s"
                  << " sample=" << report.sample_seconds << "s pattern=" << report.pattern_seconds << "s\n";
    }
    return motifs.empty() ? 1 : 0;
}

// cmd_verify (tools/pms8.cpp:193-256): one line per candidate, `motif\tPASS\t
// offsets` or `motif\tFAIL`; exit 0 if all pass, 1 otherwise, 2 on bad input.
// The scan runs on the GPU (pms8g_verify_motifs).
int cmd_verify(const std::vector<std::string>& args) {
    std::string input, motifs_path, alphabet;
    std::optional<int> l, d;
    int device = -1;
    for (size_t i = 0; i < args.size(); ++i) {
        const std::string& a = args[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= args.size()) throw Usage(a + " needs a value");
            return args[++i];
        };
        if (a == "-l") l = to_int(a, val());
        else if (a == "-d") d = to_int(a, val());
        else if (a == "-M" || a == "--motifs") motifs_path = val();
        else if (a == "--alphabet") alphabet = val();
        else if (a == "--device") device = to_int(a, val());
        else if (!a.empty() && a[0] == '-') throw Usage("unknown option " + a);
        else if (input.empty()) input = a;
        else throw Usage("unexpected argument " + a);
    }
    if (input.empty()) throw Usage("verify: input file required");
    if (motifs_path.empty()) throw Usage("verify: --motifs is required");
    const pms8g::SequenceFile file = pms8g::read_sequences(input);
    auto meta_int = [&](const char* key) -> std::optional<int> {
        auto it = file.metadata.find(key);
        if (it == file.metadata.end()) return std::nullopt;
        return std::stoi(it->second);
    };
    if (!l) l = meta_int("l");
    if (!d) d = meta_int("d");
    if (!l || !d) {
        std::cerr << "error: -l and -d are required (no l/d metadata in " << input << ")\n";
        return 2;
    }
    if (alphabet.empty()) {
        auto it = file.metadata.find("alphabet");
        alphabet = it != file.metadata.end() ? it->second : "dna";
    }
    pms8g::Problem problem;
    problem.sequences = file.sequences;
    problem.motif_length = *l;
    problem.max_mismatches = *d;
    problem.alphabet = pms8g::alphabet_symbols(alphabet);
    problem.alphabet_name = alphabet;
    problem.validate();
    const pms8g::SequenceFile motif_file = pms8g::read_plain(motifs_path);
    // the reference reports the motifs before the first malformed one, then
    // fails on it (tools/pms8.cpp:219-253): scan that prefix in one batch
    std::vector<std::string> good;
    std::string bad_msg;
    for (const std::string& motif : motif_file.sequences) {
        if (static_cast<int>(motif.size()) != *l) {
            bad_msg = "motif " + motif + " has length " + std::to_string(motif.size()) + ", expected l=" +
                      std::to_string(*l);
            break;
        }
        for (char c : motif)
            if (bad_msg.empty() && problem.alphabet.find(c) == std::string::npos)
                bad_msg = "motif " + motif + " contains symbol '" + std::string(1, c) + "' outside alphabet " +
                          alphabet;
        if (!bad_msg.empty()) break;
        good.push_back(motif);
    }
    const std::vector<pms8g::MotifCheck> checks = pms8g::verify_motifs(problem, good, device);
    bool all_pass = true;
    for (size_t i = 0; i < checks.size(); ++i) {
        const std::string& motif = good[i];
        if (checks[i].pass) {
            std::cout << motif << "\tPASS\t";
            for (size_t k = 0; k < checks[i].witness_offsets.size(); ++k)
                std::cout << (k ? "," : "") << checks[i].witness_offsets[k];
            std::cout << "\n";
        } else {
            std::cout << motif << "\tFAIL\n";
            all_pass = false;
        }
    }
    if (!bad_msg.empty()) {
        std::cerr << "error: " << bad_msg << "\n";
        return 2;
    }
    return all_pass ? 0 : 1;
}

int cmd_generate(const std::vector<std::string>& args) {
    int l = -1, d = -1, n = 20, m = 600;
    std::string alphabet = "dna", mutation = "atmost", output = "instance.fa";
    uint64_t seed = 0;
    for (size_t i = 0; i < args.size(); ++i) {
        const std::string& a = args[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= args.size()) throw Usage(a + " needs a value");
            return args[++i];
        };
        if (a == "-l") l = to_int(a, val());
        else if (a == "-d") d = to_int(a, val());
        else if (a == "-n") n = to_int(a, val());
        else if (a == "-m") m = to_int(a, val());
        else if (a == "--alphabet") alphabet = val();
        else if (a == "--seed") seed = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--mutation") {
            mutation = val();
            if (mutation != "atmost" && mutation != "exact") throw Usage("--mutation: atmost or exact");
        } else if (a == "-o" || a == "--output") output = val();
        else throw Usage("unknown option " + a);
    }
    if (l < 0 || d < 0) throw Usage("generate: -l and -d are required");
    const std::string sym = pms8g::alphabet_symbols(alphabet);
    std::vector<uint8_t> codes(static_cast<size_t>(n) * m), motif(l > 0 ? l : 1);
    std::vector<int32_t> pos(n > 0 ? n : 1);
    if (pms8g_generate(n, m, l, d, static_cast<int>(sym.size()), seed, mutation == "exact", codes.data(),
                       motif.data(), pos.data()) != PMS8G_OK)
        throw std::invalid_argument("need 1 <= l <= m, 0 <= d <= l, n >= 1");
    std::vector<std::string> seqs(n), names(n);
    std::string motif_s(l, ' '), positions;
    for (int p = 0; p < l; ++p) motif_s[p] = sym[motif[p]];
    for (int i = 0; i < n; ++i) {
        seqs[i].resize(m);
        for (int j = 0; j < m; ++j) seqs[i][j] = sym[codes[static_cast<size_t>(i) * m + j]];
        names[i] = "seq_" + std::to_string(i) + " pos=" + std::to_string(pos[i]);
        positions += (i ? "," : "") + std::to_string(pos[i]);
    }
    // metadata lines as cmd_generate writes them (tools/pms8.cpp:82-97)
    std::vector<std::pair<std::string, std::string>> meta{
        {"format", "pms8-planted-instance-v1"}, {"n", std::to_string(n)}, {"m", std::to_string(m)},
        {"l", std::to_string(l)}, {"d", std::to_string(d)}, {"alphabet", alphabet},
        {"seed", std::to_string(seed)}, {"mutation", mutation}, {"motif", motif_s}, {"positions", positions}};
    pms8g::write_fasta(output, names, seqs, meta);
    std::cout << motif_s << "\n";
    std::cerr << "wrote " << output << " (" << n << " sequences of length " << m << ")\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    std::string command;
    for (int i = 0; i < argc; ++i) command += (i ? " " : "") + std::string(argv[i]);
    try {
        if (args.empty()) throw Usage("a subcommand is required: solve | verify | generate");
        const std::string sub = args[0];
        args.erase(args.begin());
        if (sub == "solve") return cmd_solve(args, command);
        if (sub == "generate") return cmd_generate(args);
        if (sub == "verify") return cmd_verify(args);
        throw Usage("unknown subcommand " + sub);
    } catch (const Usage& e) {
        std::cerr << "usage error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
