// tests/helpers/json_ref.cpp — TEST INFRASTRUCTURE: prints the `pms8 solve
// --format json` document for given report values with nlohmann::json (the
// library the reference CLI uses, tools/pms8.cpp:31-60,171-176), so
// tests/test_report_json.py can compare pms8g_report_json's bytes with it.
// Input on stdin, one token per line:
//   alphabet command n m l d threshold workers subproblems motif_count
//   wall sample pattern pair row book packed lookup stacks nbh visited emitted
//   count motif...
#include <iostream>
#include <string>
#include <vector>

#include "nlohmann/json.hpp"

int main() {
    using nlohmann::json;
    std::string alphabet, command;
    std::getline(std::cin, alphabet);
    std::getline(std::cin, command);
    long long n, m, l, d, thr, workers, sub, mc;
    double wall, sample, pattern;
    unsigned long long pair, row, book, packed, lookup;
    long long stacks, nbh, visited, emitted, count;
    std::cin >> n >> m >> l >> d >> thr >> workers >> sub >> mc >> wall >> sample >> pattern >> pair >> row >> book >>
        packed >> lookup >> stacks >> nbh >> visited >> emitted >> count;
    std::vector<std::string> motifs(static_cast<size_t>(count));
    for (auto& s : motifs) std::cin >> s;
    const unsigned long long tracked = pair + row + book + packed;
    json rep;
    rep["n"] = n;
    rep["m"] = m;
    rep["l"] = l;
    rep["d"] = d;
    rep["alphabet"] = alphabet;
    rep["threshold"] = thr;
    rep["workers"] = workers;
    rep["subproblems"] = sub;
    rep["motif_count"] = mc;
    rep["wall_seconds"] = wall;
    rep["sample_seconds"] = sample;
    rep["pattern_seconds"] = pattern;
    rep["memory"]["pair_matrix_words"] = pair;
    rep["memory"]["row_matrix_words"] = row;
    rep["memory"]["row_bookkeeping_words"] = book;
    rep["memory"]["packed_words"] = packed;
    rep["memory"]["lookup_table_words"] = lookup;
    rep["memory"]["tracked_total_words"] = tracked;
    rep["memory"]["tracked_total_bytes"] = tracked * 8;
    rep["counters"]["stacks_explored"] = stacks;
    rep["counters"]["neighborhoods"] = nbh;
    rep["counters"]["neighbors_visited"] = visited;
    rep["counters"]["motifs_emitted"] = emitted;
    rep["command"] = command;
    json out;
    out["motifs"] = motifs;
    out["report"] = rep;
    std::cout << out.dump(2) << "\n";
    return 0;
}
