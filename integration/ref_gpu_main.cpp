// integration/ref_gpu_main.cpp — TEST INFRASTRUCTURE: a reference-side caller
// of run_parallel_gpu. Generates the planted instance with the reference's own
// generator (src/instance.cpp:22-73) and prints the motif set, one per line,
// then `REPORT threshold workers motif_count stacks_explored`.
//   pms8ref_gpu l d seed [workers]
#include <cstdio>
#include <cstdlib>

#include "pms8/instance.hpp"
#include "pms8/parallel.hpp"

namespace pms8 {
MotifSet run_parallel_gpu(const Problem&, const SolverConfig&, const ParallelOptions&, RunReport*);
}

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    pms8::PlantedInstanceSpec spec;
    spec.l = std::atoi(argv[1]);
    spec.d = std::atoi(argv[2]);
    spec.seed = std::strtoull(argv[3], nullptr, 10);
    spec.mutation = pms8::MutationMode::exactly_d;
    const auto inst = pms8::generate_planted_instance(spec);
    pms8::ParallelOptions par;
    par.workers = argc > 4 ? std::atoi(argv[4]) : 1;
    pms8::RunReport rep;
    try {
        const auto motifs = pms8::run_parallel_gpu(inst.problem, pms8::SolverConfig{}, par, &rep);
        for (const auto& m : motifs) std::printf("%s\n", m.c_str());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    std::printf("REPORT %d %d %lld %lld\n", rep.threshold, rep.workers, (long long)rep.motif_count,
                (long long)rep.counters.stacks_explored);
    return 0;
}
