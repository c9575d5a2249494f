// Runs the reference's epoch pipeline (pipeline.hpp run_epoch: beacon paths,
// distinct check, aggregation, GKR, dist_sumcheck, DistPc) and prints its
// report without timings. Built twice by oracle/Makefile: against the plain
// reference (epoch_cpu) and with include/dropin first (epoch_gpu: gkr_prove,
// pcs::commit / open on the B200 prover); tests/test_gpu_dropin.py compares
// the two reports byte for byte, with and without tamper hooks.
// usage: epoch_{cpu,gpu} [validators blocks workers seed [tamper hooks...]]
#include <cstdlib>
#include <iostream>

#include "dgkr/pipeline.hpp"

int main(int argc, char** argv) {
    dgkr::pipeline::EpochConfig cfg;
    cfg.record_timings = false;
    if (argc > 4) {
        cfg.validators = std::strtoull(argv[1], nullptr, 10);
        cfg.blocks = std::strtoull(argv[2], nullptr, 10);
        cfg.workers = std::strtoull(argv[3], nullptr, 10);
        cfg.seed = std::strtoull(argv[4], nullptr, 10);
        for (int i = 5; i < argc; ++i) cfg.tamper_hooks.push_back(argv[i]);
    }
    const auto rep = dgkr::pipeline::run_epoch(cfg);
    std::cout << rep.to_json().dump() << "\n";
    return 0;
}
