// simulate_main.cpp — `rlsim simulate <config.json>` without the CLI11 front end
// (reference proj/tools/main.cpp:59-78, run_table_command): load_config ->
// run_experiment -> the result table as JSON lines on stdout.  Linked twice:
// against the reference's own losses.cpp (oracle/_ref/rlsim_simulate_ref, the CPU
// reference) and against integration/rlsim_gpu_shim.cpp
// (integration/_build/rlsim_simulate_gpu, the same experiment with every
// loss_and_grad / grpo_advantages call on the GPU).
#include <cstdio>
#include <exception>
#include <string>

#include "rlsim/experiment.hpp"

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <config.json>\n", argv[0]);
        return 2;
    }
    try {
        const rlsim::ExperimentConfig cfg = rlsim::load_config(argv[1]);
        const rlsim::ResultTable table = rlsim::run_experiment(cfg, "");
        std::fputs(table.to_jsonl().c_str(), stdout);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
