// tests/orch_driver.cpp — TEST INFRASTRUCTURE (the drop-in parity harness).
//
// Runs the reference's Orchestrator (proj/include/marlsim/orchestrator.hpp,
// unmodified) end to end and dumps what tests/test_gpu_dropin.py compares.
// oracle/Makefile compiles it twice from the same source:
//   oracle/_ref/orch_stock  — the stock reference build (CPU TrainingEngine);
//   oracle/_ref/orch_b200   — with -I dropin first, so orchestrator.hpp's
//                             #include "marlsim/training.hpp" resolves to the
//                             B200 drop-in (dropin/marlsim/training.hpp).
// Usage: orch_{stock,b200} <out_dir> <steps> <static_allocation 0|1> <training_slots> [vocab feat]
// Writes <out_dir>/<agent>.w0 / .w (f64 V x D, initial / final weights) and
// <out_dir>/events.ndjson (activate / suspend / micro_grad / update records).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "marlsim/orchestrator.hpp"

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s out_dir steps static_allocation training_slots\n", argv[0]);
        return 2;
    }
    const std::string out = argv[1];
    marlsim::RunConfig cfg;
    cfg.steps = std::atoi(argv[2]);
    cfg.static_allocation = std::atoi(argv[3]) != 0;
    cfg.training_slots = std::atoi(argv[4]);
    if (argc >= 7) {
        cfg.model.vocab_size = static_cast<std::size_t>(std::atoll(argv[5]));
        cfg.model.feature_dim = static_cast<std::size_t>(std::atoll(argv[6]));
    }
    try {
        marlsim::Orchestrator orch(cfg);
        orch.run();
        for (const std::string& agent : cfg.agents) {
            const marlsim::Matrix w0 = orch.trainer().initial_model(agent).weights();
            const marlsim::Matrix w = orch.final_weights(agent);
            std::ofstream(out + "/" + agent + ".w0", std::ios::binary)
                .write(reinterpret_cast<const char*>(w0.a.data()), static_cast<std::streamsize>(w0.a.size() * 8));
            std::ofstream(out + "/" + agent + ".w", std::ios::binary)
                .write(reinterpret_cast<const char*>(w.a.data()), static_cast<std::streamsize>(w.a.size() * 8));
        }
        std::ofstream ev(out + "/events.ndjson");
        for (const auto& r : orch.log().records()) {
            if (r.kind != "micro_grad" && r.kind != "update" && r.kind != "activate" && r.kind != "suspend") continue;
            marlsim::Json j = r.payload;
            j["t"] = r.t;
            j["kind"] = r.kind;
            ev << j.dump() << "\n";
        }
    } catch (const marlsim::Error& e) {
        std::fprintf(stderr, "marlsim error: %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
