// TEST INFRASTRUCTURE ONLY - runs the reference tuning engine (Algorithm 1, scheduler.cpp:240-290)
// on a model file and prints its convergence curve plus an exact digest of every family model.
// Linked twice by oracle/Makefile:
//   engine_ref   - with the reference's own costmodel.o + family.o
//   engine_b200  - with libfamtune_b200.so in their place (the drop-in: every fit / predict /
//                  family lookup of the unchanged scheduler runs through the B200 library)
//   engine_b200_batched - -DFS_BATCHED_ENGINE: famtune::gpu::BatchedTuningEngine (the batched
//                  caller, paper_2201_00194_b200/host/batched_engine.cpp) on the drop-in
// tests/test_engine_e2e.py requires the outputs to be byte-identical. The loop's wall time goes
// to stderr ("engine_wall_s <seconds>").
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "famtune/costmodel.hpp"
#include "famtune/family.hpp"
#include "famtune/graph.hpp"
#include "famtune/scheduler.hpp"
#include "famtune/simbackend.hpp"
#ifdef FS_BATCHED_ENGINE
#include "famtune/batched_engine.hpp"
using Engine = famtune::gpu::BatchedTuningEngine;
#else
using Engine = famtune::TuningEngine;
#endif

using namespace famtune;

static std::uint64_t fnv(const void* p, std::size_t n, std::uint64_t h) {
  const auto* c = static_cast<const unsigned char*>(p);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= c[i];
    h *= 1099511628211ULL;
  }
  return h;
}

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: %s model.json budget seed algo(0-2) foresee(0/1) trees\n", argv[0]);
    return 2;
  }
  const auto model = load_model(argv[1]);
  const std::int64_t budget = std::atoll(argv[2]);
  const std::uint64_t seed = std::strtoull(argv[3], nullptr, 10);
  const int algo = std::atoi(argv[4]);
  const bool foresee = std::atoi(argv[5]) != 0;
  const int trees = std::atoi(argv[6]);
  const auto truth = build_registry(ClusterAlgo::ByCoreOp, model.subgraphs);
  SimBackend backend(model, make_landscape(model, truth, seed), seed);
  TuneOptions opt;
  opt.budget = budget;
  opt.seed = seed;
  opt.cost_model.trees = trees;
  const ClusterAlgo ca = algo == 1 ? ClusterAlgo::ByOpCount : algo == 2 ? ClusterAlgo::ByOpSequence : ClusterAlgo::ByCoreOp;
  const auto t0 = std::chrono::steady_clock::now();
  Engine engine(backend, foresee ? make_foresee_policy(ca) : make_baseline_policy(ca), opt);
  const auto state = engine.run();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::fprintf(stderr, "engine_wall_s %.6f\n", wall);
  std::fputs(curve_to_csv(state).c_str(), stdout);
  std::fputs(engine.registry().to_csv().c_str(), stdout);
  for (const auto& m : engine.models()) {
    std::uint64_t h = 14695981039346656037ULL;
    h = fnv(&m.base_prediction, sizeof(double), h);
    std::size_t nodes = 0;
    for (const auto& t : m.trees)
      for (const auto& nd : t.nodes) {
        h = fnv(&nd.feature, sizeof nd.feature, h);
        h = fnv(&nd.threshold, sizeof nd.threshold, h);
        h = fnv(&nd.left, sizeof nd.left, h);
        h = fnv(&nd.right, sizeof nd.right, h);
        h = fnv(&nd.value, sizeof nd.value, h);
        ++nodes;
      }
    std::printf("model family=%d samples=%zu trees=%zu nodes=%zu digest=%016llx\n", m.family_id, m.training_set.size(),
                m.trees.size(), nodes, static_cast<unsigned long long>(h));
  }
  return 0;
}
