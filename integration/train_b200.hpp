// Reference-side drop-in for the MORLAX training step on B200.
// A maintainer adds integration/train_b200.{hpp,cpp} next to proj/src/train.cpp
// and links libmorlax_b200.so; cmd_train (tools/cmd_train.cpp:36) then calls
// train_b200 in place of train. Same signatures and exception types as the
// reference entry points they replace.
#pragma once

#include <string>
#include <vector>

#include "morlax/pareto.hpp"
#include "morlax/trainer.hpp"

namespace morlax {

// train() (include/morlax/trainer.hpp:256-257; src/train.cpp:55-229) on the GPU
Checkpoint train_b200(const RunConfig& cfg, const TrainOptions& opts, const IterationCallback& callback = {});

// nondominated_filter (include/morlax/pareto.hpp:21-30; src/pareto.cpp:38-77) on the GPU
std::vector<ObjectiveVector> nondominated_filter_b200(const std::vector<ObjectiveVector>& points);

// evaluate_params (include/morlax/trainer.hpp:271-276; src/evaluate.cpp:17-101) on the GPU
EvalTable evaluate_params_b200(const HypernetSpec& spec, const HypernetParams& params, const std::string& env_name,
                               int grid_resolution, int episodes_per_point, const Rng& rng);

}  // namespace morlax
