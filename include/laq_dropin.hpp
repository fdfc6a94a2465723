// laq_dropin.hpp -- C++ extensions of the drop-in (integration/laq_dropin*.cpp)
// to the reference's unchanged API (proj/include/laq/cli.hpp).
//
// The paper chooses between the fused operator (the model pushed through the
// join, Y = sum_j I_j (B_j W_j)) and the non-fused one (materialize, then
// predict) with its complexity analysis: Eq. 2 for linear models, Eq. 4 for
// trees (fusion.cpp:199-219), fuse iff ratio > threshold (decide_fusion,
// fusion.cpp:221-224).  The reference only evaluates the model in `laq cost`
// (cli.cpp:709-741) and leaves the pipeline mode to the user (cli.cpp:648-652);
// run_auto lets the cost model pick the plan a PipelineRunner executes.
#pragma once

#include "laq/cli.hpp"
#include "laq/fusion.hpp"

namespace laq::cli {

struct PlanChoice {
  bool fused = true;
  double ratio = 0.0;           // speedup_ratio_linear / _tree
  fusion::CostInputs inputs;    // i = target rows, k, l, p, dim rows
};

// The cost-model plan for a runner; prepares the joins first (i = join rows).
PlanChoice plan_pipeline(PipelineRunner& runner, StageTimes& st, double threshold = 1.0);

// run_fused or run_nonfused, whichever plan_pipeline picks.
PipelineResult run_auto(PipelineRunner& runner, StageTimes& st, double threshold = 1.0,
                        PlanChoice* chosen = nullptr);

}  // namespace laq::cli
