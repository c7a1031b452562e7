// convert.hpp — C-ABI struct <-> planner type conversions shared by the
// planner and executor entry points.
#pragma once
#include <string>

#include "host/planner.hpp"
#include "memo.h"

namespace memo {

char* dup_string(const std::string& s);
ModelConfig from_c(const memo_model_config& c);
void to_c(const ModelConfig& m, memo_model_config& c);
HardwareConfig from_c(const memo_hardware_config& h);
Skeletal from_c(const memo_skeletal_sizes& s);
SwapDecision from_c(const memo_swap_plan& s);
void to_c(const SwapDecision& d, memo_swap_plan& s);
Timing from_c(const memo_timing_model& t);
Timeline from_c(const memo_schedule_event* ev, std::size_t n, std::uint64_t n_layers);

}  // namespace memo
