// Timeline exporters (reference report.hpp:38-53) and the measured timing model.
#pragma once

#include <string>

#include "schedule.hpp"

namespace bfpp {

std::string chrome_trace_json(const Timeline& timeline, const TaskGraph& graph);
std::string gantt_svg(const Timeline& timeline, const TaskGraph& graph);
// Per-kind mean task durations of a (measured) timeline as the simulator's TimingModel.
TimingModel measured_timing_model(const TaskGraph& graph, const Timeline& timeline);

}  // namespace bfpp
