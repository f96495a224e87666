// rnnwave/trace.hpp -- the schedule-trace value types of the reference API
// (proj/include/rnnwave/scheduler.hpp:35, 180-192): sched::TaskPhase, sched::TraceRecord and
// sched::ScheduleTrace, which Engine::set_trace_sink fills from the device's stamps
// (rw_trace_records). When the reference's own scheduler.hpp is on the include path (a caller
// that also uses its build_graph / validate_trace / write_trace_csv), its definitions are used,
// so both can be included in one translation unit.
#pragma once

#if __has_include("rnnwave/scheduler.hpp")
#include "rnnwave/scheduler.hpp"
#else
#include <cstdint>
#include <vector>

namespace rnnwave::sched {

enum class TaskPhase { InputGemm, RecurrentStep };

struct TraceRecord {
  int task_id = 0;
  int layer = 0;
  int block = 0;
  int step_k = 0;
  TaskPhase phase = TaskPhase::InputGemm;
  int worker = 0;
  std::int64_t start_ns = 0;
  std::int64_t end_ns = 0;
};

using ScheduleTrace = std::vector<TraceRecord>;

}  // namespace rnnwave::sched
#endif
