// trigger.cuh — device trigger stage (Algorithm 1).
#pragma once

#include "objects.h"

namespace csg {

struct WinStat {
  uint32_t n_rec;
  uint32_t n_comp;
  uint32_t has_state;
  uint32_t pad;
  unsigned long long bytes;
  double min_end;
  double max_end;
};

struct TrigParams {
  double delta;
  double drop;
  double inflate;
  double alpha;
  int32_t warmup;
  int32_t pad;
};

inline TrigParams trig_params(const csg_trigger_config& c) {
  TrigParams p;
  p.delta = c.delta_ms;
  p.drop = c.throughput_drop_factor;
  p.inflate = c.interval_inflation_factor;
  p.alpha = c.ema_alpha;
  p.warmup = c.warmup_windows;
  p.pad = 0;
  return p;
}

void trigger_window_stats(csg_store* s, const double* d_ticks, int32_t T,
                          const int32_t* d_sampled, int32_t S, double delta,
                          WinStat* d_out);
int32_t trigger_ticks(csg_store* s, double I, double delta, DevBuf& ticks);
// Returns the number of tripped ticks; events[0..n) in tick order.
int32_t trigger_run(csg_store* s, const double* d_ticks, int32_t T,
                    const int32_t* d_sampled, int32_t S, const TrigParams& p,
                    DevBuf& events);
void trigger_evaluate_single(csg_store* s, const int32_t* sampled, int32_t S,
                             double t, csg_trigger_state* state,
                             const TrigParams& p, int* tripped,
                             csg_trigger_event* event);

}  // namespace csg
