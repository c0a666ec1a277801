/* synth_host.c — host side of the synthetic generators (see synth.h). */
#include "synth.h"

void synth_fill_host(const synth_recipe *p, uint64_t start, uint64_t n, uint64_t *out) {
  if (p->kind == SYN_RUNS) {
    uint64_t x = p->add;
    for (uint64_t i = 0; i < start; ++i) x += synth_run_inc(p->seed, i);
    for (uint64_t i = 0; i < n; ++i) {
      x += synth_run_inc(p->seed, start + i);
      out[i] = x;
    }
    return;
  }
  for (uint64_t i = 0; i < n; ++i) out[i] = synth_value(p, start + i);
}
