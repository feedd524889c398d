/*
 * libinvaskit probe exports: measurement hooks used by tools/ (not part of the
 * drop-in boundary in invaskit.h, not bound by the Python package).
 */
#ifndef INVASKIT_PROBE_H
#define INVASKIT_PROBE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Time the 16-column LU panel kernel on `count` random T x T nodes (rank
 * padding tp, panel width w), `reps` launches; ms = mean launch time, clk =
 * CTA 0's phase clocks. tools/panel_probe.py. */
int ks_probe_panel(int T, int tp, int w, int count, int reps, double* ms, long long* clk);

/* Per-step timeline of the last persistent-LU launch recorded with
 * KS_SLAB_TRACE=1 (tools/slab_trace.py); returns entries written. */
int ks_slab_trace(long long* out, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* INVASKIT_PROBE_H */
