/*
 * pf_pipes.h -- issue-rate microbenchmarks (lib/libpf_pipes.so).
 *
 * Measurement support, not part of the reference's interface: the per-pipe
 * peaks that bench.py's roofline.pipes divides by (the paper reports pipe
 * utilisation against such peaks).
 */
#ifndef PF_PIPES_H
#define PF_PIPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* number of instruction kinds and their names: hfma2, hadd2, ffma, dfma,
 * imad, iadd3, lop3, lds, ldg (L1 hit), mufu_ex2, f2f_f16_f64, i2f */
int pf_pipe_count(void);
const char* pf_pipe_name(int i);
const char* pf_pipe_error(void);
/* out[pf_pipe_count()]: warp-instructions per SM per clock, 32 warps per SM */
int pf_pipe_peaks(double* out, int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* PF_PIPES_H */
