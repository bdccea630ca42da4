/*
 * tierflow_b200_tuning.h — tuning hooks of the fused update kernel: the 40
 * measured launch configurations and element-math forms of DESIGN.md §5.1
 * (register / TMA / cp.async / verified-fast-path variants), every one
 * bit-identical to the shipped kernel. No reference counterpart.
 *
 * Library: paper_2509_02480_b200/lib/libtierflow_b200_tuning.so, built with
 * `python -m paper_2509_02480_b200.build --tuning` (also by __graft_entry__.
 * build() for the tests and sweeps). The product library
 * libtierflow_b200.so does not contain these kernels; the update path never
 * loads this one.
 */
#ifndef TIERFLOW_B200_TUNING_H
#define TIERFLOW_B200_TUNING_H

#include "tierflow_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Kernel tuning hook (no reference counterpart): the fused kernel in launch
 * configuration `variant` (0 = the shipped default; 1..count-1 F16/F16 only). */
int tfg_adam_variant_count(int* count);
int tfg_adam_fused_variant(int variant, float* p, float* m, float* v, const uint16_t* grad, uint16_t* param16,
                           uint64_t n, const tfg_adam_hyper* hyper, uint64_t t, unsigned long long* counters,
                           void* stream);

/* The fused reduce + update (tfg_adam_fused_multi) in form `variant`:
 * 0 = the staged n-source kernel (2, 4 or 8 sources), 1 = the register
 * n-source kernel. F16/F16. */
int tfg_adam_fused_multi_variant(int variant, float* p, float* m, float* v, const void* const* grads, int n_sources,
                                 uint16_t* param16, uint64_t n, const tfg_adam_hyper* hyper, uint64_t t,
                                 unsigned long long* counters, void* stream);

/* Self-test of the second verified fast path (variants 44-46): the largest
 * relative error of its approximate step against the exact chain over n
 * random (m, v, t), and the elements whose P/m/v bits differ from the
 * shipped kernel (must be 0). */
int tfg_selftest_fast_step(uint64_t n, uint64_t seed, double* worst_rel_err, uint64_t* mismatches);
/* Self-test of variant 47's in-range sqrt / division against the library's
 * __dsqrt_rn / __ddiv_rn on n random operand pairs: mismatches (must be 0). */
int tfg_selftest_fast_rn(uint64_t n, uint64_t seed, uint64_t* mismatches);

#ifdef __cplusplus
}
#endif

#endif /* TIERFLOW_B200_TUNING_H */
