/*
 * oracle/heatbem_oracle_q.c -- quad-precision build of the CPU oracle
 * (TEST INFRASTRUCTURE ONLY).  Same source as heatbem_oracle.c with every
 * internal quantity in __float128 (libquadmath erfq/expq/sqrtq): the exact
 * value of the reference's quadrature, used to measure how far the
 * reference's own fp64 result and the GPU result each are from it.
 * Exported symbols carry a _q suffix.
 */
#include <quadmath.h>
#define HB_REAL __float128
#define HB_ERF erfq
#define HB_EXP expq
#define HB_SQRT sqrtq
#define HB_PI M_PIq
#define HB_SYM(name) name##_q
#define HB_WITH_PASS 0
#include "heatbem_oracle.c"
