/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Instantiates oracle_impl.h for
 * double (suffix _d) and float (suffix _f).  Build (see oracle/build.sh):
 *   gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -fPIC -shared
 * (x86-64 SSE arithmetic, no FMA contraction, no FTZ/DAZ).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SUF)

#define T double
#define SUF d
#define ABS fabs
#define SQRT sqrt
#define NEXTAFTER nextafter
#include "oracle_impl.h"
#undef T
#undef SUF
#undef ABS
#undef SQRT
#undef NEXTAFTER

#define T float
#define SUF f
#define ABS fabsf
#define SQRT sqrtf
#define NEXTAFTER nextafterf
#include "oracle_impl.h"
#undef T
#undef SUF
#undef ABS
#undef SQRT
#undef NEXTAFTER

int or_version(void) { return 1; }

#ifdef _OPENMP
#include <omp.h>
void or_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
int or_get_threads(void) { return omp_get_max_threads(); }
#else
void or_set_threads(int n) { (void)n; }
int or_get_threads(void) { return 1; }
#endif
