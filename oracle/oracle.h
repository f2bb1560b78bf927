/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY (see oracle_impl.h).  C ABI of the
 * plain CPU oracle for the adaptive solver of arXiv 2007.11208.  Declares its
 * own types; it deliberately does not include anything from include/ or
 * paper_2007_11208_b200/ (the oracle and the CUDA path share no code).
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

/* literal detection flags */
#define OR_BANDED 0x1u
#define OR_LOWER  0x2u
#define OR_UPPER  0x4u
#define OR_SPD    0x8u
/* solve flags */
#define OR_F_CHOL_FAILED   (1u << 8)
#define OR_F_SINGULAR      (1u << 9)
#define OR_F_RCOND_LOW     (1u << 10)
#define OR_F_FALLBACK      (1u << 11)
#define OR_F_POORLY_COND   (1u << 12)
#define OR_F_NONFINITE     (1u << 13)
#define OR_F_SVD_NOCONV    (1u << 14)
#define OR_F_RANK_DEF      (1u << 15)
#define OR_F_SYMMETRIC     (1u << 16)   /* exact symmetry (only with OR_OPT_SYM_INDEF) */
/* methods */
#define OR_M_BAND 1
#define OR_M_TRI_LOWER 2
#define OR_M_TRI_UPPER 3
#define OR_M_CHOL 4
#define OR_M_LU 5
#define OR_M_SVD 6
#define OR_M_LDLT 7   /* symmetric indefinite LDL^T, Bunch-Kaufman (OR_OPT_SYM_INDEF) */
/* options */
#define OR_OPT_NO_FALLBACK  0x1u
#define OR_OPT_FORCE_METHOD 0x2u
#define OR_OPT_CHECK_FINITE 0x4u
#define OR_OPT_FULLSCAN     0x8u
#define OR_OPT_SYM_INDEF    0x20u  /* exactly symmetric, not (or failed) sympd -> LDL^T (Z30) */
/* errors */
#define OR_ERR_SINGULAR_NO_FALLBACK 1
#define OR_ERR_SVD_NOT_CONVERGED    2
#define OR_ERR_NONFINITE            3

typedef struct {
    uint32_t flags;       /* OR_BANDED | OR_LOWER | OR_UPPER | OR_SPD (literal, each evaluated) */
    int32_t pad;
    int64_t kl, ku;       /* exact band extent */
    double max_diag;      /* Fig. 4 max_diag (0 if a diagonal entry <= 0 stopped pass 1) */
} or_structure;

typedef struct {
    uint32_t flags;
    int32_t force_method;
    double rcond_threshold;  /* < 0: 0.5 eps */
    double lsq_cutoff;       /* < 0: n eps */
    int32_t max_sweeps;      /* <= 0: 30 */
    int32_t pad;
} or_options;

typedef struct {
    uint32_t flags;          /* detection bits 0-3, method bits 4-7, solve bits 8-15 */
    int32_t method;          /* final method (6 = SVD after a fallback) */
    int32_t primary_method;  /* the structured/LU path that ran */
    int32_t sweeps;
    int64_t kl, ku;          /* -1 unless banded (or FULLSCAN) */
    double rcond, anorm;
    int64_t rank;            /* -1 unless the fallback ran */
    int64_t info;            /* 1 + first singular column, 0 otherwise */
    int64_t chol_fail_col;
} or_report;

#endif
