// gf_internal.h -- error plumbing shared by the C-ABI translation units.
#pragma once
#include "../../include/gatefit_b200.h"

void gf_set_error(const char *fmt, ...);
int gf_fail(int code, const char *fmt, ...);

#ifdef __CUDACC__
#include "gf_common.cuh"
// fast paths of the public kernel ops for arity / support sizes 8 and 16
// (gf_hessian.cu); row / col: per support position, slot orientation
int gf_fast_hole_apply(const void *psi, void *out, int k, int lo, int hi, const int *row, const int *col, int arity,
                       void *stream);
int gf_fast_array_apply(const void *in, void *out, int k, int arity, int lo, int hi, const gf::Mat4 &g, int sparse,
                        void *stream);
int gf_fast_hole_array(const void *bra, const void *arr, int k, int arity, int lo, int hi, const int *row,
                       const int *col, int ncols, void *out, void *stream);
#endif
