// gf_internal.h -- error plumbing shared by the C-ABI translation units.
#pragma once
#include "../../include/gatefit_b200.h"

void gf_set_error(const char *fmt, ...);
int gf_fail(int code, const char *fmt, ...);
