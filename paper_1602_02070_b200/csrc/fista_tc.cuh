// fista_tc.cuh -- the tensor-core L~_r Z product of the fp32 FISTA path
// (gram_tc.cu), used by fista.cu.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace cpcag_cuda {

struct FistaTcPlan {
  i64 rr = 0, rc = 0, ld = 0;
  int np = 0, nkc = 0, S = 0;
  size_t smem = 0;
  CUtensorMap mAh{}, mAl{}, mBh{}, mBl{};
};

// rr >= 128, rc <= 256 and every k slice within the kernel's chunk budget.
bool fista_tc_supported(i64 rr, i64 rc, int S);
// Splits the dense (symmetric) L~_r into Ah/Al (ld x rr, ld = rr rounded up
// to 4) and builds the tensor maps (Zh/Zl: ld x rc, filled per iteration).
void fista_tc_setup(Ctx* c, i64 rr, i64 rc, int S, const float* Lr_dense, float* Ah, float* Al, float* Zh, float* Zl,
                    FistaTcPlan* pl);
// part1[s] = L~_r Z over the s-th k slice (Z split into Zh/Zl first); skipped
// when *done.
void fista_tc_part1(Ctx* c, const FistaTcPlan& pl, const float* Z, float* Zh, float* Zl, double* part1, const int* done);

}  // namespace cpcag_cuda
