// fista_persist.cuh -- single-kernel FISTA for the fp32 dense path
// (fista_persist.cu).
#pragma once

#include "common.cuh"

namespace cpcag_cuda {

struct FistaPersistOut {
  i64 iterations;
  int converged, err;
  double frc;
  unsigned long long prof_ns[5];  // CTA 0: phase A, barrier wait, reduce, tile GEMM, element-wise
};

// CPCAG_FISTA_PERSIST=0 disables the path (the per-kernel path then runs).
bool fista_persist_enabled();

// Runs the whole solve (fp32 or fp64); false when the shape does not fit the tiling (the
// caller then takes the per-kernel path).  Dr/Dc are the dense, exactly
// symmetric operators; trace_dev receives one objective value per iteration.
template <typename T>
bool fista_persist_run(Ctx* c, const T* Y, i64 rr, i64 rc, const T* Dr, const T* Dc, const cpcag_frpcag_config& cfg,
                       double step, T* X, double* trace_dev, FistaPersistOut* res);

}  // namespace cpcag_cuda
