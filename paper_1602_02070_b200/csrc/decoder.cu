// decoder.cu -- the graph-regularised alternate decoder (decoders.cpp:145-186):
// conjugate gradient on the normal operator
//     A(X) = gbar_c X Lc + gbar_r Lr X + M o X,   b = scatter(Xt),  X0 = 0,
// with the reference recurrence of detail::pcg_core (solvers.hpp:33-74,
// identity preconditioner: z = r, rho = <r, r>).
//
// Precision.  fp64 data: every vector fp64, per-entry arithmetic of the apply
// bit-identical to the reference loop.  fp32 data: X is stored in fp32, the
// Krylov vectors R, P, AP in fp64 (operator values rounded to fp32, products
// and sums in fp64).  tools/cfg3_precision.py measured at config 3
// (4096 x 200000, 100 unconverged iterations): fp32 P, R or AP each put the
// solution 7-8e-4 from the fp64 solve, fp32 X and fp32 operator values stay
// within 1.3e-6 / 8e-8.  `krylov_precision = CPCAG_F32` keeps every vector in
// fp32 (the faster path for well-conditioned systems, e.g. config 1).
//
// HBM layout: X, R, P, AP are p x n column-major; the mask and b are never
// materialised (rsel[i] / csel[c] give the position of row i / column c in
// the plan, or -1).  One CG iteration is four kernels, every scalar on the
// device:
//   lc pass   U = P Lc                  (row bands: the gathered band of P is
//                                        in shared memory when n is small,
//                                        resident in L2 otherwise)
//   lr pass   AP = gc U + gr Lr P + M o P, <P, AP>   (column tiles of P
//                                        staged in shared memory)
//   residual  alpha = rho / <P, AP>; R -= alpha AP, ||R||^2
//   update    beta = ||R||^2 / rho; X += alpha P, P = R + beta P, stop test
// U holds the unscaled X Lc sums, so AP = gc * x1 + gr * x2 (+ P) rounds
// exactly like decoders.cpp:160-170 (bit-identical in fp64).
#include <algorithm>
#include <cstdio>
#include <memory>
#include <numeric>
#include <string>
#include <type_traits>
#include <vector>

#include "decoder.cuh"

namespace cpcag_cuda {

// ------------------------------------------------------------------ the solver
// The operator plans of one decode: pulls of L_r / L_c in the value type
// and the apply plans of the CG (TK iterates) and of the true residual (TX).
template <typename TX, typename TK, typename TV>
struct DecodePrep : DecodePrepBase {
  Pull<TV> pr{}, pc{};
  ApplyPlan apK, apX;
  i64 p = 0, n = 0;
  RowOrder<TV> ro;  // the solve's row order (two-pass path, hub-heavy row graphs)
  const Csr* Lr = nullptr;
  const Csr* Lc = nullptr;
};

template <typename TX, typename TK, typename TV>
void decode_prepare(Ctx* c, i64 p, i64 n, Csr* Lr, Csr* Lc, DecodePrep<TX, TK, TV>& d) {
  d.pr = make_pull<TV>(c, Lr, false);
  d.pc = make_pull<TV>(c, Lc, true);
  std::vector<i64> rpr;
  std::vector<int> cir;
  std::vector<TV> vr;
  host_pull<TV>(c, d.pr, p, Lr->nnz, rpr, cir, &vr);
  const bool exact = sizeof(TX) == 8;
  {
    const bool two_pass = c->apply_path == 1 ||
                          (c->apply_path == 0 && p * n * static_cast<i64>(sizeof(TK)) > (i64{96} << 20));
    if (d.ro.build(c, p, two_pass, sizeof(TX), rpr, cir, vr)) d.pr = d.ro.pull;
  }
  HostPull<TV> lcp;
  host_pull<TV>(c, d.pc, n, Lc->nnz, lcp.rp, lcp.ci, &lcp.v);
  trace_mark(c, "decode: operator copies");
  plan_apply<TK, TK, TV>(c, d.apK, p, n, n, 0, rpr, cir, vr, exact, &lcp);
  trace_mark(c, "decode: plan K");
  // the true residual reuses the CG's operator plan when X and the iterates share a type
  if constexpr (!std::is_same<TX, TK>::value) plan_apply<TX, TK, TV>(c, d.apX, p, n, n, 0, rpr, cir, vr, exact, &lcp);
  trace_mark(c, "decode: plans");
  d.p = p;
  d.n = n;
  d.Lr = Lr;
  d.Lc = Lc;
}

template <typename TX, typename TK, typename TV>
void decode_impl(Ctx* c, const TX* Xt, i64 rho_r, i64 rho_c, i64 p, i64 n, Csr* Lr, Csr* Lc, double gbar_r,
                 double gbar_c, const Plan& pl_in, const cpcag_decoder_config& cfg, TX* X, int* converged,
                 i64* iterations, DecodePrepBase* prep_in) {
  const i64 N = p * n;
  auto* prep = dynamic_cast<DecodePrep<TX, TK, TV>*>(prep_in);
  DecodePrep<TX, TK, TV> local;
  if (!prep || prep->p != p || prep->n != n || prep->Lr != Lr || prep->Lc != Lc) {
    decode_prepare<TX, TK, TV>(c, p, n, Lr, Lc, local);
    prep = &local;
  }
  const Pull<TV> pr = prep->pr, pc = prep->pc;
  constexpr bool same_plan = std::is_same<TX, TK>::value;
  const ApplyPlan& apK = prep->apK;
  const ApplyPlan& apR = same_plan ? prep->apK : prep->apX;
  DevBuf<TK> R(c, N), P(c, N), AP(c, N), U(c, N);
  DevBuf<CgState> st(c, 1);
  st.zero(c);
  // the solve runs in the prepared row order
  DevBuf<int> rsel_perm;
  Plan pl = pl_in;
  if (prep->ro.on) pl.rsel = prep->ro.permute_rsel(c, pl_in.rsel, rsel_perm);
  const unsigned nbv = stride_blocks(c, std::max<i64>(N, 1));
  // the CG vector kernels: one wave of 8 x 256 threads per SM (4 vectors in flight per thread)
  const unsigned nbw = static_cast<unsigned>(std::max<i64>(1, std::min<i64>(c->num_sms * 8, (N + 1023) / 1024)));
  size_t nparts = std::max<size_t>({static_cast<size_t>(nbv), lr_blocks(apK), lr_blocks(apR)});
  DevBuf<double> part(c, std::max<size_t>(nparts, 1));
  cg_init_k<TK, TX, TX><<<nbv, kBlock, 0, c->stream>>>(p, n, 0, pl, Xt, X, R.p, P.p, part.p, st.p);
  launched(c);
  cg_start_k<<<1, 1, 0, c->stream>>>(st.p, cfg.pcg_tol, cfg.pcg_max_iter);
  launched(c);
  CgState host = read_back(c, st.p);
  trace_mark(c, "decode: init");
  if (host.zero_rhs) {  // solvers.hpp:40-44: x = b = 0
    *converged = 1;
    *iterations = 0;
    return;
  }
  const TK gr = static_cast<TK>(gbar_r), gc = static_cast<TK>(gbar_c);
  const Combine<TK, TX> cbK{U.p, AP.p, gr, gc, pl, nullptr, part.p, st.p};
  const Combine<TK, TX> none{nullptr, nullptr, gr, gc, pl, nullptr, nullptr, st.p};
  const bool vecK = reinterpret_cast<uintptr_t>(R.p) % 16 == 0 && reinterpret_cast<uintptr_t>(AP.p) % 16 == 0;
  const bool vecU = vecK && reinterpret_cast<uintptr_t>(X) % 16 == 0 && reinterpret_cast<uintptr_t>(P.p) % 16 == 0;
  i64 launched_it = 0;
  const i64 chunk = 32;
  while (!host.done && launched_it < cfg.pcg_max_iter) {
    // exactly the iterations that can still run (no launch past max_iter)
    const i64 todo = std::min<i64>(chunk, cfg.pcg_max_iter - launched_it);
    // a side-stream job holding an SM: the persistent slab grid leaves it out
    // (its 148th CTA would otherwise queue behind another and double the pass)
    if (c->side_job_running) {
      const bool busy = cudaEventQuery(c->join_ev) == cudaErrorNotReady;
      (void)cudaGetLastError();
      c->sm_reserve = busy ? 1 : 0;
    }
    for (i64 k = 0; k < todo; ++k) {
      launch_apply<TK, TK, TV, TX>(c, apK, pr, pc, P.p, U.p, cbK);
      {
        KScope ks_(c, "cg_residual");
        if (vecK)
          launch_pdl(cg_residual_k<TK, true>, dim3(nbw), dim3(kBlock), 0, c->stream, N, R.p, AP.p, part.p, st.p);
        else
          cg_residual_k<TK, false><<<nbv, kBlock, 0, c->stream>>>(N, R.p, AP.p, part.p, st.p);
        launched(c);
      }
      {
        KScope ks_(c, "cg_update");
        if (vecU)
          launch_pdl(cg_update_k<TK, TX, true>, dim3(nbw), dim3(kBlock), 0, c->stream, N, X, P.p, R.p, st.p);
        else
          cg_update_k<TK, TX, false><<<nbv, kBlock, 0, c->stream>>>(N, X, P.p, R.p, st.p);
        launched(c);
      }
    }
    launched_it += todo;
    host = read_back(c, st.p);
  }
  trace_mark(c, "decode: CG iterations");
  if (host.err) runtime("pcg: breakdown (nonpositive curvature) at iteration " + std::to_string(host.err_it));
  // true residual ||b - A x|| / ||b|| (solvers.hpp:69-72), x in its stored precision
  {
    KScope ks_(c, "cg_true_residual");
    CUDA_OK(cudaMemsetAsync(&st.p->done, 0, sizeof(int), c->stream));
    const Combine<TK, TX> cbR{U.p, nullptr, gr, gc, pl, Xt, part.p, st.p};
    launch_apply<TX, TK, TV, TX>(c, apR, pr, pc, X, U.p, cbR);
  }
  if (prep->ro.on) prep->ro.restore_rows(c, X, n);  // rows of X back to the caller's order
  host = read_back(c, st.p);
  const double rel = host.norm_b > 0.0 ? std::sqrt(host.curv) / host.norm_b : 0.0;
  *converged = rel <= cfg.pcg_tol ? 1 : 0;
  *iterations = host.it;
}

template <typename T>
void alternate_decode_device(Ctx* c, const T* Xt, i64 rho_r, i64 rho_c, const i64* om_r_host,
                             const i64* om_c_host, i64 p, i64 n, Csr* Lr, Csr* Lc, double lk1_r,
                             double lk1_c, const cpcag_decoder_config& cfg, T* X, int* converged,
                             i64* iterations, DecodePrepBase* prep) {
  if (Lr->rows != p || Lc->rows != n || Lr->cols != p || Lc->cols != n)
    invalid("alternate decoder: Laplacians do not match plan");
  if (cfg.gamma <= 0.0) invalid("alternate decoder: gamma must be positive");
  if (p > INT32_MAX / 2 || n > INT32_MAX / 2) invalid("alternate decoder: dimension too large");
  {
    std::vector<char> seen_r(static_cast<size_t>(p), 0), seen_c(static_cast<size_t>(n), 0);
    for (i64 k = 0; k < rho_r; ++k) {
      const i64 r = om_r_host[k];
      if (r < 0 || r >= p || seen_r[r]) invalid("alternate decoder: Xt does not match plan");
      seen_r[r] = 1;
    }
    for (i64 k = 0; k < rho_c; ++k) {
      const i64 q = om_c_host[k];
      if (q < 0 || q >= n || seen_c[q]) invalid("alternate decoder: Xt does not match plan");
      seen_c[q] = 1;
    }
  }
  const double gbar_r = cfg.gamma / lk1_r;
  const double gbar_c = cfg.gamma / lk1_c;
  if (p * n == 0) {
    *converged = 1;
    *iterations = 0;
    return;
  }
  DevBuf<i64> omr(c, rho_r), omc(c, rho_c);
  if (rho_r) CUDA_OK(cudaMemcpyAsync(omr.p, om_r_host, sizeof(i64) * rho_r, cudaMemcpyHostToDevice, c->stream));
  if (rho_c) CUDA_OK(cudaMemcpyAsync(omc.p, om_c_host, sizeof(i64) * rho_c, cudaMemcpyHostToDevice, c->stream));
  DevBuf<int> rsel(c, p), csel(c, n);
  fill_sel_k<<<blocks_for(p), kBlock, 0, c->stream>>>(p, rsel.p);
  launched(c);
  fill_sel_k<<<blocks_for(n), kBlock, 0, c->stream>>>(n, csel.p);
  launched(c);
  if (rho_r) {
    scatter_sel_k<<<blocks_for(rho_r), kBlock, 0, c->stream>>>(omr.p, rho_r, rsel.p);
    launched(c);
  }
  if (rho_c) {
    scatter_sel_k<<<blocks_for(rho_c), kBlock, 0, c->stream>>>(omc.p, rho_c, csel.p);
    launched(c);
  }
  const Plan pl{rsel.p, csel.p, rho_r};
  if constexpr (sizeof(T) == 8) {
    decode_impl<double, double, double>(c, Xt, rho_r, rho_c, p, n, Lr, Lc, gbar_r, gbar_c, pl, cfg, X, converged,
                                        iterations, prep);
  } else {
    if (cfg.krylov_precision == CPCAG_F32)
      decode_impl<float, float, float>(c, Xt, rho_r, rho_c, p, n, Lr, Lc, gbar_r, gbar_c, pl, cfg, X, converged,
                                       iterations, prep);
    else
      decode_impl<float, double, float>(c, Xt, rho_r, rho_c, p, n, Lr, Lc, gbar_r, gbar_c, pl, cfg, X, converged,
                                        iterations, prep);
  }
}

template void alternate_decode_device<double>(Ctx*, const double*, i64, i64, const i64*, const i64*, i64, i64,
                                              Csr*, Csr*, double, double, const cpcag_decoder_config&,
                                              double*, int*, i64*, DecodePrepBase*);
template void alternate_decode_device<float>(Ctx*, const float*, i64, i64, const i64*, const i64*, i64, i64,
                                             Csr*, Csr*, double, double, const cpcag_decoder_config&,
                                             float*, int*, i64*, DecodePrepBase*);

// The plans alternate_decode_device<T> will use, built now (same type
// selection); null when the shapes leave nothing to plan.
template <typename T>
std::unique_ptr<DecodePrepBase> alternate_decode_prepare(Ctx* c, i64 p, i64 n, Csr* Lr, Csr* Lc,
                                                         const cpcag_decoder_config& cfg) {
  if (Lr->rows != p || Lc->rows != n || Lr->cols != p || Lc->cols != n || p * n == 0) return nullptr;
  if (p > INT32_MAX / 2 || n > INT32_MAX / 2) return nullptr;
  auto make = [&](auto* tag) -> std::unique_ptr<DecodePrepBase> {
    using D = std::remove_pointer_t<decltype(tag)>;
    auto d = std::make_unique<D>();
    decode_prepare(c, p, n, Lr, Lc, *d);
    return d;
  };
  if constexpr (sizeof(T) == 8) {
    return make(static_cast<DecodePrep<double, double, double>*>(nullptr));
  } else {
    if (cfg.krylov_precision == CPCAG_F32) return make(static_cast<DecodePrep<float, float, float>*>(nullptr));
    return make(static_cast<DecodePrep<float, double, float>*>(nullptr));
  }
}
template std::unique_ptr<DecodePrepBase> alternate_decode_prepare<double>(Ctx*, i64, i64, Csr*, Csr*,
                                                                          const cpcag_decoder_config&);
template std::unique_ptr<DecodePrepBase> alternate_decode_prepare<float>(Ctx*, i64, i64, Csr*, Csr*,
                                                                         const cpcag_decoder_config&);

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_cuda_alternate_decode(cpcag_ctx ctx, int precision, const void* Xt, int64_t rho_r,
                                           int64_t rho_c, const int64_t* omega_r, const int64_t* omega_c,
                                           int64_t p, int64_t n, cpcag_csr Lr, cpcag_csr Lc,
                                           double lambda_k1_r, double lambda_k1_c,
                                           const cpcag_decoder_config* cfg, void* X, int* converged,
                                           int64_t* iterations) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!cfg || !converged || !iterations) invalid("null argument");
      std::vector<i64> omr(static_cast<size_t>(std::max<int64_t>(rho_r, 0)));
      std::vector<i64> omc(static_cast<size_t>(std::max<int64_t>(rho_c, 0)));
      auto fetch = [&](std::vector<i64>& dst, const int64_t* src) {
        if (dst.empty()) return;
        if (is_device_ptr(src))
          CUDA_OK(cudaMemcpy(dst.data(), src, sizeof(i64) * dst.size(), cudaMemcpyDeviceToHost));
        else
          std::copy(src, src + dst.size(), dst.begin());
      };
      fetch(omr, omega_r);
      fetch(omc, omega_c);
      InView<T> xt(c, static_cast<const T*>(Xt), static_cast<size_t>(rho_r * rho_c));
      OutView<T> x(c, static_cast<T*>(X), static_cast<size_t>(p * n));
      alternate_decode_device<T>(c, xt.d, rho_r, rho_c, omr.data(), omc.data(), p, n, as_csr(Lr), as_csr(Lc),
                                 lambda_k1_r, lambda_k1_c, *cfg, x.d, converged, iterations);
      x.flush(c);
      sync(c);
    });
  };
  if (precision == CPCAG_F64) return run(double{});
  if (precision == CPCAG_F32) return run(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}

// The decoder's operator alone (the lambda of decoders.cpp:160-170): AP =
// gbar_c P Lc + gbar_r Lr P + M o P and <P, AP>, through the same two passes
// the CG runs (fp64: bit-identical per entry to the reference loop).
namespace cpcag_cuda {
template <typename T>
void decoder_apply_device(Ctx* c, const T* P, i64 p, i64 n, Csr* Lr, Csr* Lc, const std::vector<i64>& omr,
                          const std::vector<i64>& omc, double gbar_r, double gbar_c, T* AP, double* dot) {
  if (Lr->rows != p || Lc->rows != n || Lr->cols != p || Lc->cols != n)
    invalid("alternate decoder: Laplacians do not match plan");
  std::vector<int> rs(static_cast<size_t>(p), -1), cs(static_cast<size_t>(n), -1);
  for (size_t k = 0; k < omr.size(); ++k) {
    if (omr[k] < 0 || omr[k] >= p || rs[omr[k]] >= 0) invalid("alternate decoder: Xt does not match plan");
    rs[omr[k]] = static_cast<int>(k);
  }
  for (size_t k = 0; k < omc.size(); ++k) {
    if (omc[k] < 0 || omc[k] >= n || cs[omc[k]] >= 0) invalid("alternate decoder: Xt does not match plan");
    cs[omc[k]] = static_cast<int>(k);
  }
  DevBuf<int> rsel(c, std::max<i64>(p, 1)), csel(c, std::max<i64>(n, 1));
  if (p) CUDA_OK(cudaMemcpyAsync(rsel.p, rs.data(), sizeof(int) * p, cudaMemcpyHostToDevice, c->stream));
  if (n) CUDA_OK(cudaMemcpyAsync(csel.p, cs.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
  const Plan pl{rsel.p, csel.p, static_cast<i64>(omr.size())};
  const Pull<T> pr = make_pull<T>(c, Lr, false), pc = make_pull<T>(c, Lc, true);
  std::vector<i64> rpr;
  std::vector<int> cir;
  std::vector<T> vr;
  host_pull<T>(c, pr, p, Lr->nnz, rpr, cir, &vr);
  ApplyPlan ap;
  HostPull<T> lcp;
  host_pull<T>(c, pc, n, Lc->nnz, lcp.rp, lcp.ci, &lcp.v);
  plan_apply<T, T, T>(c, ap, p, n, n, 0, rpr, cir, vr, sizeof(T) == 8, &lcp);
  DevBuf<T> U(c, std::max<i64>(p * n, 1));
  DevBuf<CgState> st(c, 1);
  st.zero(c);
  DevBuf<double> part(c, std::max<size_t>(lr_blocks(ap), 1));
  const T gr = static_cast<T>(gbar_r), gc = static_cast<T>(gbar_c);
  const Combine<T, T> none{nullptr, nullptr, gr, gc, pl, nullptr, nullptr, st.p};
  const Combine<T, T> cb{U.p, AP, gr, gc, pl, nullptr, part.p, st.p};
  launch_apply<T, T, T, T>(c, ap, pr, pc, P, U.p, cb);
  *dot = read_back(c, st.p).curv;
}
}  // namespace cpcag_cuda

extern "C" int cpcag_cuda_decoder_apply(cpcag_ctx ctx, int precision, const void* P, int64_t p, int64_t n,
                                        cpcag_csr Lr, cpcag_csr Lc, const int64_t* omega_r, int64_t rho_r,
                                        const int64_t* omega_c, int64_t rho_c, double gbar_r, double gbar_c,
                                        void* AP, double* dot) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!P || !AP || !dot) invalid("null argument");
      std::vector<i64> omr(static_cast<size_t>(std::max<int64_t>(rho_r, 0))), omc(static_cast<size_t>(std::max<int64_t>(rho_c, 0)));
      auto fetch = [&](std::vector<i64>& dst, const int64_t* src) {
        if (dst.empty()) return;
        if (is_device_ptr(src))
          CUDA_OK(cudaMemcpy(dst.data(), src, sizeof(i64) * dst.size(), cudaMemcpyDeviceToHost));
        else
          std::copy(src, src + dst.size(), dst.begin());
      };
      fetch(omr, omega_r);
      fetch(omc, omega_c);
      InView<T> pv(c, static_cast<const T*>(P), static_cast<size_t>(p * n));
      OutView<T> ap(c, static_cast<T*>(AP), static_cast<size_t>(p * n));
      decoder_apply_device<T>(c, pv.d, p, n, as_csr(Lr), as_csr(Lc), omr, omc, gbar_r, gbar_c, ap.d, dot);
      ap.flush(c);
      sync(c);
    });
  };
  if (precision == CPCAG_F64) return run(double{});
  if (precision == CPCAG_F32) return run(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}
