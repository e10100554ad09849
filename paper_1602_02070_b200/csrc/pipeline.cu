// pipeline.cu -- run_pipeline for the low-rank task with the alternate
// decoder (pipeline.cpp:228-350), device resident end to end:
//   graphs -> plan -> subsample -> kron -> solve (FISTA) -> decode.
// Stage failures are re-raised as runtime errors tagged "stage <name>: ..."
// (pipeline.cpp:24-39); stage times are device event intervals on the
// context stream.
#include <algorithm>
#include <memory>

#include <cstdlib>
#include <string>

#include "common.cuh"
#include "frpcag.cuh"

namespace cpcag_cuda {

struct StageTimer {
  Ctx* c;
  cudaEvent_t a, b;
  explicit StageTimer(Ctx* ctx) : c(ctx) {
    CUDA_OK(cudaEventCreate(&a));
    CUDA_OK(cudaEventCreate(&b));
  }
  ~StageTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  template <class F>
  double run(const char* name, F&& body) {
    CUDA_OK(cudaEventRecord(a, c->stream));
    try {
      body();
    } catch (const Error& e) {
      if (e.status == CPCAG_ERR_CUDA) throw;
      fail(CPCAG_ERR_RUNTIME, std::string("stage ") + name + ": " + e.what());
    }
    CUDA_OK(cudaEventRecord(b, c->stream));
    CUDA_OK(cudaEventSynchronize(b));
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }
};

template <typename T>
__global__ void scatter_full_k(const T* __restrict__ Xt, i64 rho_r, i64 rho_c, const i64* __restrict__ om_r,
                               const i64* __restrict__ om_c, i64 p, T* __restrict__ X) {
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= rho_r) return;
  for (i64 j = blockIdx.y; j < rho_c; j += gridDim.y) X[om_r[i] + om_c[j] * p] = Xt[i + j * rho_r];
}

template <typename T>
void run_pipeline_device(Ctx* c, const T* Y, i64 p, i64 n, Csr* Wr, Csr* Wc, const cpcag_pipeline_config& cfg,
                         T* Xt_out, T* X_out, i64* om_r_out, i64* om_c_out, double* objective,
                         cpcag_pipeline_report* rep, const cpcag_pipeline_factors* factors) {
  std::memset(rep, 0, sizeof(*rep));
  rep->p = p;
  rep->n = n;
  StageTimer tm(c);
  std::unique_ptr<Csr> Lr, Lc, Wr_own, Wc_own;
  DevBuf<double> deg_r(c, std::max<i64>(p, 1)), deg_c(c, std::max<i64>(n, 1));

  rep->stage_ms[0] = tm.run("graphs", [&] {
    Csr* L = nullptr;
    Csr* W = nullptr;
    double s2 = 0.0;
    if (Wr) {
      graph_from_adjacency_device(c, Wr, cfg.laplacian, &L, deg_r.p);
    } else {
      knn_graph_device<T>(c, Y, p, n, true, cfg.knn, cfg.laplacian, cfg.sigma2, &W, &L, deg_r.p, &s2);
      Wr_own.reset(W);
    }
    Lr.reset(L);
    if (Wc) {
      graph_from_adjacency_device(c, Wc, cfg.laplacian, &L, deg_c.p);
    } else {
      knn_graph_device<T>(c, Y, p, n, false, cfg.knn, cfg.laplacian, cfg.sigma2, &W, &L, deg_c.p, &s2);
      Wc_own.reset(W);
    }
    Lc.reset(L);
    if (Lr->rows != p || Lc->rows != n) invalid("graph sizes do not match the data matrix");
  });

  std::vector<i64> om_r, om_c;
  rep->stage_ms[1] = tm.run("plan", [&] {
    if (cfg.a < 1 || cfg.b < 1) invalid("downsampling factors must be integers >= 1");
    i64 rho_r = cfg.rho_r_override > 0 ? cfg.rho_r_override : (p + cfg.b - 1) / cfg.b;
    i64 rho_c = cfg.rho_c_override > 0 ? cfg.rho_c_override : (n + cfg.a - 1) / cfg.a;
    rho_r = std::min(rho_r, p);
    rho_c = std::min(rho_c, n);
    if (rho_r < 1 || rho_r > p) invalid("draw_plan: rho_r out of range [1, " + std::to_string(p) + "]");
    if (rho_c < 1 || rho_c > n) invalid("draw_plan: rho_c out of range [1, " + std::to_string(n) + "]");
    om_r = draw_indices(p, rho_r, HostRng::derive(cfg.seed, 0x726f7773ULL));
    om_c = draw_indices(n, rho_c, HostRng::derive(cfg.seed, 0x636f6c73ULL));
  });
  const i64 rho_r = static_cast<i64>(om_r.size()), rho_c = static_cast<i64>(om_c.size());
  rep->rho_r = rho_r;
  rep->rho_c = rho_c;
  const bool full = rho_r == p && rho_c == n;

  DevBuf<i64> om_r_d(c, rho_r), om_c_d(c, rho_c);
  CUDA_OK(cudaMemcpyAsync(om_r_d.p, om_r.data(), sizeof(i64) * rho_r, cudaMemcpyHostToDevice, c->stream));
  CUDA_OK(cudaMemcpyAsync(om_c_d.p, om_c.data(), sizeof(i64) * rho_c, cudaMemcpyHostToDevice, c->stream));
  DevBuf<T> Yt(c, rho_r * rho_c);
  rep->stage_ms[2] = tm.run("subsample", [&] {
    subsample_device<T>(c, Y, p, om_r_d.p, rho_r, om_c_d.p, rho_c, Yt.p);
  });

  std::unique_ptr<Csr> Lr_s, Lc_s;
  rep->stage_ms[3] = tm.run("kron", [&] {
    Lr_s.reset(kron_reduce_device(c, Lr.get(), om_r, cfg.kron_pcg_tol, 1e-12));
    Lr_s->sym = 1;
    Lc_s.reset(kron_reduce_device(c, Lc.get(), om_c, cfg.kron_pcg_tol, 1e-12));
    Lc_s->sym = 1;
  });

  // The decoder's operator planning (host work, ~1 ms at config 1) runs
  // while the device iterates the spectral norms of the solve stage; the
  // decode stage builds the plans itself if that did not happen.
  const bool want_x = cfg.task != CPCAG_TASK_CLUSTER;
  std::unique_ptr<DecodePrepBase> dprep;
  IdleWorkScope idle_scope(c);
  if (want_x && !full && cfg.decoder_variant == CPCAG_DECODER_ALTERNATE)
    c->idle_work = [&] {
      try {
        dprep = alternate_decode_prepare<T>(c, p, n, Lr.get(), Lc.get(), cfg.decoder);
      } catch (const Error& e) {
        if (e.status == CPCAG_ERR_CUDA) throw;
        dprep.reset();  // the decode stage plans again and reports the error there
      }
    };

  rep->stage_ms[4] = tm.run("solve", [&] {
    fista_device<T>(c, Yt.p, rho_r, rho_c, Lr_s.get(), Lc_s.get(), cfg.frpcag, Xt_out, objective, &rep->trace);
  });

  // pipeline.cpp:319-320: the detected rank of the compressed solution (its
  // singular values only), outside the stage timers as in the reference.
  // Gram matrices of order <= 110 (config 1: 100) go through the one-CTA
  // Jacobi job on the side stream; when nothing downstream needs the rank
  // (alternate decoder, both spectral gaps given, no clustering) the job runs
  // beside the decoder and is read after it.
  trace_mark(c, "pipeline: stages to solve");
  const i64 q_rank = std::min(rho_r, rho_c);
  DevBuf<double> A_rank(c, std::max<i64>(rho_r * rho_c, 1));
  RankJob rank_job;
  const bool rank_small = q_rank > 0 && q_rank <= 110;
  const bool rank_later = rank_small && cfg.decoder_variant == CPCAG_DECODER_ALTERNATE && cfg.lambda_k1_r > 0.0 &&
                          cfg.lambda_k1_c > 0.0 && cfg.task == CPCAG_TASK_LOWRANK;
  if (rank_small) {
    to_f64_device(c, Xt_out, rho_r * rho_c, A_rank.p);
    rank_job_start(c, rank_job, A_rank.p, rho_r, rho_c, side_stream(c));
    if (!rank_later) rep->detected_rank = detect_rank_host(rank_job_finish(c, rank_job), cfg.approx.rank_threshold);
  } else {
    DevBuf<double> sv(c, std::max<i64>(q_rank, 1));
    if (rho_r * rho_c) {
      to_f64_device(c, Xt_out, rho_r * rho_c, A_rank.p);
      gram_svd_device(c, A_rank.p, rho_r, rho_c, 0, sv.p, nullptr, nullptr);
    }
    std::vector<double> hs(static_cast<size_t>(q_rank));
    if (q_rank) CUDA_OK(cudaMemcpyAsync(hs.data(), sv.p, sizeof(double) * q_rank, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    rep->detected_rank = detect_rank_host(hs, cfg.approx.rank_threshold);
  }
  trace_mark(c, "pipeline: detected rank");
  rep->has_factors = 0;
  rep->factors_k = 0;

  if (want_x) rep->stage_ms[5] = tm.run("decode", [&] {
    run_idle_work(c);
    if (full) {
      // pipeline.cpp:327-337: no compression, scatter back through the plan.
      dim3 g(blocks_for(rho_r), static_cast<unsigned>(std::min<i64>(rho_c, 65535)));
      scatter_full_k<T><<<g, kBlock, 0, c->stream>>>(Xt_out, rho_r, rho_c, om_r_d.p, om_c_d.p, p, X_out);
      launched(c);
      rep->decoder_converged = 1;
      rep->decoder_iterations = 0;
      return;
    }
    if (cfg.decoder_variant == CPCAG_DECODER_APPROX) {
      i64 k = 0;
      approx_decode_device<T>(c, Xt_out, rho_r, rho_c, om_r, om_c, p, n, Lr.get(), Lc.get(), cfg.approx, X_out,
                              factors ? factors->U : nullptr, factors ? factors->sigma : nullptr,
                              factors ? factors->V : nullptr, factors ? factors->k_cap : 0, &k);
      rep->factors_k = k;
      rep->has_factors = 1;
      rep->decoder_converged = 1;
      rep->decoder_iterations = 0;
      return;
    }
    if (cfg.decoder_variant != CPCAG_DECODER_ALTERNATE)
      invalid("run_pipeline: decoder variant not supported on the device path (alternate or approx)");
    // pipeline.cpp:343-349: gaps from the k+1 smallest eigenvalues of the full
    // Laplacians, k = max(1, detected rank), unless the caller supplies them.
    double lk1_r = cfg.lambda_k1_r, lk1_c = cfg.lambda_k1_c;
    if (!(lk1_r > 0.0) || !(lk1_c > 0.0)) {
      const i64 k = std::max<i64>(1, rep->detected_rank);
      std::vector<double> ev(static_cast<size_t>(k + 1));
      // The reference's dense solver where it is feasible; Lanczos beyond
      // (n > 46340: cfg3/cfg4 graphs) or when CPCAG_GAP_LANCZOS=1.
      const char* gl = std::getenv("CPCAG_GAP_LANCZOS");
      auto smallest_eigs = [&](Csr* L, i64 order, double* out) {
        if (L->rows > 46340 || (gl && std::string(gl) == "1")) {
          sym_eigvals_lanczos(c, L, order, 1e-10, 5000, 0, out, nullptr);
        } else {
          DevBuf<double> e(c, order);
          sym_eig_device(c, L, order, e.p, nullptr);
          CUDA_OK(cudaMemcpyAsync(out, e.p, sizeof(double) * order, cudaMemcpyDeviceToHost, c->stream));
          sync(c);
        }
      };
      if (!(lk1_r > 0.0)) {
        smallest_eigs(Lr.get(), k + 1, ev.data());
        lk1_r = spectral_gap_host(ev.data(), k + 1, k).lambda_k1;
      }
      if (!(lk1_c > 0.0)) {
        smallest_eigs(Lc.get(), k + 1, ev.data());
        lk1_c = spectral_gap_host(ev.data(), k + 1, k).lambda_k1;
      }
    }
    rep->lambda_k1_r = lk1_r;
    rep->lambda_k1_c = lk1_c;
    int conv = 0;
    i64 it = 0;
    alternate_decode_device<T>(c, Xt_out, rho_r, rho_c, om_r.data(), om_c.data(), p, n, Lr.get(), Lc.get(), lk1_r,
                               lk1_c, cfg.decoder, X_out, &conv, &it, dprep.get());
    rep->decoder_converged = conv;
    rep->decoder_iterations = it;
  });
  // pipeline.cpp:371-388: k-means on the compressed solution's columns
  // (seed mix(seed ^ "kmean")), then decode_labels over the column graph
  if (cfg.task == CPCAG_TASK_CLUSTER || cfg.task == CPCAG_TASK_BOTH) {
    rep->cluster_ms = tm.run("cluster", [&] {
      const i64 k = cfg.n_clusters > 0 ? cfg.n_clusters : std::max<i64>(1, rep->detected_rank);
      DevBuf<double> Xd(c, static_cast<size_t>(std::max<i64>(rho_r * rho_c, 1)));
      to_f64_device(c, Xt_out, rho_r * rho_c, Xd.p);
      DevBuf<int> sl(c, static_cast<size_t>(std::max<i64>(rho_c, 1))), lab(c, static_cast<size_t>(n));
      kmeans_device(c, Xd.p, rho_r, rho_c, k, cfg.kmeans_restarts,
                    HostRng::mix(cfg.seed ^ 0x6b6d65616eULL), 100, sl.p, nullptr);
      decode_labels_device(c, Lc.get(), om_c, sl.p, k, cfg.decoder.pcg_tol, cfg.decoder.pcg_max_iter, n, lab.p);
      if (factors && factors->labels)
        CUDA_OK(cudaMemcpyAsync(factors->labels, lab.p, sizeof(int) * n, cudaMemcpyDefault, c->stream));
      rep->n_clusters = k;
    });
  }
  if (rank_later) rep->detected_rank = detect_rank_host(rank_job_finish(c, rank_job), cfg.approx.rank_threshold);
  if (om_r_out) std::copy(om_r.begin(), om_r.end(), om_r_out);
  if (om_c_out) std::copy(om_c.begin(), om_c.end(), om_c_out);
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_cuda_run_pipeline(cpcag_ctx ctx, int precision, const void* Y, int64_t p, int64_t n,
                                       cpcag_csr W_r, cpcag_csr W_c, const cpcag_pipeline_config* cfg, void* Xt,
                                       void* X, int64_t* omega_r, int64_t* omega_c, double* objective,
                                       cpcag_pipeline_report* report, const cpcag_pipeline_factors* factors) {
  auto run = [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!cfg || !report || !Xt || (!X && cfg->task != CPCAG_TASK_CLUSTER)) invalid("null argument");
      if (p < 1 || n < 1) invalid("run_pipeline: empty data matrix");
      i64 rho_r = cfg->rho_r_override > 0 ? cfg->rho_r_override : (cfg->b >= 1 ? (p + cfg->b - 1) / cfg->b : p);
      i64 rho_c = cfg->rho_c_override > 0 ? cfg->rho_c_override : (cfg->a >= 1 ? (n + cfg->a - 1) / cfg->a : n);
      rho_r = std::min<i64>(rho_r, p);
      rho_c = std::min<i64>(rho_c, n);
      InView<T> y(c, static_cast<const T*>(Y), static_cast<size_t>(p * n));
      OutView<T> xt(c, static_cast<T*>(Xt), static_cast<size_t>(std::max<i64>(rho_r, 1) * std::max<i64>(rho_c, 1)));
      OutView<T> x(c, static_cast<T*>(X), X ? static_cast<size_t>(p * n) : 0);
      run_pipeline_device<T>(c, y.d, p, n, W_r ? as_csr(W_r) : nullptr, W_c ? as_csr(W_c) : nullptr, *cfg, xt.d, x.d,
                             omega_r, omega_c, objective, report, factors);
      xt.flush(c);
      x.flush(c);
      sync(c);
    });
  };
  if (precision == CPCAG_F64) return run(double{});
  if (precision == CPCAG_F32) return run(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}
