// sharded.cu -- the alternate decoder (decoders.cpp:145-186) split over the
// GPUs of one node by column blocks of X, one process per GPU,
// NCCL over NVLink.  Rank g owns columns [bounds[g], bounds[g+1]).
//
// Per CG iteration (the reference recurrence, solvers.hpp:33-74):
//   1. pack the columns of P other ranks' L_c rows reference (the halo plan,
//      built once from L_c's structure) and exchange them with one grouped
//      ncclSend/ncclRecv on a second stream, received straight into the
//      local column space [own block | halo];
//   2. meanwhile, on the compute stream, the lr pass x2 = L_r P_own (L_r is
//      replicated, the pass is block-local);
//   3. the lc pass over the local column space combines
//      AP = gc x1 + gr x2 (+ P) and the partial <P, AP>;
//   4. ncclAllReduce of <P, AP> (device scalar), R -= alpha AP,
//      ncclAllReduce of ||R||^2, X += alpha P, P = R + beta P.
// Every scalar stays on the device and every rank computes identical
// alpha / beta / stop decisions, so the host only polls the done flag per
// chunk of iterations.  The local L_c rows keep the reference's entry order
// (indices remapped into the local space), so each entry of AP is the one-GPU
// decoder's value bit for bit; only the dot products' summation order differs.
//
// cpcag_cuda_alternate_decode_sharded_emulated runs all ranks in one process
// on one device (the exchange becomes device copies, the all-reduce a
// fixed-order sum), phase by phase: no kernel ever waits for another, so the
// multi-rank logic is testable with one GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include "decoder.cuh"
#include "frpcag.cuh"
#include "fista_dense.cuh"

namespace cpcag_cuda {

// NCCL is resolved at run time (dlopen of libnccl.so.2, the copy already in
// the process if the caller's framework loaded one): linking it would bind
// the system library first and break a later `import torch`, whose bundled
// NCCL is newer.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("nccl: cannot load libnccl.so.2 (") + dlerror() + ")";
      return;
    }
    auto get = [&](const char* name) {
      void* f = dlsym(h, name);
      if (!f && err.empty()) err = std::string("nccl: missing symbol ") + name;
      return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(get("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(get("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(get("ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(get("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(get("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(get("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(get("ncclRecv"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(get("ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(get("ncclGetErrorString"));
  });
  if (!err.empty()) runtime(err);
  return api;
}

#define NCCL_OK(expr)                                                                                        \
  do {                                                                                                       \
    ncclResult_t _r = (expr);                                                                                \
    if (_r != ncclSuccess) ::cpcag_cuda::runtime(std::string("nccl: ") + nccl().GetErrorString(_r));      \
  } while (0)

// ------------------------------------------------------------------ halo plan (host)
struct HaloPlan {
  int G = 1, rank = 0;
  i64 n = 0, c0 = 0, c1 = 0;
  std::vector<i64> recv_cols;  // global ids this rank receives, grouped by owner (ascending), sorted
  std::vector<i64> recv_off;   // G + 1
  std::vector<i64> send_cols;  // local ids (j - c0) this rank sends, grouped by destination
  std::vector<i64> send_off;   // G + 1
};

HaloPlan make_halo_plan(const i64* rp, const int* ci, i64 n, const i64* bounds, int G, int rank) {
  for (int g = 0; g < G; ++g)
    if (bounds[g] < 0 || bounds[g] > bounds[g + 1] || bounds[g + 1] > n)
      invalid("sharded decoder: column bounds must be ascending within [0, n]");
  if (bounds[0] != 0 || bounds[G] != n) invalid("sharded decoder: column bounds must cover [0, n)");
  HaloPlan h;
  h.G = G;
  h.rank = rank;
  h.n = n;
  h.c0 = bounds[rank];
  h.c1 = bounds[rank + 1];
  std::vector<int> stamp(static_cast<size_t>(n), -1);
  std::vector<std::vector<i64>> need(static_cast<size_t>(G));
  for (int q = 0; q < G; ++q) {
    const i64 a = bounds[q], e = bounds[q + 1];
    for (i64 c = a; c < e; ++c)
      for (i64 k = rp[c]; k < rp[c + 1]; ++k) {
        const i64 j = ci[k];
        if ((j < a || j >= e) && stamp[j] != q) {
          stamp[j] = q;
          need[q].push_back(j);
        }
      }
    std::sort(need[q].begin(), need[q].end());
  }
  h.recv_off.assign(static_cast<size_t>(G) + 1, 0);
  h.recv_cols = need[rank];
  for (int s = 0, k = 0; s < G; ++s) {
    while (k < static_cast<int>(h.recv_cols.size()) && h.recv_cols[k] < bounds[s + 1]) ++k;
    h.recv_off[s + 1] = k;
  }
  h.send_off.assign(static_cast<size_t>(G) + 1, 0);
  for (int d = 0; d < G; ++d) {
    if (d != rank)
      for (const i64 j : need[d])
        if (j >= h.c0 && j < h.c1) h.send_cols.push_back(j - h.c0);
    h.send_off[d + 1] = static_cast<i64>(h.send_cols.size());
  }
  return h;
}

// ------------------------------------------------------------------ kernels
template <typename T>
__global__ void pack_cols_k(i64 p, i64 ncols, const int* __restrict__ idx, const T* __restrict__ src,
                            T* __restrict__ dst) {
  const i64 N = p * ncols;
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < N; q += (i64)gridDim.x * blockDim.x) {
    const i64 c = q / p, i = q - c * p;
    dst[q] = src[static_cast<i64>(idx[c]) * p + i];
  }
}

// Fixed-order sum of one double over `nr` ranks' states (emulated all-reduce).
__global__ void emu_allreduce_k(CgState** st, int nr, int field) {
  double s = 0.0;
  for (int r = 0; r < nr; ++r) s += field == 0 ? st[r]->rho : (field == 1 ? st[r]->curv : st[r]->rho_next);
  for (int r = 0; r < nr; ++r) {
    if (field == 0) st[r]->rho = s;
    else if (field == 1) st[r]->curv = s;
    else st[r]->rho_next = s;
  }
}

// ------------------------------------------------------------------ one rank's state
template <typename TX, typename TK, typename TV>
struct Shard {
  Ctx* c = nullptr;
  HaloPlan hp;
  i64 p = 0, n = 0, nb = 0, nh = 0, nsend = 0;
  Pull<TV> pr{};   // L_r (replicated)
  Pull<TV> pcl{};  // local rows of L_c, indices in [own | halo] space
  DevBuf<i64> lrp;
  DevBuf<int> lci;
  DevBuf<TV> lv;
  DevBuf<int> send_idx;
  ApplyPlan apK, apX;
  RowOrder<TV> ro;
  DevBuf<int> rsel_perm;
  DevBuf<TK> Ploc, R, AP, U, sendK;
  DevBuf<TX> Xloc, sendX;
  DevBuf<CgState> st;
  DevBuf<double> part;
  Plan pl{};
  TX* X = nullptr;  // caller's block (p x nb)
  const TX* Xt = nullptr;

  void build(Ctx* ctx, const HaloPlan& h, i64 p_, i64 n_, Csr* Lr, Csr* Lc, const std::vector<i64>& rpc,
             const std::vector<int>& cic, const std::vector<TV>& vc, const std::vector<i64>& rpr,
             const std::vector<int>& cir, const std::vector<TV>& vr, const Plan& plan, TX* Xblock, const TX* Xt_) {
    c = ctx;
    hp = h;
    p = p_;
    n = n_;
    nb = h.c1 - h.c0;
    nh = static_cast<i64>(h.recv_cols.size());
    nsend = static_cast<i64>(h.send_cols.size());
    pl = plan;
    X = Xblock;
    Xt = Xt_;
    pr = make_pull<TV>(c, Lr, false);
    (void)Lc;
    // local L_c rows: own columns first, then the halo in receive order
    std::vector<int> pos(static_cast<size_t>(n), -1);
    for (i64 j = h.c0; j < h.c1; ++j) pos[j] = static_cast<int>(j - h.c0);
    for (i64 q = 0; q < nh; ++q) pos[h.recv_cols[q]] = static_cast<int>(nb + q);
    std::vector<i64> hrp(static_cast<size_t>(nb) + 1, 0);
    for (i64 r = 0; r < nb; ++r) hrp[r + 1] = hrp[r] + (rpc[h.c0 + r + 1] - rpc[h.c0 + r]);
    const i64 lnnz = hrp[nb];
    std::vector<int> hci(static_cast<size_t>(lnnz));
    std::vector<TV> hv(static_cast<size_t>(lnnz));
    for (i64 r = 0; r < nb; ++r) {
      const i64 k0 = rpc[h.c0 + r];
      for (i64 k = k0; k < rpc[h.c0 + r + 1]; ++k) {
        hci[hrp[r] + (k - k0)] = pos[cic[k]];
        hv[hrp[r] + (k - k0)] = vc[k];
      }
    }
    lrp.alloc(c, static_cast<size_t>(nb) + 1);
    lci.alloc(c, std::max<i64>(lnnz, 1));
    lv.alloc(c, std::max<i64>(lnnz, 1));
    CUDA_OK(cudaMemcpyAsync(lrp.p, hrp.data(), sizeof(i64) * (nb + 1), cudaMemcpyHostToDevice, c->stream));
    if (lnnz) {
      CUDA_OK(cudaMemcpyAsync(lci.p, hci.data(), sizeof(int) * lnnz, cudaMemcpyHostToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(lv.p, hv.data(), sizeof(TV) * lnnz, cudaMemcpyHostToDevice, c->stream));
    }
    pcl = Pull<TV>{lrp.p, lci.p, lv.p};
    std::vector<int> sidx(h.send_cols.begin(), h.send_cols.end());
    send_idx.alloc(c, std::max<i64>(nsend, 1));
    if (nsend) CUDA_OK(cudaMemcpyAsync(send_idx.p, sidx.data(), sizeof(int) * nsend, cudaMemcpyHostToDevice, c->stream));
    // the solve's row order (every rank derives the same one from L_r, so
    // exchanged columns agree): hub-heavy row graphs run in degree-sorted rows
    std::vector<i64> rpr2(rpr);
    std::vector<int> cir2(cir);
    std::vector<TV> vr2(vr);
    if (ro.build(c, p, true, sizeof(TX), rpr2, cir2, vr2)) {
      pr = ro.pull;
      pl.rsel = ro.permute_rsel(c, plan.rsel, rsel_perm);
    }
    plan_apply<TK, TK, TV>(c, apK, p, nb, nb + nh, h.c0, rpr2, cir2, vr2, sizeof(TX) == 8);
    plan_apply<TX, TK, TV>(c, apX, p, nb, nb + nh, h.c0, rpr2, cir2, vr2, sizeof(TX) == 8);
    const i64 N = p * nb;
    Ploc.alloc(c, static_cast<size_t>(std::max<i64>(p * (nb + nh), 1)));
    R.alloc(c, std::max<i64>(N, 1));
    AP.alloc(c, std::max<i64>(N, 1));
    U.alloc(c, std::max<i64>(N, 1));
    sendK.alloc(c, std::max<i64>(p * nsend, 1));
    st.alloc(c, 1);
    st.zero(c);
    size_t nparts = stride_blocks(c, std::max<i64>(N, 1));
    nparts = std::max<size_t>({nparts, lr_blocks(apK), lr_blocks(apX), lc_blocks(apK, 128 / sizeof(TK)),
                               lc_blocks(apX, 128 / sizeof(TX))});
    part.alloc(c, nparts);
    sync(c);
  }

  i64 N() const { return p * nb; }
  unsigned nbv() const { return stride_blocks(c, std::max<i64>(N(), 1)); }
  void finish() {  // the block's rows of X back to the caller's order
    if (ro.on) ro.restore_rows(c, X, nb);
  }

  void init_partial() {  // X = 0, R = P_own = b, st->rho = ||b_block||^2
    cg_init_k<TK, TX, TX><<<nbv(), kBlock, 0, c->stream>>>(p, nb, hp.c0, pl, Xt, X, R.p, Ploc.p, part.p, st.p);
    launched(c);
  }
  void start(double tol, i64 max_iter) {
    cg_start_k<<<1, 1, 0, c->stream>>>(st.p, tol, max_iter);
    launched(c);
  }
  void pack(cudaStream_t s) {  // P columns other ranks need
    if (!nsend) return;
    KScope ks_(c, "shard_pack");
    pack_cols_k<TK><<<stride_blocks(c, p * nsend), kBlock, 0, s>>>(p, nsend, send_idx.p, Ploc.p, sendK.p);
    launched(c);
  }
  // A rank without halo columns has no exchange to hide: it applies the
  // operator in the single-GPU order (L_c pass into U, then the L_r pass
  // combining), whose combine is cheaper than the one in the gather-bound
  // L_c pass (config 3 at one rank: 23.7 + 19.4 ms against 18.7 + 21.3 ms).
  bool local_order() const { return nh == 0 && nsend == 0; }
  void lr_local(TK gr, TK gc) {
    if (local_order()) return;  // lc_combine runs both passes
    const Combine<TK, TX> none{nullptr, nullptr, gr, gc, pl, nullptr, nullptr, st.p};
    launch_lr<TK, TK, TV, TX>(c, apK, pr, Ploc.p, U.p, none, false);
  }
  void zero_curv() {  // a rank without columns contributes 0 to the all-reduced dot
    CUDA_OK(cudaMemsetAsync(&st.p->curv, 0, sizeof(double), c->stream));
  }
  void lc_combine(TK gr, TK gc) {
    if (nb == 0) return zero_curv();
    const Combine<TK, TX> cb{U.p, AP.p, gr, gc, pl, nullptr, part.p, st.p};
    if (local_order()) {
      const Combine<TK, TX> none{nullptr, nullptr, gr, gc, pl, nullptr, nullptr, st.p};
      launch_lc<TK, TK, TV, TX>(c, apK, pcl, Ploc.p, U.p, none, false);
      launch_lr<TK, TK, TV, TX>(c, apK, pr, Ploc.p, nullptr, cb, true);
      return;
    }
    launch_lc<TK, TK, TV, TX>(c, apK, pcl, Ploc.p, nullptr, cb, true);
  }
  // the CG vector kernels: one wave of 8 x 256 threads per SM, 16-byte vectors when the buffers allow
  unsigned nbw() const {
    return static_cast<unsigned>(std::max<i64>(1, std::min<i64>(c->num_sms * 8, (N() + 1023) / 1024)));
  }
  static bool al16(const void* q) { return reinterpret_cast<uintptr_t>(q) % 16 == 0; }
  void residual() {
    KScope ks_(c, "cg_residual");
    if (al16(R.p) && al16(AP.p))
      cg_residual_k<TK, true><<<nbw(), kBlock, 0, c->stream>>>(N(), R.p, AP.p, part.p, st.p);
    else
      cg_residual_k<TK, false><<<nbv(), kBlock, 0, c->stream>>>(N(), R.p, AP.p, part.p, st.p);
    launched(c);
  }
  void update() {
    KScope ks_(c, "cg_update");
    if (al16(R.p) && al16(X) && al16(Ploc.p))
      cg_update_k<TK, TX, true><<<nbw(), kBlock, 0, c->stream>>>(N(), X, Ploc.p, R.p, st.p);
    else
      cg_update_k<TK, TX, false><<<nbv(), kBlock, 0, c->stream>>>(N(), X, Ploc.p, R.p, st.p);
    launched(c);
  }
  // true residual: X halo first (Xloc = [X own | X halo]), then x1 -> U and the combine in residual mode
  void prepare_x_halo() {
    Xloc.alloc(c, static_cast<size_t>(std::max<i64>(p * (nb + nh), 1)));
    sendX.alloc(c, std::max<i64>(p * nsend, 1));
    if (N()) CUDA_OK(cudaMemcpyAsync(Xloc.p, X, sizeof(TX) * N(), cudaMemcpyDeviceToDevice, c->stream));
    if (nsend)
      pack_cols_k<TX><<<stride_blocks(c, p * nsend), kBlock, 0, c->stream>>>(p, nsend, send_idx.p, Xloc.p, sendX.p);
    launched(c);
    CUDA_OK(cudaMemsetAsync(&st.p->done, 0, sizeof(int), c->stream));
  }
  void true_residual_partial(TK gr, TK gc) {
    if (nb == 0) return zero_curv();
    const Combine<TK, TX> none{nullptr, nullptr, gr, gc, pl, nullptr, nullptr, st.p};
    const Combine<TK, TX> cbR{U.p, nullptr, gr, gc, pl, Xt, part.p, st.p};
    launch_lc<TX, TK, TV, TX>(c, apX, pcl, Xloc.p, U.p, none, false);
    launch_lr<TX, TK, TV, TX>(c, apX, pr, Xloc.p, nullptr, cbR, true);
  }
};

template <typename T>
ncclDataType_t nccl_type() {
  return sizeof(T) == 8 ? ncclDouble : ncclFloat;
}

struct Comm {
  ncclComm_t nc = nullptr;
  int rank = 0, size = 1, device = 0;
  cudaStream_t s_comm = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_x0 = nullptr, ev_x1 = nullptr;
  ~Comm() {
    if (nc) nccl().CommDestroy(nc);
    if (s_comm) cudaStreamDestroy(s_comm);
    if (ev_pack) cudaEventDestroy(ev_pack);
    if (ev_x0) cudaEventDestroy(ev_x0);
    if (ev_x1) cudaEventDestroy(ev_x1);
  }
};

template <typename T>
void nccl_exchange(Comm* cm, const HaloPlan& h, i64 p, const T* sendbuf, T* recv_base, cudaStream_t s) {
  NCCL_OK(nccl().GroupStart());
  for (int q = 0; q < h.G; ++q) {
    if (q == h.rank) continue;
    const i64 ns = h.send_off[q + 1] - h.send_off[q], nr = h.recv_off[q + 1] - h.recv_off[q];
    if (ns) NCCL_OK(nccl().Send(sendbuf + h.send_off[q] * p, static_cast<size_t>(ns * p), nccl_type<T>(), q, cm->nc, s));
    if (nr) NCCL_OK(nccl().Recv(recv_base + h.recv_off[q] * p, static_cast<size_t>(nr * p), nccl_type<T>(), q, cm->nc, s));
  }
  NCCL_OK(nccl().GroupEnd());
}

// Common set-up of one rank: plan arrays, rsel/csel, the halo plan, the shard.
struct Setup {
  DevBuf<int> rsel, csel;
  Plan pl{};
};

void setup_plan(Ctx* c, Setup& s, i64 p, i64 n, const std::vector<i64>& omr, const std::vector<i64>& omc) {
  std::vector<int> rs(static_cast<size_t>(p), -1), cs(static_cast<size_t>(n), -1);
  for (size_t k = 0; k < omr.size(); ++k) {
    if (omr[k] < 0 || omr[k] >= p || rs[omr[k]] >= 0) invalid("alternate decoder: Xt does not match plan");
    rs[omr[k]] = static_cast<int>(k);
  }
  for (size_t k = 0; k < omc.size(); ++k) {
    if (omc[k] < 0 || omc[k] >= n || cs[omc[k]] >= 0) invalid("alternate decoder: Xt does not match plan");
    cs[omc[k]] = static_cast<int>(k);
  }
  s.rsel.alloc(c, std::max<i64>(p, 1));
  s.csel.alloc(c, std::max<i64>(n, 1));
  if (p) CUDA_OK(cudaMemcpyAsync(s.rsel.p, rs.data(), sizeof(int) * p, cudaMemcpyHostToDevice, c->stream));
  if (n) CUDA_OK(cudaMemcpyAsync(s.csel.p, cs.data(), sizeof(int) * n, cudaMemcpyHostToDevice, c->stream));
  s.pl = Plan{s.rsel.p, s.csel.p, static_cast<i64>(omr.size())};
}

// NCCL driver: this process's rank.
template <typename TX, typename TK, typename TV>
void decode_sharded_nccl(Ctx* c, Comm* cm, const TX* Xt, const std::vector<i64>& omr, const std::vector<i64>& omc,
                         i64 p, i64 n, Csr* Lr, Csr* Lc, double gbar_r, double gbar_c,
                         const cpcag_decoder_config& cfg, const i64* bounds, TX* Xblock, int* converged,
                         i64* iterations, cpcag_shard_stats* stats) {
  Setup su;
  setup_plan(c, su, p, n, omr, omc);
  std::vector<i64> rpc, rpr;
  std::vector<int> cic, cir;
  std::vector<TV> vc, vr;
  const Pull<TV> pcg = make_pull<TV>(c, Lc, true), prg = make_pull<TV>(c, Lr, false);
  host_pull(c, pcg, n, Lc->nnz, rpc, cic, &vc);
  host_pull<TV>(c, prg, p, Lr->nnz, rpr, cir, &vr);
  const HaloPlan hp = make_halo_plan(rpc.data(), cic.data(), n, bounds, cm->size, cm->rank);
  Shard<TX, TK, TV> sh;
  sh.build(c, hp, p, n, Lr, Lc, rpc, cic, vc, rpr, cir, vr, su.pl, Xblock, Xt);
  const TK gr = static_cast<TK>(gbar_r), gc = static_cast<TK>(gbar_c);
  double* rho = &sh.st.p->rho;
  double* curv = &sh.st.p->curv;
  double* rnext = &sh.st.p->rho_next;
  sh.init_partial();
  NCCL_OK(nccl().AllReduce(rho, rho, 1, ncclDouble, ncclSum, cm->nc, c->stream));
  sh.start(cfg.pcg_tol, cfg.pcg_max_iter);
  CgState host = read_back(c, sh.st.p);
  if (stats) {
    stats->halo_cols = sh.nh;
    stats->send_cols = sh.nsend;
    stats->exchange_ms = 0.0;
    stats->bytes_per_iteration = static_cast<double>((sh.nh + sh.nsend) * p) * sizeof(TK);
  }
  if (host.zero_rhs) {
    *converged = 1;
    *iterations = 0;
    return;
  }
  const bool timing = stats && stats->measure_exchange;
  std::vector<cudaEvent_t> evs;
  i64 done_it = 0;
  const i64 chunk = 32;
  while (!host.done && done_it < cfg.pcg_max_iter) {
    const i64 todo = std::min<i64>(chunk, cfg.pcg_max_iter - done_it);
    if (timing && evs.size() < static_cast<size_t>(2 * todo)) {
      while (evs.size() < static_cast<size_t>(2 * todo)) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreate(&e));
        evs.push_back(e);
      }
    }
    for (i64 k = 0; k < todo; ++k) {
      // 1. halo exchange on the comm stream, overlapped with 2. the block-local lr pass
      CUDA_OK(cudaEventRecord(cm->ev_pack, c->stream));
      CUDA_OK(cudaStreamWaitEvent(cm->s_comm, cm->ev_pack, 0));
      if (timing) CUDA_OK(cudaEventRecord(evs[2 * k], cm->s_comm));
      sh.pack(cm->s_comm);
      if (sh.nsend || sh.nh) nccl_exchange<TK>(cm, hp, p, sh.sendK.p, sh.Ploc.p + sh.nb * p, cm->s_comm);
      if (timing) CUDA_OK(cudaEventRecord(evs[2 * k + 1], cm->s_comm));
      CUDA_OK(cudaEventRecord(cm->ev_x1, cm->s_comm));
      sh.lr_local(gr, gc);
      CUDA_OK(cudaStreamWaitEvent(c->stream, cm->ev_x1, 0));
      // 3. lc pass + combine, 4. the CG scalars
      sh.lc_combine(gr, gc);
      NCCL_OK(nccl().AllReduce(curv, curv, 1, ncclDouble, ncclSum, cm->nc, c->stream));
      sh.residual();
      NCCL_OK(nccl().AllReduce(rnext, rnext, 1, ncclDouble, ncclSum, cm->nc, c->stream));
      sh.update();
    }
    done_it += todo;
    host = read_back(c, sh.st.p);
    if (timing)
      for (i64 k = 0; k < todo; ++k) {
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, evs[2 * k], evs[2 * k + 1]));
        stats->exchange_ms += ms;
      }
  }
  for (auto e : evs) cudaEventDestroy(e);
  if (host.err) runtime("pcg: breakdown (nonpositive curvature) at iteration " + std::to_string(host.err_it));
  sh.prepare_x_halo();
  if (sh.nsend || sh.nh) nccl_exchange<TX>(cm, hp, p, sh.sendX.p, sh.Xloc.p + sh.nb * p, c->stream);
  sh.true_residual_partial(gr, gc);
  NCCL_OK(nccl().AllReduce(curv, curv, 1, ncclDouble, ncclSum, cm->nc, c->stream));
  sh.finish();
  host = read_back(c, sh.st.p);
  const double rel = host.norm_b > 0.0 ? std::sqrt(host.curv) / host.norm_b : 0.0;
  *converged = rel <= cfg.pcg_tol ? 1 : 0;
  *iterations = host.it;
}

// Emulated driver: all ranks on one device, phase by phase.
template <typename TX, typename TK, typename TV>
void decode_sharded_emulated(Ctx* c, int G, const TX* Xt, const std::vector<i64>& omr, const std::vector<i64>& omc,
                             i64 p, i64 n, Csr* Lr, Csr* Lc, double gbar_r, double gbar_c,
                             const cpcag_decoder_config& cfg, const i64* bounds, TX* X, int* converged,
                             i64* iterations, cpcag_shard_stats* stats) {
  Setup su;
  setup_plan(c, su, p, n, omr, omc);
  std::vector<i64> rpc, rpr;
  std::vector<int> cic, cir;
  std::vector<TV> vc, vr;
  const Pull<TV> pcg = make_pull<TV>(c, Lc, true), prg = make_pull<TV>(c, Lr, false);
  host_pull(c, pcg, n, Lc->nnz, rpc, cic, &vc);
  host_pull<TV>(c, prg, p, Lr->nnz, rpr, cir, &vr);
  std::vector<std::unique_ptr<Shard<TX, TK, TV>>> sh;
  for (int g = 0; g < G; ++g) {
    sh.emplace_back(new Shard<TX, TK, TV>());
    sh[g]->build(c, make_halo_plan(rpc.data(), cic.data(), n, bounds, G, g), p, n, Lr, Lc, rpc, cic, vc, rpr,
                 cir, vr, su.pl, X + bounds[g] * p, Xt);
  }
  std::vector<CgState*> hst(static_cast<size_t>(G));
  for (int g = 0; g < G; ++g) hst[g] = sh[g]->st.p;
  DevBuf<CgState*> dst(c, static_cast<size_t>(G));
  CUDA_OK(cudaMemcpyAsync(dst.p, hst.data(), sizeof(CgState*) * G, cudaMemcpyHostToDevice, c->stream));
  auto allreduce = [&](int field) {
    emu_allreduce_k<<<1, 1, 0, c->stream>>>(dst.p, G, field);
    launched(c);
  };
  // copies of the packed columns into each receiver's halo slots
  auto exchange = [&](bool xmode) {
    for (int g = 0; g < G; ++g) xmode ? (void)0 : sh[g]->pack(c->stream);
    for (int d = 0; d < G; ++d)
      for (int s = 0; s < G; ++s) {
        if (s == d) continue;
        const HaloPlan& hs = sh[s]->hp;
        const HaloPlan& hd = sh[d]->hp;
        const i64 cnt = hd.recv_off[s + 1] - hd.recv_off[s];
        if (cnt != hs.send_off[d + 1] - hs.send_off[d]) runtime("sharded decoder: halo plan mismatch");
        if (!cnt) continue;
        if (xmode)
          CUDA_OK(cudaMemcpyAsync(sh[d]->Xloc.p + (sh[d]->nb + hd.recv_off[s]) * p,
                                  sh[s]->sendX.p + hs.send_off[d] * p, sizeof(TX) * cnt * p, cudaMemcpyDeviceToDevice,
                                  c->stream));
        else
          CUDA_OK(cudaMemcpyAsync(sh[d]->Ploc.p + (sh[d]->nb + hd.recv_off[s]) * p,
                                  sh[s]->sendK.p + hs.send_off[d] * p, sizeof(TK) * cnt * p, cudaMemcpyDeviceToDevice,
                                  c->stream));
      }
  };
  const TK gr = static_cast<TK>(gbar_r), gc = static_cast<TK>(gbar_c);
  for (auto& s : sh) s->init_partial();
  allreduce(0);
  for (auto& s : sh) s->start(cfg.pcg_tol, cfg.pcg_max_iter);
  CgState host = read_back(c, sh[0]->st.p);
  if (stats) {
    stats->halo_cols = sh[0]->nh;
    stats->send_cols = sh[0]->nsend;
    stats->exchange_ms = 0.0;
    stats->bytes_per_iteration = static_cast<double>((sh[0]->nh + sh[0]->nsend) * p) * sizeof(TK);
  }
  if (host.zero_rhs) {
    *converged = 1;
    *iterations = 0;
    return;
  }
  i64 done_it = 0;
  while (!host.done && done_it < cfg.pcg_max_iter) {
    const i64 todo = std::min<i64>(32, cfg.pcg_max_iter - done_it);
    for (i64 k = 0; k < todo; ++k) {
      exchange(false);
      for (auto& s : sh) s->lr_local(gr, gc);
      for (auto& s : sh) s->lc_combine(gr, gc);
      allreduce(1);
      for (auto& s : sh) s->residual();
      allreduce(2);
      for (auto& s : sh) s->update();
    }
    done_it += todo;
    host = read_back(c, sh[0]->st.p);
  }
  if (host.err) runtime("pcg: breakdown (nonpositive curvature) at iteration " + std::to_string(host.err_it));
  for (auto& s : sh) s->prepare_x_halo();
  exchange(true);
  for (auto& s : sh) s->true_residual_partial(gr, gc);
  allreduce(1);
  for (auto& s : sh) s->finish();
  host = read_back(c, sh[0]->st.p);
  const double rel = host.norm_b > 0.0 ? std::sqrt(host.curv) / host.norm_b : 0.0;
  *converged = rel <= cfg.pcg_tol ? 1 : 0;
  *iterations = host.it;
}

template <typename F>
void dispatch_precision(int precision, const cpcag_decoder_config& cfg, F&& f) {
  if (precision == CPCAG_F64)
    f(double{}, double{}, double{});
  else if (precision == CPCAG_F32 && cfg.krylov_precision == CPCAG_F32)
    f(float{}, float{}, float{});
  else if (precision == CPCAG_F32)
    f(float{}, double{}, float{});
  else
    invalid("unknown precision flag");
}

void check_sharded_args(i64 p, i64 n, Csr* Lr, Csr* Lc, const cpcag_decoder_config* cfg, int G) {
  if (!cfg) invalid("null argument");
  if (Lr->rows != p || Lc->rows != n || Lr->cols != p || Lc->cols != n)
    invalid("alternate decoder: Laplacians do not match plan");
  if (cfg->gamma <= 0.0) invalid("alternate decoder: gamma must be positive");
  if (G < 1) invalid("sharded decoder: at least one rank");
}

std::vector<i64> fetch_list(const int64_t* src, i64 k) {
  std::vector<i64> v(static_cast<size_t>(std::max<i64>(k, 0)));
  if (v.empty()) return v;
  if (is_device_ptr(src))
    CUDA_OK(cudaMemcpy(v.data(), src, sizeof(i64) * v.size(), cudaMemcpyDeviceToHost));
  else
    std::copy(src, src + v.size(), v.begin());
  return v;
}


// ------------------------------------------------------------------ column-sharded FISTA (frpcag.cpp:62-112)
// the compressed problem (rows x cols) split into contiguous
// column blocks, one per rank.  Per iteration a rank
//   1. forms its block of S = prox(Z - step grad g(Z)) from the full Z
//      (the Z L_c term reads every column of Z: the Kron-reduced L_c is dense),
//   2. all-gathers S (grouped send/recv of the blocks, ragged blocks allowed),
//   3. sums its block's share of the objective's three terms and of
//      ||Z||^2, ||Z_next - Z||^2 (one kernel, fixed order),
//   4. all-reduces those five scalars on the device,
//   5. decides (one thread: trace, t, coef, stop) and forms the full
//      Z_next = S + coef (S - S_prev) locally (elementwise, no exchange).
// The state lives on the device; the host polls it every kShfPoll iterations.
// S is bit-identical to the single-GPU CSR path (same element formulas); only
// the five scalars are summed in another order.
struct ShfState {
  double t, coef, frc;
  i64 j, iterations;
  int done, converged, err, pad;
  i64 err_j;
  unsigned cnt[2];
};
constexpr int kShfPoll = 16;

template <typename T>
__global__ void shf_grad_prox_k(i64 rows, i64 c0, i64 c1, Pull<T> Lr, Pull<T> Lc, T s_r, T s_c, int use_r,
                                int use_c, int loss, T step, const T* __restrict__ Z, const T* __restrict__ Y,
                                T* __restrict__ S, const ShfState* st) {
  if (st->done) return;
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (i64 c = c0 + blockIdx.y; c < c1; c += gridDim.y) {
    const i64 at = i + c * rows;
    const T g = grad_elem(Lr, Lc, s_r, s_c, use_r, use_c, Z, rows, i, c);
    const T arg = sub_rn(Z[at], mul_rn(step, g));
    S[at] = loss == CPCAG_LOSS_L2 ? prox_l2_elem(arg, Y[at], step) : prox_l1_elem(arg, Y[at], step);
  }
}

// scal[0..4] = this block's {data term, <S, S L_c>, <S, L_r S>, ||Z||^2, ||Z_next - Z||^2}.
template <typename T>
__global__ void shf_block_sums_k(i64 rows, i64 c0, i64 c1, Pull<T> Lr, Pull<T> Lc, int use_r, int use_c, int loss,
                                 const T* __restrict__ S, const T* __restrict__ Sp, const T* __restrict__ Z,
                                 const T* __restrict__ Y, double* partials, double* scal, ShfState* st) {
  if (st->done) return;
  const double t = st->t;
  const T coef = static_cast<T>((t - 1.0) / (0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t))));
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (i < rows) {
    for (i64 c = c0 + blockIdx.y; c < c1; c += gridDim.y) {
      const i64 at = i + c * rows;
      const T sv = S[at];
      const double x = static_cast<double>(sv);
      const double e = static_cast<double>(Y[at]) - x;
      s[0] += loss == CPCAG_LOSS_L2 ? e * e : fabs(e);
      if (use_c) s[1] += static_cast<double>(pull_right(Lc.rp[c], Lc.rp[c + 1], Lc.ci, Lc.v, S, rows, i)) * x;
      if (use_r) s[2] += static_cast<double>(pull_left(Lr.rp[i], Lr.rp[i + 1], Lr.ci, Lr.v, S + c * rows)) * x;
      const T zn = add_rn(sv, mul_rn(coef, sub_rn(sv, Sp[at])));
      const T z = Z[at];
      const double zd = static_cast<double>(z);
      const double dd = static_cast<double>(sub_rn(zn, z));
      s[3] += zd * zd;
      s[4] += dd * dd;
    }
  }
  double tot[5];
  if (grid_sum_last<5>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 5; ++q) scal[q] = tot[q];
  }
}

// Dense-operator forms of the two block kernels (Kron-reduced Laplacians are
// near dense; fista_dense.cuh): one 32 x 32 output tile per CTA, tiles of the
// block's columns only; fp64 sums run over k in ascending order with explicit
// multiply then add, i.e. the CSR-order sums plus exact zeros.
template <typename T>
__global__ void __launch_bounds__(256) shf_dense_grad_prox_k(i64 rr, i64 rc, i64 b0, i64 b1, const T* __restrict__ Lr,
                                                             const T* __restrict__ Lc, T s_r, T s_c, int use_r,
                                                             int use_c, int loss, T step, const T* __restrict__ Z,
                                                             const T* __restrict__ Y, T* __restrict__ S,
                                                             const ShfState* st) {
  if (st->done) return;
  const i64 i0 = static_cast<i64>(blockIdx.x) * kDT, c0 = b0 + static_cast<i64>(blockIdx.y) * kDT;
  T acc1[2][2], acc2[2][2];
  dual_gemm_tile(Lr, Lc, Z, rr, rc, use_r, use_c, i0, c0, acc1, acc2);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const i64 i = i0 + ty + 16 * a, c = c0 + tx + 16 * b;
      if (i >= rr || c >= b1) continue;
      const i64 at = i + c * rr;
      T g = T(0);
      if (use_c) g = add_rn(g, mul_rn(s_c, acc2[a][b]));
      if (use_r) g = add_rn(g, mul_rn(s_r, acc1[a][b]));
      const T arg = sub_rn(Z[at], mul_rn(step, g));
      S[at] = loss == CPCAG_LOSS_L2 ? prox_l2_elem(arg, Y[at], step) : prox_l1_elem(arg, Y[at], step);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) shf_dense_block_sums_k(i64 rr, i64 rc, i64 b0, i64 b1,
                                                              const T* __restrict__ Lr, const T* __restrict__ Lc,
                                                              int use_r, int use_c, int loss, const T* __restrict__ S,
                                                              const T* __restrict__ Sp, const T* __restrict__ Z,
                                                              const T* __restrict__ Y, double* partials, double* scal,
                                                              ShfState* st) {
  if (st->done) return;
  const double t = st->t;
  const T coef = static_cast<T>((t - 1.0) / (0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t))));
  const i64 i0 = static_cast<i64>(blockIdx.x) * kDT, c0 = b0 + static_cast<i64>(blockIdx.y) * kDT;
  T acc1[2][2], acc2[2][2];
  dual_gemm_tile(Lr, Lc, S, rr, rc, use_r, use_c, i0, c0, acc1, acc2);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const i64 i = i0 + ty + 16 * a, c = c0 + tx + 16 * b;
      if (i >= rr || c >= b1) continue;
      const i64 at = i + c * rr;
      const T sv = S[at];
      const double x = static_cast<double>(sv);
      const double e = static_cast<double>(Y[at]) - x;
      s[0] += loss == CPCAG_LOSS_L2 ? e * e : fabs(e);
      s[1] += static_cast<double>(acc2[a][b]) * x;
      s[2] += static_cast<double>(acc1[a][b]) * x;
      const T zn = add_rn(sv, mul_rn(coef, sub_rn(sv, Sp[at])));
      const T z = Z[at];
      const double zd = static_cast<double>(z);
      const double dd = static_cast<double>(sub_rn(zn, z));
      s[3] += zd * zd;
      s[4] += dd * dd;
    }
  double tot[5];
  if (grid_sum_last<5>(s, partials, &st->cnt[0], tot) && threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 5; ++q) scal[q] = tot[q];
  }
}

// frpcag.cpp:84-110 on the all-reduced scalars (identical on every rank).
__global__ void shf_decide_k(const double* scal, double gamma_r, double gamma_c, double tol, i64 max_iter,
                             double* trace, ShfState* st) {
  if (st->done) return;
  double val = scal[0];
  if (gamma_c != 0.0) val += gamma_c * scal[1];
  if (gamma_r != 0.0) val += gamma_r * scal[2];
  const i64 j = st->j;
  if (!isfinite(val)) {
    st->err = 1;
    st->err_j = j;
    st->done = 1;
    return;
  }
  trace[j - 1] = val;
  st->iterations = j;
  const double t = st->t;
  const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
  st->coef = (t - 1.0) / tn;
  const double denom = scal[3], change = scal[4];
  st->frc = denom > 0.0 ? change / denom : change;
  if (change < tol * denom) {
    st->converged = 1;
    st->done = 1;
    return;
  }
  st->t = tn;
  st->j = j + 1;
  if (st->j > max_iter) st->done = 1;
}

template <typename T>
__global__ void shf_update_k(i64 N, const T* __restrict__ S, const T* __restrict__ Sp, T* __restrict__ Z,
                             const ShfState* st) {
  if (st->done) return;
  const T coef = static_cast<T>(st->coef);
  for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < N; q += (i64)gridDim.x * blockDim.x) {
    const T sv = S[q];
    Z[q] = add_rn(sv, mul_rn(coef, sub_rn(sv, Sp[q])));
  }
}

// Emulated all-reduce: rank-ordered sum of the G five-scalar records, written to all.
__global__ void shf_emu_allreduce_k(double* scal_all, int G) {
  const int q = threadIdx.x;
  if (q >= 5) return;
  double s = 0.0;
  for (int g = 0; g < G; ++g) s += scal_all[5 * g + q];
  for (int g = 0; g < G; ++g) scal_all[5 * g + q] = s;
}

double shf_step(Ctx* c, Csr* Lr, Csr* Lc, const cpcag_frpcag_config& cfg) {
  if (cfg.step > 0.0) return cfg.step;
  // frpcag.cpp:70-75, computed by every rank on the whole (replicated) Laplacians.
  double nc = 0.0, nr = 0.0;
  if (cfg.gamma_c != 0.0 && cfg.gamma_r != 0.0)
    power_norm_pair(c, Lc, Lr, 1e-7, 42, 50000, &nc, &nr);
  else if (cfg.gamma_c != 0.0)
    nc = power_norm(c, Lc, 1e-7, 42, 50000);
  else if (cfg.gamma_r != 0.0)
    nr = power_norm(c, Lr, 1e-7, 42, 50000);
  const double beta = 2.0 * cfg.gamma_c * nc + 2.0 * cfg.gamma_r * nr;
  return beta > 0.0 ? 1.0 / beta : 1.0;
}

void shf_check(i64 rows, i64 cols, Csr* Lr, Csr* Lc, const cpcag_frpcag_config* cfg, const i64* bd, int G) {
  if (!cfg) invalid("null argument");
  frpcag_check_dims(rows, cols, Lr, Lc);
  if (cfg->gamma_r < 0.0 || cfg->gamma_c < 0.0) invalid("fista: negative regularization weight");
  if (cfg->tol <= 0.0) invalid("fista: stopping tolerance must be positive");
  if (cfg->max_iter < 1) invalid("fista: max_iter must be >= 1");
  if (G < 1) invalid("sharded fista: at least one rank");
  if (bd[0] != 0 || bd[G] != cols) invalid("sharded fista: bounds must run from 0 to cols");
  for (int g = 0; g < G; ++g)
    if (bd[g + 1] < bd[g]) invalid("sharded fista: bounds must ascend");
}

// One rank's buffers and the three block-local launches of an iteration.
template <typename T>
struct ShfRank {
  i64 rows = 0, cols = 0, c0 = 0, c1 = 0;
  DevBuf<T> S[2], Z;
  DevBuf<double> part, trace;
  DevBuf<ShfState> st;
  double* scal = nullptr;
  dim3 grid, gd;
  unsigned nb1 = 1;
  const T *Dr = nullptr, *Dc = nullptr;  // dense images of Lr, Lc (null: CSR pulls)

  void init(Ctx* c, const T* Y, i64 r, i64 cl, i64 b0, i64 b1, i64 max_iter, double* scal_dev) {
    rows = r, cols = cl, c0 = b0, c1 = b1, scal = scal_dev;
    const i64 N = rows * cols;
    S[0].alloc(c, N), S[1].alloc(c, N), Z.alloc(c, N);
    CUDA_OK(cudaMemcpyAsync(S[0].p, Y, sizeof(T) * N, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_OK(cudaMemcpyAsync(Z.p, Y, sizeof(T) * N, cudaMemcpyDeviceToDevice, c->stream));
    trace.alloc(c, max_iter);
    ShfState init{};
    init.t = 1.0;
    init.j = 1;
    st.alloc(c, 1);
    CUDA_OK(cudaMemcpyAsync(st.p, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    const unsigned gx = blocks_for(std::max<i64>(rows, 1));
    const i64 ycap = std::max<i64>(1, (static_cast<i64>(c->num_sms) * 16) / gx);
    grid = dim3(gx, static_cast<unsigned>(std::max<i64>(1, std::min<i64>({c1 - c0, ycap, 65535}))));
    nb1 = stride_blocks(c, N);
    gd = dim3(static_cast<unsigned>((rows + kDT - 1) / kDT),
              static_cast<unsigned>(std::max<i64>(1, (c1 - c0 + kDT - 1) / kDT)));
    part.alloc(c, 5 * std::max(static_cast<size_t>(grid.x) * grid.y, static_cast<size_t>(gd.x) * gd.y));
  }
  void grad_prox(Ctx* c, const Pull<T>& pr, const Pull<T>& pc, const cpcag_frpcag_config& cfg, T step, const T* Y,
                 i64 j) {
    if (c1 == c0) return;
    KScope ks_(c, "shf_grad_prox");
    if (Dr) {
      shf_dense_grad_prox_k<T><<<gd, 256, 0, c->stream>>>(
          rows, cols, c0, c1, Dr, Dc, static_cast<T>(2.0 * cfg.gamma_r), static_cast<T>(2.0 * cfg.gamma_c),
          cfg.gamma_r != 0.0, cfg.gamma_c != 0.0, cfg.loss, step, Z.p, Y, S[j & 1].p, st.p);
      launched(c);
      return;
    }
    shf_grad_prox_k<T><<<grid, kBlock, 0, c->stream>>>(
        rows, c0, c1, pr, pc, static_cast<T>(2.0 * cfg.gamma_r), static_cast<T>(2.0 * cfg.gamma_c),
        cfg.gamma_r != 0.0, cfg.gamma_c != 0.0, cfg.loss, step, Z.p, Y, S[j & 1].p, st.p);
    launched(c);
  }
  void block_sums(Ctx* c, const Pull<T>& pr, const Pull<T>& pc, const cpcag_frpcag_config& cfg, const T* Y, i64 j) {
    KScope ks_(c, "shf_block_sums");
    if (Dr) {
      shf_dense_block_sums_k<T><<<gd, 256, 0, c->stream>>>(rows, cols, c0, c1, Dr, Dc, cfg.gamma_r != 0.0,
                                                           cfg.gamma_c != 0.0, cfg.loss, S[j & 1].p,
                                                           S[(j - 1) & 1].p, Z.p, Y, part.p, scal, st.p);
      launched(c);
      return;
    }
    shf_block_sums_k<T><<<grid, kBlock, 0, c->stream>>>(rows, c0, c1, pr, pc, cfg.gamma_r != 0.0, cfg.gamma_c != 0.0,
                                                        cfg.loss, S[j & 1].p, S[(j - 1) & 1].p, Z.p, Y, part.p, scal,
                                                        st.p);
    launched(c);
  }
  void decide_update(Ctx* c, const cpcag_frpcag_config& cfg, i64 j) {
    KScope ks_(c, "shf_update");
    shf_decide_k<<<1, 1, 0, c->stream>>>(scal, cfg.gamma_r, cfg.gamma_c, cfg.tol, cfg.max_iter, trace.p, st.p);
    launched(c);
    shf_update_k<T><<<nb1, kBlock, 0, c->stream>>>(rows * cols, S[j & 1].p, S[(j - 1) & 1].p, Z.p, st.p);
    launched(c);
  }
};

template <typename T>
void shf_finish(Ctx* c, ShfRank<T>& R, const ShfState& host, double step, T* X, i64 col0, i64 col1,
                double* objective_host, cpcag_solve_trace* trace) {
  if (host.err)
    runtime("fista: diverged (non-finite objective at iteration " + std::to_string(host.err_j) +
            "); step too large");
  const i64 J = host.iterations;
  if (col1 > col0)
    CUDA_OK(cudaMemcpyAsync(X, R.S[J & 1].p + col0 * R.rows, sizeof(T) * R.rows * (col1 - col0),
                            cudaMemcpyDeviceToDevice, c->stream));
  if (objective_host && J > 0)
    CUDA_OK(cudaMemcpyAsync(objective_host, R.trace.p, sizeof(double) * J, cudaMemcpyDefault, c->stream));
  sync(c);
  trace->iterations = J;
  trace->converged = host.converged;
  trace->final_rel_change = host.frc;
  trace->step = step;
}

void shf_empty(const cpcag_frpcag_config& cfg, double step, double* objective_host, cpcag_solve_trace* trace) {
  // As the single-GPU path: every norm is zero, 0 < 0 is false, max_iter zero objectives.
  if (objective_host) std::fill(objective_host, objective_host + cfg.max_iter, 0.0);
  trace->iterations = cfg.max_iter;
  trace->converged = 0;
  trace->final_rel_change = 0.0;
  trace->step = step;
}

// Dense images when both Laplacians are >= 25 % full and exactly symmetric
// (the one-GPU path's rule, fista.cu).
template <typename T>
bool shf_densify(Ctx* c, Csr* Lr, Csr* Lc, DevBuf<T>& Dr, DevBuf<T>& Dc) {
  if (!(dense_worthwhile(Lr) && dense_worthwhile(Lc) && csr_symmetric(c, Lr) && csr_symmetric(c, Lc))) return false;
  densify<T>(c, Lr, Dr);
  densify<T>(c, Lc, Dc);
  return true;
}

template <typename T>
void fista_sharded_nccl(Ctx* c, Comm* cm, const T* Y, i64 rows, i64 cols, Csr* Lr, Csr* Lc,
                        const cpcag_frpcag_config& cfg, const i64* bd, T* X_block, double* objective_host,
                        cpcag_solve_trace* trace) {
  const double step = shf_step(c, Lr, Lc, cfg);
  if (rows * cols == 0) return shf_empty(cfg, step, objective_host, trace);
  const int G = cm->size, me = cm->rank;
  DevBuf<double> scal(c, 5);
  ShfRank<T> R;
  R.init(c, Y, rows, cols, bd[me], bd[me + 1], cfg.max_iter, scal.p);
  DevBuf<T> Dr, Dc;
  if (shf_densify<T>(c, Lr, Lc, Dr, Dc)) R.Dr = Dr.p, R.Dc = Dc.p;
  const Pull<T> pr = make_pull<T>(c, Lr, false), pc = make_pull<T>(c, Lc, true);
  ShfState host{};
  for (i64 j0 = 1; j0 <= cfg.max_iter; j0 += kShfPoll) {
    const i64 j1 = std::min<i64>(cfg.max_iter, j0 + kShfPoll - 1);
    for (i64 j = j0; j <= j1; ++j) {
      R.grad_prox(c, pr, pc, cfg, static_cast<T>(step), Y, j);
      if (G > 1) {  // all-gather of the S blocks
        T* S = R.S[j & 1].p;
        NCCL_OK(nccl().GroupStart());
        for (int q = 0; q < G; ++q) {
          if (q == me) continue;
          const i64 mine = (bd[me + 1] - bd[me]) * rows, theirs = (bd[q + 1] - bd[q]) * rows;
          if (mine) NCCL_OK(nccl().Send(S + bd[me] * rows, static_cast<size_t>(mine), nccl_type<T>(), q, cm->nc, c->stream));
          if (theirs) NCCL_OK(nccl().Recv(S + bd[q] * rows, static_cast<size_t>(theirs), nccl_type<T>(), q, cm->nc, c->stream));
        }
        NCCL_OK(nccl().GroupEnd());
      }
      R.block_sums(c, pr, pc, cfg, Y, j);
      if (G > 1) NCCL_OK(nccl().AllReduce(scal.p, scal.p, 5, ncclDouble, ncclSum, cm->nc, c->stream));
      R.decide_update(c, cfg, j);
    }
    host = read_back(c, R.st.p);
    if (host.done) break;
  }
  shf_finish(c, R, host, step, X_block, bd[me], bd[me + 1], objective_host, trace);
}

template <typename T>
void fista_sharded_emulated(Ctx* c, int G, const T* Y, i64 rows, i64 cols, Csr* Lr, Csr* Lc,
                            const cpcag_frpcag_config& cfg, const i64* bd, T* X, double* objective_host,
                            cpcag_solve_trace* trace) {
  const double step = shf_step(c, Lr, Lc, cfg);
  if (rows * cols == 0) return shf_empty(cfg, step, objective_host, trace);
  DevBuf<double> scal(c, 5 * static_cast<size_t>(G));
  std::vector<ShfRank<T>> R(static_cast<size_t>(G));
  for (int g = 0; g < G; ++g) R[g].init(c, Y, rows, cols, bd[g], bd[g + 1], cfg.max_iter, scal.p + 5 * g);
  DevBuf<T> Dr, Dc;
  if (shf_densify<T>(c, Lr, Lc, Dr, Dc))
    for (int g = 0; g < G; ++g) R[g].Dr = Dr.p, R[g].Dc = Dc.p;
  const Pull<T> pr = make_pull<T>(c, Lr, false), pc = make_pull<T>(c, Lc, true);
  ShfState host{};
  for (i64 j0 = 1; j0 <= cfg.max_iter; j0 += kShfPoll) {
    const i64 j1 = std::min<i64>(cfg.max_iter, j0 + kShfPoll - 1);
    for (i64 j = j0; j <= j1; ++j) {
      for (int g = 0; g < G; ++g) R[g].grad_prox(c, pr, pc, cfg, static_cast<T>(step), Y, j);
      for (int g = 0; g < G; ++g)  // the all-gather as device copies of rank g's block to every other rank
        for (int q = 0; q < G; ++q)
          if (q != g && bd[g + 1] > bd[g])
            CUDA_OK(cudaMemcpyAsync(R[q].S[j & 1].p + bd[g] * rows, R[g].S[j & 1].p + bd[g] * rows,
                                    sizeof(T) * rows * (bd[g + 1] - bd[g]), cudaMemcpyDeviceToDevice, c->stream));
      for (int g = 0; g < G; ++g) R[g].block_sums(c, pr, pc, cfg, Y, j);
      shf_emu_allreduce_k<<<1, 32, 0, c->stream>>>(scal.p, G);
      launched(c);
      for (int g = 0; g < G; ++g) R[g].decide_update(c, cfg, j);
    }
    host = read_back(c, R[0].st.p);
    if (host.done) break;
  }
  shf_finish(c, R[G - 1], host, step, X, 0, cols, objective_host, trace);
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_halo_plan(const int64_t* row_ptr, const int64_t* col_idx, int64_t n, const int64_t* bounds,
                               int nranks, int rank, int64_t* recv_counts, int64_t* send_counts, int64_t* recv_cols,
                               int64_t* send_cols) {
  return guard([&] {
    if (!row_ptr || !bounds || !recv_counts || !send_counts) invalid("null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) invalid("sharded decoder: rank out of range");
    std::vector<int> ci(static_cast<size_t>(row_ptr[n]));
    for (size_t k = 0; k < ci.size(); ++k) ci[k] = static_cast<int>(col_idx[k]);
    const HaloPlan h = make_halo_plan(row_ptr, ci.data(), n, bounds, nranks, rank);
    for (int q = 0; q < nranks; ++q) {
      recv_counts[q] = h.recv_off[q + 1] - h.recv_off[q];
      send_counts[q] = h.send_off[q + 1] - h.send_off[q];
    }
    if (recv_cols) std::copy(h.recv_cols.begin(), h.recv_cols.end(), recv_cols);
    if (send_cols) std::copy(h.send_cols.begin(), h.send_cols.end(), send_cols);
  });
}

extern "C" int cpcag_cuda_comm_unique_id(void* id_out) {
  return guard([&] {
    if (!id_out) invalid("null argument");
    ncclUniqueId id;
    NCCL_OK(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

extern "C" int cpcag_cuda_comm_create(cpcag_ctx ctx, const void* id, int nranks, int rank, cpcag_comm* out) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!id || !out) invalid("null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) invalid("sharded decoder: rank out of range");
    auto cm = std::make_unique<Comm>();
    cm->rank = rank;
    cm->size = nranks;
    cm->device = c->device;
    CUDA_OK(cudaSetDevice(c->device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    NCCL_OK(nccl().CommInitRank(&cm->nc, nranks, uid, rank));
    CUDA_OK(cudaStreamCreateWithFlags(&cm->s_comm, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&cm->ev_pack, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&cm->ev_x1, cudaEventDisableTiming));
    *out = reinterpret_cast<cpcag_comm>(cm.release());
  });
}

extern "C" int cpcag_cuda_comm_destroy(cpcag_comm comm) {
  return guard([&] { delete reinterpret_cast<Comm*>(comm); });
}

extern "C" int cpcag_cuda_alternate_decode_sharded(cpcag_ctx ctx, cpcag_comm comm, int precision, const void* Xt,
                                                   int64_t rho_r, int64_t rho_c, const int64_t* omega_r,
                                                   const int64_t* omega_c, int64_t p, int64_t n, cpcag_csr Lr,
                                                   cpcag_csr Lc, double lambda_k1_r, double lambda_k1_c,
                                                   const cpcag_decoder_config* cfg, const int64_t* bounds,
                                                   void* X_block, int* converged, int64_t* iterations,
                                                   cpcag_shard_stats* stats) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    Comm* cm = reinterpret_cast<Comm*>(comm);
    if (!cm || !bounds || !converged || !iterations) invalid("null argument");
    Csr *A = as_csr(Lr), *B = as_csr(Lc);
    check_sharded_args(p, n, A, B, cfg, cm->size);
    const std::vector<i64> omr = fetch_list(omega_r, rho_r), omc = fetch_list(omega_c, rho_c);
    std::vector<i64> bd(bounds, bounds + cm->size + 1);
    const i64 nb = bd[cm->rank + 1] - bd[cm->rank];
    dispatch_precision(precision, *cfg, [&](auto tx, auto tk, auto tv) {
      using TX = decltype(tx);
      using TK = decltype(tk);
      using TV = decltype(tv);
      InView<TX> xt(c, static_cast<const TX*>(Xt), static_cast<size_t>(rho_r * rho_c));
      OutView<TX> x(c, static_cast<TX*>(X_block), static_cast<size_t>(p * nb));
      decode_sharded_nccl<TX, TK, TV>(c, cm, xt.d, omr, omc, p, n, A, B, cfg->gamma / lambda_k1_r,
                                      cfg->gamma / lambda_k1_c, *cfg, bd.data(), x.d, converged, iterations, stats);
      x.flush(c);
      sync(c);
    });
  });
}

extern "C" int cpcag_cuda_alternate_decode_sharded_emulated(cpcag_ctx ctx, int nranks, int precision, const void* Xt,
                                                            int64_t rho_r, int64_t rho_c, const int64_t* omega_r,
                                                            const int64_t* omega_c, int64_t p, int64_t n,
                                                            cpcag_csr Lr, cpcag_csr Lc, double lambda_k1_r,
                                                            double lambda_k1_c, const cpcag_decoder_config* cfg,
                                                            const int64_t* bounds, void* X, int* converged,
                                                            int64_t* iterations, cpcag_shard_stats* stats) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!bounds || !converged || !iterations) invalid("null argument");
    Csr *A = as_csr(Lr), *B = as_csr(Lc);
    check_sharded_args(p, n, A, B, cfg, nranks);
    const std::vector<i64> omr = fetch_list(omega_r, rho_r), omc = fetch_list(omega_c, rho_c);
    std::vector<i64> bd(bounds, bounds + nranks + 1);
    dispatch_precision(precision, *cfg, [&](auto tx, auto tk, auto tv) {
      using TX = decltype(tx);
      using TK = decltype(tk);
      using TV = decltype(tv);
      InView<TX> xt(c, static_cast<const TX*>(Xt), static_cast<size_t>(rho_r * rho_c));
      OutView<TX> x(c, static_cast<TX*>(X), static_cast<size_t>(p * n));
      decode_sharded_emulated<TX, TK, TV>(c, nranks, xt.d, omr, omc, p, n, A, B, cfg->gamma / lambda_k1_r,
                                          cfg->gamma / lambda_k1_c, *cfg, bd.data(), x.d, converged, iterations,
                                          stats);
      x.flush(c);
      sync(c);
    });
  });
}

template <typename F>
static int shf_dispatch(int precision, F&& f) {
  if (precision == CPCAG_F64) return f(double{});
  if (precision == CPCAG_F32) return f(float{});
  set_last_error("unknown precision flag");
  return CPCAG_ERR_INVALID_ARGUMENT;
}

template <typename T, typename Body>
static void shf_call(Ctx* c, const void* Y, int64_t rows, int64_t cols, const cpcag_frpcag_config* cfg, void* X,
                     int64_t x_elems, double* objective, cpcag_solve_trace* trace, Body&& body) {
  InView<T> y(c, static_cast<const T*>(Y), static_cast<size_t>(rows * cols));
  OutView<T> x(c, static_cast<T*>(X), static_cast<size_t>(x_elems));
  std::vector<double> obj_host;
  double* obj_dst = objective;
  if (objective && is_device_ptr(objective)) {
    obj_host.resize(static_cast<size_t>(std::max<int64_t>(cfg->max_iter, 1)));
    obj_dst = obj_host.data();
  }
  body(y.d, x.d, obj_dst);
  x.flush(c);
  if (!obj_host.empty() && trace->iterations > 0)
    CUDA_OK(cudaMemcpyAsync(objective, obj_host.data(), sizeof(double) * trace->iterations, cudaMemcpyHostToDevice,
                            c->stream));
  sync(c);
}

extern "C" int cpcag_cuda_fista_sharded(cpcag_ctx ctx, cpcag_comm comm, int precision, const void* Y, int64_t rows,
                                        int64_t cols, cpcag_csr Lr, cpcag_csr Lc, const cpcag_frpcag_config* cfg,
                                        const int64_t* bounds, void* X_block, double* objective,
                                        cpcag_solve_trace* trace) {
  return shf_dispatch(precision, [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      Comm* cm = reinterpret_cast<Comm*>(comm);
      if (!cm || !bounds || !trace) invalid("null argument");
      shf_check(rows, cols, as_csr(Lr), as_csr(Lc), cfg, bounds, cm->size);
      const int64_t nb = bounds[cm->rank + 1] - bounds[cm->rank];
      shf_call<T>(c, Y, rows, cols, cfg, X_block, rows * nb, objective, trace, [&](const T* y, T* x, double* obj) {
        fista_sharded_nccl<T>(c, cm, y, rows, cols, as_csr(Lr), as_csr(Lc), *cfg, bounds, x, obj, trace);
      });
    });
  });
}

extern "C" int cpcag_cuda_fista_sharded_emulated(cpcag_ctx ctx, int nranks, int precision, const void* Y, int64_t rows,
                                                 int64_t cols, cpcag_csr Lr, cpcag_csr Lc,
                                                 const cpcag_frpcag_config* cfg, const int64_t* bounds, void* X,
                                                 double* objective, cpcag_solve_trace* trace) {
  return shf_dispatch(precision, [&](auto tag) {
    using T = decltype(tag);
    return guard([&] {
      Ctx* c = as_ctx(ctx);
      if (!bounds || !trace) invalid("null argument");
      if (nranks < 1) invalid("sharded fista: at least one rank");
      shf_check(rows, cols, as_csr(Lr), as_csr(Lc), cfg, bounds, nranks);
      shf_call<T>(c, Y, rows, cols, cfg, X, rows * cols, objective, trace, [&](const T* y, T* x, double* obj) {
        fista_sharded_emulated<T>(c, nranks, y, rows, cols, as_csr(Lr), as_csr(Lc), *cfg, bounds, x, obj, trace);
      });
    });
  });
}
