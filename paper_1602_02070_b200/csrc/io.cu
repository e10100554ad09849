// io.cu -- the GLR1 binary container straight to/from HBM (SURVEY §8f row
// 3: the data format on either side of the path).  Layout (io.cpp:16-20,
// 39-75, 88-188): magic "GLR1", little-endian u64 block kind (1 dense, 2
// CSR, 3 factors), little-endian u64 dimensions, then raw arrays:
//   dense   rows, cols, rows*cols fp64 column-major          (io.cpp:88-118)
//   CSR     rows, cols, nnz, row_ptr u64[rows+1], col_idx u64[nnz],
//           values fp64[nnz]                                  (io.cpp:151-188)
//   factors p, n, k, scale flag, U fp64[p*k], sigma fp64[k],
//           V fp64[n*k]                                       (io.cpp:200-230)
//
// Dense blocks stream through two 32 MB pinned buffers: the file read of
// chunk i+1 overlaps the H2D copy (and, for fp32 destinations, the fp64 ->
// fp32 narrowing kernel) of chunk i, so a 32 GB config-4 matrix lands in HBM
// as fp32 at file-read speed without a host-side conversion pass.  Saves run
// the reverse (fp32 -> fp64 widening on the device, D2H, write).  Error texts
// are the reference's ("<path>: not a GLR1 container (bad magic)", ...), as
// std::runtime_error.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"

namespace cpcag_cuda {

namespace {

constexpr uint64_t kDense = 1, kCsr = 2, kFactors = 3;
constexpr size_t kChunk = size_t{32} << 20;  // bytes per pinned staging buffer

[[noreturn]] void io_fail(const std::string& path, const std::string& what) { runtime(path + ": " + what); }

struct File {
  std::FILE* f = nullptr;
  std::string path;
  File(const std::string& p, bool write) : path(p) {
    f = std::fopen(p.c_str(), write ? "wb" : "rb");
    if (!f) io_fail(p, write ? "cannot open for writing" : "cannot open for reading");
  }
  ~File() {
    if (f) std::fclose(f);
  }
  void put_u64(uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
    if (std::fwrite(b, 1, 8, f) != 8) io_fail(path, "write failed");
  }
  uint64_t get_u64() {
    unsigned char b[8];
    if (std::fread(b, 1, 8, f) != 8) io_fail(path, "truncated header");
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return v;
  }
  void read(void* dst, size_t bytes, const char* what = "truncated data section") {
    if (bytes && std::fread(dst, 1, bytes, f) != bytes) io_fail(path, what);
  }
  void write(const void* src, size_t bytes) {
    if (bytes && std::fwrite(src, 1, bytes, f) != bytes) io_fail(path, "write failed");
  }
  uint64_t open_glr1() {
    char m[4];
    if (std::fread(m, 1, 4, f) != 4 || std::memcmp(m, "GLR1", 4) != 0) io_fail(path, "not a GLR1 container (bad magic)");
    return get_u64();
  }
  void header(uint64_t kind) {
    write("GLR1", 4);
    put_u64(kind);
  }
  void close() {
    if (f && std::fclose(f) != 0) {
      f = nullptr;
      io_fail(path, "write failed");
    }
    f = nullptr;
  }
};

struct PinnedPair {
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  explicit PinnedPair(size_t bytes) {
    for (int i = 0; i < 2; ++i) {
      CUDA_OK(cudaHostAlloc(&buf[i], bytes, cudaHostAllocDefault));
      CUDA_OK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
  }
  ~PinnedPair() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
};

__global__ void narrow_k(i64 n, const double* __restrict__ src, float* __restrict__ dst) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += gridDim.x * (i64)blockDim.x)
    dst[i] = static_cast<float>(src[i]);
}
__global__ void widen_k(i64 n, const float* __restrict__ src, double* __restrict__ dst) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += gridDim.x * (i64)blockDim.x)
    dst[i] = static_cast<double>(src[i]);
}

bool on_device(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// count fp64 values from the file into dst (fp64 or fp32, host or device).
void read_values(Ctx* c, File& f, i64 count, int precision, void* dst) {
  if (count <= 0) return;
  const bool dev = on_device(dst);
  if (!dev) {
    if (precision == CPCAG_F64) {
      f.read(dst, sizeof(double) * count);
    } else {
      std::vector<double> tmp(std::min<i64>(count, static_cast<i64>(kChunk / 8)));
      float* o = static_cast<float*>(dst);
      for (i64 at = 0; at < count;) {
        const i64 m = std::min<i64>(count - at, static_cast<i64>(tmp.size()));
        f.read(tmp.data(), sizeof(double) * m);
        for (i64 q = 0; q < m; ++q) o[at + q] = static_cast<float>(tmp[q]);
        at += m;
      }
    }
    return;
  }
  PinnedPair pp(kChunk);
  DevBuf<double> stage[2];
  if (precision == CPCAG_F32)
    for (auto& s : stage) s.alloc(c, kChunk / 8);
  const i64 per = static_cast<i64>(kChunk / 8);
  int b = 0;
  for (i64 at = 0; at < count; at += per, b ^= 1) {
    const i64 m = std::min<i64>(count - at, per);
    CUDA_OK(cudaEventSynchronize(pp.ev[b]));  // the previous copy out of this buffer is done
    f.read(pp.buf[b], sizeof(double) * m);
    if (precision == CPCAG_F64) {
      CUDA_OK(cudaMemcpyAsync(static_cast<double*>(dst) + at, pp.buf[b], sizeof(double) * m, cudaMemcpyHostToDevice,
                              c->stream));
    } else {
      CUDA_OK(cudaMemcpyAsync(stage[b].p, pp.buf[b], sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
      narrow_k<<<stride_blocks(c, m), kBlock, 0, c->stream>>>(m, stage[b].p, static_cast<float*>(dst) + at);
      launched(c);
    }
    CUDA_OK(cudaEventRecord(pp.ev[b], c->stream));
  }
  sync(c);
}

// count values of src (fp64 or fp32, host or device) to the file as fp64.
void write_values(Ctx* c, File& f, i64 count, int precision, const void* src) {
  if (count <= 0) return;
  if (!on_device(src)) {
    if (precision == CPCAG_F64) {
      f.write(src, sizeof(double) * count);
    } else {
      std::vector<double> tmp(std::min<i64>(count, static_cast<i64>(kChunk / 8)));
      const float* s = static_cast<const float*>(src);
      for (i64 at = 0; at < count;) {
        const i64 m = std::min<i64>(count - at, static_cast<i64>(tmp.size()));
        for (i64 q = 0; q < m; ++q) tmp[q] = static_cast<double>(s[at + q]);
        f.write(tmp.data(), sizeof(double) * m);
        at += m;
      }
    }
    return;
  }
  PinnedPair pp(kChunk);
  DevBuf<double> stage[2];
  if (precision == CPCAG_F32)
    for (auto& s : stage) s.alloc(c, kChunk / 8);
  const i64 per = static_cast<i64>(kChunk / 8);
  // issue chunk 0, then for each chunk: issue the next, wait for this one, write it
  auto issue = [&](i64 at, int b) {
    const i64 m = std::min<i64>(count - at, per);
    if (precision == CPCAG_F64) {
      CUDA_OK(cudaMemcpyAsync(pp.buf[b], static_cast<const double*>(src) + at, sizeof(double) * m,
                              cudaMemcpyDeviceToHost, c->stream));
    } else {
      widen_k<<<stride_blocks(c, m), kBlock, 0, c->stream>>>(m, static_cast<const float*>(src) + at, stage[b].p);
      launched(c);
      CUDA_OK(cudaMemcpyAsync(pp.buf[b], stage[b].p, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_OK(cudaEventRecord(pp.ev[b], c->stream));
  };
  issue(0, 0);
  int b = 0;
  for (i64 at = 0; at < count; at += per, b ^= 1) {
    if (at + per < count) issue(at + per, b ^ 1);
    CUDA_OK(cudaEventSynchronize(pp.ev[b]));
    f.write(pp.buf[b], sizeof(double) * std::min<i64>(count - at, per));
  }
}

void check_prec(int precision) {
  if (precision != CPCAG_F32 && precision != CPCAG_F64) invalid("unknown precision flag");
}

}  // namespace

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

extern "C" int cpcag_glr1_info(const char* path, int64_t* kind, int64_t* dims) {
  return guard([&] {
    if (!path || !kind || !dims) invalid("null argument");
    File f(path, false);
    const uint64_t k = f.open_glr1();
    *kind = static_cast<int64_t>(k);
    const int nd = k == kDense ? 2 : (k == kCsr ? 3 : (k == kFactors ? 4 : 0));
    if (!nd) io_fail(path, "unknown GLR1 block kind " + std::to_string(k));
    for (int i = 0; i < nd; ++i) dims[i] = static_cast<int64_t>(f.get_u64());
  });
}

extern "C" int cpcag_cuda_load_matrix_glr1(cpcag_ctx ctx, const char* path, int precision, void* out, int64_t rows,
                                           int64_t cols) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    check_prec(precision);
    if (!path) invalid("null argument");
    File f(path, false);
    if (f.open_glr1() != kDense) io_fail(path, "not a dense-matrix block");
    const auto r = static_cast<int64_t>(f.get_u64()), cc = static_cast<int64_t>(f.get_u64());
    if (r != rows || cc != cols)
      invalid(std::string(path) + ": dimension mismatch (file " + std::to_string(r) + " x " + std::to_string(cc) +
              ", buffer " + std::to_string(rows) + " x " + std::to_string(cols) + ")");
    if (r * cc > 0 && !out) invalid("null argument");
    read_values(c, f, r * cc, precision, out);
  });
}

extern "C" int cpcag_cuda_save_matrix_glr1(cpcag_ctx ctx, const char* path, int precision, const void* M, int64_t rows,
                                           int64_t cols) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    check_prec(precision);
    if (!path || (rows * cols > 0 && !M)) invalid("null argument");
    if (rows < 0 || cols < 0) invalid("negative dimensions");
    File f(path, true);
    f.header(kDense);
    f.put_u64(static_cast<uint64_t>(rows));
    f.put_u64(static_cast<uint64_t>(cols));
    write_values(c, f, rows * cols, precision, M);
    f.close();
  });
}

// load_sparse (io.cpp:164-188): the reference rebuilds through
// SparseMatrix::from_triplets, which sorts by (row, col), sums duplicates and
// drops exact zeros; canonical files take the direct path, others are
// canonicalised the same way here.
extern "C" int cpcag_cuda_load_sparse_glr1(cpcag_ctx ctx, const char* path, cpcag_csr* out) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!path || !out) invalid("null argument");
    File f(path, false);
    if (f.open_glr1() != kCsr) io_fail(path, "not a CSR block");
    const auto rows = static_cast<int64_t>(f.get_u64()), cols = static_cast<int64_t>(f.get_u64()),
               nnz = static_cast<int64_t>(f.get_u64());
    std::vector<int64_t> rp(static_cast<size_t>(rows) + 1), ci(static_cast<size_t>(nnz));
    std::vector<double> v(static_cast<size_t>(nnz));
    for (auto& x : rp) x = static_cast<int64_t>(f.get_u64());
    for (auto& x : ci) x = static_cast<int64_t>(f.get_u64());
    f.read(v.data(), sizeof(double) * nnz);
    if (rp.front() != 0 || rp.back() != nnz) io_fail(path, "inconsistent row pointers");
    bool canonical = true;
    for (int64_t r = 0; r < rows; ++r) {
      if (rp[r] > rp[r + 1]) io_fail(path, "row pointers not monotone");
      for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
        if (ci[k] < 0 || ci[k] >= cols) invalid("sparse: triplet index out of range");  // sparse.cpp:14-15
        if (!std::isfinite(v[k])) invalid("sparse: non-finite entry");
        if ((k > rp[r] && ci[k] <= ci[k - 1]) || v[k] == 0.0) canonical = false;
      }
    }
    if (!canonical) {
      std::vector<int64_t> nrp(static_cast<size_t>(rows) + 1, 0), nci;
      std::vector<double> nv;
      nci.reserve(static_cast<size_t>(nnz));
      nv.reserve(static_cast<size_t>(nnz));
      std::vector<int64_t> ord;
      for (int64_t r = 0; r < rows; ++r) {
        ord.resize(static_cast<size_t>(rp[r + 1] - rp[r]));
        std::iota(ord.begin(), ord.end(), rp[r]);
        std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return ci[a] < ci[b]; });
        for (size_t q = 0; q < ord.size();) {
          double s = 0.0;
          size_t e = q;
          for (; e < ord.size() && ci[ord[e]] == ci[ord[q]]; ++e) s += v[ord[e]];
          if (std::fabs(s) > 0.0) {
            nci.push_back(ci[ord[q]]);
            nv.push_back(s);
          }
          q = e;
        }
        nrp[r + 1] = static_cast<int64_t>(nci.size());
      }
      rp.swap(nrp);
      ci.swap(nci);
      v.swap(nv);
    }
    const int st = cpcag_csr_create(ctx, rows, cols, static_cast<int64_t>(v.size()), rp.data(), ci.data(), v.data(), out);
    if (st != CPCAG_OK) fail(st, cpcag_cuda_last_error());
    (void)c;
  });
}

extern "C" int cpcag_cuda_save_sparse_glr1(cpcag_ctx ctx, cpcag_csr A, const char* path) {
  return guard([&] {
    as_ctx(ctx);
    if (!path) invalid("null argument");
    int64_t rows = 0, cols = 0, nnz = 0;
    if (cpcag_csr_info(A, &rows, &cols, &nnz) != CPCAG_OK) fail(CPCAG_ERR_INVALID_ARGUMENT, cpcag_cuda_last_error());
    std::vector<int64_t> rp(static_cast<size_t>(rows) + 1), ci(static_cast<size_t>(nnz));
    std::vector<double> v(static_cast<size_t>(nnz));
    const int st = cpcag_csr_export(ctx, A, rp.data(), ci.data(), v.data());
    if (st != CPCAG_OK) fail(st, cpcag_cuda_last_error());
    File f(path, true);
    f.header(kCsr);
    f.put_u64(static_cast<uint64_t>(rows));
    f.put_u64(static_cast<uint64_t>(cols));
    f.put_u64(static_cast<uint64_t>(nnz));
    for (auto x : rp) f.put_u64(static_cast<uint64_t>(x));
    for (auto x : ci) f.put_u64(static_cast<uint64_t>(x));
    f.write(v.data(), sizeof(double) * v.size());
    f.close();
  });
}

extern "C" int cpcag_cuda_save_factors_glr1(cpcag_ctx ctx, const char* path, int64_t p, int64_t n, int64_t k,
                                            int scale_applied, const double* U, const double* sigma, const double* V) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!path || (k > 0 && (!U || !sigma || !V))) invalid("null argument");
    if (p < 0 || n < 0 || k < 0) invalid("negative dimensions");
    File f(path, true);
    f.header(kFactors);
    f.put_u64(static_cast<uint64_t>(p));
    f.put_u64(static_cast<uint64_t>(n));
    f.put_u64(static_cast<uint64_t>(k));
    f.put_u64(scale_applied ? 1 : 0);
    write_values(c, f, p * k, CPCAG_F64, U);
    write_values(c, f, k, CPCAG_F64, sigma);
    write_values(c, f, n * k, CPCAG_F64, V);
    f.close();
  });
}

extern "C" int cpcag_cuda_load_factors_glr1(cpcag_ctx ctx, const char* path, int64_t p, int64_t n, int64_t k,
                                            int* scale_applied, double* U, double* sigma, double* V) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (!path) invalid("null argument");
    File f(path, false);
    if (f.open_glr1() != kFactors) io_fail(path, "not a factors block");
    const auto fp = static_cast<int64_t>(f.get_u64()), fn = static_cast<int64_t>(f.get_u64()),
               fk = static_cast<int64_t>(f.get_u64());
    const uint64_t sc = f.get_u64();
    if (fp != p || fn != n || fk != k) invalid(std::string(path) + ": factor dimensions do not match the buffers");
    if (scale_applied) *scale_applied = sc != 0;
    if (k > 0 && (!U || !sigma || !V)) invalid("null argument");
    read_values(c, f, p * k, CPCAG_F64, U);
    read_values(c, f, k, CPCAG_F64, sigma);
    read_values(c, f, n * k, CPCAG_F64, V);
  });
}
