// types.hpp -- the reference's dense types (proj/core/include/cpcag/types.hpp:10-16)
// without Eigen: column-major fp64 Matrix and Vector with the subset of the
// Eigen interface the cpcag API and its callers use (rows/cols/size/data,
// (i, j) indexing, Zero).  Storage is contiguous column-major, exactly the
// C-ABI's dense layout, so calls pass data() straight through.
#pragma once

#include <cstdint>
#include <algorithm>
#include <initializer_list>
#include <stdexcept>
#include <vector>

namespace cpcag {

using Index = std::int64_t;
using IndexList = std::vector<Index>;

class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : r_(rows), c_(cols), v_(static_cast<size_t>(rows * cols), 0.0) {
    if (rows < 0 || cols < 0) throw std::invalid_argument("Matrix: negative dimension");
  }
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  // Row-major initializer, e.g. Matrix::from_rows({{1, 2}, {3, 4}}).
  static Matrix from_rows(std::initializer_list<std::initializer_list<double>> rows) {
    const Index r = static_cast<Index>(rows.size());
    const Index c = r ? static_cast<Index>(rows.begin()->size()) : 0;
    Matrix m(r, c);
    Index i = 0;
    for (const auto& row : rows) {
      if (static_cast<Index>(row.size()) != c) throw std::invalid_argument("Matrix: ragged rows");
      Index j = 0;
      for (double x : row) m(i, j++) = x;
      ++i;
    }
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(i + j * r_)]; }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};

class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(static_cast<size_t>(n), 0.0) {}
  Vector(std::initializer_list<double> xs) : v_(xs) {}
  static Vector Zero(Index n) { return Vector(n); }
  Index size() const { return static_cast<Index>(v_.size()); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }

 private:
  std::vector<double> v_;
};

}  // namespace cpcag
