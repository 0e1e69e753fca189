// loraserve_compat_testing.hpp -- the reference's host-side test utilities
// (matrix.hpp:105-164) for code written against loraserve_compat.hpp: the
// fp64-accumulating gemm_reference oracle, the tolerance metric and the
// elementwise helpers reference tests use to build expected values.  Test
// infrastructure only: the operator path (loraserve_compat.hpp) never calls
// these.
#pragma once

#include <algorithm>
#include <cmath>

#include "loraserve_compat.hpp"

namespace loraserve {

namespace detail {
template <typename T>
void same_shape(ConstMatSpan<T> a, ConstMatSpan<T> b, const char* op) {
  if (a.rows != b.rows || a.cols != b.cols) throw ShapeError(a.rows, a.cols, b.rows, b.cols, op);
}
}  // namespace detail

// Naive product with 64-bit accumulation: the oracle every test referees with.
template <typename T>
Matrix<T> gemm_reference(ConstMatSpan<T> a, ConstMatSpan<T> b) {
  if (a.cols != b.rows) throw ShapeError(a.rows, a.cols, b.rows, b.cols, "gemm_reference");
  Matrix<T> c(a.rows, b.cols);
  for (std::size_t i = 0; i < a.rows; ++i) {
    for (std::size_t j = 0; j < b.cols; ++j) {
      double acc = 0.0;
      for (std::size_t p = 0; p < a.cols; ++p) acc += double(a(i, p)) * double(b(p, j));
      c(i, j) = static_cast<T>(acc);
    }
  }
  return c;
}

template <typename T>
void add_inplace(MatSpan<T> target, ConstMatSpan<T> delta) {
  detail::same_shape<T>(target, delta, "add_inplace");
  for (std::size_t i = 0, e = target.rows * target.cols; i < e; ++i) target.data[i] += delta.data[i];
}

template <typename T>
void sub_inplace(MatSpan<T> target, ConstMatSpan<T> delta) {
  detail::same_shape<T>(target, delta, "sub_inplace");
  for (std::size_t i = 0, e = target.rows * target.cols; i < e; ++i) target.data[i] -= delta.data[i];
}

template <typename T>
double max_abs_diff(ConstMatSpan<T> a, ConstMatSpan<T> b) {
  detail::same_shape<T>(a, b, "max_abs_diff");
  double w = 0.0;
  for (std::size_t i = 0, e = a.rows * a.cols; i < e; ++i) w = std::max(w, std::abs(double(a.data[i]) - double(b.data[i])));
  return w;
}

template <typename T>
double max_abs(ConstMatSpan<T> a) {
  double w = 0.0;
  for (std::size_t i = 0, e = a.rows * a.cols; i < e; ++i) w = std::max(w, std::abs(double(a.data[i])));
  return w;
}

}  // namespace loraserve
