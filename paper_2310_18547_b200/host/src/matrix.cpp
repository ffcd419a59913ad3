// matrix.cpp -- Matrix utilities of the drop-in (host, fp64).
#include <cmath>
#include <stdexcept>

#include "lorasim/matrix.hpp"

namespace lorasim {

Matrix matmul(const Matrix& a, const Matrix& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("matmul: inner dimensions differ");
  Matrix out(a.rows(), b.cols());
  const std::size_t n = b.cols();
  for (std::size_t i = 0; i < a.rows(); ++i) {
    double* orow = out.data().data() + i * n;
    for (std::size_t k = 0; k < a.cols(); ++k) {
      const double s = a(i, k);
      const double* brow = b.data().data() + k * n;
      for (std::size_t j = 0; j < n; ++j) orow[j] += s * brow[j];
    }
  }
  return out;
}

double max_abs_diff(const Matrix& a, const Matrix& b) {
  if (!a.same_shape(b)) throw std::invalid_argument("max_abs_diff: shape mismatch");
  double worst = 0.0;
  const auto& x = a.data();
  const auto& y = b.data();
  for (std::size_t i = 0; i < x.size(); ++i) worst = std::fmax(worst, std::fabs(x[i] - y[i]));
  return worst;
}

}  // namespace lorasim
