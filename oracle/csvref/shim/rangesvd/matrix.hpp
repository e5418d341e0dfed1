// Stand-in for the reference's rangesvd/matrix.hpp (which pulls in Eigen, absent
// from this image).  csv.hpp only needs DenseMatrix for read_csv_matrix; the
// CsvReader / read_csv_rows code under test does not touch it.  Test tooling
// only (oracle/csvref), never part of the product.
#pragma once
#include <cstddef>
#include <vector>
#include <rangesvd/errors.hpp>
namespace rangesvd {
class DenseMatrix {
public:
    DenseMatrix(std::size_t r, std::size_t c) : r_(r), c_(c), v_(r * c) {}
    double& operator()(std::size_t i, std::size_t j) { return v_[i * c_ + j]; }
    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
private:
    std::size_t r_, c_;
    std::vector<double> v_;
};
}  // namespace rangesvd
