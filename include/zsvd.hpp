// zsvd.hpp — drop-in C++ API for the rangesvd storage/query hot path, backed by
// the B200 C ABI (zsvd.h).  Reference users replace
//     #include <rangesvd/rangesvd.hpp>
// with
//     #include <zsvd.hpp>
// and link libzsvd.so; the hot-path names below keep the reference's
// signatures and exception types:
//
//   rangesvd::DenseMatrix            matrix.hpp:19-133   (row-major fp64; map() is a plain view)
//   rangesvd::SvdFactors             svd.hpp:30-40
//   rangesvd::orthonormality_defect  svd.hpp:48-58
//   rangesvd::validate_factors       svd.hpp:63-85
//   rangesvd::thin_svd               svd.hpp:90-131
//   rangesvd::truncate_rank          svd.hpp:135-164
//   rangesvd::reconstruct            svd.hpp:167-174
//   rangesvd::canonical_sign         svd.hpp:179-203
//   rangesvd::OpenBlock/SealedBlock  store.hpp:26-37
//   open_block_from_row / incremental_update / reorthonormalize   store.hpp:55-127
//   rangesvd::BlockStore             store.hpp:161-249   (ctor, append, sealed(), open(),
//                                                          snapshot, from_parts)
//   rangesvd::StoreSnapshot          store.hpp:135-156   (open, block_factors)
//   rangesvd::TimeRange::resolve     query.hpp:34-51
//   rangesvd::trim_block             query.hpp:64-89
//   rangesvd::stitch                 query.hpp:150-157
//   rangesvd::range_query (3 forms)  query.hpp:163-201
//   errors                           errors.hpp:9-68
//
// Additions: a FIXED_RANK truncation policy (BASELINE configs), device
// selection, and bulk append of many rows in one call.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <initializer_list>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "zsvd.h"

#ifndef ZSVD_NO_RANGESVD_NAMESPACE
namespace rangesvd {

// ------------------------------------------------------------ errors.hpp
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class InvalidInputError : public Error {
public:
    using Error::Error;
};
class InvalidParameterError : public Error {
public:
    using Error::Error;
};
class RangeError : public Error {
public:
    using Error::Error;
};
class DeviceError : public Error {
public:
    using Error::Error;
};
class IoError : public Error {  // errors.hpp:52
public:
    using Error::Error;
};
class FormatError : public Error {  // errors.hpp:58
public:
    using Error::Error;
};
class CorruptionError : public Error {  // errors.hpp:65
public:
    using Error::Error;
};
class ParseError : public Error {  // errors.hpp:34-45: "line N: what"
public:
    ParseError(std::size_t line, const std::string& what) : Error(what), line_(line) {}
    std::size_t line() const { return line_; }

private:
    std::size_t line_;
};
class SchemaError : public Error {  // errors.hpp:47
public:
    using Error::Error;
};

namespace detail {
inline void check(int code) {
    if (code == ZSVD_OK) return;
    char buf[4096];
    zsvd_last_error(buf, sizeof buf);
    switch (code) {
        case ZSVD_ERR_PARSE: throw ParseError(zsvd_last_error_line(), buf);
        case ZSVD_ERR_SCHEMA: throw SchemaError(buf);
        case ZSVD_ERR_INVALID_INPUT: throw InvalidInputError(buf);
        case ZSVD_ERR_INVALID_PARAMETER: throw InvalidParameterError(buf);
        case ZSVD_ERR_RANGE: throw RangeError(buf);
        case ZSVD_ERR_LOGIC: throw std::logic_error(buf);
        case ZSVD_ERR_IO: throw IoError(buf);
        case ZSVD_ERR_FORMAT: throw FormatError(buf);
        case ZSVD_ERR_CORRUPTION: throw CorruptionError(buf);
        default: throw DeviceError(buf);
    }
}
struct FactorsDeleter {
    void operator()(zsvd_factors* f) const { zsvd_factors_release(f); }
};
using FactorsPtr = std::unique_ptr<zsvd_factors, FactorsDeleter>;
}  // namespace detail

// ------------------------------------------------------------ matrix.hpp
/// Read-only row-major view (what DenseMatrix::map() returns here in place of
/// the reference's Eigen::Map): rows(), cols(), operator()(i, j).
struct MatrixView {
    const double* ptr = nullptr;
    std::size_t nrows = 0, ncols = 0;
    std::size_t rows() const { return nrows; }
    std::size_t cols() const { return ncols; }
    double operator()(std::size_t i, std::size_t j) const { return ptr[i * ncols + j]; }
};

class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(rows * cols, 0.0) {}
    DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data)
        : rows_(rows), cols_(cols), data_(std::move(data)) {
        if (data_.size() != rows_ * cols_) throw InvalidInputError("matrix data length does not match rows x cols");
        for (double v : data_)
            if (!(v - v == 0.0)) throw InvalidInputError("matrix entries must be finite");
    }
    static DenseMatrix from_rows(std::initializer_list<std::initializer_list<double>> rows) {
        std::vector<double> data;
        const std::size_t nr = rows.size(), nc = nr == 0 ? 0 : rows.begin()->size();
        for (const auto& r : rows) {
            if (r.size() != nc) throw InvalidInputError("from_rows: ragged row lengths");
            data.insert(data.end(), r.begin(), r.end());
        }
        return DenseMatrix(nr, nc, std::move(data));
    }
    static DenseMatrix from_row(std::span<const double> row) {
        return DenseMatrix(1, row.size(), std::vector<double>(row.begin(), row.end()));
    }
    /// Evaluates any matrix-like value (rows(), cols(), operator()(i, j)), e.g.
    /// a MatrixView or a caller's own expression type (matrix.hpp:59-70).
    template <typename Expr>
    static DenseMatrix from_expr(const Expr& e) {
        DenseMatrix m((std::size_t)e.rows(), (std::size_t)e.cols());
        for (std::size_t i = 0; i < m.rows_; ++i)
            for (std::size_t j = 0; j < m.cols_; ++j) m(i, j) = e((decltype(e.rows()))i, (decltype(e.cols()))j);
        if (!m.all_finite()) throw InvalidInputError("matrix expression produced non-finite entries");
        return m;
    }
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
    MatrixView map() const { return MatrixView{data_.data(), rows_, cols_}; }
    bool all_finite() const {
        for (double v : data_)
            if (!std::isfinite(v)) return false;
        return true;
    }
    double frobenius_norm() const {
        double sum = 0.0;
        for (double v : data_) sum += v * v;
        return std::sqrt(sum);
    }
    DenseMatrix left_cols(std::size_t k) const {
        DenseMatrix out(rows_, k);
        for (std::size_t i = 0; i < rows_; ++i)
            for (std::size_t j = 0; j < k; ++j) out(i, j) = (*this)(i, j);
        return out;
    }
    double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
    double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
    std::span<const double> values() const { return data_; }
    std::span<const double> row(std::size_t i) const { return {data_.data() + i * cols_, cols_}; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    DenseMatrix middle_rows(std::size_t first, std::size_t count) const {
        DenseMatrix out(count, cols_);
        std::copy(data_.begin() + first * cols_, data_.begin() + (first + count) * cols_, out.data_.begin());
        return out;
    }
    bool operator==(const DenseMatrix&) const = default;

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

// --------------------------------------------------------------- svd.hpp
struct SvdFactors {
    DenseMatrix u;
    std::vector<double> sigma;
    DenseMatrix v;
    std::size_t rank() const { return sigma.size(); }
    std::size_t left_rows() const { return u.rows(); }
    std::size_t right_rows() const { return v.rows(); }
    bool operator==(const SvdFactors&) const = default;
};

inline SvdFactors make_empty_factors(std::size_t rows, std::size_t cols) {
    return SvdFactors{DenseMatrix(rows, 0), {}, DenseMatrix(cols, 0)};
}

/// svd.hpp:22, :25.
inline constexpr double kNumericalRankCutoff = 1e-12;
inline constexpr double kOrthonormalityTol = 1e-10;

/// orthonormality_defect (svd.hpp:48-58): max |M^T M - I|, on the GPU.
inline double orthonormality_defect(const DenseMatrix& m);
/// validate_factors (svd.hpp:63-85).
inline void validate_factors(const SvdFactors& f, double defect_tol = kOrthonormalityTol);

/// Truncation policy: ENERGY(xi) is the reference's; FIXED_RANK(k) the BASELINE configs'.
struct Truncation {
    zsvd_truncation t;
    static Truncation energy(double xi) { return {{ZSVD_POLICY_ENERGY, xi, 0}}; }
    static Truncation fixed_rank(std::size_t k) { return {{ZSVD_POLICY_FIXED_RANK, 1.0, (uint64_t)k}}; }
};

namespace detail {
inline SvdFactors download(zsvd_factors* f) {
    std::size_t m = 0, n = 0, k = 0;
    check(zsvd_factors_shape(f, &m, &n, &k));
    SvdFactors out{DenseMatrix(m, k), std::vector<double>(k), DenseMatrix(n, k)};
    check(zsvd_factors_copy(f, out.u.data(), out.sigma.data(), out.v.data()));
    return out;
}
inline FactorsPtr upload(const SvdFactors& f) {
    zsvd_factors* h = nullptr;
    check(zsvd_factors_upload(f.u.data(), f.sigma.data(), f.v.data(), f.u.rows(), f.v.rows(), f.rank(), &h));
    return FactorsPtr(h);
}
}  // namespace detail

inline double orthonormality_defect(const DenseMatrix& m) {
    if (m.rows() < m.cols())
        throw InvalidInputError("orthonormality_defect: matrix must be tall (rows >= cols)");
    if (m.cols() == 0) return 0.0;
    double d = 0.0;
    detail::check(zsvd_orthonormality_defect(m.data(), m.rows(), m.cols(), m.cols(), ZSVD_MEM_HOST, &d));
    return d;
}

inline void validate_factors(const SvdFactors& f, double defect_tol) {
    const std::size_t k = f.rank();
    if (f.u.cols() != k || f.v.cols() != k) throw InvalidInputError("factors: rank mismatch between u, sigma and v");
    if (k > std::min(f.u.rows(), f.v.rows())) throw InvalidInputError("factors: rank exceeds matrix dimensions");
    for (std::size_t i = 0; i < k; ++i) {
        if (!std::isfinite(f.sigma[i]) || f.sigma[i] < 0.0)
            throw InvalidInputError("factors: singular values must be finite and non-negative");
        if (i + 1 < k && f.sigma[i] < f.sigma[i + 1])
            throw InvalidInputError("factors: singular values must be non-increasing");
    }
    if (!f.u.all_finite() || !f.v.all_finite()) throw InvalidInputError("factors: non-finite entries");
    if (orthonormality_defect(f.u) > defect_tol || orthonormality_defect(f.v) > defect_tol)
        throw InvalidInputError("factors: singular vectors are not orthonormal");
}

/// reconstruct (svd.hpp:167-174): U diag(sigma) V^T on the GPU; rank 0 gives zeros.
inline DenseMatrix reconstruct(const SvdFactors& f) {
    DenseMatrix out(f.left_rows(), f.right_rows());
    if (f.rank() == 0 || out.size() == 0) return out;
    auto d = detail::upload(f);
    detail::check(zsvd_reconstruct(d.get(), out.data(), ZSVD_MEM_HOST));
    if (!out.all_finite()) throw InvalidInputError("matrix expression produced non-finite entries");
    return out;
}

inline SvdFactors thin_svd(const DenseMatrix& a) {
    if (a.rows() < 1 || a.cols() < 1)
        throw InvalidInputError("thin_svd: matrix must have at least one row and one column");
    zsvd_factors* h = nullptr;
    detail::check(zsvd_thin_svd(a.data(), a.rows(), a.cols(), ZSVD_MEM_HOST, &h));
    detail::FactorsPtr p(h);
    return detail::download(h);
}

inline SvdFactors truncate_rank(const SvdFactors& f, Truncation t) {
    auto d = detail::upload(f);
    zsvd_factors* h = nullptr;
    detail::check(zsvd_truncate(d.get(), t.t, &h));
    detail::FactorsPtr p(h);
    return detail::download(h);
}
inline SvdFactors truncate_rank(const SvdFactors& f, double xi) { return truncate_rank(f, Truncation::energy(xi)); }

inline SvdFactors canonical_sign(SvdFactors f) {
    auto d = detail::upload(f);
    zsvd_factors* h = nullptr;
    detail::check(zsvd_canonical_sign(d.get(), &h));
    detail::FactorsPtr p(h);
    return detail::download(h);
}

// ------------------------------------------------------------- query.hpp
inline SvdFactors trim_block(const SvdFactors& block, std::size_t keep_from, std::size_t keep_to, Truncation t) {
    auto d = detail::upload(block);
    zsvd_factors* h = nullptr;
    detail::check(zsvd_trim_block(d.get(), keep_from, keep_to, t.t, &h));
    detail::FactorsPtr p(h);
    return detail::download(h);
}
inline SvdFactors trim_block(const SvdFactors& block, std::size_t keep_from, std::size_t keep_to, double xi) {
    return trim_block(block, keep_from, keep_to, Truncation::energy(xi));
}

inline SvdFactors stitch(const std::vector<SvdFactors>& parts, Truncation t) {
    std::vector<detail::FactorsPtr> held;
    std::vector<zsvd_factors*> raw;
    for (const auto& p : parts) {
        held.push_back(detail::upload(p));
        raw.push_back(held.back().get());
    }
    zsvd_factors* h = nullptr;
    detail::check(zsvd_stitch(raw.data(), raw.size(), t.t, &h));
    detail::FactorsPtr p(h);
    return detail::download(h);
}
inline SvdFactors stitch(const std::vector<SvdFactors>& parts, double xi) {
    return stitch(parts, Truncation::energy(xi));
}

// ------------------------------------------------------------- store.hpp
class BlockStore;

/// store.hpp:23.
inline constexpr std::size_t kReorthCadence = 64;

/// The block being filled (store.hpp:26-30); u has rows_seen rows.
struct OpenBlock {
    std::size_t index = 0;
    std::size_t rows_seen = 0;
    SvdFactors factors;
};

/// A finished block (store.hpp:34-37).
struct SealedBlock {
    std::size_t index = 0;
    SvdFactors factors;
};

namespace detail {
inline void check_row(std::span<const double> row, std::size_t num_columns) {  // store.hpp:41-50
    if (row.size() != num_columns) throw InvalidInputError("row has wrong number of columns");
    for (double v : row)
        if (!std::isfinite(v)) throw InvalidInputError("row entries must be finite");
}
}  // namespace detail

/// open_block_from_row (store.hpp:55-57): the thin SVD of the first row.
inline OpenBlock open_block_from_row(std::size_t index, std::span<const double> row) {
    return OpenBlock{index, 1, thin_svd(DenseMatrix::from_row(row))};
}

/// incremental_update (store.hpp:63-97): the SVD of [diag(sigma) V^T ; row]
/// with U_new = [[U, 0], [0, 1]] U_inner, numerical-rank cutoff only.  On the
/// GPU this is exactly a stitch (query.hpp:95-144) of the block's factors and
/// the row as a one-row part (u = [1], sigma = 1, v = row^T) with no
/// truncation (FIXED_RANK(c) keeps min(c, numerical rank)).
inline OpenBlock incremental_update(const OpenBlock& block, std::span<const double> row, std::size_t capacity) {
    if (block.rows_seen >= capacity) throw std::logic_error("incremental_update: block is already full");
    const std::size_t cols = block.factors.right_rows();
    detail::check_row(row, cols);
    SvdFactors rowpart{DenseMatrix(1, 1, {1.0}), {1.0}, DenseMatrix(cols, 1, std::vector<double>(row.begin(), row.end()))};
    SvdFactors inner = stitch({block.factors, rowpart}, Truncation::fixed_rank(cols));
    return OpenBlock{block.index, block.rows_seen + 1, std::move(inner)};
}

/// reorthonormalize (store.hpp:102-127): if U has lost orthonormality
/// (defect > 1e-10), refactor.  Here: the thin SVD of U diag(sigma) V^T,
/// rebuilt on the device — equal in exact arithmetic to the reference's
/// Q * thin_svd(R diag(sigma) V^T).
inline OpenBlock reorthonormalize(OpenBlock block) {
    const std::size_t k = block.factors.rank();
    if (k == 0 || orthonormality_defect(block.factors.u) <= kOrthonormalityTol) return block;
    auto d = detail::upload(block.factors);
    zsvd_factors* h = nullptr;
    detail::check(zsvd_refactor(d.get(), &h));
    detail::FactorsPtr p(h);
    block.factors = detail::download(h);
    return block;
}

struct TimeRange {
    std::size_t first_row = 0, last_row = 0, start_block = 0, end_block = 0;
    std::size_t skip_front = 0, keep_front = 0, keep_back = 0, skip_back = 0;
    std::size_t length() const { return last_row - first_row + 1; }
    static TimeRange resolve(std::size_t first, std::size_t last, const class StoreSnapshot& snap);
};

struct RangeSvd {
    SvdFactors factors;
    std::size_t rows() const { return factors.left_rows(); }
    std::size_t rank() const { return factors.rank(); }
};

namespace detail {
inline SvdFactors snapshot_block(zsvd_snapshot* s, std::size_t i) {
    zsvd_factors* h = nullptr;
    check(zsvd_snapshot_block(s, i, &h));
    FactorsPtr p(h);
    return download(h);
}
/// Host copies of a snapshot's blocks, fetched on first use and shared by
/// copies of the snapshot (blocks are immutable once the snapshot exists).
struct SnapshotCache {
    std::shared_ptr<zsvd_snapshot> h;
    std::mutex mu;
    std::map<std::size_t, SvdFactors> blocks;
    std::optional<OpenBlock> open;
    const SvdFactors& block(std::size_t i) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = blocks.find(i);
        if (it == blocks.end()) it = blocks.emplace(i, snapshot_block(h.get(), i)).first;
        return it->second;
    }
};
}  // namespace detail

/// The snapshot's open block (store.hpp:141, std::optional<OpenBlock> there):
/// has_value() is free; the factors are downloaded on first dereference.
class SnapshotOpenBlock {
public:
    bool has_value() const { return rows_ > 0; }
    explicit operator bool() const { return has_value(); }
    const OpenBlock& value() const {
        if (!has_value()) throw std::bad_optional_access();
        std::lock_guard<std::mutex> lk(cache_->mu);
        if (!cache_->open) cache_->open = OpenBlock{index_, rows_, detail::snapshot_block(cache_->h.get(), index_)};
        return *cache_->open;
    }
    const OpenBlock& operator*() const { return value(); }
    const OpenBlock* operator->() const { return &value(); }

private:
    friend class BlockStore;
    std::shared_ptr<detail::SnapshotCache> cache_;
    std::size_t index_ = 0, rows_ = 0;
};

class StoreSnapshot {
public:
    std::size_t block_size = 0, num_columns = 0, total_rows = 0, sealed_count = 0, open_rows = 0;
    double energy_threshold = 1.0;
    SnapshotOpenBlock open;
    std::size_t block_count() const { return sealed_count + (open_rows ? 1 : 0); }
    std::size_t block_rows(std::size_t i) const { return i < sealed_count ? block_size : open_rows; }
    /// store.hpp:150-155 (host copy, fetched once per snapshot).
    const SvdFactors& block_factors(std::size_t i) const {
        if (i >= block_count()) throw RangeError("block index out of range");
        return cache_->block(i);
    }
    zsvd_snapshot* handle() const { return h_.get(); }

private:
    friend class BlockStore;
    struct Del {
        void operator()(zsvd_snapshot* s) const { zsvd_snapshot_release(s); }
    };
    std::shared_ptr<zsvd_snapshot> h_;
    std::shared_ptr<detail::SnapshotCache> cache_;
};

inline TimeRange TimeRange::resolve(std::size_t first, std::size_t last, const StoreSnapshot& snap) {
    zsvd_time_range r{};
    detail::check(zsvd_resolve(snap.handle(), first, last, &r));
    return TimeRange{r.first_row, r.last_row, r.start_block, r.end_block,
                     r.skip_front, r.keep_front, r.keep_back, r.skip_back};
}

class BlockStore {
public:
    BlockStore(std::size_t block_size, std::size_t num_columns, double energy_threshold, int device = 0)
        : BlockStore(block_size, num_columns, Truncation::energy(energy_threshold), device) {}
    BlockStore(std::size_t block_size, std::size_t num_columns, Truncation t, int device = 0) : trunc_(t) {
        zsvd_store* s = nullptr;
        detail::check(zsvd_store_create_ex(block_size, num_columns, t.t, device, &s));
        h_.reset(s);
    }
    /// Adopts a store handle (load_store).
    explicit BlockStore(zsvd_store* s) : trunc_(Truncation::energy(1.0)) {
        h_.reset(s);
        trunc_ = Truncation{info().truncation};
    }
    std::size_t block_size() const { return info().block_size; }
    std::size_t num_columns() const { return info().num_columns; }
    double energy_threshold() const { return trunc_.t.xi; }
    std::size_t total_rows() const { return info().total_rows; }
    std::size_t sealed_count() const { return info().sealed_count; }
    Truncation truncation() const { return trunc_; }

    /// Consumes one time tick (store.hpp:182).
    void append(std::span<const double> row) {
        if (row.size() != num_columns()) throw InvalidInputError("row has wrong number of columns");
        detail::check(zsvd_store_append(h_.get(), row.data(), 1, row.size(), ZSVD_MEM_HOST));
    }
    /// Appends nrows rows at once (row stride ld); validated before any state change.
    void append_rows(const double* rows, std::size_t nrows, std::size_t ld, int memory = ZSVD_MEM_HOST) {
        detail::check(zsvd_store_append(h_.get(), rows, nrows, ld, memory));
    }

    /// Factors of block i (sealed, or the open tail when i == sealed_count()).
    SvdFactors block(std::size_t i) const {
        std::size_t k = 0;
        detail::check(zsvd_store_block_rank(h_.get(), i, &k));
        const auto inf = info();
        const std::size_t rows = i < inf.sealed_count ? inf.block_size : inf.open_rows;
        SvdFactors f{DenseMatrix(rows, k), std::vector<double>(k), DenseMatrix(inf.num_columns, k)};
        detail::check(zsvd_store_block_copy(h_.get(), i, f.u.data(), f.sigma.data(), f.v.data()));
        return f;
    }

    StoreSnapshot snapshot() const {
        zsvd_snapshot* s = nullptr;
        detail::check(zsvd_snapshot_create(h_.get(), &s));
        StoreSnapshot snap;
        snap.h_ = std::shared_ptr<zsvd_snapshot>(s, StoreSnapshot::Del{});
        zsvd_store_info inf{};
        detail::check(zsvd_snapshot_info_get(s, &inf));
        snap.block_size = inf.block_size;
        snap.num_columns = inf.num_columns;
        snap.total_rows = inf.total_rows;
        snap.sealed_count = inf.sealed_count;
        snap.open_rows = inf.open_rows;
        snap.energy_threshold = trunc_.t.xi;
        snap.cache_ = std::make_shared<detail::SnapshotCache>();
        snap.cache_->h = snap.h_;
        snap.open.cache_ = snap.cache_;
        snap.open.index_ = inf.sealed_count;
        snap.open.rows_ = inf.open_rows;
        return snap;
    }

    /// sealed() (store.hpp:178): host copies of the sealed blocks, downloaded
    /// once each (sealed blocks are immutable) and kept in a deque, so
    /// references stay valid while the store grows, as in the reference.
    const std::deque<SealedBlock>& sealed() const {
        const auto inf = info();
        if (inf.sealed_count < sealed_cache_.size()) sealed_cache_.clear();  // reset()
        while (sealed_cache_.size() < inf.sealed_count) {
            const std::size_t i = sealed_cache_.size();
            sealed_cache_.push_back(SealedBlock{i, block(i)});
        }
        return sealed_cache_;
    }
    /// open() (store.hpp:179): the open block's factors (untruncated,
    /// numerical-rank cutoff only), or nullopt when no block is open.
    const std::optional<OpenBlock>& open() const {
        const auto inf = info();
        if (inf.open_rows == 0) {
            open_cache_.reset();
        } else if (!open_cache_ || open_cache_total_ != inf.total_rows || open_cache_->rows_seen != inf.open_rows) {
            open_cache_ = OpenBlock{inf.sealed_count, inf.open_rows, block(inf.sealed_count)};
            open_cache_total_ = inf.total_rows;
        }
        return open_cache_;
    }

    /// from_parts (store.hpp:206-231): rebuilds a store from persisted parts;
    /// counts and shapes must be consistent (InvalidInputError otherwise).
    static BlockStore from_parts(std::size_t block_size, std::size_t num_columns, Truncation t,
                                 const std::deque<SealedBlock>& sealed, const std::optional<OpenBlock>& open,
                                 int device = 0) {
        if (block_size < 1 || num_columns < 1)
            throw InvalidParameterError("block size and column count must be at least 1");
        if (t.t.policy == ZSVD_POLICY_ENERGY && (!(t.t.xi > 0.0) || t.t.xi > 1.0))
            throw InvalidParameterError("energy threshold must lie in (0, 1]");
        std::vector<zsvd_block_factors> parts;
        for (std::size_t i = 0; i < sealed.size(); ++i) {
            const SvdFactors& f = sealed[i].factors;
            if (sealed[i].index != i || f.left_rows() != block_size || f.right_rows() != num_columns ||
                f.u.cols() != f.rank() || f.v.cols() != f.rank())
                throw InvalidInputError("from_parts: inconsistent sealed block");
            parts.push_back({sealed[i].index, f.left_rows(), f.rank(), f.u.data(), f.sigma.data(), f.v.data()});
        }
        zsvd_block_factors op{};
        if (open) {
            const SvdFactors& f = open->factors;
            if (open->index != sealed.size() || open->rows_seen < 1 || open->rows_seen > block_size ||
                f.left_rows() != open->rows_seen || f.right_rows() != num_columns || f.u.cols() != f.rank() ||
                f.v.cols() != f.rank())
                throw InvalidInputError("from_parts: inconsistent open block");
            op = {open->index, open->rows_seen, f.rank(), f.u.data(), f.sigma.data(), f.v.data()};
        }
        zsvd_store* s = nullptr;
        detail::check(zsvd_store_from_parts(block_size, num_columns, t.t, device, parts.data(), parts.size(),
                                            open ? &op : nullptr, &s));
        return BlockStore(s);
    }
    static BlockStore from_parts(std::size_t block_size, std::size_t num_columns, double energy_threshold,
                                 const std::deque<SealedBlock>& sealed, const std::optional<OpenBlock>& open) {
        return from_parts(block_size, num_columns, Truncation::energy(energy_threshold), sealed, open);
    }

    zsvd_store* handle() const { return h_.get(); }
    zsvd_store_info info() const {
        zsvd_store_info i{};
        detail::check(zsvd_store_info_get(h_.get(), &i));
        return i;
    }

private:
    struct Del {
        void operator()(zsvd_store* s) const { zsvd_store_destroy(s); }
    };
    std::unique_ptr<zsvd_store, Del> h_;
    Truncation trunc_;
    mutable std::deque<SealedBlock> sealed_cache_;
    mutable std::optional<OpenBlock> open_cache_;
    mutable std::size_t open_cache_total_ = 0;
};

inline RangeSvd range_query(const StoreSnapshot& snap, std::size_t first, std::size_t last, Truncation t) {
    zsvd_factors* h = nullptr;
    detail::check(zsvd_range_query(snap.handle(), first, last, t.t, &h));
    detail::FactorsPtr p(h);
    return RangeSvd{detail::download(h)};
}
inline RangeSvd range_query(const StoreSnapshot& snap, std::size_t first, std::size_t last, double xi) {
    return range_query(snap, first, last, Truncation::energy(xi));
}
inline RangeSvd range_query(const BlockStore& store, std::size_t first, std::size_t last, double xi) {
    return range_query(store.snapshot(), first, last, xi);
}
inline RangeSvd range_query(const BlockStore& store, std::size_t first, std::size_t last) {
    return range_query(store.snapshot(), first, last, store.truncation());
}

/// naive_range_svd (analysis.hpp:49-66), on the GPU.
inline SvdFactors naive_range_svd(const StoreSnapshot& snap, std::size_t first, std::size_t last) {
    zsvd_factors* h = nullptr;
    detail::check(zsvd_naive_range_svd(snap.handle(), first, last, &h));
    detail::FactorsPtr p(h);
    return detail::download(h);
}

/// reconstruction_error (analysis.hpp:20-37), on the GPU.
inline double reconstruction_error(const DenseMatrix& raw, const SvdFactors& f) {
    if (raw.rows() != f.left_rows() || raw.cols() != f.right_rows())
        throw InvalidInputError("reconstruction_error: shape mismatch");
    zsvd_factors* h = nullptr;
    detail::check(zsvd_factors_upload(f.u.data(), f.sigma.data(), f.v.data(), f.left_rows(), f.right_rows(),
                                      f.rank(), &h));
    detail::FactorsPtr p(h);
    double e = 0.0;
    detail::check(zsvd_reconstruction_error(raw.data(), raw.rows(), raw.cols(), ZSVD_MEM_HOST, h, &e));
    return e;
}

/// oracle_range_svd (analysis.hpp:40-45): thin SVD of the raw row slice.
inline SvdFactors oracle_range_svd(const DenseMatrix& raw, std::size_t first, std::size_t last) {
    if (last < first || last >= raw.rows()) throw RangeError("oracle_range_svd: range out of bounds");
    return thin_svd(raw.middle_rows(first, last - first + 1));
}

/// serialize.hpp:147: header bytes of the v1 format.
inline constexpr std::size_t kHeaderBytes = 4 + 4 + 4 + 4 + 8 + 8 + 8 + 1;

/// serialized_size (serialize.hpp:150-161): exact size of save_store's output
/// (FIXED_RANK stores: the v2 header's extra rank field).
inline std::size_t serialized_size(const BlockStore& store) {
    const auto inf = store.info();
    const std::size_t c = inf.num_columns;
    auto factors_bytes = [c](std::size_t rows, std::size_t k) { return 4 + 8 * k * (rows + 1 + c); };
    std::size_t n = kHeaderBytes + (inf.truncation.policy == ZSVD_POLICY_FIXED_RANK ? 8 : 0);
    for (std::size_t i = 0; i <= inf.sealed_count; ++i) {
        if (i == inf.sealed_count && inf.open_rows == 0) break;
        std::size_t k = 0;
        detail::check(zsvd_store_block_rank(store.handle(), i, &k));
        n += i < inf.sealed_count ? 8 + factors_bytes(inf.block_size, k) : 16 + factors_bytes(inf.open_rows, k);
    }
    return n;
}

/// save_store / load_store (serialize.hpp:162-254): the ZSVD v1 file format.
inline void save_store(const BlockStore& store, const std::string& path) {
    detail::check(zsvd_store_save(store.handle(), path.c_str()));
}
inline BlockStore load_store(const std::string& path, int device = 0) {
    zsvd_store* s = nullptr;
    detail::check(zsvd_store_load(path.c_str(), device, &s));
    return BlockStore(s);
}

/// analysis.hpp:70-74.
struct SearchHit {
    std::size_t window_start = 0;
    double similarity = 0.0;  // |cosine| of leading left singular vectors, in [0, 1]
};

namespace detail {
/// leading_vector_similarity (analysis.hpp:77-96): |cos| between the leading
/// left singular vectors of two host-resident answers; 0 when either has rank 0.
inline double leading_vector_similarity(const SvdFactors& a, const SvdFactors& b) {
    if (a.rank() == 0 || b.rank() == 0) return 0.0;
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (std::size_t i = 0; i < a.left_rows(); ++i) {
        const double x = a.u(i, 0), y = b.u(i, 0);
        dot += x * y;
        na += x * x;
        nb += y * y;
    }
    if (na == 0.0 || nb == 0.0) return 0.0;
    return std::fabs(dot) / (std::sqrt(na) * std::sqrt(nb));
}
}  // namespace detail

/// similar_range_search (analysis.hpp:106-148): every window is queried on the
/// GPU in batches; same ordering, ties and error types as the reference.
inline std::vector<SearchHit> similar_range_search(const StoreSnapshot& snap, std::size_t base_first,
                                                   std::size_t base_last, std::size_t stride,
                                                   std::size_t top_n, Truncation t) {
    std::vector<uint64_t> starts(top_n > 0 ? top_n : 1);
    std::vector<double> sims(top_n > 0 ? top_n : 1);
    std::size_t n = 0;
    detail::check(zsvd_similar_range_search(snap.handle(), base_first, base_last, stride, top_n, t.t,
                                            starts.data(), sims.data(), &n));
    std::vector<SearchHit> hits(n);
    for (std::size_t i = 0; i < n; ++i) hits[i] = SearchHit{(std::size_t)starts[i], sims[i]};
    return hits;
}
inline std::vector<SearchHit> similar_range_search(const StoreSnapshot& snap, std::size_t base_first,
                                                   std::size_t base_last, std::size_t stride,
                                                   std::size_t top_n, double xi) {
    return similar_range_search(snap, base_first, base_last, stride, top_n, Truncation::energy(xi));
}
inline std::vector<SearchHit> similar_range_search(const BlockStore& store, std::size_t base_first,
                                                   std::size_t base_last, std::size_t stride,
                                                   std::size_t top_n, double xi) {
    return similar_range_search(store.snapshot(), base_first, base_last, stride, top_n, xi);
}
inline std::vector<SearchHit> similar_range_search(const BlockStore& store, std::size_t base_first,
                                                   std::size_t base_last, std::size_t stride,
                                                   std::size_t top_n) {
    return similar_range_search(store.snapshot(), base_first, base_last, stride, top_n, store.truncation());
}

// ------------------------------------------------------------ csv.hpp
/// CsvOptions (csv.hpp:22-27).
struct CsvOptions {
    std::optional<std::size_t> expected_cols;
    bool drop_timestamp = false;
};

/// CsvReader (csv.hpp:67-150).  The whole file is read and parsed on the GPU
/// when the reader is constructed (IoError if it cannot be opened, like the
/// reference constructor); next() then yields the rows in file order and
/// throws the reader's ParseError / SchemaError where the reference would,
/// after the rows before it.
class CsvReader {
public:
    explicit CsvReader(const std::string& path, CsvOptions options = {}, int device = 0) {
        zsvd_csv_options o{options.expected_cols ? (int64_t)*options.expected_cols : -1,
                           options.drop_timestamp ? 1 : 0};
        zsvd_csv* h = nullptr;
        detail::check(zsvd_csv_read(path.c_str(), o, device, &h));
        h_.reset(h);
        detail::check(zsvd_csv_info(h, &rows_, &cols_, &error_, &error_line_));
        char buf[4096];
        zsvd_csv_error_message(h, buf, sizeof buf);
        message_ = buf;
    }
    /// Next row, or nullopt at end of input.
    std::optional<std::vector<double>> next() {
        if (next_ < rows_) {
            std::vector<double> row(cols_);
            detail::check(zsvd_csv_rows_copy(h_.get(), next_, 1, row.data()));
            ++next_;
            return row;
        }
        raise();
        return std::nullopt;
    }
    /// Columns per row; 0 until the first data row has been read.
    std::size_t cols() const { return next_ > 0 ? cols_ : 0; }

    // beyond the reference: the whole parsed file at once
    std::size_t rows_before_error() const { return rows_; }
    std::size_t file_cols() const { return cols_; }
    zsvd_csv* handle() const { return h_.get(); }
    void raise() const {
        if (error_ == ZSVD_ERR_PARSE) throw ParseError(error_line_, message_);
        if (error_ == ZSVD_ERR_SCHEMA) throw SchemaError(message_);
    }

private:
    struct Deleter {
        void operator()(zsvd_csv* h) const { zsvd_csv_release(h); }
    };
    std::unique_ptr<zsvd_csv, Deleter> h_;
    std::size_t rows_ = 0, cols_ = 0, error_line_ = 0, next_ = 0;
    int error_ = ZSVD_OK;
    std::string message_;
};

/// read_csv_rows (csv.hpp:153-161).
inline std::vector<std::vector<double>> read_csv_rows(const std::string& path, CsvOptions options = {}) {
    CsvReader r(path, options);
    r.raise();
    std::vector<std::vector<double>> rows(r.rows_before_error(), std::vector<double>(r.file_cols()));
    for (std::size_t i = 0; i < rows.size(); ++i)
        detail::check(zsvd_csv_rows_copy(r.handle(), i, 1, rows[i].data()));
    return rows;
}

/// read_csv_matrix (csv.hpp:164-177): no data rows -> InvalidInputError.
inline DenseMatrix read_csv_matrix(const std::string& path, CsvOptions options = {}) {
    CsvReader r(path, options);
    r.raise();
    if (r.rows_before_error() == 0) throw InvalidInputError("'" + path + "' contains no data rows");
    DenseMatrix m(r.rows_before_error(), r.file_cols());
    detail::check(zsvd_csv_rows_copy(r.handle(), 0, m.rows(), m.data()));
    return m;
}

/// Appends every row of a CSV file to the store straight from HBM (the
/// cmd_ingest loop, commands.hpp:119-123); all or nothing.
inline std::size_t append_csv(BlockStore& store, const std::string& path, CsvOptions options = {}) {
    CsvReader r(path, options, store.info().device);
    std::size_t n = 0;
    detail::check(zsvd_store_append_csv(store.handle(), r.handle(), &n));
    return n;
}

}  // namespace rangesvd
#endif
