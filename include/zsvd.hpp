// zsvd.hpp — drop-in C++ API for the rangesvd storage/query hot path, backed by
// the B200 C ABI (zsvd.h).  Reference users replace
//     #include <rangesvd/rangesvd.hpp>
// with
//     #include <zsvd.hpp>
// and link libzsvd.so; the hot-path names below keep the reference's
// signatures and exception types:
//
//   rangesvd::DenseMatrix            matrix.hpp:19-133   (row-major fp64 subset)
//   rangesvd::SvdFactors             svd.hpp:30-40
//   rangesvd::thin_svd               svd.hpp:90-131
//   rangesvd::truncate_rank          svd.hpp:135-164
//   rangesvd::canonical_sign         svd.hpp:179-203
//   rangesvd::BlockStore             store.hpp:161-249   (ctor, append, snapshot, accessors)
//   rangesvd::StoreSnapshot          store.hpp:135-156
//   rangesvd::TimeRange::resolve     query.hpp:34-51
//   rangesvd::trim_block             query.hpp:64-89
//   rangesvd::stitch                 query.hpp:150-157
//   rangesvd::range_query (3 forms)  query.hpp:163-201
//   errors                           errors.hpp:9-68
//
// Additions: a FIXED_RANK truncation policy (BASELINE configs), device
// selection, and bulk append of many rows in one call.
#pragma once

#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <memory>
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
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return data_.size(); }
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

class StoreSnapshot {
public:
    std::size_t block_size = 0, num_columns = 0, total_rows = 0, sealed_count = 0, open_rows = 0;
    double energy_threshold = 1.0;
    std::size_t block_count() const { return sealed_count + (open_rows ? 1 : 0); }
    std::size_t block_rows(std::size_t i) const { return i < sealed_count ? block_size : open_rows; }
    zsvd_snapshot* handle() const { return h_.get(); }

private:
    friend class BlockStore;
    struct Del {
        void operator()(zsvd_snapshot* s) const { zsvd_snapshot_release(s); }
    };
    std::shared_ptr<zsvd_snapshot> h_;
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
        return snap;
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
