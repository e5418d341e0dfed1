// zsvd_internal.h — host/device shared descriptors of the B200 Zoom-SVD engine.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

namespace zsvd {

// Reference constants (kept identical): svd.hpp:22, svd.hpp:25.
constexpr double kNumericalRankCutoff = 1e-12;
constexpr double kOrthonormalityTol = 1e-10;

// Widest matrix side (after transposing wide inputs) the smem engine handles.
constexpr int kQMax = 64;
constexpr int kEngineThreads = 256;

enum TruncKind : int32_t { TRUNC_NONE = -1, TRUNC_ENERGY = 0, TRUNC_FIXED = 1 };

struct Trunc {
    int32_t kind;
    int32_t k;
    double xi;
};

// Per-task status codes written by the engine.
enum TaskStatus : int32_t {
    TASK_OK = 0,
    TASK_NEEDS_FALLBACK = 1,  // CholeskyQR2 rejected (ill-conditioned / rank-deficient)
    TASK_DONE_FALLBACK = 2,
    TASK_UNSUPPORTED = 3,     // q > kQMax
    TASK_CAPACITY = 4,        // resulting rank exceeds the output capacity
};

// One thin SVD problem A (m x n) -> U (m x k), sigma (k), V (nv x k).
// A(i, j) = a[i * lda + j] * (colscale ? colscale[j] : 1).
// n (and m) may be read from device memory at run time (trim of a slot whose
// rank lives in the slot header; stitch whose stack height is data dependent).
struct SvdTask {
    const double* a;
    int64_t lda;
    const double* colscale;
    const double* n_from;   // if non-null: n = (int)n_from[0]
    const int32_t* m_from;  // if non-null: m = m_from[0]
    int32_t m, n;

    double* u;
    int64_t ldu;
    double* s;
    double* v;
    int64_t ldv;
    double* k_out;          // rank written as a double (slot-header convention)
    int32_t kcap;           // columns available in u / s / v

    // Epilogue: V_final = vpre (nvpre x n, row-major, ldvpre) * V_inner (trim).
    const double* vpre;
    int64_t ldvpre;
    int32_t nvpre;

    Trunc trunc;
    int32_t sign;           // apply canonical_sign to the output
    int32_t qr_only;        // factor A = Q R only: U = Q, sigma = 1, V = vpre diag(vscale) R^T
                            // (no SVD): a no-op truncation's trim in stack form (mid2_body)
    const double* vscale;   // qr_only: the trim's sigma, applied to vpre's columns instead of
                            // to A (the fallback re-applies it to A as colscale)
    int32_t gram_only;      // the task's Gram partials come from gram_parts_kernel (no data
                            // rows): mid-1 flags a second CholeskyQR pass as a fallback
    int32_t direct;         // set by the eigen phase (svd_engine.cu eig_body): mid-2 starts its Jacobi
                            // from the Gram's leading eigenvectors (X in the stage area)
    int32_t status;         // TaskStatus, written by the engine
    int32_t sweeps;         // Jacobi sweeps used (diagnostics)
    int32_t reason;         // why the fast path was rejected (diagnostics)
    int32_t krank;          // rank chosen by the mid-2 phase
    int32_t onepass;        // set by mid-1: R1 is accurate enough, skip the second QR pass
    int32_t nsplit;         // row splits of the pass kernels
    int32_t rows_per_split; // multiple of 32
    double* ws;             // per-task workspace (workspace_doubles(nsplit))
    int32_t* nonfinite;     // if non-null: mid-1 sets it to 1 when a diagonal entry of the
                            // Gram is not finite (storage: the input held NaN / Inf)
    int64_t clk[8];         // phase timestamps, clock64 (diagnostics)
};

// Narrow-engine task workspace (svd_engine.cu phases): nsplit partial Q x Q
// Grams (row-major, ld kQMax), R1, the inverted diagonal blocks, M (U = W M),
// sigma, a stage area.  gram_stitch.cu writes the partials and reads M / sigma.
constexpr int kWsQ2 = kQMax * kQMax;
__host__ __device__ constexpr int64_t ws_off_r1(int nsplit) { return (int64_t)nsplit * kWsQ2; }
__host__ __device__ constexpr int64_t ws_off_dinv(int nsplit) { return ws_off_r1(nsplit) + kWsQ2; }
__host__ __device__ constexpr int64_t ws_off_m(int nsplit) { return ws_off_dinv(nsplit) + 16 * kQMax; }
__host__ __device__ constexpr int64_t ws_off_sig(int nsplit) { return ws_off_m(nsplit) + kWsQ2; }
__host__ __device__ constexpr int64_t ws_off_stage(int nsplit) { return ws_off_sig(nsplit) + kQMax; }
__host__ __device__ constexpr int64_t ws_total(int nsplit) { return ws_off_stage(nsplit) + kWsQ2; }

// One part of a Gram stitch (gram_stitch.cu): a stored block's factors, or a
// row slice of them (the head / tail of a range, whose rows enter the Gram
// through C = U_s^T U_s instead of a trim SVD).
struct GramPart {
    const double* u;       // first U row of the part (ld ldu)
    const double* s;       // sigma
    const double* v;       // V (c x rank, ld ldv)
    const double* k_from;  // rank (double), device
    int64_t ldu, ldv;
    int64_t rows;          // rows of the part in the answer
    int32_t slice;         // 1: row slice (head / tail)
    int32_t pad;
};
struct GramItem {           // work item of gram_parts_kernel
    int32_t part;
    int32_t row0, nrows;    // slice rows [row0, row0 + nrows) of the part (slices only)
    int32_t pad;
};

// Launch geometry of the wide path (wide_engine.cu): every task of a batch has
// p <= p_bound rows and q <= q_bound columns after transposing; nsplit = row
// splits of the Gram kernels.
struct WParams {
    int32_t p_bound;
    int32_t q_bound;
    int32_t nsplit;
    int32_t pad;  // max inner sweeps of a pair solve (0: until converged)
    double tol1;  // pass-1 relative rotation threshold
};

// Sealed-block slot layout inside the store arena (doubles):
//   [0] rank k (as double) | sigma[kcap] | V (c x kcap) | U (b x kcap)
struct SlotLayout {
    int64_t stride;
    int64_t off_s, off_v, off_u;
    int32_t b, c, kcap;
};

// One part of a stitched query (query.hpp:95-144): U (rows x k, ld), sigma, V (c x k, ld).
struct PartDesc {
    const double* u;
    const double* s;
    const double* v;
    const double* k_from;   // rank (double) in device memory
    int64_t ldu, ldv;
    int64_t rows;
};

// One item of the similarity reduction of similar_range_search (analysis.hpp:
// 89-103): a part of a stitched window (its rows of the window's leading left
// singular vector are U_p * U_inner[band, 0]) or a single-block window (the
// column 0 of its trim's U).
struct SimItem {
    const double* u;       // U rows of the item (ld ldu)
    int64_t ldu;
    const double* w;       // U_inner (ld ldw), or null for single-block windows
    int64_t ldw;
    const int32_t* band;   // band offset of the part in U_inner, or null
    const double* k_from;  // rank of the part / trim
    int64_t rows;          // rows of the item
    int64_t row0;          // first row of the item within the window
};

// Programmatic dependent launch: kernels of the engine / query chains are
// launched with programmatic stream serialisation and wait here, before any
// global-memory access, for the previous kernel's completion and memory flush
// (only its launch and block scheduling overlap; a no-op for ordinary launches).
#define ZSVD_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

// Host helpers defined in zsvd_api.cu, shared by csv_ingest.cu.
int set_error(int code, const std::string& msg, size_t line = 0);  // returns code
void count_launches(uint64_t n);
int ensure_device(int dev);

}  // namespace zsvd
