// mdgemm.hpp -- C++ API of the B200-native mixed-datatype gemm.
//
// Source-compatible with the reference engine's public headers
// (/root/reference/proj/include/mdgemm/{dtypes,kernels,packing,config,
// dispatch,case_label}.hpp): the same namespace, type names, enumerators,
// member names and function signatures, so code written against the
// reference recompiles unchanged.  What differs is underneath: MatrixView
// bases may be device pointers (or host pointers, which gemm() stages through
// HBM), and gemm() executes on an sm_100a GPU through the C ABI in
// include/mdgemm_b200.h.  The per-file forwarding headers in this directory
// keep the reference's include paths working.
#pragma once

#include <complex>
#include <cstddef>
#include <memory>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mdgemm {

// ------------------------------------------------------------------ errors
// dtypes.hpp:14-20.  ScalarPolicyError marks an alpha the case cannot honor.
struct Error : std::runtime_error {
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
struct ScalarPolicyError : Error {
  explicit ScalarPolicyError(const std::string& what) : Error(what) {}
};

// --------------------------------------------------------------- datatypes
enum class Domain : std::uint8_t { Real, Complex };
enum class Precision : std::uint8_t { Single, Double };

// Unit roundoff 2^-24 / 2^-53 (dtypes.hpp:25-28).
constexpr double eps_of(Precision p) { return p == Precision::Double ? 0x1p-53 : 0x1p-24; }
constexpr std::size_t real_size(Precision p) { return p == Precision::Double ? 8u : 4u; }

struct Datatype {
  Domain domain = Domain::Real;
  Precision precision = Precision::Double;
  friend constexpr bool operator==(Datatype x, Datatype y) {
    return x.domain == y.domain && x.precision == y.precision;
  }
  friend constexpr bool operator!=(Datatype x, Datatype y) { return !(x == y); }
};

inline constexpr Datatype dt_s{Domain::Real, Precision::Single};
inline constexpr Datatype dt_d{Domain::Real, Precision::Double};
inline constexpr Datatype dt_c{Domain::Complex, Precision::Single};
inline constexpr Datatype dt_z{Domain::Complex, Precision::Double};

constexpr std::size_t dtype_size(Datatype t) {
  return (t.domain == Domain::Complex ? 2u : 1u) * real_size(t.precision);
}

char dtype_letter(Datatype t);
Datatype dtype_from_letter(char ch);
char precision_letter(Precision p);
Precision precision_from_letter(char ch);
std::string to_string(Datatype t);

enum class CaseId : std::uint8_t { C0, C1a, C1b, C1c, C2ab, C2ac, C2bc, C3 };
const char* to_string(CaseId c);

// ------------------------------------------------------------------ scalars
// Payload in double, exactly representable in the scalar's precision.
struct Scalar {
  double re = 0.0;
  double im = 0.0;
  Datatype dtype = dt_d;

  bool is_real() const { return dtype.domain == Domain::Real; }
  bool is_zero() const { return re == 0.0 && im == 0.0; }
  bool is_one() const { return re == 1.0 && im == 0.0; }
  std::complex<double> value() const { return {re, im}; }

  static Scalar real_value(double v, Precision p = Precision::Double);
  static Scalar complex_value(double r, double i, Precision p = Precision::Double);
};

Scalar typecast_scalar(Scalar s, Datatype target);
Scalar project_scalar(Scalar s, Precision p);

// ------------------------------------------------------------------- views
enum class Part : std::uint8_t { Re, Im };
enum class FlattenAxis : std::uint8_t { Rows, Cols };
enum class StorageKind : std::uint8_t { ColumnStored, RowStored, GeneralStored };

struct MatrixView {
  std::byte* base = nullptr;
  std::int64_t m = 0;
  std::int64_t n = 0;
  std::int64_t rs = 0;
  std::int64_t cs = 0;
  Datatype dtype = dt_d;
  bool conj = false;
  Precision comp_prec = Precision::Double;
  Datatype target_dtype = dt_d;

  static MatrixView make(void* base, std::int64_t m, std::int64_t n, std::int64_t rs,
                         std::int64_t cs, Datatype dtype);

  std::byte* elem_ptr(std::int64_t i, std::int64_t j) const {
    return base + static_cast<std::size_t>(i * rs + j * cs) * dtype_size(dtype);
  }
  MatrixView with_conj(bool c) const {
    MatrixView v = *this;
    v.conj = c;
    return v;
  }
  MatrixView with_comp_prec(Precision p) const {
    MatrixView v = *this;
    v.comp_prec = p;
    return v;
  }
};

MatrixView induced_transpose(MatrixView v);
MatrixView real_projection(MatrixView v, Part part);
bool can_flatten(const MatrixView& v, FlattenAxis axis);
MatrixView real_flatten(MatrixView v, FlattenAxis axis);
MatrixView slice(MatrixView v, std::int64_t i0, std::int64_t j0, std::int64_t mm,
                 std::int64_t nn);
StorageKind storage_kind(const MatrixView& v);

// Host-memory element access (the views must hold host pointers).
std::complex<double> load_elem(const MatrixView& v, std::int64_t i, std::int64_t j);
void store_elem(const MatrixView& v, std::int64_t i, std::int64_t j, std::complex<double> value);

std::pair<const std::byte*, const std::byte*> byte_range(const MatrixView& v);
bool ranges_overlap(const MatrixView& a, const MatrixView& b);

// ------------------------------------------------------ microkernel metadata
enum class Preference : std::uint8_t { Column, Row };
enum class PairAxis : std::uint8_t { None, Rows, Cols };
enum class OneMVariant : std::uint8_t { Column, Row };

struct UkrDescriptor {
  Precision precision = Precision::Double;
  int mr = 4;
  int nr = 4;
  Preference preference = Preference::Column;
};

inline constexpr int kMaxUkrDim = 32;

class FlopCounter {
 public:
  void add(std::uint64_t n) { flops_ += n; }
  void merge(const FlopCounter& other) { flops_ += other.flops_; }
  void reset() { flops_ = 0; }
  std::uint64_t value() const { return flops_; }

 private:
  std::uint64_t flops_ = 0;
};

// ------------------------------------------------------------------ packing
enum class PackFormat : std::uint8_t { Standard, OneE, OneR };
enum class Side : std::uint8_t { Left, Right };

// Bytes of the packed block (packing.hpp:101-102).
std::size_t packed_bytes(const MatrixView& src, Side side, PackFormat format, Datatype target,
                         std::int64_t reg_block);

// Device pack: typecast/conj/scale/format `src` (device memory) into `dst`
// (device memory, packed_bytes() long) in the reference's panel layout.
// B200 counterpart of pack_block_into (packing.hpp:118-120).
void pack_block_device(void* dst, const MatrixView& src, Side side, PackFormat format, bool conj,
                       Scalar scale, Datatype target, std::int64_t reg_block,
                       void* stream = nullptr);

// The reference's pack seam (packing.hpp:27-130) on the device.  A packed
// operand block: zero-padded register panels over one dimension, contiguous
// along the other; the packed logical matrix is the operand after format
// expansion.  The panels are produced by the sm_100a pack kernels (byte for
// byte the reference's pack); `storage` may be host or device memory, the
// source view too (host sources are staged through HBM).  Synchronous.
class PackedBlock {
 public:
  PackedBlock() = default;
  PackedBlock(const PackedBlock&) = delete;
  PackedBlock& operator=(const PackedBlock&) = delete;
  PackedBlock(PackedBlock&&) = default;
  PackedBlock& operator=(PackedBlock&&) = default;

  std::span<const std::byte> buf() const { return buf_; }
  Datatype dtype() const { return dtype_; }
  PackFormat format() const { return format_; }
  Side side() const { return side_; }
  // panel geometry in packed-logical units (complex elements for a
  // Standard-packed complex operand, real elements otherwise)
  std::int64_t panel_dim() const { return panel_dim_; }
  std::int64_t panels() const { return panels_; }
  std::int64_t panel_len() const { return panel_len_; }
  std::int64_t logical_rows() const { return logical_rows_; }
  std::int64_t logical_cols() const { return logical_cols_; }
  std::int64_t padded_rows() const { return side_ == Side::Left ? panels_ * panel_dim_ : logical_rows_; }
  std::int64_t padded_cols() const { return side_ == Side::Right ? panels_ * panel_dim_ : logical_cols_; }
  // element (i, j) of the zero-padded packed logical matrix
  std::complex<double> packed_element(std::int64_t i, std::int64_t j) const;
  // as real register panels: a Standard-packed complex block doubles its panel dimension
  std::int64_t kernel_panel_dim() const { return panel_dim_ * (dtype_.domain == Domain::Complex ? 2 : 1); }
  std::int64_t kernel_panel_len() const { return panel_len_; }
  Precision kernel_precision() const { return dtype_.precision; }
  const std::byte* panel_ptr(std::int64_t p) const { return buf_.data() + static_cast<std::size_t>(p) * panel_bytes(); }
  std::size_t panel_bytes() const { return static_cast<std::size_t>(panel_dim_ * panel_len_) * dtype_size(dtype_); }

 private:
  friend PackedBlock pack_block_panels(std::span<std::byte>, const MatrixView&, Side, PackFormat, bool, Scalar,
                                       Datatype, std::int64_t, std::int64_t, std::int64_t);
  friend PackedBlock pack_block(const MatrixView&, Side, PackFormat, bool, Scalar, Datatype, std::int64_t);
  std::span<std::byte> buf_;
  std::vector<std::byte> owned_;
  Datatype dtype_ = dt_d;
  PackFormat format_ = PackFormat::Standard;
  Side side_ = Side::Left;
  std::int64_t panel_dim_ = 0, panels_ = 0, panel_len_ = 0, logical_rows_ = 0, logical_cols_ = 0;
};

// packing.hpp:101-130: pack into a fresh host buffer / into caller storage /
// only panels [panel_begin, panel_end) of it (other panels' bytes untouched).
PackedBlock pack_block(const MatrixView& src, Side side, PackFormat format, bool conj, Scalar scale, Datatype target,
                       std::int64_t reg_block);
PackedBlock pack_block_into(std::span<std::byte> storage, const MatrixView& src, Side side, PackFormat format,
                            bool conj, Scalar scale, Datatype target, std::int64_t reg_block);
PackedBlock pack_block_panels(std::span<std::byte> storage, const MatrixView& src, Side side, PackFormat format,
                              bool conj, Scalar scale, Datatype target, std::int64_t reg_block,
                              std::int64_t panel_begin, std::int64_t panel_end);

// ------------------------------------------------------------------- config
struct BlockingParams {
  std::int64_t mc = 0;
  std::int64_t nc = 0;
  std::int64_t kc = 0;
  int mr = 0;
  int nr = 0;
  int threads = 1;
};

enum class CTempMode : std::uint8_t { Auto, On, Off };

// B200 extension: which device arithmetic gemm() uses (see mdgemm_b200.h).
enum class Numerics : std::uint8_t { Fast, Exact };
// The default of Config::numerics: FAST, or the environment's
// MDGEMM_GPU_NUMERICS (fast | exact) -- so code that never touches the key
// (the reference's own tests, built against this header) can run either
// arithmetic.
Numerics default_numerics();

struct Config {
  BlockingParams single_params{128, 1024, 256, 8, 8, 1};
  BlockingParams double_params{64, 512, 128, 4, 4, 1};
  int threads = 1;
  Preference preference = Preference::Column;
  CTempMode ctemp = CTempMode::Auto;
  Numerics numerics = default_numerics();
  // B200 extension (gpu.splitk = auto | off): FAST calls whose tile grid
  // fills less than half of the GPU may split the inner dimension over
  // several CTAs (deterministic, but a different summation order than the
  // unsplit grid); off keeps every FAST result bitwise independent of the
  // grid, sharding and batching.
  bool splitk = true;

  static Config defaults() { return Config{}; }
  static Config load(const std::optional<std::string>& file = std::nullopt, bool apply_env = true);
  void set(const std::string& key, const std::string& value);
  void validate() const;

  BlockingParams blocking(Precision p) const {
    BlockingParams bp = p == Precision::Double ? double_params : single_params;
    bp.threads = threads;
    return bp;
  }
  UkrDescriptor ukr(Precision p) const {
    const BlockingParams& bp = p == Precision::Double ? double_params : single_params;
    return UkrDescriptor{p, bp.mr, bp.nr, preference};
  }
  std::string describe() const;
};

// ----------------------------------------------------------------- dispatch
CaseId classify_case(Domain c, Domain a, Domain b);
Precision resolve_comp_precision(const MatrixView& c);
std::uint64_t flops_of_case(CaseId case_id, std::int64_t m, std::int64_t n, std::int64_t k);
std::pair<Scalar, Scalar> apply_scalar_policy(Scalar alpha, Scalar beta, CaseId case_id,
                                              Precision comp_prec, Precision c_storage_prec);

enum class UkrPath : std::uint8_t { Direct, Temp, OneMColumn, OneMRow };
enum class MacroMode : std::uint8_t { Standard, AccumulateTypecast };

struct CTempDescriptor {
  std::int64_t rows = 0;
  std::int64_t cols = 0;
  Precision precision = Precision::Double;
  enum class Mode : std::uint8_t { CopyBack, AccumulateBack } mode = Mode::AccumulateBack;
};

struct ExecutionPlan {
  CaseId case_id = CaseId::C0;
  bool logical_transpose = false;
  Precision comp_prec = Precision::Double;
  std::int64_t m = 0, n = 0, k = 0;

  MatrixView a, b, c;
  PackFormat format_a = PackFormat::Standard;
  PackFormat format_b = PackFormat::Standard;
  bool conj_a = false;
  bool conj_b = false;
  Datatype target_dtype_a = dt_d;
  Datatype target_dtype_b = dt_d;
  std::int64_t reg_block_a = 0;
  std::int64_t reg_block_b = 0;

  Scalar alpha{};
  Scalar beta{};
  Scalar pack_scale_a{1.0, 0.0, dt_d};
  Scalar pack_scale_b{1.0, 0.0, dt_d};

  MacroMode macro_mode = MacroMode::Standard;
  UkrPath ukr_path = UkrPath::Direct;
  PairAxis pair_axis = PairAxis::None;
  std::optional<CTempDescriptor> ctemp;

  BlockingParams params{};
  UkrDescriptor ukr{};
};

ExecutionPlan plan(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta,
                   const MatrixView& c, const Config& cfg);

// C := alpha*op(A,B) + beta*C on the GPU (dispatch.hpp:89-91).  Synchronous.
void gemm(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta,
          const MatrixView& c, const Config& cfg = Config::defaults(), FlopCounter* fc = nullptr);

// A list of gemm() calls, equivalent to calling gemm() on each in order.
// Host operand windows are copied into HBM once per batch and stay resident
// (calls sharing an operand reuse the device copy; a host C goes back once,
// after its last writer); copies overlap the kernels of neighbouring calls,
// and calls touching disjoint memory run concurrently.  Synchronous.  B200
// extension.
struct GemmCall {
  Scalar alpha;
  MatrixView a, b;
  Scalar beta;
  MatrixView c;
};
void gemm_batch(const std::vector<GemmCall>& calls, const Config& cfg = Config::defaults(),
                FlopCounter* fc = nullptr);
// Same, forked from and joined back into `stream` (a cudaStream_t) without
// synchronising; host operands must stay valid until the stream completes.
void gemm_batch_async(const std::vector<GemmCall>& calls, const Config& cfg, void* stream,
                      FlopCounter* fc = nullptr);

// Bytes the batch runner has copied host->device and device->host so far
// (process-wide counters).
void staging_bytes(uint64_t* h2d, uint64_t* d2h);

// Device-pointer variant ordered on `stream` (a cudaStream_t); returns
// without synchronising.
void gemm_async(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta,
                const MatrixView& c, const Config& cfg, void* stream, FlopCounter* fc = nullptr);

// Runs an already-built plan on device operands (the boundary the reference's
// dispatch.cpp:359-388 crosses).
void execute(const ExecutionPlan& p, Numerics numerics, void* stream, FlopCounter* fc = nullptr,
             bool allow_splitk = true);

// ------------------------------------------------------------ multi-GPU
// C and B split into column panels, A broadcast once over
// NVLink / NVSwitch (NCCL, loaded at run time), no reduction.

// Columns [*j0, *j0 + *nb) of n owned by `rank` of `world`: equal panels,
// multiples of `align` columns, the last one shorter (or empty).
void shard_columns(std::int64_t n, int world, int rank, std::int64_t align, std::int64_t* j0, std::int64_t* nb);

// A communicator of one process per GPU (NCCL, on the current device).
struct CommId {
  unsigned char bytes[128];
};
class Communicator {
 public:
  static CommId unique_id();                          // on one rank; share it with the others
  Communicator(const CommId& id, int nranks, int rank);  // collective over the ranks
  ~Communicator();
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  int size() const;
  int rank() const;
  int device() const;
  struct Impl;

 private:
  std::unique_ptr<Impl> impl_;
  friend void gemm_sharded(Communicator&, int, Scalar, const MatrixView&, const MatrixView&, Scalar,
                           const MatrixView&, const Config&, void*, FlopCounter*);
};

// This rank's column panel of C := beta*C + alpha*A*B: `a` is the root's A
// (on other ranks the same geometry; base null = the library receives it),
// b_panel / c_panel this rank's device column panels (shard_columns).  A
// goes to every rank by broadcast while each rank packs its B panel.
// Ordered on `stream` (a cudaStream_t), no host synchronisation.  A shard
// never takes split-K.
void gemm_sharded(Communicator& comm, int root, Scalar alpha, const MatrixView& a, const MatrixView& b_panel,
                  Scalar beta, const MatrixView& c_panel, const Config& cfg = Config::defaults(),
                  void* stream = nullptr, FlopCounter* fc = nullptr);

// The whole call over several GPUs of this process: A, B, C anywhere (host
// or device memory); column panels of B and C go to `devices`, A is
// broadcast from the first one, C panels come back.  Synchronous.
void gemm_multi(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta, const MatrixView& c,
                const Config& cfg, const std::vector<int>& devices, FlopCounter* fc = nullptr);

// --------------------------------------------------------------- case labels
struct CaseLabel {
  Datatype c = dt_d;
  Datatype a = dt_d;
  Datatype b = dt_d;
  Precision comp = Precision::Double;

  CaseId case_id() const { return classify_case(c.domain, a.domain, b.domain); }
  std::string str() const;
  static CaseLabel parse(const std::string& s);
  static std::vector<CaseLabel> all();
};

}  // namespace mdgemm
