// The planner: reduces any of the 128 storage/computation datatype
// combinations to one real product over packed panels.  Host-only; the
// decisions are those of the reference (dispatch.cpp:11-305), re-expressed
// here as a few small decision functions.
#include "mdgemm/mdgemm.hpp"

namespace mdgemm {

CaseId classify_case(Domain c, Domain a, Domain b) {
  // Index by (C complex, A complex, B complex) -> case (dispatch.cpp:11-31).
  static const CaseId table[8] = {
      CaseId::C0,   // r r r
      CaseId::C1b,  // r r c
      CaseId::C1a,  // r c r
      CaseId::C2ab, // r c c
      CaseId::C1c,  // c r r
      CaseId::C2bc, // c r c
      CaseId::C2ac, // c c r
      CaseId::C3,   // c c c
  };
  const int idx = (c == Domain::Complex ? 4 : 0) | (a == Domain::Complex ? 2 : 0) |
                  (b == Domain::Complex ? 1 : 0);
  return table[idx];
}

Precision resolve_comp_precision(const MatrixView& c) { return c.comp_prec; }

std::uint64_t flops_of_case(CaseId id, std::int64_t m, std::int64_t n, std::int64_t k) {
  // 2/4/8 mnk by how many components take part (dispatch.cpp:35-54).
  std::uint64_t factor = 2;
  if (id == CaseId::C2ab || id == CaseId::C2ac || id == CaseId::C2bc) factor = 4;
  if (id == CaseId::C3) factor = 8;
  return factor * static_cast<std::uint64_t>(m) * static_cast<std::uint64_t>(n) *
         static_cast<std::uint64_t>(k);
}

namespace {

// Cases whose update touches only real data project beta to real.
bool beta_is_projected(CaseId id) {
  return id == CaseId::C0 || id == CaseId::C1a || id == CaseId::C1b || id == CaseId::C1c ||
         id == CaseId::C2ab;
}

CaseId mirrored(CaseId id) {
  switch (id) {
    case CaseId::C1a: return CaseId::C1b;
    case CaseId::C1b: return CaseId::C1a;
    case CaseId::C2ac: return CaseId::C2bc;
    case CaseId::C2bc: return CaseId::C2ac;
    default: return id;
  }
}

// Operation transposition (dispatch.cpp:126-143): run C' = B' A' when that
// puts the output in the microkernel's preferred orientation.
bool wants_flip(CaseId id, Preference pref, const MatrixView& c) {
  if (id == CaseId::C1c) return false;
  if (id == CaseId::C2ac) return pref == Preference::Row;
  if (id == CaseId::C2bc) return pref == Preference::Column;
  const StorageKind sk = storage_kind(c);
  return pref == Preference::Column ? sk == StorageKind::RowStored : sk == StorageKind::ColumnStored;
}

}  // namespace

std::pair<Scalar, Scalar> apply_scalar_policy(Scalar alpha, Scalar beta, CaseId id,
                                              Precision comp_prec, Precision c_storage_prec) {
  Scalar a;
  if (id == CaseId::C3) {
    a = typecast_scalar(alpha, Datatype{alpha.dtype.domain, comp_prec});
  } else {
    if (id != CaseId::C0 && alpha.im != 0.0)
      throw ScalarPolicyError(std::string("case ") + to_string(id) +
                              " does not support alpha with a nonzero imaginary part");
    a = project_scalar(alpha, comp_prec);
  }
  const Scalar b = beta_is_projected(id)
                       ? project_scalar(beta, c_storage_prec)
                       : typecast_scalar(beta, Datatype{beta.dtype.domain, c_storage_prec});
  return {a, b};
}

ExecutionPlan plan(Scalar alpha, const MatrixView& a, const MatrixView& b, Scalar beta,
                   const MatrixView& c, const Config& cfg) {
  cfg.validate();
  if (a.m != c.m || b.n != c.n || a.n != b.m)
    throw Error("gemm: dimension mismatch: C is " + std::to_string(c.m) + "x" +
                std::to_string(c.n) + ", A is " + std::to_string(a.m) + "x" + std::to_string(a.n) +
                ", B is " + std::to_string(b.m) + "x" + std::to_string(b.n));

  const Precision comp = resolve_comp_precision(c);
  const CaseId given = classify_case(c.dtype.domain, a.dtype.domain, b.dtype.domain);
  const auto [alpha_e, beta_e] = apply_scalar_policy(alpha, beta, given, comp, c.dtype.precision);
  const Preference pref = cfg.preference;
  const bool col_pref = pref == Preference::Column;

  ExecutionPlan p;
  p.logical_transpose = wants_flip(given, pref, c);
  const bool flip = p.logical_transpose;
  const MatrixView A = flip ? induced_transpose(b) : a;
  const MatrixView B = flip ? induced_transpose(a) : b;
  const MatrixView C = flip ? induced_transpose(c) : c;
  p.case_id = flip ? mirrored(given) : given;
  p.comp_prec = comp;
  p.params = cfg.blocking(comp);
  p.ukr = cfg.ukr(comp);
  p.alpha = alpha_e;
  p.beta = beta_e;

  const CaseId id = p.case_id;
  const std::int64_t m = C.m, n = C.n, k = A.n;
  MatrixView ea = A, eb = B, ec = C;
  std::int64_t me = m, ne = n, ke = k;
  PairAxis pair = PairAxis::None;

  // Per-case reduction to real panels (dispatch.cpp:167-211).
  switch (id) {
    case CaseId::C0:
      break;
    case CaseId::C1a:
      ea = real_projection(A, Part::Re);
      break;
    case CaseId::C1b:
      eb = real_projection(B, Part::Re);
      break;
    case CaseId::C1c:
      ec = real_projection(C, Part::Re);
      break;
    case CaseId::C2ab:  // Re(A conj(B)) along a doubled inner dimension
      p.format_a = p.format_b = PackFormat::OneR;
      p.conj_b = true;
      ke = 2 * k;
      break;
    case CaseId::C2ac:
      pair = PairAxis::Rows;
      me = 2 * m;
      break;
    case CaseId::C2bc:
      pair = PairAxis::Cols;
      ne = 2 * n;
      break;
    case CaseId::C3:  // 1m: 1e on the alpha-carrying side, 1r on the other
      p.format_a = col_pref ? PackFormat::OneE : PackFormat::OneR;
      p.format_b = col_pref ? PackFormat::OneR : PackFormat::OneE;
      pair = col_pref ? PairAxis::Rows : PairAxis::Cols;
      (col_pref ? me : ne) *= 2;
      ke = 2 * k;
      break;
  }

  p.target_dtype_a = Datatype{ea.dtype.domain, comp};
  p.target_dtype_b = Datatype{eb.dtype.domain, comp};
  // A complex operand packed Standard counts panel rows in complex elements.
  const bool a_halves = p.format_a == PackFormat::Standard && ea.dtype.domain == Domain::Complex;
  const bool b_halves = p.format_b == PackFormat::Standard && eb.dtype.domain == Domain::Complex;
  p.reg_block_a = a_halves ? p.ukr.mr / 2 : p.ukr.mr;
  p.reg_block_b = b_halves ? p.ukr.nr / 2 : p.ukr.nr;

  // Alpha rides with exactly one packed operand (dispatch.cpp:229-235).
  const Scalar unit = Scalar::real_value(1.0, comp);
  const bool alpha_on_b = id == CaseId::C3 && !col_pref;
  p.pack_scale_a = alpha_on_b ? unit : alpha_e;
  p.pack_scale_b = alpha_on_b ? alpha_e : unit;

  p.macro_mode = comp != c.dtype.precision ? MacroMode::AccumulateTypecast : MacroMode::Standard;

  // Output path: first match wins (dispatch.cpp:245-266).
  bool flattened = false;
  UkrPath path = UkrPath::Direct;
  if (id == CaseId::C3) {
    path = col_pref ? UkrPath::OneMColumn : UkrPath::OneMRow;
  } else if (p.macro_mode == MacroMode::AccumulateTypecast || id == CaseId::C1c) {
    path = UkrPath::Temp;
  } else if (id == CaseId::C2ac || id == CaseId::C2bc) {
    const FlattenAxis ax = id == CaseId::C2ac ? FlattenAxis::Rows : FlattenAxis::Cols;
    flattened = can_flatten(ec, ax);
    if (flattened && beta_e.im == 0.0) {
      ec = real_flatten(ec, ax);
      pair = PairAxis::None;
    } else {
      path = UkrPath::Temp;
    }
  }

  // Intermediate output buffer (dispatch.cpp:273-294).
  bool unreachable_image = false;
  if (id == CaseId::C2ac || id == CaseId::C2bc) unreachable_image = !flattened;
  if (id == CaseId::C3) unreachable_image = !can_flatten(ec, col_pref ? FlattenAxis::Rows : FlattenAxis::Cols);
  const bool triggered = p.macro_mode == MacroMode::AccumulateTypecast ||
                         (id == CaseId::C1c && k > p.params.kc) || unreachable_image;
  const bool gate_open = cfg.ctemp == CTempMode::On || (cfg.ctemp == CTempMode::Auto && p.params.threads == 1);
  if (triggered && gate_open) {
    CTempDescriptor ct;
    ct.rows = me;
    ct.cols = ne;
    ct.precision = comp;
    ct.mode = beta_e.is_zero() ? CTempDescriptor::Mode::CopyBack : CTempDescriptor::Mode::AccumulateBack;
    p.ctemp = ct;
  }

  p.a = ea;
  p.b = eb;
  p.c = ec;
  p.m = me;
  p.n = ne;
  p.k = ke;
  p.ukr_path = path;
  p.pair_axis = pair;
  return p;
}

}  // namespace mdgemm
