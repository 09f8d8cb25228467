// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).
//
// A C-ABI wrapper around the reference CPU engine compiled from its own
// sources under /root/reference/proj/src (see oracle/Makefile, which builds
// them with -Dmdgemm=mdgemm_ref so the reference's namespace cannot collide
// with anything else).  The result, oracle/_ref/libmdgemm_ref.so, is used by
// tests/ to pin the C restatement in oracle/mdg_oracle.c and by bench.py's
// CPU-baseline / --impl reference legs.  It is never linked into the product.
//
// Every function takes the same plain-data structs the product ABI uses
// (include/mdgemm_b200.h) with HOST pointers.
#include "mdgemm/bench.hpp"
#include "mdgemm/case_label.hpp"
#include "mdgemm/config.hpp"
#include "mdgemm/dispatch.hpp"
#include "mdgemm/matrix.hpp"
#include "mdgemm/oracle.hpp"
#include "mdgemm/packing.hpp"
#include "mdgemm/rng.hpp"

#include "mdgemm_b200.h"

#include <cstring>
#include <exception>
#include <string>
#include <vector>

using namespace mdgemm;  // expands to mdgemm_ref under -Dmdgemm=mdgemm_ref

namespace {

thread_local std::string g_err;

Datatype dt_of(int32_t code) {
  switch (code) {
    case MDG_DT_S: return dt_s;
    case MDG_DT_D: return dt_d;
    case MDG_DT_C: return dt_c;
    case MDG_DT_Z: return dt_z;
  }
  throw Error("ref_shim: bad datatype code " + std::to_string(code));
}

int32_t code_of(Datatype t) {
  if (t.domain == Domain::Real) return t.precision == Precision::Single ? MDG_DT_S : MDG_DT_D;
  return t.precision == Precision::Single ? MDG_DT_C : MDG_DT_Z;
}

Precision prec_of(int32_t p) { return p == MDG_PREC_SINGLE ? Precision::Single : Precision::Double; }
int32_t pcode(Precision p) { return p == Precision::Single ? MDG_PREC_SINGLE : MDG_PREC_DOUBLE; }

MatrixView view_in(const mdg_view_t* v) {
  MatrixView out = MatrixView::make(v->base, v->m, v->n, v->rs, v->cs, dt_of(v->dtype));
  out.conj = v->conj != 0;
  out.comp_prec = prec_of(v->comp_prec);
  return out;
}

mdg_view_t view_out(const MatrixView& v) {
  mdg_view_t o{};
  o.base = v.base;
  o.m = v.m; o.n = v.n; o.rs = v.rs; o.cs = v.cs;
  o.dtype = code_of(v.dtype);
  o.conj = v.conj;
  o.comp_prec = pcode(v.comp_prec);
  o.target_dtype = code_of(v.target_dtype);
  return o;
}

Scalar scalar_in(mdg_scalar_t s) { return Scalar{s.re, s.im, dt_of(s.dtype)}; }
mdg_scalar_t scalar_out(const Scalar& s) {
  mdg_scalar_t o{};
  o.re = s.re; o.im = s.im; o.dtype = code_of(s.dtype);
  return o;
}

Config config_in(const mdg_config_t* c) {
  Config cfg;
  if (!c) return cfg;
  cfg.single_params = BlockingParams{c->single_params.mc, c->single_params.nc,
                                     c->single_params.kc, c->single_params.mr,
                                     c->single_params.nr, 1};
  cfg.double_params = BlockingParams{c->double_params.mc, c->double_params.nc,
                                     c->double_params.kc, c->double_params.mr,
                                     c->double_params.nr, 1};
  cfg.threads = c->threads;
  cfg.preference = c->preference == MDG_PREF_ROW ? Preference::Row : Preference::Column;
  cfg.ctemp = c->ctemp == MDG_CTEMP_ON ? CTempMode::On
            : c->ctemp == MDG_CTEMP_OFF ? CTempMode::Off : CTempMode::Auto;
  return cfg;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return MDG_OK;
  } catch (const ScalarPolicyError& e) {
    g_err = e.what();
    return MDG_ERR_SCALAR_POLICY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MDG_ERR;
  }
}

Rng rng_path(uint64_t seed, const char* const* tags, const uint64_t* salts, int n) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) r = tags && tags[i] ? r.split(std::string_view(tags[i])) : r.split(salts[i]);
  return r;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_config_defaults(mdg_config_t* out) {
  return guarded([&] {
    Config c = Config::defaults();
    out->single_params = {c.single_params.mc, c.single_params.nc, c.single_params.kc,
                          c.single_params.mr, c.single_params.nr};
    out->double_params = {c.double_params.mc, c.double_params.nc, c.double_params.kc,
                          c.double_params.mr, c.double_params.nr};
    out->threads = c.threads;
    out->preference = MDG_PREF_COLUMN;
    out->ctemp = MDG_CTEMP_AUTO;
    out->numerics = MDG_NUMERICS_FAST;
  });
}

int ref_plan(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
             const mdg_view_t* c, const mdg_config_t* cfg, mdg_plan_t* out) {
  return guarded([&] {
    ExecutionPlan p = plan(scalar_in(alpha), view_in(a), view_in(b), scalar_in(beta),
                           view_in(c), config_in(cfg));
    mdg_plan_t o{};
    o.case_id = static_cast<int32_t>(p.case_id);
    o.logical_transpose = p.logical_transpose;
    o.comp_prec = pcode(p.comp_prec);
    o.m = p.m; o.n = p.n; o.k = p.k;
    o.a = view_out(p.a); o.b = view_out(p.b); o.c = view_out(p.c);
    o.format_a = static_cast<int32_t>(p.format_a);
    o.format_b = static_cast<int32_t>(p.format_b);
    o.conj_a = p.conj_a; o.conj_b = p.conj_b;
    o.target_dtype_a = code_of(p.target_dtype_a);
    o.target_dtype_b = code_of(p.target_dtype_b);
    o.reg_block_a = p.reg_block_a; o.reg_block_b = p.reg_block_b;
    o.alpha = scalar_out(p.alpha); o.beta = scalar_out(p.beta);
    o.pack_scale_a = scalar_out(p.pack_scale_a);
    o.pack_scale_b = scalar_out(p.pack_scale_b);
    o.macro_mode = static_cast<int32_t>(p.macro_mode);
    o.ukr_path = static_cast<int32_t>(p.ukr_path);
    o.pair_axis = static_cast<int32_t>(p.pair_axis);
    o.has_ctemp = p.ctemp.has_value();
    if (p.ctemp) {
      o.ctemp_rows = p.ctemp->rows;
      o.ctemp_cols = p.ctemp->cols;
      o.ctemp_precision = pcode(p.ctemp->precision);
      o.ctemp_mode = p.ctemp->mode == CTempDescriptor::Mode::CopyBack ? MDG_CTEMP_COPY_BACK
                                                                       : MDG_CTEMP_ACCUMULATE_BACK;
    }
    o.params = {p.params.mc, p.params.nc, p.params.kc, p.params.mr, p.params.nr};
    o.threads = p.params.threads;
    o.ukr_precision = pcode(p.ukr.precision);
    o.ukr_mr = p.ukr.mr; o.ukr_nr = p.ukr.nr;
    o.ukr_preference = p.ukr.preference == Preference::Row ? MDG_PREF_ROW : MDG_PREF_COLUMN;
    *out = o;
  });
}

int ref_gemm(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
             const mdg_view_t* c, const mdg_config_t* cfg, uint64_t* flops) {
  return guarded([&] {
    FlopCounter fc;
    gemm(scalar_in(alpha), view_in(a), view_in(b), scalar_in(beta), view_in(c), config_in(cfg), &fc);
    if (flops) *flops = fc.value();
  });
}

size_t ref_packed_bytes(const mdg_view_t* src, int32_t side, int32_t format, int32_t target,
                        int64_t reg_block) {
  size_t r = 0;
  int rc = guarded([&] {
    r = packed_bytes(view_in(src), static_cast<Side>(side), static_cast<PackFormat>(format),
                     dt_of(target), reg_block);
  });
  return rc == MDG_OK ? r : 0;
}

int ref_pack(const mdg_view_t* src, int32_t side, int32_t format, int32_t conj,
             mdg_scalar_t scale, int32_t target, int64_t reg_block, void* dst, size_t cap) {
  return guarded([&] {
    pack_block_into(std::span<std::byte>(static_cast<std::byte*>(dst), cap), view_in(src),
                    static_cast<Side>(side), static_cast<PackFormat>(format), conj != 0,
                    scalar_in(scale), dt_of(target), reg_block);
  });
}

// oracle_gemm (oracle.cpp:92-140) into a caller-provided column-stored
// buffer of c_in's datatype.
int ref_oracle_gemm(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b,
                    mdg_scalar_t beta, const mdg_view_t* c_in, int32_t comp_prec,
                    void* out, size_t cap) {
  return guarded([&] {
    MatrixView cv = view_in(c_in);
    CaseId id = classify_case(cv.dtype.domain, view_in(a).dtype.domain, view_in(b).dtype.domain);
    Matrix r = oracle_gemm(scalar_in(alpha), view_in(a), view_in(b), scalar_in(beta), cv, id,
                           prec_of(comp_prec));
    if (r.size_bytes() > cap) throw Error("ref_oracle_gemm: output buffer too small");
    std::memcpy(out, r.data(), r.size_bytes());
  });
}

// The reference's per-element acceptance criterion: max_violation of c_impl
// against oracle_gemm under tolerance(8(k+2)eps_comp + 4eps_out)*magnitude
// (acceptance.cpp:54-64, oracle.cpp:142-206).
int ref_violation(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b,
                  mdg_scalar_t beta, const mdg_view_t* c_before, const mdg_view_t* c_after,
                  int32_t comp_prec, double* violation) {
  return guarded([&] {
    MatrixView av = view_in(a), bv = view_in(b), cb = view_in(c_before), ca = view_in(c_after);
    CaseId id = classify_case(cb.dtype.domain, av.dtype.domain, bv.dtype.domain);
    Matrix want = oracle_gemm(scalar_in(alpha), av, bv, scalar_in(beta), cb, id, prec_of(comp_prec));
    ErrorBoundParams bp{av.n, eps_of(prec_of(comp_prec)), eps_of(cb.dtype.precision),
                        magnitude_matrix(scalar_in(alpha), av, bv, scalar_in(beta), cb, id)};
    Matrix tol = tolerance(bp);
    *violation = max_violation(ca, want.view(), tol.view());
  });
}

int ref_fill_uniform_path(const mdg_view_t* v, uint64_t seed, const char* const* tags,
                          const uint64_t* salts, int32_t n) {
  return guarded([&] { fill_uniform(view_in(v), rng_path(seed, tags, salts, n)); });
}

// run_bench (bench.cpp:13-51): warm-up + best of `trials`.
int ref_run_bench(const char* label, int64_t m, int64_t n, int64_t k, int32_t trials,
                  const mdg_config_t* cfg, uint64_t seed, double* best_seconds, double* gflops) {
  return guarded([&] {
    BenchResult r = run_bench(CaseLabel::parse(label), m, n, k, trials, config_in(cfg), seed);
    *best_seconds = r.best_seconds;
    *gflops = r.gflops;
  });
}

uint64_t ref_flops_of_case(int32_t case_id, int64_t m, int64_t n, int64_t k) {
  return flops_of_case(static_cast<CaseId>(case_id), m, n, k);
}

}  // extern "C"
