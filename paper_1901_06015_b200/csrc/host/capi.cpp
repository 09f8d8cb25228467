// The C ABI (include/mdgemm_b200.h): plain-data conversions around the C++
// API, with the reference's exceptions mapped to status codes.
#include <cstring>
#include <exception>

#include "driver.hpp"
#include "profile.hpp"
#include "mdgemm_b200.h"

using namespace mdgemm;

namespace {

thread_local std::string g_last_error;

Datatype dt_from(int32_t code) {
  switch (code) {
    case MDG_DT_S: return dt_s;
    case MDG_DT_D: return dt_d;
    case MDG_DT_C: return dt_c;
    case MDG_DT_Z: return dt_z;
  }
  throw Error("unknown datatype code " + std::to_string(code));
}

int32_t dt_to(Datatype t) {
  return (t.domain == Domain::Complex ? 2 : 0) + (t.precision == Precision::Double ? 1 : 0);
}

Precision prec_from(int32_t p) {
  if (p == MDG_PREC_SINGLE) return Precision::Single;
  if (p == MDG_PREC_DOUBLE) return Precision::Double;
  throw Error("unknown precision code " + std::to_string(p));
}
int32_t prec_to(Precision p) { return p == Precision::Double ? MDG_PREC_DOUBLE : MDG_PREC_SINGLE; }

MatrixView view_from(const mdg_view_t* v) {
  if (!v) throw Error("null view");
  MatrixView out = MatrixView::make(v->base, v->m, v->n, v->rs, v->cs, dt_from(v->dtype));
  out.conj = v->conj != 0;
  out.comp_prec = prec_from(v->comp_prec);
  return out;
}

mdg_view_t view_to(const MatrixView& v) {
  mdg_view_t o{};
  o.base = v.base;
  o.m = v.m;
  o.n = v.n;
  o.rs = v.rs;
  o.cs = v.cs;
  o.dtype = dt_to(v.dtype);
  o.conj = v.conj ? 1 : 0;
  o.comp_prec = prec_to(v.comp_prec);
  o.target_dtype = dt_to(v.target_dtype);
  return o;
}

Scalar scalar_from(const mdg_scalar_t& s) { return Scalar{s.re, s.im, dt_from(s.dtype)}; }
mdg_scalar_t scalar_to(const Scalar& s) {
  mdg_scalar_t o{};
  o.re = s.re;
  o.im = s.im;
  o.dtype = dt_to(s.dtype);
  return o;
}

BlockingParams blocking_from(const mdg_blocking_t& b) { return BlockingParams{b.mc, b.nc, b.kc, b.mr, b.nr, 1}; }
mdg_blocking_t blocking_to(const BlockingParams& b) { return mdg_blocking_t{b.mc, b.nc, b.kc, b.mr, b.nr}; }

Config config_from(const mdg_config_t* c) {
  Config cfg;
  if (!c) return cfg;
  cfg.single_params = blocking_from(c->single_params);
  cfg.double_params = blocking_from(c->double_params);
  cfg.threads = c->threads;
  cfg.preference = c->preference == MDG_PREF_ROW ? Preference::Row : Preference::Column;
  cfg.ctemp = c->ctemp == MDG_CTEMP_ON ? CTempMode::On : c->ctemp == MDG_CTEMP_OFF ? CTempMode::Off : CTempMode::Auto;
  cfg.numerics = c->numerics == MDG_NUMERICS_EXACT ? Numerics::Exact : Numerics::Fast;
  cfg.splitk = c->splitk != 0;
  return cfg;
}

void config_to(const Config& cfg, mdg_config_t* o) {
  o->single_params = blocking_to(cfg.single_params);
  o->double_params = blocking_to(cfg.double_params);
  o->threads = cfg.threads;
  o->preference = cfg.preference == Preference::Row ? MDG_PREF_ROW : MDG_PREF_COLUMN;
  o->ctemp = cfg.ctemp == CTempMode::On ? MDG_CTEMP_ON : cfg.ctemp == CTempMode::Off ? MDG_CTEMP_OFF : MDG_CTEMP_AUTO;
  o->numerics = cfg.numerics == Numerics::Exact ? MDG_NUMERICS_EXACT : MDG_NUMERICS_FAST;
  o->splitk = cfg.splitk ? 1 : 0;
  o->reserved = 0;
}

ExecutionPlan plan_from(const mdg_plan_t* q) {
  ExecutionPlan p;
  p.case_id = static_cast<CaseId>(q->case_id);
  p.logical_transpose = q->logical_transpose != 0;
  p.comp_prec = prec_from(q->comp_prec);
  p.m = q->m;
  p.n = q->n;
  p.k = q->k;
  p.a = view_from(&q->a);
  p.b = view_from(&q->b);
  p.c = view_from(&q->c);
  p.format_a = static_cast<PackFormat>(q->format_a);
  p.format_b = static_cast<PackFormat>(q->format_b);
  p.conj_a = q->conj_a != 0;
  p.conj_b = q->conj_b != 0;
  p.target_dtype_a = dt_from(q->target_dtype_a);
  p.target_dtype_b = dt_from(q->target_dtype_b);
  p.reg_block_a = q->reg_block_a;
  p.reg_block_b = q->reg_block_b;
  p.alpha = scalar_from(q->alpha);
  p.beta = scalar_from(q->beta);
  p.pack_scale_a = scalar_from(q->pack_scale_a);
  p.pack_scale_b = scalar_from(q->pack_scale_b);
  p.macro_mode = static_cast<MacroMode>(q->macro_mode);
  p.ukr_path = static_cast<UkrPath>(q->ukr_path);
  p.pair_axis = static_cast<PairAxis>(q->pair_axis);
  if (q->has_ctemp) {
    CTempDescriptor ct;
    ct.rows = q->ctemp_rows;
    ct.cols = q->ctemp_cols;
    ct.precision = prec_from(q->ctemp_precision);
    ct.mode = q->ctemp_mode == MDG_CTEMP_COPY_BACK ? CTempDescriptor::Mode::CopyBack
                                                   : CTempDescriptor::Mode::AccumulateBack;
    p.ctemp = ct;
  }
  p.params = blocking_from(q->params);
  p.params.threads = q->threads;
  p.ukr = UkrDescriptor{prec_from(q->ukr_precision), q->ukr_mr, q->ukr_nr,
                        q->ukr_preference == MDG_PREF_ROW ? Preference::Row : Preference::Column};
  return p;
}

void plan_to(const ExecutionPlan& p, mdg_plan_t* o) {
  std::memset(o, 0, sizeof(*o));
  o->case_id = static_cast<int32_t>(p.case_id);
  o->logical_transpose = p.logical_transpose ? 1 : 0;
  o->comp_prec = prec_to(p.comp_prec);
  o->m = p.m;
  o->n = p.n;
  o->k = p.k;
  o->a = view_to(p.a);
  o->b = view_to(p.b);
  o->c = view_to(p.c);
  o->format_a = static_cast<int32_t>(p.format_a);
  o->format_b = static_cast<int32_t>(p.format_b);
  o->conj_a = p.conj_a;
  o->conj_b = p.conj_b;
  o->target_dtype_a = dt_to(p.target_dtype_a);
  o->target_dtype_b = dt_to(p.target_dtype_b);
  o->reg_block_a = p.reg_block_a;
  o->reg_block_b = p.reg_block_b;
  o->alpha = scalar_to(p.alpha);
  o->beta = scalar_to(p.beta);
  o->pack_scale_a = scalar_to(p.pack_scale_a);
  o->pack_scale_b = scalar_to(p.pack_scale_b);
  o->macro_mode = static_cast<int32_t>(p.macro_mode);
  o->ukr_path = static_cast<int32_t>(p.ukr_path);
  o->pair_axis = static_cast<int32_t>(p.pair_axis);
  o->has_ctemp = p.ctemp.has_value();
  if (p.ctemp) {
    o->ctemp_rows = p.ctemp->rows;
    o->ctemp_cols = p.ctemp->cols;
    o->ctemp_precision = prec_to(p.ctemp->precision);
    o->ctemp_mode = p.ctemp->mode == CTempDescriptor::Mode::CopyBack ? MDG_CTEMP_COPY_BACK : MDG_CTEMP_ACCUMULATE_BACK;
  }
  o->params = blocking_to(p.params);
  o->threads = p.params.threads;
  o->ukr_precision = prec_to(p.ukr.precision);
  o->ukr_mr = p.ukr.mr;
  o->ukr_nr = p.ukr.nr;
  o->ukr_preference = p.ukr.preference == Preference::Row ? MDG_PREF_ROW : MDG_PREF_COLUMN;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return MDG_OK;
  } catch (const ScalarPolicyError& e) {
    g_last_error = e.what();
    return MDG_ERR_SCALAR_POLICY;
  } catch (const CudaFailure& e) {
    g_last_error = e.what();
    return MDG_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MDG_ERR;
  } catch (...) {
    g_last_error = "unknown failure";
    return MDG_ERR;
  }
}

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
uint64_t splitmix(uint64_t z) {
  z += kGamma;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" {

int mdg_abi_version(void) { return MDG_ABI_VERSION; }

const char* mdg_last_error(void) { return g_last_error.c_str(); }

int mdg_config_defaults(mdg_config_t* out) {
  return guarded([&] { config_to(Config::defaults(), out); });
}

int mdg_config_set(mdg_config_t* cfg, const char* key, const char* value) {
  return guarded([&] {
    Config c = config_from(cfg);
    c.set(key ? key : "", value ? value : "");
    config_to(c, cfg);
  });
}

int mdg_config_load(mdg_config_t* out, const char* path_or_null, int apply_env) {
  return guarded([&] {
    const std::optional<std::string> path = path_or_null ? std::optional<std::string>(path_or_null) : std::nullopt;
    config_to(Config::load(path, apply_env != 0), out);
  });
}

int mdg_config_validate(const mdg_config_t* cfg) {
  return guarded([&] { config_from(cfg).validate(); });
}

int mdg_view_make(void* base, int64_t m, int64_t n, int64_t rs, int64_t cs, int32_t dtype, mdg_view_t* out) {
  return guarded([&] { *out = view_to(MatrixView::make(base, m, n, rs, cs, dt_from(dtype))); });
}

int32_t mdg_classify_case(int32_t c_complex, int32_t a_complex, int32_t b_complex) {
  auto dom = [](int32_t x) { return x ? Domain::Complex : Domain::Real; };
  return static_cast<int32_t>(classify_case(dom(c_complex), dom(a_complex), dom(b_complex)));
}

uint64_t mdg_flops_of_case(int32_t case_id, int64_t m, int64_t n, int64_t k) {
  return flops_of_case(static_cast<CaseId>(case_id), m, n, k);
}

int mdg_apply_scalar_policy(mdg_scalar_t alpha, mdg_scalar_t beta, int32_t case_id, int32_t comp_prec,
                            int32_t c_storage_prec, mdg_scalar_t* alpha_out, mdg_scalar_t* beta_out) {
  return guarded([&] {
    const auto [a, b] = apply_scalar_policy(scalar_from(alpha), scalar_from(beta), static_cast<CaseId>(case_id),
                                            prec_from(comp_prec), prec_from(c_storage_prec));
    *alpha_out = scalar_to(a);
    *beta_out = scalar_to(b);
  });
}

int mdg_plan(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta, const mdg_view_t* c,
             const mdg_config_t* cfg, mdg_plan_t* out) {
  return guarded([&] {
    const ExecutionPlan p =
        plan(scalar_from(alpha), view_from(a), view_from(b), scalar_from(beta), view_from(c), config_from(cfg));
    plan_to(p, out);
  });
}

int mdg_execute(const mdg_plan_t* p, int32_t numerics, void* stream, uint64_t* flops_out) {
  return guarded([&] {
    FlopCounter fc;
    execute(plan_from(p), (numerics & 0xff) == MDG_NUMERICS_EXACT ? Numerics::Exact : Numerics::Fast, stream, &fc,
            (numerics & MDG_EXEC_NO_SPLITK) == 0);
    if (flops_out) *flops_out = fc.value();
  });
}

int mdg_gemm(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta, const mdg_view_t* c,
             const mdg_config_t* cfg, uint64_t* flops_out) {
  return guarded([&] {
    FlopCounter fc;
    gemm(scalar_from(alpha), view_from(a), view_from(b), scalar_from(beta), view_from(c), config_from(cfg), &fc);
    if (flops_out) *flops_out = fc.value();
  });
}

static std::vector<GemmCall> call_list(int32_t count, const mdg_gemm_call_t* calls) {
  if (count < 0 || (count > 0 && !calls)) throw Error("mdg_gemm_batch: bad call list");
  std::vector<GemmCall> list;
  list.reserve(static_cast<size_t>(count));
  for (int32_t i = 0; i < count; ++i)
    list.push_back(GemmCall{scalar_from(calls[i].alpha), view_from(&calls[i].a), view_from(&calls[i].b),
                            scalar_from(calls[i].beta), view_from(&calls[i].c)});
  return list;
}

int mdg_gemm_batch(int32_t count, const mdg_gemm_call_t* calls, const mdg_config_t* cfg, uint64_t* flops_out) {
  return guarded([&] {
    FlopCounter fc;
    gemm_batch(call_list(count, calls), config_from(cfg), &fc);
    if (flops_out) *flops_out = fc.value();
  });
}

int mdg_dual_schedule(int32_t count, const mdg_gemm_call_t* calls, const mdg_config_t* cfg, int32_t capacity,
                      int32_t* pieces, int32_t* npieces, int32_t* call_tiles) {
  return guarded([&] {
    std::vector<int32_t> tiles;
    const std::vector<DualPiece> out = dual_schedule_pieces(call_list(count, calls), config_from(cfg), &tiles);
    *npieces = static_cast<int32_t>(out.size());
    for (size_t x = 0; x < out.size() && static_cast<int32_t>(x) < capacity; ++x) {
      int32_t* q = pieces + 5 * x;
      q[0] = out[x].unit;
      q[1] = out[x].call;
      q[2] = out[x].t0;
      q[3] = out[x].t1;
      q[4] = out[x].group;
    }
    if (call_tiles)
      for (int32_t i = 0; i < count; ++i) call_tiles[i] = tiles[static_cast<size_t>(i)];
  });
}

int mdg_gemm_batch_async(int32_t count, const mdg_gemm_call_t* calls, const mdg_config_t* cfg, void* stream,
                         uint64_t* flops_out) {
  return guarded([&] {
    FlopCounter fc;
    gemm_batch_async(call_list(count, calls), config_from(cfg), stream, &fc);
    if (flops_out) *flops_out = fc.value();
  });
}

int mdg_gemm_async(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
                   const mdg_view_t* c, const mdg_config_t* cfg, void* stream, uint64_t* flops_out) {
  return guarded([&] {
    FlopCounter fc;
    gemm_async(scalar_from(alpha), view_from(a), view_from(b), scalar_from(beta), view_from(c), config_from(cfg),
               stream, &fc);
    if (flops_out) *flops_out = fc.value();
  });
}

size_t mdg_packed_bytes(const mdg_view_t* src, int32_t side, int32_t format, int32_t target_dtype, int64_t reg_block,
                        int64_t panel_len) {
  size_t bytes = 0;
  const int rc = guarded([&] {
    bytes = pack_geometry(view_from(src), static_cast<Side>(side), static_cast<PackFormat>(format),
                          dt_from(target_dtype), reg_block, panel_len)
                .bytes;
  });
  return rc == MDG_OK ? bytes : 0;
}

int mdg_pack_operand(const mdg_view_t* src, int32_t side, int32_t format, int32_t conj, mdg_scalar_t scale,
                     int32_t target_dtype, int64_t reg_block, int64_t panel_len, void* dst, void* stream) {
  return guarded([&] {
    pack_block_device_padded(dst, view_from(src), static_cast<Side>(side), static_cast<PackFormat>(format),
                             conj != 0, scalar_from(scale), dt_from(target_dtype), reg_block, panel_len, stream);
  });
}

int mdg_fill_uniform(const mdg_view_t* v, uint64_t rng_state, void* stream) {
  return guarded([&] {
    const MatrixView mv = view_from(v);
    prof::Scope scope(MDG_KERNEL_FILL, static_cast<cudaStream_t>(stream),
                      static_cast<double>(mv.m) * mv.n * dtype_size(mv.dtype));
    cuda_check(mdg::launch_fill_uniform(to_dview(view_from(v)), rng_state, device_sms(), static_cast<cudaStream_t>(stream)),
               "fill_uniform");
  });
}

int mdg_fill_normal(const mdg_view_t* v, uint64_t rng_state, void* stream) {
  return guarded([&] {
    const MatrixView mv = view_from(v);
    prof::Scope scope(MDG_KERNEL_FILL, static_cast<cudaStream_t>(stream),
                      static_cast<double>(mv.m) * mv.n * dtype_size(mv.dtype));
    cuda_check(mdg::launch_fill_normal(to_dview(mv), rng_state, device_sms(), static_cast<cudaStream_t>(stream)),
               "fill_normal");
  });
}

uint64_t mdg_rng_split_tag(uint64_t state, const char* tag) {
  uint64_t h = state ^ kGamma;
  for (const char* p = tag; p && *p; ++p) h = splitmix(h ^ static_cast<uint64_t>(static_cast<unsigned char>(*p)));
  return h;
}

uint64_t mdg_rng_split_salt(uint64_t state, uint64_t salt) { return splitmix(state ^ salt); }

int mdg_shard_columns(int64_t n, int32_t world, int32_t rank, int64_t align, int64_t* j0, int64_t* nb) {
  return guarded([&] {
    if (!j0 || !nb) throw Error("mdg_shard_columns: bad arguments");
    shard_columns(n, world, rank, align, j0, nb);
  });
}

int mdg_comm_unique_id(uint8_t* id) {
  return guarded([&] {
    if (!id) throw Error("mdg_comm_unique_id: null id");
    const CommId c = Communicator::unique_id();
    std::memcpy(id, c.bytes, sizeof(c.bytes));
  });
}

int mdg_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, mdg_comm_t* out) {
  return guarded([&] {
    if (!id || !out) throw Error("mdg_comm_init: bad arguments");
    CommId c;
    std::memcpy(c.bytes, id, sizeof(c.bytes));
    *out = reinterpret_cast<mdg_comm_t>(new Communicator(c, nranks, rank));
  });
}

int mdg_comm_destroy(mdg_comm_t comm) {
  return guarded([&] { delete reinterpret_cast<Communicator*>(comm); });
}

int mdg_gemm_sharded(mdg_comm_t comm, int32_t root, mdg_scalar_t alpha, const mdg_view_t* a,
                     const mdg_view_t* b_panel, mdg_scalar_t beta, const mdg_view_t* c_panel,
                     const mdg_config_t* cfg, void* stream, uint64_t* flops_out) {
  return guarded([&] {
    if (!comm) throw Error("mdg_gemm_sharded: null communicator");
    FlopCounter fc;
    gemm_sharded(*reinterpret_cast<Communicator*>(comm), root, scalar_from(alpha), view_from(a), view_from(b_panel),
                 scalar_from(beta), view_from(c_panel), config_from(cfg), stream, &fc);
    if (flops_out) *flops_out = fc.value();
  });
}

int mdg_gemm_multi(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
                   const mdg_view_t* c, const mdg_config_t* cfg, int32_t ndev, const int32_t* devices,
                   uint64_t* flops_out) {
  return guarded([&] {
    if (ndev < 1) throw Error("mdg_gemm_multi: ndev must be at least 1");
    std::vector<int> devs(static_cast<size_t>(ndev));
    for (int32_t i = 0; i < ndev; ++i) devs[i] = devices ? devices[i] : i;
    FlopCounter fc;
    gemm_multi(scalar_from(alpha), view_from(a), view_from(b), scalar_from(beta), view_from(c), config_from(cfg), devs,
               &fc);
    if (flops_out) *flops_out = fc.value();
  });
}

int mdg_trim_workspace(uint64_t keep_bytes) {
  return guarded([&] { trim_workspace(static_cast<size_t>(keep_bytes)); });
}

uint64_t mdg_launch_count(void) { return prof::launches(); }

void mdg_staging_bytes(uint64_t* h2d, uint64_t* d2h) { mdgemm::staging_bytes(h2d, d2h); }

int mdg_profile_begin(void) {
  return guarded([&] { prof::begin(); });
}

int mdg_profile_end(mdg_kernel_stats_t* out) {
  return guarded([&] { prof::end(out); });
}

}  // extern "C"
