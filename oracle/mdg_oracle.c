/*
 * mdg_oracle.c -- TEST INFRASTRUCTURE ONLY: CPU restatement of the reference
 * mixed-datatype gemm (arXiv 1901.06015 / /root/reference/proj) used as the
 * checker by tests/ and as the "port" CPU baseline.  Compiled with
 * -ffp-contract=off so every multiply and add rounds separately, exactly as
 * the reference's x86-64 build evaluates them.  Parity of this file is
 * pinned against the reference library built from its own sources
 * (oracle/_ref) and against the reference tests' known answers.
 */
#include "mdg_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------ datatypes */

static int is_cplx(int32_t dt) { return dt == MDG_DT_C || dt == MDG_DT_Z; }
static int is_sgl(int32_t dt) { return dt == MDG_DT_S || dt == MDG_DT_C; }
static int32_t prec_of(int32_t dt) { return is_sgl(dt) ? MDG_PREC_SINGLE : MDG_PREC_DOUBLE; }
static int32_t mkdt(int cplx, int32_t prec) { return (cplx ? 2 : 0) + (prec == MDG_PREC_DOUBLE ? 1 : 0); }
static size_t dsize(int32_t dt) { return (size_t)(is_sgl(dt) ? 4 : 8) * (is_cplx(dt) ? 2 : 1); }
static size_t rsize(int32_t prec) { return prec == MDG_PREC_SINGLE ? 4 : 8; }

/* dtypes.cpp:54-56 */
static double rnd(double v, int32_t prec) { return prec == MDG_PREC_SINGLE ? (double)(float)v : v; }

static char* eptr(const mdg_view_t* v, int64_t i, int64_t j) {
  return (char*)v->base + (size_t)(i * v->rs + j * v->cs) * dsize(v->dtype);
}

/* load_elem (dtypes.cpp:176-193) */
static void load(const mdg_view_t* v, int64_t i, int64_t j, double* re, double* im) {
  const char* p = eptr(v, i, j);
  switch (v->dtype) {
    case MDG_DT_S: *re = *(const float*)p; *im = 0.0; break;
    case MDG_DT_D: *re = *(const double*)p; *im = 0.0; break;
    case MDG_DT_C: *re = ((const float*)p)[0]; *im = ((const float*)p)[1]; break;
    default: *re = ((const double*)p)[0]; *im = ((const double*)p)[1]; break;
  }
  if (v->conj) *im = -*im;
}

/* store_elem (dtypes.cpp:195-213), value already validated */
static void store(const mdg_view_t* v, int64_t i, int64_t j, double re, double im) {
  char* p = eptr(v, i, j);
  switch (v->dtype) {
    case MDG_DT_S: *(float*)p = (float)re; break;
    case MDG_DT_D: *(double*)p = re; break;
    case MDG_DT_C: ((float*)p)[0] = (float)re; ((float*)p)[1] = (float)im; break;
    default: ((double*)p)[0] = re; ((double*)p)[1] = im; break;
  }
}

/* complex<double> product as GCC evaluates it: separate multiplies/adds,
 * Annex G recovery (libgcc __muldc3) when both parts come out NaN. */
static double box(int inf, double s) { return copysign(inf ? 1.0 : 0.0, s); }
static void cmul(double a, double b, double c, double d, double* x, double* y) {
  double ac = a * c, bd = b * d, ad = a * d, bc = b * c;
  *x = ac - bd;
  *y = ad + bc;
  if (isnan(*x) && isnan(*y)) {
    int recalc = 0;
    if (isinf(a) || isinf(b)) {
      a = box(isinf(a), a);
      b = box(isinf(b), b);
      if (isnan(c)) c = copysign(0.0, c);
      if (isnan(d)) d = copysign(0.0, d);
      recalc = 1;
    }
    if (isinf(c) || isinf(d)) {
      c = box(isinf(c), c);
      d = box(isinf(d), d);
      if (isnan(a)) a = copysign(0.0, a);
      if (isnan(b)) b = copysign(0.0, b);
      recalc = 1;
    }
    if (!recalc && (isinf(ac) || isinf(bd) || isinf(ad) || isinf(bc))) {
      if (isnan(a)) a = copysign(0.0, a);
      if (isnan(b)) b = copysign(0.0, b);
      if (isnan(c)) c = copysign(0.0, c);
      if (isnan(d)) d = copysign(0.0, d);
      recalc = 1;
    }
    if (recalc) {
      *x = INFINITY * (a * c - b * d);
      *y = INFINITY * (a * d + b * c);
    }
  }
}

/* ------------------------------------------------------------------ rng */

#define GAMMA 0x9e3779b97f4a7c15ULL

static uint64_t mix(uint64_t z) { /* rng.hpp:19-24 */
  z += GAMMA;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_rng_split_tag(uint64_t state, const char* tag) { /* rng.hpp:34-39 */
  uint64_t h = state ^ GAMMA;
  for (const unsigned char* p = (const unsigned char*)tag; p && *p; ++p) h = mix(h ^ (uint64_t)*p);
  return h;
}

uint64_t orc_rng_split_salt(uint64_t state, uint64_t salt) { return mix(state ^ salt); } /* rng.hpp:41 */

static double next_uniform(uint64_t* s) { /* rng.hpp:26-31 */
  *s += GAMMA;
  const uint64_t x = mix(*s);
  return 2.0 * ((double)(x >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
}

int orc_fill_uniform(const mdg_view_t* v, uint64_t state) { /* rng.hpp:49-56 */
  uint64_t s = state;
  for (int64_t j = 0; j < v->n; ++j)
    for (int64_t i = 0; i < v->m; ++i) {
      const double re = next_uniform(&s);
      const double im = is_cplx(v->dtype) ? next_uniform(&s) : 0.0;
      store(v, i, j, re, im);
    }
  return MDG_OK;
}

/* --------------------------------------------------------------- config */

int orc_config_defaults(mdg_config_t* o) { /* config.hpp:38-41 */
  memset(o, 0, sizeof *o);
  o->single_params = (mdg_blocking_t){128, 1024, 256, 8, 8};
  o->double_params = (mdg_blocking_t){64, 512, 128, 4, 4};
  o->threads = 1;
  o->preference = MDG_PREF_COLUMN;
  o->ctemp = MDG_CTEMP_AUTO;
  o->numerics = MDG_NUMERICS_FAST;
  o->splitk = 1;
  return MDG_OK;
}

static int check_blocking(const mdg_blocking_t* b, const char* which) { /* config.cpp:135-153 */
  if (b->mr < 2 || b->nr < 2 || b->mr > 32 || b->nr > 32)
    return fail(MDG_ERR, "config: %s blocking invalid: mr/nr must lie in [2, 32]", which);
  if (b->mr % 2 || b->nr % 2) return fail(MDG_ERR, "config: %s blocking invalid: mr/nr must be even", which);
  if (b->mc < b->mr || b->nc < b->nr || b->kc < 2)
    return fail(MDG_ERR, "config: %s blocking invalid: mc/nc/kc too small", which);
  if (b->mc % b->mr) return fail(MDG_ERR, "config: %s blocking invalid: mc must be a multiple of mr", which);
  if (b->nc % b->nr) return fail(MDG_ERR, "config: %s blocking invalid: nc must be a multiple of nr", which);
  if (b->mc % 2 || b->nc % 2 || b->kc % 2)
    return fail(MDG_ERR, "config: %s blocking invalid: mc/nc/kc must be even", which);
  return MDG_OK;
}

int orc_config_validate(const mdg_config_t* c) {
  int rc = check_blocking(&c->single_params, "single");
  if (rc) return rc;
  rc = check_blocking(&c->double_params, "double");
  if (rc) return rc;
  if (c->threads < 1 || c->threads > 1024) return fail(MDG_ERR, "config: gemm.threads must lie in [1, 1024]");
  return MDG_OK;
}

/* ---------------------------------------------------------------- views */

static mdg_view_t transpose(mdg_view_t v) { /* dtypes.cpp:113-117 */
  int64_t t = v.m; v.m = v.n; v.n = t;
  t = v.rs; v.rs = v.cs; v.cs = t;
  return v;
}

static mdg_view_t real_proj(mdg_view_t v, int im_part) { /* dtypes.cpp:119-129 */
  const int32_t p = prec_of(v.dtype);
  v.dtype = mkdt(0, p);
  v.base = (char*)v.base + (im_part ? rsize(p) : 0);
  v.rs *= 2;
  v.cs *= 2;
  v.conj = 0;
  return v;
}

static int can_flatten(const mdg_view_t* v, int rows_axis) { /* dtypes.cpp:131-135 */
  if (!is_cplx(v->dtype)) return 0;
  return rows_axis ? v->rs == 1 : v->cs == 1;
}

static mdg_view_t real_flat(mdg_view_t v, int rows_axis) { /* dtypes.cpp:137-155 */
  v.dtype = mkdt(0, prec_of(v.dtype));
  v.conj = 0;
  if (rows_axis) { v.m *= 2; v.rs = 1; v.cs *= 2; }
  else { v.n *= 2; v.cs = 1; v.rs *= 2; }
  return v;
}

enum { SK_COL, SK_ROW, SK_GEN };
static int storage_kind(const mdg_view_t* v) { /* dtypes.cpp:168-174 */
  if (v->rs == 1 && v->cs >= (v->m > 1 ? v->m : 1)) return SK_COL;
  if (v->cs == 1 && v->rs >= (v->n > 1 ? v->n : 1)) return SK_ROW;
  return SK_GEN;
}

static void byte_range(const mdg_view_t* v, const char** lo, const char** hi) { /* dtypes.cpp:215-220 */
  *lo = (const char*)v->base;
  *hi = *lo;
  if (v->m == 0 || v->n == 0) return;
  *hi = eptr(v, v->m - 1, v->n - 1) + dsize(v->dtype);
}

static int overlap(const mdg_view_t* a, const mdg_view_t* b) {
  const char *alo, *ahi, *blo, *bhi;
  byte_range(a, &alo, &ahi);
  byte_range(b, &blo, &bhi);
  return alo < bhi && blo < ahi;
}

/* -------------------------------------------------------------- scalars */

static mdg_scalar_t sc_make(double re, double im, int32_t dt) {
  mdg_scalar_t s;
  memset(&s, 0, sizeof s);
  s.re = re; s.im = im; s.dtype = dt;
  return s;
}

static int typecast_sc(mdg_scalar_t s, int32_t target, mdg_scalar_t* out) { /* dtypes.cpp:68-76 */
  if (!is_cplx(target) && s.im != 0.0)
    return fail(MDG_ERR, "typecast_scalar: nonzero imaginary part cannot convert to a real datatype");
  const int32_t p = prec_of(target);
  *out = sc_make(rnd(s.re, p), is_cplx(target) ? rnd(s.im, p) : 0.0, target);
  return MDG_OK;
}

static mdg_scalar_t project_sc(mdg_scalar_t s, int32_t prec) { return sc_make(rnd(s.re, prec), 0.0, mkdt(0, prec)); }
static int sc_zero(mdg_scalar_t s) { return s.re == 0.0 && s.im == 0.0; }
static int sc_one(mdg_scalar_t s) { return s.re == 1.0 && s.im == 0.0; }

/* ------------------------------------------------------------- planning */

int32_t orc_classify_case(int32_t c, int32_t a, int32_t b) { /* dispatch.cpp:11-31 */
  if (!c) {
    if (a && b) return MDG_CASE_2AB;
    if (a) return MDG_CASE_1A;
    if (b) return MDG_CASE_1B;
    return MDG_CASE_0;
  }
  if (a && b) return MDG_CASE_3;
  if (a) return MDG_CASE_2AC;
  if (b) return MDG_CASE_2BC;
  return MDG_CASE_1C;
}

uint64_t orc_flops_of_case(int32_t id, int64_t m, int64_t n, int64_t k) { /* dispatch.cpp:35-54 */
  const uint64_t mnk = (uint64_t)m * (uint64_t)n * (uint64_t)k;
  if (id == MDG_CASE_3) return 8 * mnk;
  if (id == MDG_CASE_2AB || id == MDG_CASE_2AC || id == MDG_CASE_2BC) return 4 * mnk;
  return 2 * mnk;
}

static const char* case_name(int32_t id) {
  static const char* n[] = {"0", "1a", "1b", "1c", "2ab", "2ac", "2bc", "3"};
  return id >= 0 && id < 8 ? n[id] : "?";
}

static int scalar_policy(mdg_scalar_t alpha, mdg_scalar_t beta, int32_t id, int32_t comp, int32_t cprec,
                         mdg_scalar_t* ae, mdg_scalar_t* be) { /* dispatch.cpp:56-85 */
  int rc;
  if (id == MDG_CASE_0) {
    *ae = project_sc(alpha, comp);
  } else if (id == MDG_CASE_3) {
    rc = typecast_sc(alpha, mkdt(is_cplx(alpha.dtype), comp), ae);
    if (rc) return rc;
  } else {
    if (alpha.im != 0.0)
      return fail(MDG_ERR_SCALAR_POLICY, "case %s does not support alpha with a nonzero imaginary part",
                  case_name(id));
    *ae = project_sc(alpha, comp);
  }
  const int projects = id == MDG_CASE_0 || id == MDG_CASE_1A || id == MDG_CASE_1B || id == MDG_CASE_1C ||
                       id == MDG_CASE_2AB;
  if (projects) {
    *be = project_sc(beta, cprec);
    return MDG_OK;
  }
  return typecast_sc(beta, mkdt(is_cplx(beta.dtype), cprec), be);
}

static int32_t mirror(int32_t id) {
  switch (id) {
    case MDG_CASE_1A: return MDG_CASE_1B;
    case MDG_CASE_1B: return MDG_CASE_1A;
    case MDG_CASE_2AC: return MDG_CASE_2BC;
    case MDG_CASE_2BC: return MDG_CASE_2AC;
    default: return id;
  }
}

int orc_plan(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta, const mdg_view_t* c,
             const mdg_config_t* cfg, mdg_plan_t* out) { /* dispatch.cpp:106-305 */
  int rc = orc_config_validate(cfg);
  if (rc) return rc;
  if (a->m != c->m || b->n != c->n || a->n != b->m)
    return fail(MDG_ERR, "gemm: dimension mismatch: C is %lldx%lld, A is %lldx%lld, B is %lldx%lld", (long long)c->m,
                (long long)c->n, (long long)a->m, (long long)a->n, (long long)b->m, (long long)b->n);
  const int32_t comp = c->comp_prec;
  const int32_t in_case = orc_classify_case(is_cplx(c->dtype), is_cplx(a->dtype), is_cplx(b->dtype));
  mdg_scalar_t ae, be;
  rc = scalar_policy(alpha, beta, in_case, comp, prec_of(c->dtype), &ae, &be);
  if (rc) return rc;
  const int colpref = cfg->preference == MDG_PREF_COLUMN;

  int flip;
  if (in_case == MDG_CASE_2AC) flip = !colpref;
  else if (in_case == MDG_CASE_2BC) flip = colpref;
  else if (in_case == MDG_CASE_1C) flip = 0;
  else {
    const int sk = storage_kind(c);
    flip = (colpref && sk == SK_ROW) || (!colpref && sk == SK_COL);
  }
  const mdg_view_t A = flip ? transpose(*b) : *a;
  const mdg_view_t B = flip ? transpose(*a) : *b;
  const mdg_view_t C = flip ? transpose(*c) : *c;
  const int32_t id = flip ? mirror(in_case) : in_case;
  const int64_t m = C.m, n = C.n, k = A.n;

  mdg_plan_t p;
  memset(&p, 0, sizeof p);
  p.case_id = id;
  p.logical_transpose = flip;
  p.comp_prec = comp;
  const mdg_blocking_t bp = comp == MDG_PREC_SINGLE ? cfg->single_params : cfg->double_params;
  p.params = bp;
  p.threads = cfg->threads;
  p.ukr_precision = comp;
  p.ukr_mr = bp.mr;
  p.ukr_nr = bp.nr;
  p.ukr_preference = cfg->preference;
  p.alpha = ae;
  p.beta = be;

  mdg_view_t ea = A, eb = B, ec = C;
  int32_t fa = MDG_FMT_STANDARD, fb = MDG_FMT_STANDARD, pair = MDG_PAIR_NONE;
  int conjb = 0;
  int64_t me = m, ne = n, ke = k;
  switch (id) {
    case MDG_CASE_1A: ea = real_proj(A, 0); break;
    case MDG_CASE_1B: eb = real_proj(B, 0); break;
    case MDG_CASE_1C: ec = real_proj(C, 0); break;
    case MDG_CASE_2AB: fa = fb = MDG_FMT_ONER; conjb = 1; ke = 2 * k; break;
    case MDG_CASE_2AC: pair = MDG_PAIR_ROWS; me = 2 * m; break;
    case MDG_CASE_2BC: pair = MDG_PAIR_COLS; ne = 2 * n; break;
    case MDG_CASE_3:
      if (colpref) { fa = MDG_FMT_ONEE; fb = MDG_FMT_ONER; pair = MDG_PAIR_ROWS; me = 2 * m; }
      else { fa = MDG_FMT_ONER; fb = MDG_FMT_ONEE; pair = MDG_PAIR_COLS; ne = 2 * n; }
      ke = 2 * k;
      break;
    default: break;
  }
  p.format_a = fa;
  p.format_b = fb;
  p.conj_a = 0;
  p.conj_b = conjb;
  p.target_dtype_a = mkdt(is_cplx(ea.dtype), comp);
  p.target_dtype_b = mkdt(is_cplx(eb.dtype), comp);
  p.reg_block_a = (fa == MDG_FMT_STANDARD && is_cplx(ea.dtype)) ? bp.mr / 2 : bp.mr;
  p.reg_block_b = (fb == MDG_FMT_STANDARD && is_cplx(eb.dtype)) ? bp.nr / 2 : bp.nr;

  const mdg_scalar_t unit = sc_make(rnd(1.0, comp), 0.0, mkdt(0, comp));
  p.pack_scale_a = unit;
  p.pack_scale_b = unit;
  if (id == MDG_CASE_3 && !colpref) p.pack_scale_b = ae;
  else p.pack_scale_a = ae;

  p.macro_mode = comp != prec_of(c->dtype) ? MDG_MACRO_ACCUMULATE_TYPECAST : MDG_MACRO_STANDARD;

  int flatten_ok = 0;
  int32_t path = MDG_PATH_DIRECT;
  if (id == MDG_CASE_3) {
    path = colpref ? MDG_PATH_ONEM_COLUMN : MDG_PATH_ONEM_ROW;
  } else if (p.macro_mode == MDG_MACRO_ACCUMULATE_TYPECAST) {
    path = MDG_PATH_TEMP;
  } else if (id == MDG_CASE_1C) {
    path = MDG_PATH_TEMP;
  } else if (id == MDG_CASE_2AC || id == MDG_CASE_2BC) {
    const int rows_axis = id == MDG_CASE_2AC;
    flatten_ok = can_flatten(&ec, rows_axis);
    if (flatten_ok && be.im == 0.0) {
      ec = real_flat(ec, rows_axis);
      pair = MDG_PAIR_NONE;
      path = MDG_PATH_DIRECT;
    } else {
      path = MDG_PATH_TEMP;
    }
  }

  const int trig_cast = p.macro_mode == MDG_MACRO_ACCUMULATE_TYPECAST;
  const int trig_strided = id == MDG_CASE_1C && k > bp.kc;
  int trig_orient = 0;
  if ((id == MDG_CASE_2AC || id == MDG_CASE_2BC) && !flatten_ok) trig_orient = 1;
  if (id == MDG_CASE_3) trig_orient = !can_flatten(&ec, colpref);
  const int trig = trig_cast || trig_strided || trig_orient;
  const int engaged = cfg->ctemp != MDG_CTEMP_OFF && trig && (cfg->ctemp == MDG_CTEMP_ON || cfg->threads == 1);
  if (engaged) {
    p.has_ctemp = 1;
    p.ctemp_rows = me;
    p.ctemp_cols = ne;
    p.ctemp_precision = comp;
    p.ctemp_mode = sc_zero(be) ? MDG_CTEMP_COPY_BACK : MDG_CTEMP_ACCUMULATE_BACK;
  }
  p.a = ea;
  p.b = eb;
  p.c = ec;
  p.m = me;
  p.n = ne;
  p.k = ke;
  p.ukr_path = path;
  p.pair_axis = pair;
  *out = p;
  return MDG_OK;
}

/* -------------------------------------------------------------- packing */

typedef struct {
  int32_t block_dt;
  int64_t rows, cols, panels, len, lpad;
} geom_t;

static int geometry(const mdg_view_t* src, int32_t side, int32_t fmt, int32_t target, int64_t rb, int64_t plen,
                    geom_t* g) { /* packing.cpp:27-67 */
  if (rb < 1) return fail(MDG_ERR, "pack_block: reg_block must be at least 1");
  const int left = side == MDG_SIDE_LEFT;
  switch (fmt) {
    case MDG_FMT_STANDARD:
      if (is_cplx(target) != is_cplx(src->dtype))
        return fail(MDG_ERR, "pack_block: Standard packing cannot change the domain");
      g->block_dt = target;
      g->rows = src->m;
      g->cols = src->n;
      break;
    case MDG_FMT_ONEE:
      if (!is_cplx(src->dtype)) return fail(MDG_ERR, "pack_block: OneE requires a complex source");
      if (rb % 2) return fail(MDG_ERR, "pack_block: OneE requires an even reg_block");
      g->block_dt = mkdt(0, prec_of(target));
      g->rows = 2 * src->m;
      g->cols = 2 * src->n;
      break;
    case MDG_FMT_ONER:
      if (!is_cplx(src->dtype)) return fail(MDG_ERR, "pack_block: OneR requires a complex source");
      g->block_dt = mkdt(0, prec_of(target));
      g->rows = left ? src->m : 2 * src->m;
      g->cols = left ? 2 * src->n : src->n;
      break;
    default:
      return fail(MDG_ERR, "pack_block: unknown format");
  }
  const int64_t extent = left ? g->rows : g->cols;
  g->panels = (extent + rb - 1) / rb;
  g->len = left ? g->cols : g->rows;
  g->lpad = plen > g->len ? plen : g->len;
  return MDG_OK;
}

size_t orc_packed_bytes(const mdg_view_t* src, int32_t side, int32_t format, int32_t target, int64_t rb,
                        int64_t plen) {
  geom_t g;
  if (geometry(src, side, format, target, rb, plen, &g)) return 0;
  return (size_t)(g.panels * rb * g.lpad) * dsize(g.block_dt);
}

static void put(void* dst, int32_t dt, int64_t idx, double re, double im) { /* packing.cpp:70-89 */
  switch (dt) {
    case MDG_DT_S: ((float*)dst)[idx] = (float)re; break;
    case MDG_DT_D: ((double*)dst)[idx] = re; break;
    case MDG_DT_C: ((float*)dst)[2 * idx] = (float)re; ((float*)dst)[2 * idx + 1] = (float)im; break;
    default: ((double*)dst)[2 * idx] = re; ((double*)dst)[2 * idx + 1] = im; break;
  }
}

int orc_pack(const mdg_view_t* src, int32_t side, int32_t fmt, int32_t conj, mdg_scalar_t scale, int32_t target,
             int64_t rb, int64_t plen, void* dst) { /* packing.cpp:114-230 */
  if (scale.im != 0.0 && fmt == MDG_FMT_STANDARD)
    return fail(MDG_ERR, "pack_block: complex scale requires OneE or OneR format");
  geom_t g;
  int rc = geometry(src, side, fmt, target, rb, plen, &g);
  if (rc) return rc;
  memset(dst, 0, (size_t)(g.panels * rb * g.lpad) * dsize(g.block_dt));
  const int do_conj = (src->conj != 0) != (conj != 0);
  const int32_t tp = prec_of(target);
  const int unit = sc_one(scale);
  mdg_view_t raw = *src;
  raw.conj = 0;
  const int64_t PD = rb, L = g.lpad;
  const int left = side == MDG_SIDE_LEFT;
#define OFF_L(p, r, col) ((p) * PD * L + (col) * PD + (r))
#define OFF_R(p, c, row) ((p) * PD * L + (row) * PD + (c))
#define PROCESS(i, j, re, im)                                         \
  do {                                                                \
    load(&raw, (i), (j), &re, &im);                                   \
    if (do_conj) im = -im;                                            \
    re = rnd(re, tp);                                                 \
    im = rnd(im, tp);                                                 \
    if (!unit) {                                                      \
      double x_, y_;                                                  \
      cmul(re, im, scale.re, scale.im, &x_, &y_);                     \
      re = rnd(x_, tp);                                               \
      im = rnd(y_, tp);                                               \
    }                                                                 \
  } while (0)
  for (int64_t p = 0; p < g.panels; ++p) {
    if (fmt == MDG_FMT_STANDARD) {
      const int64_t outer = left ? src->n : src->m;
      for (int64_t l = 0; l < outer; ++l)
        for (int64_t w = 0; w < PD; ++w) {
          const int64_t x = p * PD + w;
          double re = 0.0, im = 0.0;
          if (left ? x < src->m : x < src->n) {
            if (left) PROCESS(x, l, re, im);
            else PROCESS(l, x, re, im);
          }
          put(dst, g.block_dt, left ? OFF_L(p, w, l) : OFF_R(p, w, l), re, im);
        }
    } else if (fmt == MDG_FMT_ONEE) {
      const int64_t pdc = PD / 2, outer = left ? src->n : src->m;
      for (int64_t lc = 0; lc < outer; ++lc)
        for (int64_t wc = 0; wc < pdc; ++wc) {
          const int64_t x = p * pdc + wc;
          double re = 0.0, im = 0.0;
          if (left ? x < src->m : x < src->n) {
            if (left) PROCESS(x, lc, re, im);
            else PROCESS(lc, x, re, im);
          }
          if (left) {
            put(dst, g.block_dt, OFF_L(p, 2 * wc, 2 * lc), re, 0.0);
            put(dst, g.block_dt, OFF_L(p, 2 * wc, 2 * lc + 1), -im, 0.0);
            put(dst, g.block_dt, OFF_L(p, 2 * wc + 1, 2 * lc), im, 0.0);
            put(dst, g.block_dt, OFF_L(p, 2 * wc + 1, 2 * lc + 1), re, 0.0);
          } else {
            put(dst, g.block_dt, OFF_R(p, 2 * wc, 2 * lc), re, 0.0);
            put(dst, g.block_dt, OFF_R(p, 2 * wc + 1, 2 * lc), im, 0.0);
            put(dst, g.block_dt, OFF_R(p, 2 * wc, 2 * lc + 1), -im, 0.0);
            put(dst, g.block_dt, OFF_R(p, 2 * wc + 1, 2 * lc + 1), re, 0.0);
          }
        }
    } else { /* 1r */
      const int64_t outer = left ? src->n : src->m;
      for (int64_t lc = 0; lc < outer; ++lc)
        for (int64_t w = 0; w < PD; ++w) {
          const int64_t x = p * PD + w;
          double re = 0.0, im = 0.0;
          if (left ? x < src->m : x < src->n) {
            if (left) PROCESS(x, lc, re, im);
            else PROCESS(lc, x, re, im);
          }
          if (left) {
            put(dst, g.block_dt, OFF_L(p, w, 2 * lc), re, 0.0);
            put(dst, g.block_dt, OFF_L(p, w, 2 * lc + 1), im, 0.0);
          } else {
            put(dst, g.block_dt, OFF_R(p, w, 2 * lc), re, 0.0);
            put(dst, g.block_dt, OFF_R(p, w, 2 * lc + 1), im, 0.0);
          }
        }
    }
  }
#undef PROCESS
#undef OFF_L
#undef OFF_R
  return MDG_OK;
}

/* ------------------------------------------------------------ execution */

/* accumulate_element (kernels.cpp:79-95) */
static void combine(const mdg_view_t* c, int64_t i, int64_t j, mdg_scalar_t beta, double tre, double tim) {
  const int32_t sp = prec_of(c->dtype);
  const double cre = rnd(tre, sp), cim = rnd(tim, sp);
  double rre, rim;
  if (sc_zero(beta)) {
    rre = cre;
    rim = cim;
  } else {
    double xre, xim;
    load(c, i, j, &xre, &xim);
    if (sc_one(beta)) {
      rre = rnd(xre + cre, sp);
      rim = rnd(xim + cim, sp);
    } else {
      double bre, bim;
      cmul(beta.re, beta.im, xre, xim, &bre, &bim);
      rre = rnd(rnd(bre, sp) + cre, sp);
      rim = rnd(rnd(bim, sp) + cim, sp);
    }
  }
  if (!is_cplx(c->dtype)) rim = 0.0;
  store(c, i, j, rre, rim);
}

typedef struct {
  const void* a;
  const void* b;
  int64_t pda, pdb, k;
} panels_t;

/* Element (r, l) of Ã and (l, c) of B̃ in the real computation precision. */
#define PANEL_AT(T, base, pd, len, r, l) (((const T*)(base))[((r) / (pd)) * (pd) * (len) + (l) * (pd) + (r) % (pd)])

static double sum_d(const panels_t* P, int64_t r, int64_t c, int64_t lo, int64_t hi, double seed) {
  double acc = seed; /* kernels.cpp:26-35, T = double */
  for (int64_t l = lo; l < hi; ++l)
    acc += PANEL_AT(double, P->a, P->pda, P->k, r, l) * PANEL_AT(double, P->b, P->pdb, P->k, c, l);
  return acc;
}

static float sum_s(const panels_t* P, int64_t r, int64_t c, int64_t lo, int64_t hi, float seed) {
  float acc = seed; /* kernels.cpp:26-35, T = float */
  for (int64_t l = lo; l < hi; ++l)
    acc += PANEL_AT(float, P->a, P->pda, P->k, r, l) * PANEL_AT(float, P->b, P->pdb, P->k, c, l);
  return acc;
}

static double sum_t(int single, const panels_t* P, int64_t r, int64_t c, int64_t lo, int64_t hi) {
  return single ? (double)sum_s(P, r, c, lo, hi, 0.0f) : sum_d(P, r, c, lo, hi, 0.0);
}

static uint64_t flops_of_plan(const mdg_plan_t* p, int direct_ukr) { /* kernels.cpp:73-76 summed over tiles */
  const uint64_t MR = (uint64_t)p->ukr_mr, NR = (uint64_t)p->ukr_nr;
  const uint64_t tiles = (uint64_t)((p->m + p->ukr_mr - 1) / p->ukr_mr) * (uint64_t)((p->n + p->ukr_nr - 1) / p->ukr_nr);
  uint64_t f = 2 * MR * NR * (uint64_t)p->k * tiles;
  if (direct_ukr && p->beta.re != 0.0 && p->beta.re != 1.0) f += MR * NR * tiles;
  return f;
}

int orc_gemm(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta, const mdg_view_t* c,
             const mdg_config_t* cfg, uint64_t* flops) { /* dispatch.cpp:350-389 */
  if (flops) *flops = 0;
  if (overlap(c, a) || overlap(c, b)) return fail(MDG_ERR, "gemm: C must not alias A or B");
  mdg_plan_t p;
  int rc = orc_plan(alpha, a, b, beta, c, cfg, &p);
  if (rc) return rc;
  if (p.m == 0 || p.n == 0) return MDG_OK;
  if (p.k == 0) { /* beta_pass, dispatch.cpp:311-317 */
    if (!(p.beta.re == 1.0 && p.beta.im == 0.0))
      for (int64_t j = 0; j < p.c.n; ++j)
        for (int64_t i = 0; i < p.c.m; ++i) combine(&p.c, i, j, p.beta, 0.0, 0.0);
    return MDG_OK;
  }
  const size_t ba = orc_packed_bytes(&p.a, MDG_SIDE_LEFT, p.format_a, p.target_dtype_a, p.reg_block_a, 0);
  const size_t bb = orc_packed_bytes(&p.b, MDG_SIDE_RIGHT, p.format_b, p.target_dtype_b, p.reg_block_b, 0);
  void* pa = malloc(ba ? ba : 1);
  void* pb = malloc(bb ? bb : 1);
  if (!pa || !pb) {
    free(pa);
    free(pb);
    return fail(MDG_ERR, "orc_gemm: out of memory");
  }
  rc = orc_pack(&p.a, MDG_SIDE_LEFT, p.format_a, p.conj_a, p.pack_scale_a, p.target_dtype_a, p.reg_block_a, 0, pa);
  if (!rc) rc = orc_pack(&p.b, MDG_SIDE_RIGHT, p.format_b, p.conj_b, p.pack_scale_b, p.target_dtype_b, p.reg_block_b, 0, pb);
  if (rc) {
    free(pa);
    free(pb);
    return rc;
  }
  panels_t P;
  P.a = pa;
  P.b = pb;
  P.k = p.k;
  P.pda = p.reg_block_a * ((p.format_a == MDG_FMT_STANDARD && is_cplx(p.a.dtype)) ? 2 : 1);
  P.pdb = p.reg_block_b * ((p.format_b == MDG_FMT_STANDARD && is_cplx(p.b.dtype)) ? 2 : 1);
  const int single = p.comp_prec == MDG_PREC_SINGLE;

  /* Output route of the plan (gemm_core.cpp:43-70 run_tile). */
  enum { R_CTEMP, R_DIRECT, R_TEMP, R_ONEM_MIXED } route = R_TEMP;
  mdg_view_t out = p.c, flat = p.c;
  int32_t pair = p.pair_axis;
  int onem_flat = 0;
  if (p.ukr_path == MDG_PATH_ONEM_COLUMN || p.ukr_path == MDG_PATH_ONEM_ROW) {
    const int rows_axis = p.ukr_path == MDG_PATH_ONEM_COLUMN; /* kernels.cpp:139-146 */
    onem_flat = prec_of(p.c.dtype) == p.comp_prec && can_flatten(&p.c, rows_axis);
    if (onem_flat) flat = real_flat(p.c, rows_axis);
  }
  if (p.has_ctemp) {
    route = R_CTEMP;
  } else if (p.ukr_path == MDG_PATH_DIRECT) {
    route = R_DIRECT;
  } else if (onem_flat) {
    /* virtual_ukr_onem decides per KC block: with a real beta every block is
     * direct; with a complex beta only the first block goes through the
     * temp tile and later blocks (beta = 1) update the flattened C in T. */
    if (p.beta.im == 0.0) {
      route = R_DIRECT;
      out = flat;
      pair = MDG_PAIR_NONE;
    } else {
      route = R_ONEM_MIXED;
    }
  }
  const int direct = route == R_DIRECT;
  const int prow = pair == MDG_PAIR_ROWS, pcol = pair == MDG_PAIR_COLS;
  const int64_t orows = prow ? p.m / 2 : p.m, ocols = pcol ? p.n / 2 : p.n;
  const mdg_scalar_t unit = sc_make(1.0, 0.0, mkdt(0, prec_of(p.beta.dtype)));
  const int64_t KC = p.params.kc;

  for (int64_t oj = 0; oj < ocols; ++oj)
    for (int64_t oi = 0; oi < orows; ++oi) {
      const int64_t r0 = prow ? 2 * oi : oi, c0 = pcol ? 2 * oj : oj;
      const int64_t r1 = prow ? r0 + 1 : r0, c1 = pcol ? c0 + 1 : c0;
      const int two = prow || pcol;
      if (route == R_DIRECT) { /* seeded accumulators stored in T (kernels.cpp:13-24, 37-39) */
        char* cp = eptr(&out, oi, oj);
        if (single) {
          const float bt = (float)p.beta.re;
          float seed = 0.0f;
          if (bt != 0.0f) seed = bt == 1.0f ? *(float*)cp : bt * *(float*)cp;
          *(float*)cp = sum_s(&P, r0, c0, 0, p.k, seed);
        } else {
          const double bt = p.beta.re;
          double seed = 0.0;
          if (bt != 0.0) seed = bt == 1.0 ? *(double*)cp : bt * *(double*)cp;
          *(double*)cp = sum_d(&P, r0, c0, 0, p.k, seed);
        }
      } else if (route == R_CTEMP) { /* C_temp + write_back (dispatch.cpp:366-385) */
        const double t0 = sum_t(single, &P, r0, c0, 0, p.k);
        const double t1 = two ? sum_t(single, &P, r1, c1, 0, p.k) : 0.0;
        combine(&out, oi, oj, p.beta, t0, t1);
      } else if (route == R_ONEM_MIXED) {
        const int64_t hi = KC < p.k ? KC : p.k;
        combine(&out, oi, oj, p.beta, sum_t(single, &P, r0, c0, 0, hi), sum_t(single, &P, r1, c1, 0, hi));
        if (hi < p.k) { /* raw components of the stored element continue in T */
          const int64_t fi0 = prow ? r0 : oi, fj0 = prow ? oj : c0;
          const int64_t fi1 = prow ? r1 : oi, fj1 = prow ? oj : c1;
          char* q0 = eptr(&flat, fi0, fj0);
          char* q1 = eptr(&flat, fi1, fj1);
          if (single) {
            *(float*)q0 = sum_s(&P, r0, c0, hi, p.k, *(float*)q0);
            *(float*)q1 = sum_s(&P, r1, c1, hi, p.k, *(float*)q1);
          } else {
            *(double*)q0 = sum_d(&P, r0, c0, hi, p.k, *(double*)q0);
            *(double*)q1 = sum_d(&P, r1, c1, hi, p.k, *(double*)q1);
          }
        }
      } else { /* temp tile per KC block (gemm_core.cpp:125-127, kernels.cpp:97-132) */
        for (int64_t pc = 0; pc < p.k; pc += KC) {
          const int64_t hi = pc + KC < p.k ? pc + KC : p.k;
          const double t0 = sum_t(single, &P, r0, c0, pc, hi);
          const double t1 = two ? sum_t(single, &P, r1, c1, pc, hi) : 0.0;
          combine(&out, oi, oj, pc == 0 ? p.beta : unit, t0, t1);
        }
      }
    }
  free(pa);
  free(pb);
  if (flops) *flops = flops_of_plan(&p, direct);
  return MDG_OK;
}

/* --------------------------------------------------- brute-force oracle */

static int oracle_scalars(mdg_scalar_t alpha, mdg_scalar_t beta, int32_t id, int32_t comp, int32_t cprec,
                          mdg_scalar_t* ar, mdg_scalar_t* br) { /* oracle.cpp:56-74 */
  if (id != MDG_CASE_0 && id != MDG_CASE_3 && alpha.im != 0.0)
    return fail(MDG_ERR_SCALAR_POLICY, "case %s does not support alpha with a nonzero imaginary part", case_name(id));
  int rc;
  if (id == MDG_CASE_0) *ar = project_sc(alpha, comp);
  else if ((rc = typecast_sc(alpha, mkdt(is_cplx(alpha.dtype), comp), ar))) return rc;
  const int projects = id == MDG_CASE_0 || id == MDG_CASE_1A || id == MDG_CASE_1B || id == MDG_CASE_1C ||
                       id == MDG_CASE_2AB;
  if (projects) *br = project_sc(beta, cprec);
  else if ((rc = typecast_sc(beta, mkdt(is_cplx(beta.dtype), cprec), br))) return rc;
  return MDG_OK;
}

static void operand(const mdg_view_t* v, int drop_im, int64_t i, int64_t j, double* re, double* im) {
  load(v, i, j, re, im);
  if (drop_im) *im = 0.0;
}

int orc_oracle_gemm(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
                    const mdg_view_t* c_in, int32_t comp_prec, void* out_buf) { /* oracle.cpp:92-140 */
  const int32_t id = orc_classify_case(is_cplx(c_in->dtype), is_cplx(a->dtype), is_cplx(b->dtype));
  if (a->m != c_in->m || b->n != c_in->n || a->n != b->m) return fail(MDG_ERR, "oracle_gemm: dimension mismatch");
  mdg_scalar_t as, bs;
  int rc = oracle_scalars(alpha, beta, id, comp_prec, prec_of(c_in->dtype), &as, &bs);
  if (rc) return rc;
  mdg_view_t ov;
  memset(&ov, 0, sizeof ov);
  ov.base = out_buf;
  ov.m = c_in->m;
  ov.n = c_in->n;
  ov.rs = 1;
  ov.cs = c_in->m > 0 ? c_in->m : 1;
  ov.dtype = c_in->dtype;
  const int beta_zero = sc_zero(beta);
  const size_t half = rsize(prec_of(c_in->dtype));
  for (int64_t j = 0; j < c_in->n; ++j)
    for (int64_t i = 0; i < c_in->m; ++i) {
      double sre = 0.0, sim = 0.0;
      for (int64_t l = 0; l < a->n; ++l) {
        double are, aim, bre, bim, x, y;
        operand(a, id == MDG_CASE_1A, i, l, &are, &aim);
        operand(b, id == MDG_CASE_1B, l, j, &bre, &bim);
        cmul(are, aim, bre, bim, &x, &y);
        sre += x;
        sim += y;
      }
      if (id == MDG_CASE_2AB) sim = 0.0;
      if (id == MDG_CASE_1C) {
        double prev = 0.0, dummy;
        if (!beta_zero) {
          const mdg_view_t cr = real_proj(*c_in, 0);
          load(&cr, i, j, &prev, &dummy);
        }
        const double re = as.re * sre + bs.re * prev;
        const mdg_view_t orr = real_proj(ov, 0);
        store(&orr, i, j, re, 0.0);
        memcpy(eptr(&ov, i, j) + half, eptr(c_in, i, j) + half, half);
        continue;
      }
      double pre = 0.0, pim = 0.0;
      if (!beta_zero) load(c_in, i, j, &pre, &pim);
      double x1, y1, x2, y2;
      cmul(as.re, as.im, sre, sim, &x1, &y1);
      cmul(bs.re, bs.im, pre, pim, &x2, &y2);
      double tre = x1 + x2, tim = y1 + y2;
      if (!is_cplx(c_in->dtype)) tim = 0.0;
      store(&ov, i, j, tre, tim);
    }
  return MDG_OK;
}

int orc_violation(mdg_scalar_t alpha, const mdg_view_t* a, const mdg_view_t* b, mdg_scalar_t beta,
                  const mdg_view_t* c_before, const mdg_view_t* c_after, int32_t comp_prec,
                  double* violation) { /* oracle.cpp:142-206 */
  const int64_t m = c_before->m, n = c_before->n, k = a->n;
  const int32_t id = orc_classify_case(is_cplx(c_before->dtype), is_cplx(a->dtype), is_cplx(b->dtype));
  void* ref = malloc((size_t)(m * n > 0 ? m * n : 1) * dsize(c_before->dtype));
  if (!ref) return fail(MDG_ERR, "orc_violation: out of memory");
  int rc = orc_oracle_gemm(alpha, a, b, beta, c_before, comp_prec, ref);
  if (rc) {
    free(ref);
    return rc;
  }
  mdg_view_t rv = *c_before;
  rv.base = ref;
  rv.rs = 1;
  rv.cs = m > 0 ? m : 1;
  rv.conj = 0;
  mdg_scalar_t as, bs; /* magnitude model resolves scalars in double */
  rc = oracle_scalars(alpha, beta, id, MDG_PREC_DOUBLE, MDG_PREC_DOUBLE, &as, &bs);
  if (rc) {
    free(ref);
    return rc;
  }
  const double eps_c = comp_prec == MDG_PREC_SINGLE ? 0x1p-24 : 0x1p-53;
  const double eps_o = is_sgl(c_before->dtype) ? 0x1p-24 : 0x1p-53;
  const double factor = 8.0 * (double)(k + 2) * eps_c + 4.0 * eps_o;
  const int beta_zero = sc_zero(beta);
  const double abs_alpha = hypot(as.re, as.im);
  double worst = 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t l = 0; l < k; ++l) {
        double are, aim, bre, bim;
        operand(a, id == MDG_CASE_1A, i, l, &are, &aim);
        operand(b, id == MDG_CASE_1B, l, j, &bre, &bim);
        acc += hypot(are, aim) * hypot(bre, bim);
      }
      double cterm = 0.0;
      if (!beta_zero) {
        double pre, pim, x, y;
        if (id == MDG_CASE_1C) {
          const mdg_view_t cr = real_proj(*c_before, 0);
          load(&cr, i, j, &pre, &pim);
        } else {
          load(c_before, i, j, &pre, &pim);
        }
        cmul(bs.re, bs.im, pre, pim, &x, &y);
        cterm = hypot(x, y);
      }
      const double mag = abs_alpha * acc + cterm;
      const double tol = factor * mag;
      double gre, gim, wre, wim;
      load(c_after, i, j, &gre, &gim);
      load(&rv, i, j, &wre, &wim);
      const double diff = hypot(gre - wre, gim - wim);
      double v;
      if (isnan(diff) || isnan(tol)) v = INFINITY;
      else if (diff == 0.0) v = 0.0;
      else if (tol == 0.0) v = INFINITY;
      else v = diff / tol;
      if (v > worst) worst = v;
    }
  free(ref);
  *violation = worst;
  return MDG_OK;
}
