// mdgemm_b200 -- command line front end of the B200 gemm, mirroring the
// reference CLI's `test`, `bench` and `info` subcommands
// (tools/mdgemm.cpp:54-181) and its CSV contract
// `case,m,n,k,trials,best_seconds,gflops` (bench.cpp:53-64).  Operands are
// drawn from the reference's seeded Rng (Rng(seed).split(label).split("bench")
// .split("a"|"b"|"c"), bench.cpp:18-24), so a CSV row here and a row of the
// reference CLI time the same numbers.
//
//   mdgemm_b200 test  [--case L ...|all] [--size N ...] [--no-storage-sweep]
//                     [--no-scalar-sweep] [--seed S] [--config FILE]
//                     [--ctemp auto|on|off] [--numerics fast|exact]
//   mdgemm_b200 bench [--case L ...|all] [--size N | --min N --max N --step N]
//                     [--trials T] [--out FILE] [--seed S] [--config FILE]
//                     [--ctemp auto|on|off] [--numerics fast|exact] [--host]
//                     [--gpus N] [--roofline]
//   mdgemm_b200 info  [--config FILE]
//
// test  replays the reference's conformance sweep (conformance.cpp:131-206:
//       sizes, the 13x7x19 rectangle, row/general C, transposed and
//       conjugated operands, the alpha x beta grid and the complex-alpha
//       rejections) through gemm() on host operands, checking every output
//       element against the reference's per-element bound
//       8(k+2)eps_comp|mag| + 4eps_out|mag| (oracle.cpp:169-206) with a
//       brute-force complex<double> product computed here on the host.
// bench --host keeps A, B, C in host memory (gemm() stages them through HBM
//       per call, as a reference caller would); the default keeps them in
//       HBM.  --gpus N runs every point through gemm_multi() over devices
//       0..N-1 (C/B column panels, A broadcast; operands in host memory).
//       --roofline appends gpus,peak_gflops,frac_of_peak: the measured
//       per-GPU peak of the computation precision (tools/peaks.cu: 37.0
//       TFLOP/s DMMA fp64, 72.0 FFMA fp32 on this pool's B200s; override
//       with MDGEMM_PEAK_D / MDGEMM_PEAK_S in GFLOPS) times N.
#include <chrono>
#include <complex>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <limits>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "mdgemm/mdgemm.hpp"
#include "mdgemm_b200.h"

using namespace mdgemm;

namespace {

struct Args {
  std::string cmd;
  std::vector<std::string> cases;
  int64_t size = 0, min = 0, max = 0, step = 0;
  int trials = 3;
  std::string out, config, ctemp, numerics;
  uint64_t seed = 42;
  bool host = false, roofline = false, no_storage = false, no_scalars = false;
  int gpus = 0;
  std::vector<int64_t> sizes;
};

[[noreturn]] void usage(const std::string& why) {
  std::cerr << "mdgemm_b200: " << why << "\n"
            << "usage: mdgemm_b200 test  [--case L ...|all] [--size N ...] [--no-storage-sweep] [--no-scalar-sweep]\n"
               "                         [--seed S] [--config FILE] [--ctemp auto|on|off] [--numerics fast|exact]\n"
               "       mdgemm_b200 bench [--case L ...|all] [--size N | --min N --max N --step N] [--trials T]\n"
               "                         [--out FILE] [--seed S] [--config FILE] [--ctemp auto|on|off]\n"
               "                         [--numerics fast|exact] [--host] [--gpus N] [--roofline]\n"
               "       mdgemm_b200 info  [--config FILE]\n";
  std::exit(2);
}

Args parse(int argc, char** argv) {
  if (argc < 2) usage("missing subcommand");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) usage("option " + k + " needs a value");
      return argv[++i];
    };
    if (k == "--case") a.cases.push_back(val());
    else if (k == "--size") {
      a.size = std::stoll(val());
      a.sizes.push_back(a.size);
    }
    else if (k == "--min") a.min = std::stoll(val());
    else if (k == "--max") a.max = std::stoll(val());
    else if (k == "--step") a.step = std::stoll(val());
    else if (k == "--trials") a.trials = std::stoi(val());
    else if (k == "--out") a.out = val();
    else if (k == "--seed") a.seed = std::stoull(val());
    else if (k == "--config") a.config = val();
    else if (k == "--ctemp") a.ctemp = val();
    else if (k == "--numerics") a.numerics = val();
    else if (k == "--host") a.host = true;
    else if (k == "--gpus") a.gpus = std::stoi(val());
    else if (k == "--roofline") a.roofline = true;
    else if (k == "--no-storage-sweep") a.no_storage = true;
    else if (k == "--no-scalar-sweep") a.no_scalars = true;
    else usage("unknown option " + k);
  }
  if (a.gpus < 0) usage("--gpus must be >= 1");
  if (a.gpus > 0 && a.cmd == "bench") a.host = true;  // gemm_multi takes operands anywhere; keep them on the host
  return a;
}

Config resolve(const Args& a) {
  Config cfg = Config::load(a.config.empty() ? std::nullopt : std::optional<std::string>(a.config));
  if (!a.ctemp.empty()) cfg.set("ctemp.enable", a.ctemp);
  if (!a.numerics.empty()) cfg.set("gpu.numerics", a.numerics);
  cfg.validate();
  return cfg;
}

// Column-major operand in host or device memory, filled from an Rng state.
struct Operand {
  Datatype dt;
  int64_t m, n;
  bool on_host;
  std::vector<std::byte> host;
  void* dev = nullptr;

  Operand(Datatype t, int64_t rows, int64_t cols, bool h) : dt(t), m(rows), n(cols), on_host(h) {
    const size_t bytes = static_cast<size_t>(std::max<int64_t>(m * n, 1)) * dtype_size(dt);
    if (on_host) host.resize(bytes);
    else if (cudaMalloc(&dev, bytes) != cudaSuccess) throw Error("cudaMalloc failed");
  }
  ~Operand() {
    if (dev) cudaFree(dev);
  }
  void* base() { return on_host ? static_cast<void*>(host.data()) : dev; }
  size_t bytes() const { return static_cast<size_t>(std::max<int64_t>(m * n, 1)) * dtype_size(dt); }
  MatrixView view() { return MatrixView::make(base(), m, n, 1, std::max<int64_t>(m, 1), dt); }

  void fill(uint64_t state) {
    // draw on the device (bit-identical to Rng/fill_uniform), then copy down if host-resident
    void* target = dev;
    void* tmp = nullptr;
    if (on_host) {
      if (cudaMalloc(&tmp, bytes()) != cudaSuccess) throw Error("cudaMalloc failed");
      target = tmp;
    }
    mdg_view_t v{target, m, n, 1, std::max<int64_t>(m, 1),
                 (dt.domain == Domain::Complex ? 2 : 0) + (dt.precision == Precision::Double ? 1 : 0), 0,
                 dt.precision == Precision::Double ? 1 : 0, 0};
    if (mdg_fill_uniform(&v, state, nullptr) != MDG_OK) throw Error(mdg_last_error());
    if (on_host) {
      cudaMemcpy(host.data(), tmp, bytes(), cudaMemcpyDeviceToHost);
      cudaFree(tmp);
    }
    cudaDeviceSynchronize();
  }
};

void copy_operand(Operand& dst, const Operand& src) {
  if (dst.on_host) std::memcpy(dst.host.data(), src.host.data(), src.bytes());
  else cudaMemcpy(dst.dev, src.dev, src.bytes(), cudaMemcpyDeviceToDevice);
}

// Measured per-GPU peaks (GFLOPS) of the computation precision's pipe
// (profiles/peaks_r01.json, tools/peaks.cu at 1965 MHz).
double peak_gflops(Precision comp) {
  const char* env = std::getenv(comp == Precision::Double ? "MDGEMM_PEAK_D" : "MDGEMM_PEAK_S");
  if (env && *env) return std::stod(env);
  return comp == Precision::Double ? 37000.0 : 72000.0;
}

struct Row {
  std::string label;
  int64_t m, n, k;
  int trials;
  double best_seconds, gflops;
};

// run_bench conventions (bench.cpp:13-51): one warm-up, best of `trials`,
// C restored outside the timed region, gflops from flops_of_case.
Row bench_one(const CaseLabel& label, int64_t s, int trials, const Config& cfg, uint64_t seed, bool host,
              int gpus) {
  uint64_t rng = mdg_rng_split_tag(mdg_rng_split_tag(seed, label.str().c_str()), "bench");
  Operand A(label.a, s, s, host), B(label.b, s, s, host), C(label.c, s, s, host), C0(label.c, s, s, host);
  A.fill(mdg_rng_split_tag(rng, "a"));
  B.fill(mdg_rng_split_tag(rng, "b"));
  C0.fill(mdg_rng_split_tag(rng, "c"));
  copy_operand(C, C0);
  const Scalar one = Scalar::real_value(1.0);
  const MatrixView vc = C.view().with_comp_prec(label.comp);
  std::vector<int> devices;
  for (int g = 0; g < gpus; ++g) devices.push_back(g);
  auto run = [&] {
    if (gpus > 0) gemm_multi(one, A.view(), B.view(), one, vc, cfg, devices);
    else gemm(one, A.view(), B.view(), one, vc, cfg);
  };
  run();  // warm-up
  double best = std::numeric_limits<double>::infinity();
  for (int t = 0; t < trials; ++t) {
    copy_operand(C, C0);
    cudaDeviceSynchronize();
    const auto t0 = std::chrono::steady_clock::now();
    run();
    const auto t1 = std::chrono::steady_clock::now();
    best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
  }
  const double flops = static_cast<double>(flops_of_case(label.case_id(), s, s, s));
  return Row{label.str(), s, s, s, trials, best, flops / best / 1e9};
}

int cmd_bench(const Args& a) {
  const Config cfg = resolve(a);
  std::vector<CaseLabel> labels;
  for (const std::string& c : a.cases) {
    if (c == "all") {
      labels = CaseLabel::all();
      break;
    }
    labels.push_back(CaseLabel::parse(c));
  }
  if (labels.empty()) labels.push_back(CaseLabel::parse("dddd"));
  std::vector<int64_t> sizes;
  if (a.size > 0) sizes.push_back(a.size);
  else if (a.min > 0 && a.max >= a.min && a.step > 0)
    for (int64_t s = a.min; s <= a.max; s += a.step) sizes.push_back(s);
  else sizes.push_back(1024);

  std::ofstream file;
  std::ostream* os = &std::cout;
  if (!a.out.empty()) {
    file.open(a.out);
    if (!file) throw Error("cannot open output file: " + a.out);
    os = &file;
  }
  *os << "case,m,n,k,trials,best_seconds,gflops" << (a.roofline ? ",gpus,peak_gflops,frac_of_peak" : "") << "\n";
  const int ngpu = std::max(a.gpus, 1);
  for (const CaseLabel& l : labels)
    for (int64_t s : sizes) {
      const Row r = bench_one(l, s, a.trials, cfg, a.seed, a.host, a.gpus);
      std::ostringstream line;
      line << r.label << ',' << r.m << ',' << r.n << ',' << r.k << ',' << r.trials << ',' << std::setprecision(9)
           << r.best_seconds << ',' << std::setprecision(4) << r.gflops;
      if (a.roofline) {
        const double peak = peak_gflops(l.comp) * ngpu;
        line << ',' << ngpu << ',' << std::setprecision(6) << peak << ',' << std::setprecision(4) << r.gflops / peak;
      }
      *os << line.str() << "\n";
      os->flush();
    }
  return 0;
}

// ------------------------------------------------------------------ test
// The reference conformance sweep (conformance.cpp:131-206) against this
// library.  Operand draws follow run_one (conformance.cpp:46-60):
// Rng(seed).split(label).split(variant).split(m*1000003 + n*1009 + k), then
// "a" / "b" / "c", fill order j-major, i-minor (rng.hpp:49-56; the device
// generator is bit-identical).  The checker is a brute-force complex<double>
// product with the reference's scalar resolution and per-element bound
// (oracle.cpp:9-206), written here; it is the CLI's own, not the test oracle.

struct HostMat {
  Datatype dt;
  int64_t m = 0, n = 0, rs = 1, cs = 1;
  std::vector<std::byte> buf;
  MatrixView view() const { return MatrixView::make(const_cast<std::byte*>(buf.data()), m, n, rs, cs, dt); }
};

HostMat host_mat(Datatype dt, int64_t m, int64_t n, StorageKind kind) {  // Matrix::make (matrix.hpp:17-43)
  HostMat h;
  h.dt = dt;
  h.m = m;
  h.n = n;
  switch (kind) {
    case StorageKind::ColumnStored: h.rs = 1; h.cs = std::max<int64_t>(m, 1); break;
    case StorageKind::RowStored: h.cs = 1; h.rs = std::max<int64_t>(n, 1); break;
    case StorageKind::GeneralStored: h.rs = 2; h.cs = 2 * std::max<int64_t>(m, 1) + 3; break;
  }
  const int64_t span = (m > 0 && n > 0) ? (m - 1) * h.rs + (n - 1) * h.cs + 1 : 0;
  h.buf.assign(static_cast<size_t>(span) * dtype_size(dt), std::byte{0});
  return h;
}

int dt_code(Datatype dt) { return (dt.domain == Domain::Complex ? 2 : 0) + (dt.precision == Precision::Double ? 1 : 0); }

void fill_host(HostMat& h, uint64_t state) {
  if (h.buf.empty()) return;
  void* d = nullptr;
  if (cudaMalloc(&d, h.buf.size()) != cudaSuccess) throw Error("cudaMalloc failed");
  cudaMemset(d, 0, h.buf.size());
  const int code = dt_code(h.dt);
  mdg_view_t v{d, h.m, h.n, h.rs, h.cs, code, 0, h.dt.precision == Precision::Double ? 1 : 0, code};
  const int rc = mdg_fill_uniform(&v, state, nullptr);
  cudaMemcpy(h.buf.data(), d, h.buf.size(), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (rc != MDG_OK) throw Error(mdg_last_error());
}

bool beta_projects(CaseId c) {
  return c == CaseId::C0 || c == CaseId::C1a || c == CaseId::C1b || c == CaseId::C1c || c == CaseId::C2ab;
}

// Largest |impl - ref| / tol over C (max_violation, oracle.cpp:185-206); the
// reference value is rounded to C's storage precision like oracle_gemm's
// output matrix, Im of a case-1c C is the input's.
double violation(const CaseLabel& label, Scalar alpha, Scalar beta, const MatrixView& a, const MatrixView& b,
                 const MatrixView& c_in, const MatrixView& c_out) {
  const CaseId id = label.case_id();
  const std::complex<double> al =
      (id == CaseId::C0 ? project_scalar(alpha, label.comp)
                        : typecast_scalar(alpha, Datatype{alpha.dtype.domain, label.comp})).value();
  const Precision cp = label.c.precision;
  const std::complex<double> be =
      (beta_projects(id) ? project_scalar(beta, cp) : typecast_scalar(beta, Datatype{beta.dtype.domain, cp})).value();
  // the magnitude matrix resolves the scalars at double precision (oracle.cpp:146-147)
  const double mal = std::abs((id == CaseId::C0 ? project_scalar(alpha, Precision::Double)
                                                : typecast_scalar(alpha, Datatype{alpha.dtype.domain, Precision::Double}))
                                  .value());
  const std::complex<double> mbe =
      (beta_projects(id) ? project_scalar(beta, Precision::Double)
                         : typecast_scalar(beta, Datatype{beta.dtype.domain, Precision::Double})).value();
  const bool bz = beta.is_zero();
  const int64_t m = c_in.m, n = c_in.n, k = a.n;
  const double factor = 8.0 * static_cast<double>(k + 2) * eps_of(label.comp) + 4.0 * eps_of(cp);
  auto rd = [&](std::complex<double> v) {
    return cp == Precision::Single ? std::complex<double>(static_cast<float>(v.real()), static_cast<float>(v.imag())) : v;
  };
  double worst = 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      std::complex<double> sum{0.0, 0.0};
      double mag = 0.0;
      for (int64_t l = 0; l < k; ++l) {
        std::complex<double> x = load_elem(a, i, l), y = load_elem(b, l, j);
        if (id == CaseId::C1a) x = {x.real(), 0.0};
        if (id == CaseId::C1b) y = {y.real(), 0.0};
        sum += x * y;
        mag += std::abs(x) * std::abs(y);
      }
      if (id == CaseId::C2ab) sum = {sum.real(), 0.0};
      const std::complex<double> c0 = load_elem(c_in, i, j);
      std::complex<double> ref;
      double cterm = 0.0;
      if (id == CaseId::C1c) {
        const double prev = bz ? 0.0 : c0.real();
        ref = rd({al.real() * sum.real() + be.real() * prev, 0.0});
        ref = {ref.real(), c0.imag()};
        if (!bz) cterm = std::abs(mbe * std::complex<double>(c0.real(), 0.0));
      } else {
        std::complex<double> t = al * sum + be * (bz ? std::complex<double>{} : c0);
        if (c_in.dtype.domain == Domain::Real) t = {t.real(), 0.0};
        ref = rd(t);
        if (!bz) cterm = std::abs(mbe * c0);
      }
      const double tol = factor * (mal * mag + cterm);
      const double diff = std::abs(load_elem(c_out, i, j) - ref);
      double v;
      if (std::isnan(diff) || std::isnan(tol)) v = std::numeric_limits<double>::infinity();
      else if (diff == 0.0) v = 0.0;
      else if (tol == 0.0) v = std::numeric_limits<double>::infinity();
      else v = diff / tol;
      worst = std::max(worst, v);
    }
  return worst;
}

struct Variant {
  const char* name = "base";
  StorageKind c_store = StorageKind::ColumnStored;
  bool ta = false, tb = false, ca = false, cb = false;
  Scalar alpha = Scalar::real_value(1.0), beta = Scalar::real_value(1.0);
  bool reject = false;
};

struct Report {
  int64_t checks = 0;
  std::vector<std::string> failures;
};

std::string scalar_str(const Scalar& s) {
  std::ostringstream os;
  os << s.re;
  if (s.dtype.domain == Domain::Complex) os << (s.im < 0 ? "" : "+") << s.im << "i";
  return os.str();
}

void run_one(const CaseLabel& label, int64_t m, int64_t n, int64_t k, const Variant& v, uint64_t root,
             const Config& cfg, Report& rep) {
  const uint64_t rng = mdg_rng_split_salt(mdg_rng_split_tag(mdg_rng_split_tag(root, label.str().c_str()), v.name),
                                          static_cast<uint64_t>(m * 1000003 + n * 1009 + k));
  HostMat am = host_mat(label.a, v.ta ? k : m, v.ta ? m : k, StorageKind::ColumnStored);
  HostMat bm = host_mat(label.b, v.tb ? n : k, v.tb ? k : n, StorageKind::ColumnStored);
  HostMat cm = host_mat(label.c, m, n, v.c_store);
  fill_host(am, mdg_rng_split_tag(rng, "a"));
  fill_host(bm, mdg_rng_split_tag(rng, "b"));
  fill_host(cm, mdg_rng_split_tag(rng, "c"));
  MatrixView va = v.ta ? induced_transpose(am.view()) : am.view();
  MatrixView vb = v.tb ? induced_transpose(bm.view()) : bm.view();
  if (v.ca && label.a.domain == Domain::Complex) va = va.with_conj(true);
  if (v.cb && label.b.domain == Domain::Complex) vb = vb.with_conj(true);
  std::ostringstream what;
  what << label.str() << " m=" << m << " n=" << n << " k=" << k << " variant=" << v.name
       << " alpha=" << scalar_str(v.alpha) << " beta=" << scalar_str(v.beta);
  ++rep.checks;
  HostMat work = cm;
  const MatrixView vw = work.view().with_comp_prec(label.comp);
  if (v.reject) {
    bool threw = false;
    try {
      gemm(v.alpha, va, vb, v.beta, vw, cfg);
    } catch (const ScalarPolicyError&) {
      threw = true;
    }
    if (!threw) rep.failures.push_back(what.str() + ": expected scalar rejection missing");
    else if (work.buf != cm.buf) rep.failures.push_back(what.str() + ": C written by a rejected call");
    return;
  }
  try {
    gemm(v.alpha, va, vb, v.beta, vw, cfg);
  } catch (const std::exception& e) {
    rep.failures.push_back(what.str() + ": implementation raised: " + e.what());
    return;
  }
  const double viol = violation(label, v.alpha, v.beta, va, vb, cm.view(), work.view());
  if (!(viol <= 1.0)) {
    std::ostringstream os;
    os << what.str() << ": error bound exceeded violation=" << viol;
    rep.failures.push_back(os.str());
  }
}

int cmd_test(const Args& a) {
  const Config cfg = resolve(a);
  std::vector<CaseLabel> labels;
  for (const std::string& c : a.cases) {
    if (c == "all") {
      labels.clear();
      break;
    }
    labels.push_back(CaseLabel::parse(c));
  }
  if (labels.empty()) labels = CaseLabel::all();
  const std::vector<int64_t> sizes = a.sizes.empty() ? std::vector<int64_t>{7, 16, 17, 64} : a.sizes;
  const uint64_t root = a.seed;
  Report rep;
  for (const CaseLabel& label : labels) {
    for (int64_t s : sizes) run_one(label, s, s, s, Variant{}, root, cfg, rep);
    run_one(label, 13, 7, 19, Variant{.name = "rectangular"}, root, cfg, rep);
    if (!a.no_storage) {
      const int64_t s = 17;
      const bool ca = label.a.domain == Domain::Complex, cb = label.b.domain == Domain::Complex;
      run_one(label, s, s, s, Variant{.name = "c_row", .c_store = StorageKind::RowStored}, root, cfg, rep);
      run_one(label, s, s, s, Variant{.name = "c_general", .c_store = StorageKind::GeneralStored}, root, cfg, rep);
      run_one(label, s, s, s, Variant{.name = "a_transposed", .ta = true}, root, cfg, rep);
      run_one(label, s, s, s, Variant{.name = "b_transposed", .tb = true}, root, cfg, rep);
      if (ca) run_one(label, s, s, s, Variant{.name = "a_conjugated", .ca = true}, root, cfg, rep);
      if (cb) run_one(label, s, s, s, Variant{.name = "b_conjugated", .cb = true}, root, cfg, rep);
      run_one(label, s, s, s,
              Variant{.name = "row_transposed", .c_store = StorageKind::RowStored, .ta = true, .tb = true}, root, cfg,
              rep);
      run_one(label, s, s, s,
              Variant{.name = "general_mixed", .c_store = StorageKind::GeneralStored, .ta = true, .ca = true,
                      .cb = true},
              root, cfg, rep);
    }
    if (!a.no_scalars) {
      const int64_t s = 16;
      const Scalar alphas[] = {Scalar::real_value(0.0), Scalar::real_value(1.0), Scalar::real_value(-1.0),
                               Scalar::real_value(0.7)};
      const Scalar betas[] = {Scalar::real_value(0.0), Scalar::real_value(1.0), Scalar::real_value(0.3),
                              Scalar::complex_value(0.3, 0.4)};
      for (const Scalar& al : alphas)
        for (const Scalar& be : betas) run_one(label, s, s, s, Variant{.name = "scalars", .alpha = al, .beta = be}, root, cfg, rep);
      const CaseId id = label.case_id();
      run_one(label, s, s, s,
              Variant{.name = "complex_alpha", .alpha = Scalar::complex_value(0.5, 0.5),
                      .reject = id != CaseId::C0 && id != CaseId::C3},
              root, cfg, rep);
    }
  }
  std::cout << rep.checks << " checks, " << rep.failures.size() << " failures\n";
  for (size_t i = 0; i < rep.failures.size(); ++i) {
    if (i == 25) {
      std::cout << "... (" << rep.failures.size() - 25 << " more)\n";
      break;
    }
    std::cout << "FAIL " << rep.failures[i] << "\n";
  }
  return rep.failures.empty() ? 0 : 1;
}

int cmd_info(const Args& a) {
  const Config cfg = resolve(a);
  std::cout << cfg.describe();
  std::cout << "\nlabels: 128 (C, A, B over s/d/c/z; computation precision s/d)\n"
            << "domain cases: 0, 1a, 1b, 1c, 2ab, 2ac, 2bc, 3\n";
  int dev = 0, sms = 0;
  cudaDeviceProp prop{};
  if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&prop, dev) == cudaSuccess) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    std::cout << "device: " << prop.name << " (sm_" << prop.major << prop.minor << ", " << sms << " SMs, "
              << prop.totalGlobalMem / (1 << 20) << " MiB)\n";
  } else {
    std::cout << "device: none visible\n";
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const Args a = parse(argc, argv);
  try {
    if (a.cmd == "test") return cmd_test(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "info") return cmd_info(a);
    usage("unknown subcommand " + a.cmd);
  } catch (const std::exception& e) {
    std::cerr << "mdgemm_b200: " << e.what() << "\n";
    return 1;
  }
}
