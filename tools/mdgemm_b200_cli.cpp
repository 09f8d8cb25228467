// mdgemm_b200 -- command line front end of the B200 gemm, mirroring the
// reference CLI's `bench` and `info` subcommands (tools/mdgemm.cpp:86-127)
// and its CSV contract `case,m,n,k,trials,best_seconds,gflops`
// (bench.cpp:53-64).  Operands are drawn from the reference's seeded Rng
// (Rng(seed).split(label).split("bench").split("a"|"b"|"c"), bench.cpp:18-24),
// so a CSV row here and a row of the reference CLI time the same numbers.
//
//   mdgemm_b200 bench [--case L ...|all] [--size N | --min N --max N --step N]
//                     [--trials T] [--out FILE] [--seed S] [--config FILE]
//                     [--ctemp auto|on|off] [--numerics fast|exact] [--host]
//   mdgemm_b200 info  [--config FILE]
//
// --host keeps A, B, C in host memory (gemm() stages them through HBM per
// call, as a reference caller would); the default keeps them in HBM.
#include <chrono>
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
  bool host = false;
};

[[noreturn]] void usage(const std::string& why) {
  std::cerr << "mdgemm_b200: " << why << "\n"
            << "usage: mdgemm_b200 bench [--case L ...|all] [--size N | --min N --max N --step N] [--trials T]\n"
               "                         [--out FILE] [--seed S] [--config FILE] [--ctemp auto|on|off]\n"
               "                         [--numerics fast|exact] [--host]\n"
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
    else if (k == "--size") a.size = std::stoll(val());
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
    else usage("unknown option " + k);
  }
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

struct Row {
  std::string label;
  int64_t m, n, k;
  int trials;
  double best_seconds, gflops;
};

// run_bench conventions (bench.cpp:13-51): one warm-up, best of `trials`,
// C restored outside the timed region, gflops from flops_of_case.
Row bench_one(const CaseLabel& label, int64_t s, int trials, const Config& cfg, uint64_t seed, bool host) {
  uint64_t rng = mdg_rng_split_tag(mdg_rng_split_tag(seed, label.str().c_str()), "bench");
  Operand A(label.a, s, s, host), B(label.b, s, s, host), C(label.c, s, s, host), C0(label.c, s, s, host);
  A.fill(mdg_rng_split_tag(rng, "a"));
  B.fill(mdg_rng_split_tag(rng, "b"));
  C0.fill(mdg_rng_split_tag(rng, "c"));
  copy_operand(C, C0);
  const Scalar one = Scalar::real_value(1.0);
  const MatrixView vc = C.view().with_comp_prec(label.comp);
  gemm(one, A.view(), B.view(), one, vc, cfg);  // warm-up
  double best = std::numeric_limits<double>::infinity();
  for (int t = 0; t < trials; ++t) {
    copy_operand(C, C0);
    cudaDeviceSynchronize();
    const auto t0 = std::chrono::steady_clock::now();
    gemm(one, A.view(), B.view(), one, vc, cfg);
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
  *os << "case,m,n,k,trials,best_seconds,gflops\n";
  for (const CaseLabel& l : labels)
    for (int64_t s : sizes) {
      const Row r = bench_one(l, s, a.trials, cfg, a.seed, a.host);
      std::ostringstream line;
      line << r.label << ',' << r.m << ',' << r.n << ',' << r.k << ',' << r.trials << ',' << std::setprecision(9)
           << r.best_seconds << ',' << std::setprecision(4) << r.gflops;
      *os << line.str() << "\n";
      os->flush();
    }
  return 0;
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
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "info") return cmd_info(a);
    usage("unknown subcommand " + a.cmd);
  } catch (const std::exception& e) {
    std::cerr << "mdgemm_b200: " << e.what() << "\n";
    return 1;
  }
}
