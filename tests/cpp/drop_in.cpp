// Drop-in check: a caller written against the reference's public C++ API
// (mdgemm/dispatch.hpp, dispatch.hpp:84-91) with HOST buffers, linked against
// libmdgemm_b200.so instead of the reference library.
//
//   drop_in <label> <m> <n> <k> <alpha_re> <alpha_im> <beta_re> <beta_im>
//           <fast|exact> <A.bin> <B.bin> <C.bin> <out.bin>
//
// A, B, C are column-major byte images of the label's storage datatypes; the
// updated C is written to out.bin and the FlopCounter value to stdout.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <iterator>
#include <string>
#include <vector>

#include "mdgemm/dispatch.hpp"

using namespace mdgemm;

static std::vector<std::byte> slurp(const char* path) {
  std::ifstream in(path, std::ios::binary);
  std::vector<char> raw((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::vector<std::byte> out(raw.size());
  for (size_t i = 0; i < raw.size(); ++i) out[i] = std::byte(raw[i]);
  return out;
}

int main(int argc, char** argv) {
  if (argc != 14) {
    std::cerr << "usage: drop_in label m n k are aim bre bim fast|exact A B C out\n";
    return 2;
  }
  const CaseLabel label = CaseLabel::parse(argv[1]);
  const int64_t m = std::stoll(argv[2]), n = std::stoll(argv[3]), k = std::stoll(argv[4]);
  const double are = std::stod(argv[5]), aim = std::stod(argv[6]);
  const double bre = std::stod(argv[7]), bim = std::stod(argv[8]);
  Config cfg = Config::defaults();
  cfg.set("gpu.numerics", argv[9]);
  auto a = slurp(argv[10]), b = slurp(argv[11]), c = slurp(argv[12]);
  const MatrixView va = MatrixView::make(a.data(), m, k, 1, m > 0 ? m : 1, label.a);
  const MatrixView vb = MatrixView::make(b.data(), k, n, 1, k > 0 ? k : 1, label.b);
  const MatrixView vc = MatrixView::make(c.data(), m, n, 1, m > 0 ? m : 1, label.c).with_comp_prec(label.comp);
  const Scalar alpha = aim != 0.0 ? Scalar::complex_value(are, aim) : Scalar::real_value(are);
  const Scalar beta = bim != 0.0 ? Scalar::complex_value(bre, bim) : Scalar::real_value(bre);
  FlopCounter fc;
  try {
    gemm(alpha, va, vb, beta, vc, cfg, &fc);
  } catch (const ScalarPolicyError& e) {
    std::cout << "ScalarPolicyError: " << e.what() << "\n";
    return 3;
  } catch (const Error& e) {
    std::cout << "Error: " << e.what() << "\n";
    return 4;
  }
  std::ofstream out(argv[13], std::ios::binary);
  out.write(reinterpret_cast<const char*>(c.data()), static_cast<std::streamsize>(c.size()));
  std::cout << fc.value() << "\n";
  return 0;
}
