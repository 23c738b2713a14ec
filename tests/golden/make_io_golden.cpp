// make_io_golden.cpp — TEST INFRASTRUCTURE: writes the reference's result and
// wire formats (proj/src/io.cpp, unchanged, compiled in by
// make_io_golden.sh) for fixed inputs into tests/golden/io/, so that the
// restatements (paper_1907_13428_b200/io.py, include/fdeopt_b200_io.hpp) are
// checked byte for byte without /root/reference.
#include <cmath>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include "fdeopt/io.hpp"

using namespace fdeopt;

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  // dump: n = 3, field 1, 27 values incl. -0, +-inf, a subnormal, extremes
  std::vector<double> v(27);
  for (int i = 0; i < 27; ++i) v[i] = std::sin(0.37 * i) * std::pow(10.0, (i % 7) - 3);
  v[3] = -0.0;
  v[5] = std::numeric_limits<double>::infinity();
  v[6] = -std::numeric_limits<double>::infinity();
  v[7] = std::numeric_limits<double>::denorm_min();
  v[8] = std::numeric_limits<double>::max();
  dump_solution(dir + "/u.bin", 3, 1, v);
  dump_solution(dir + "/empty.bin", 0, 0, {});
  write_dump_manifest(dir + "/manifest.txt", 3, {{"y.bin", 0}, {"u.bin", 1}});
  // summary rows: formatting of every %.12g field
  SummaryRow r{12, 1728, 0.7, 1.3, 1.2999999999999998, 1e-4, 0.4, 1.618, 0.0123456789012345,
               3.5e-17, 13.4615384615, 42, 1234.5678901234567, "converged"};
  SummaryRow f{8, 512, 0.5, 1.5, 1.5, 2.5e-300, 1e+21, 1.0, std::numeric_limits<double>::infinity(),
               -std::numeric_limits<double>::infinity(), 0.0, 0, 0.1, "failed"};
  std::ofstream csv(dir + "/summary.csv");
  csv << kSummaryHeader << "\n" << summary_csv_row(r) << "\n" << summary_csv_row(f) << "\n";
  std::ofstream plain(dir + "/summary_plain.txt");
  plain << summary_plain_row(r) << "\n" << summary_plain_row(f) << "\n";
  // iteration log
  std::vector<IterRecord> hist(3);
  for (int k = 0; k < 3; ++k) {
    hist[k].iter = k + 1;
    hist[k].r_eq = 0.1 / (k + 1);
    hist[k].r_y = 1e-7 * (k + 2);
    hist[k].r_u = 2.0 / 3.0 * k;
    hist[k].dual_inf = std::pow(10.0, -k) * M_PI;
    hist[k].inner_iters = 10 + k;
    hist[k].inner_tol = 5e-6;
  }
  std::ofstream log(dir + "/iterations.csv");
  write_iteration_log(log, hist);
  return 0;
}
