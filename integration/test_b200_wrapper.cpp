// Exercises integration/qbx3d/b200.hpp compiled against the reference's own header
// (/root/reference/proj/include) and linked with libqbxg.so and the reference's compiled
// kernels.cpp (oracle/_ref/libqbxref.so).  Prints one line per check; exit code 0 = all
// passed, 77 = no CUDA device (the device-free checks still ran and passed).
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "qbx3d/b200.hpp"

namespace {
int failures = 0;
void check(bool ok, const char* what) {
  std::printf("%s %s\n", ok ? "ok  " : "FAIL", what);
  if (!ok) ++failures;
}
}  // namespace

int main() {
  using namespace qbx;
  // device-free: argument errors map to std::invalid_argument before any device work
  {
    qbxg_config cfg{};
    cfg.p_fmm = 3;
    cfg.p_qbx = 5;  // p_qbx > p_fmm
    cfg.t_f = 0.9;
    cfg.n_max = 64;
    std::vector<double> p{0, 0, 0}, c{0, 0, 1}, r{0.1};
    qbxg_geometry g{1, p.data(), 1, c.data(), r.data(), 0, nullptr, nullptr};
    bool thrown = false;
    try {
      FmmB200 f(cfg, g);
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    check(thrown, "FmmB200 with p_qbx > p_fmm throws std::invalid_argument");
    SourceEnsemble bad;
    bad.positions = {Vec3{0, 0, 0}};
    bad.weights = {NAN};
    thrown = false;
    try {
      direct_sum_b200(bad, TargetSet{{Vec3{1, 0, 0}}, {-1}});
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    check(thrown, "direct_sum_b200 on a non-finite weight throws std::invalid_argument");
  }
  int ndev = 0;
  qbxg_device_count(&ndev);
  if (ndev == 0) {
    std::printf("no CUDA device: device checks skipped\n");
    return failures ? 1 : 77;
  }
  // direct_sum: the B200 path against the reference's own compiled direct_sum
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  SourceEnsemble s;
  TargetSet t;
  for (int i = 0; i < 2000; ++i) {
    s.positions.push_back(Vec3{u(rng), u(rng), u(rng)});
    s.weights.push_back(u(rng));
    s.dipole_moments.push_back(Vec3{u(rng), u(rng), u(rng)});
  }
  for (int i = 0; i < 700; ++i) {
    t.positions.push_back(Vec3{u(rng) + 3.0, u(rng), u(rng)});
    t.association.push_back(-1);
  }
  const std::vector<double> a = direct_sum_b200(s, t), b = direct_sum(s, t);
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  check(std::sqrt(num / den) <= 1e-13, "direct_sum_b200 == qbx::direct_sum (rel l2 <= 1e-13)");
  // coincidence: both throw std::domain_error naming the same pair
  t.positions[3] = s.positions[17];
  std::string ma, mb;
  try {
    direct_sum_b200(s, t);
  } catch (const std::domain_error& e) {
    ma = e.what();
  }
  try {
    direct_sum(s, t);
  } catch (const std::domain_error& e) {
    mb = e.what();
  }
  check(!ma.empty() && ma == mb, ("coincidence: '" + ma + "' == '" + mb + "'").c_str());
  // execute: FmmB200 over a small sphere's geometry against direct_sum at conventional
  // (far) targets, where the FMM reduces to the plain potential
  {
    std::vector<double> sp, cp, cr, tp;
    std::vector<int32_t> as;
    std::vector<double> w;
    for (size_t i = 0; i < s.size(); ++i) {
      sp.insert(sp.end(), {s.positions[i].x, s.positions[i].y, s.positions[i].z});
      w.push_back(s.weights[i]);
    }
    for (int i = 0; i < 500; ++i) {
      tp.insert(tp.end(), {u(rng) * 0.3 + 4.0, u(rng) * 0.3, u(rng) * 0.3});
      as.push_back(-1);
    }
    qbxg_geometry g{int64_t(s.size()), sp.data(), 0, nullptr, nullptr, 500, tp.data(), as.data()};
    qbxg_config cfg{};
    cfg.p_fmm = 12;
    cfg.p_qbx = 3;
    cfg.t_f = 0.9;
    cfg.n_max = 32;
    cfg.kernel = QBXG_KERNEL_LAPLACE_SL;
    FmmB200 f(cfg, g);
    SourceEnsemble sl;
    sl.positions = s.positions;
    sl.weights = s.weights;
    const std::vector<double> fp = f.apply(sl);
    TargetSet ft;
    for (int i = 0; i < 500; ++i) {
      ft.positions.push_back(Vec3{tp[3 * i], tp[3 * i + 1], tp[3 * i + 2]});
      ft.association.push_back(-1);
    }
    const std::vector<double> ref = direct_sum(sl, ft);
    num = den = 0;
    for (size_t i = 0; i < fp.size(); ++i) {
      num += (fp[i] - ref[i]) * (fp[i] - ref[i]);
      den += ref[i] * ref[i];
    }
    check(std::sqrt(num / den) <= 1e-8, "FmmB200::apply at far targets == qbx::direct_sum (rel l2 <= 1e-8)");
  }
  return failures ? 1 : 0;
}
