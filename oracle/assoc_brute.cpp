// ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
// cpu_baseline may call it; the product never does).  Brute-force CPU
// restatements of
//   - Algorithm 3, target association (spec
//     associate_targets), in the paper's scatter form: every
//     source marks the targets within its danger radius, then every centre, in
//     increasing id, claims the endangered targets within r_c (1 + eps) that it
//     is strictly closer to than the best so far -- so ties go to the lowest id
//     (SPEC.md decision "ties broken by lowest center id"); endangered targets
//     left without a centre are flagged (-2);
//   - Algorithm 5, area query, as the
//     brute-force leaf scan the spec names as its oracle: every leaf whose closed
//     cube meets the closed l-inf ball, in box-id order.
// Squared distances are (dx*dx + dy*dy) + dz*dz, each operation rounded on its
// own: this file is compiled with -ffp-contract=off (oracle/Makefile).
#include <cmath>
#include <cstdint>
#include <vector>

namespace {
inline double d2(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return (dx * dx + dy * dy) + dz * dz;
}
}  // namespace

extern "C" int oracle_associate(int64_t ns, const double* spos, const double* danger, int64_t nc,
                                const double* cpos, const double* crad, const int8_t* cside, int64_t nt,
                                const double* tpos, double eps, const int8_t* side_pref, int32_t* out,
                                int64_t* n_flagged) {
  const double onep = 1.0 + eps;
  constexpr int64_t kBlock = 256;
  int64_t flagged = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : flagged)
  for (int64_t t0 = 0; t0 < nt; t0 += kBlock) {
    const int64_t t1 = t0 + kBlock < nt ? t0 + kBlock : nt;
    std::vector<uint8_t> endangered(t1 - t0, 0);
    std::vector<double> best(t1 - t0, INFINITY);
    std::vector<int32_t> who(t1 - t0, -1);
    for (int64_t s = 0; s < ns; ++s) {  // find endangered targets
      const double rd = danger[s] * danger[s];
      for (int64_t t = t0; t < t1; ++t)
        if (d2(&tpos[3 * t], &spos[3 * s]) <= rd) endangered[t - t0] = 1;
    }
    for (int64_t c = 0; c < nc; ++c) {  // find centres for endangered targets
      const double rr = crad[c] * onep, rr2 = rr * rr;
      for (int64_t t = t0; t < t1; ++t) {
        if (!endangered[t - t0]) continue;
        if (side_pref && cside && side_pref[t] != 0 && side_pref[t] != cside[c]) continue;
        const double d = d2(&tpos[3 * t], &cpos[3 * c]);
        if (d <= rr2 && d < best[t - t0]) best[t - t0] = d, who[t - t0] = int32_t(c);
      }
    }
    for (int64_t t = t0; t < t1; ++t) {  // flag targets that could not be associated
      out[t] = endangered[t - t0] ? (who[t - t0] >= 0 ? who[t - t0] : -2) : -1;
      if (out[t] == -2) ++flagged;
    }
  }
  if (n_flagged) *n_flagged = flagged;
  return 0;
}

// counts[q] always; leaves (CSR by starts) when non-null
extern "C" int oracle_area_query(int32_t nb, const double* box_center, const double* box_radius,
                                 const int32_t* child_starts, int64_t nq, const double* qc, const double* qr,
                                 int64_t* counts, const int64_t* starts, int32_t* leaves) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < nq; ++q) {
    int64_t k = 0, pos = starts ? starts[q] : 0;
    for (int32_t b = 0; b < nb; ++b) {
      if (child_starts[b + 1] != child_starts[b]) continue;  // leaves only
      const double lim = qr[q] + box_radius[b];
      if (std::fabs(qc[3 * q] - box_center[3 * b]) <= lim && std::fabs(qc[3 * q + 1] - box_center[3 * b + 1]) <= lim &&
          std::fabs(qc[3 * q + 2] - box_center[3 * b + 2]) <= lim) {
        if (leaves) leaves[pos + k] = b;
        ++k;
      }
    }
    counts[q] = k;
  }
  return 0;
}
