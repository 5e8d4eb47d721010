// Procedural inputs for BASELINE.json configs 0-4 (pinned in SURVEY.md §8d).
//
// Flat-triangle surfaces (icosphere, torus, urchin, urchin arrays), a 4x4
// Gauss-Legendre rule collapsed onto each triangle by the Duffy map, QBX
// centres at x +- r n with r = 0.5 sqrt(area) (paper Eq. (7), PAPER.md:312-316,
// with the config's radius rule instead of r = eta/2 of PAPER.md:914-917), and
// on-surface targets associated by construction (Algorithm 3 is not run).
// The urchin radius follows the config (1 + 0.2 Re Y_8^4 / max|Y_8^4|), not
// Eq. (24) of PAPER.md:2874-2880.
#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <random>
#include <unordered_map>

#include "common.hpp"

namespace qbxg {

// ---------------------------------------------------------------- RNG
Rng::Rng(uint64_t seed) : state(new std::mt19937_64(seed)) {}
Rng::~Rng() { delete static_cast<std::mt19937_64*>(state); }
uint64_t Rng::next() { return (*static_cast<std::mt19937_64*>(state))(); }
double Rng::uniform01() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }
double Rng::uniform(double a, double b) { return a + (b - a) * uniform01(); }
int64_t Rng::uniform_int(int64_t lo, int64_t hi) {
  const uint64_t span = uint64_t(hi - lo + 1);
  return lo + int64_t(next() % span);
}

namespace {

using V3 = std::array<double, 3>;
inline V3 sub(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline V3 add(const V3& a, const V3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline V3 scl(const V3& a, double s) { return {a[0] * s, a[1] * s, a[2] * s}; }
inline double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline double nrm(const V3& a) { return std::sqrt(dot(a, a)); }

struct Tri {
  V3 a, b, c;
  V3 pa, pb, pc;   // (u,v) parameters for the torus density (unused elsewhere)
  V3 outward_ref;  // point the outward normal points away from
};

// icosahedron on the unit sphere, subdivided `level` times with midpoints
// projected back onto the sphere.
void icosphere(int level, std::vector<V3>& verts, std::vector<std::array<int, 3>>& faces) {
  const double t = (1.0 + std::sqrt(5.0)) / 2.0;
  verts = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t}, {0, 1, t},
           {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
  for (auto& v : verts) v = scl(v, 1.0 / nrm(v));
  faces = {{0, 11, 5}, {0, 5, 1}, {0, 1, 7}, {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
           {11, 10, 2}, {10, 7, 6}, {7, 1, 8}, {3, 9, 4}, {3, 4, 2}, {3, 2, 6}, {3, 6, 8},
           {3, 8, 9}, {4, 9, 5}, {2, 4, 11}, {6, 2, 10}, {8, 6, 7}, {9, 8, 1}};
  for (int l = 0; l < level; ++l) {
    std::map<std::pair<int, int>, int> mid;
    auto midpoint = [&](int i, int j) {
      auto key = std::make_pair(std::min(i, j), std::max(i, j));
      auto it = mid.find(key);
      if (it != mid.end()) return it->second;
      V3 m = scl(add(verts[i], verts[j]), 0.5);
      m = scl(m, 1.0 / nrm(m));
      verts.push_back(m);
      int id = int(verts.size()) - 1;
      mid[key] = id;
      return id;
    };
    std::vector<std::array<int, 3>> nf;
    nf.reserve(faces.size() * 4);
    for (auto& f : faces) {
      int a = midpoint(f[0], f[1]), b = midpoint(f[1], f[2]), c = midpoint(f[2], f[0]);
      nf.push_back({f[0], a, c});
      nf.push_back({f[1], b, a});
      nf.push_back({f[2], c, b});
      nf.push_back({a, b, c});
    }
    faces.swap(nf);
  }
}

// Associated Legendre P_n^m(x) without the Condon-Shortley phase.
double legendre_nocs(int n, int m, double x) {
  double pmm = 1.0, s = std::sqrt(std::max(0.0, 1.0 - x * x));
  for (int i = 1; i <= m; ++i) pmm *= (2 * i - 1) * s;
  if (n == m) return pmm;
  double pm1 = x * (2 * m + 1) * pmm;
  if (n == m + 1) return pm1;
  double pn = 0;
  for (int k = m + 2; k <= n; ++k) {
    pn = ((2 * k - 1) * x * pm1 - (k + m - 1) * pmm) / (k - m);
    pmm = pm1;
    pm1 = pn;
  }
  return pn;
}

// Urchin radius rho(theta, phi) = 1 + 0.2 Re Y_8^4 / max|Y_8^4| (BASELINE.json config 2).
struct UrchinRadius {
  double inv_max;
  UrchinRadius() {
    double mx = 0;
    const int ns = 200001;
    for (int i = 0; i < ns; ++i) {
      double th = M_PI * double(i) / double(ns - 1);
      mx = std::max(mx, std::fabs(legendre_nocs(8, 4, std::cos(th))));
    }
    inv_max = 1.0 / mx;
  }
  double operator()(const V3& v) const {
    double r = nrm(v);
    double ct = v[2] / r;
    double phi = std::atan2(v[1], v[0]);
    return 1.0 + 0.2 * legendre_nocs(8, 4, ct) * std::cos(4.0 * phi) * inv_max;
  }
};

V3 rotate_quat(const std::array<double, 4>& q, const V3& v) {
  // q = (x, y, z, w)
  const double x = q[0], y = q[1], z = q[2], w = q[3];
  const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)},
                          {2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)},
                          {2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)}};
  return {R[0][0] * v[0] + R[0][1] * v[1] + R[0][2] * v[2],
          R[1][0] * v[0] + R[1][1] * v[1] + R[1][2] * v[2],
          R[2][0] * v[0] + R[2][1] * v[1] + R[2][2] * v[2]};
}

// Gauss-Legendre 4-point rule mapped to [0,1], ascending.
const double kGLx[4] = {(1.0 - 0.8611363115940526) / 2, (1.0 - 0.3399810435848563) / 2,
                        (1.0 + 0.3399810435848563) / 2, (1.0 + 0.8611363115940526) / 2};
const double kGLw[4] = {0.3478548451374538 / 2, 0.6521451548625461 / 2, 0.6521451548625461 / 2,
                        0.3478548451374538 / 2};

}  // namespace

struct Generated {
  qbxg_geometry_spec spec;
  int64_t n_triangles = 0;
  std::vector<double> src_pos, src_normal, qw, density, ctr_pos, ctr_rad, tgt_pos;
  std::vector<int32_t> assoc;
  std::vector<double> node_param;  // 2*ns, torus (u,v) of each node
  int32_t density_is_complex = 0;
  int64_t n_volume_drawn = 0;
};

void generate(const qbxg_geometry_spec& spec, Generated& g) {
  g.spec = spec;
  Rng rng(spec.seed);
  std::vector<Tri> tris;

  if (spec.surface == QBXG_SURF_ICOSPHERE || spec.surface == QBXG_SURF_URCHIN ||
      spec.surface == QBXG_SURF_URCHIN_ARRAY) {
    if (spec.level < 0 || spec.level > 9) throw InvalidArgument("geometry: icosphere level out of range");
    std::vector<V3> verts;
    std::vector<std::array<int, 3>> faces;
    icosphere(spec.level, verts, faces);
    if (spec.surface != QBXG_SURF_ICOSPHERE) {
      UrchinRadius rho;
      for (auto& v : verts) v = scl(v, rho(v));
    }
    int nx = 1, ny = 1, nz = 1;
    if (spec.surface == QBXG_SURF_URCHIN_ARRAY) {
      nx = spec.nx; ny = spec.ny; nz = spec.nz;
      if (nx < 1 || ny < 1 || nz < 1) throw InvalidArgument("geometry: bad urchin array dims");
    }
    // geometry randomness first (SURVEY.md §8d draw order): one rotation per urchin
    std::vector<std::array<double, 4>> rots;
    for (int i = 0; i < nx * ny * nz; ++i) {
      if (spec.surface == QBXG_SURF_URCHIN_ARRAY) {
        // Shoemake's uniform random rotation
        double u1 = rng.uniform01(), u2 = rng.uniform01(), u3 = rng.uniform01();
        rots.push_back({std::sqrt(1 - u1) * std::sin(2 * M_PI * u2), std::sqrt(1 - u1) * std::cos(2 * M_PI * u2),
                        std::sqrt(u1) * std::sin(2 * M_PI * u3), std::sqrt(u1) * std::cos(2 * M_PI * u3)});
      } else {
        rots.push_back({0, 0, 0, 1});
      }
    }
    for (int ix = 0; ix < nx; ++ix)
      for (int iy = 0; iy < ny; ++iy)
        for (int iz = 0; iz < nz; ++iz) {
          const int id = (ix * ny + iy) * nz + iz;
          V3 off = {0, 0, 0};
          if (spec.surface == QBXG_SURF_URCHIN_ARRAY)
            off = {(ix - 0.5 * (nx - 1)) * spec.spacing, (iy - 0.5 * (ny - 1)) * spec.spacing,
                   (iz - 0.5 * (nz - 1)) * spec.spacing};
          for (auto& f : faces) {
            Tri t;
            t.a = add(rotate_quat(rots[id], verts[f[0]]), off);
            t.b = add(rotate_quat(rots[id], verts[f[1]]), off);
            t.c = add(rotate_quat(rots[id], verts[f[2]]), off);
            t.pa = t.pb = t.pc = {0, 0, 0};
            t.outward_ref = off;
            tris.push_back(t);
          }
        }
  } else if (spec.surface == QBXG_SURF_TORUS) {
    const int nu = spec.nu, nv = spec.nv;
    if (nu < 3 || nv < 3) throw InvalidArgument("geometry: torus grid too small");
    const double Rm = 2.0, rm = 1.0;
    auto X = [&](double u, double v) -> V3 {
      return {(Rm + rm * std::cos(v)) * std::cos(u), (Rm + rm * std::cos(v)) * std::sin(u), rm * std::sin(v)};
    };
    const double du = 2 * M_PI / nu, dv = 2 * M_PI / nv;
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < nv; ++j) {
        const double u0 = i * du, v0 = j * dv;
        V3 p00 = X(u0, v0), p10 = X(u0 + du, v0), p11 = X(u0 + du, v0 + dv), p01 = X(u0, v0 + dv);
        V3 q00 = {u0, v0, 0}, q10 = {u0 + du, v0, 0}, q11 = {u0 + du, v0 + dv, 0}, q01 = {u0, v0 + dv, 0};
        Tri t1{p00, p10, p11, q00, q10, q11, {0, 0, 0}};
        Tri t2{p00, p11, p01, q00, q11, q01, {0, 0, 0}};
        tris.push_back(t1);
        tris.push_back(t2);
      }
  } else {
    throw InvalidArgument("geometry: unknown surface");
  }

  const int64_t nt = int64_t(tris.size());
  const int64_t ns = nt * 16;
  g.n_triangles = nt;
  g.src_pos.resize(3 * ns);
  g.src_normal.resize(3 * ns);
  g.qw.resize(ns);
  g.node_param.resize(2 * ns);
  g.ctr_pos.resize(6 * ns);
  g.ctr_rad.resize(2 * ns);
  std::vector<double> tri_r(nt);
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < nt; ++k) {
    const Tri& t = tris[k];
    V3 e1 = sub(t.b, t.a), e2 = sub(t.c, t.a);
    V3 cr = cross(e1, e2);
    const double area = 0.5 * nrm(cr);
    V3 n = scl(cr, 1.0 / nrm(cr));
    V3 centroid = scl(add(add(t.a, t.b), t.c), 1.0 / 3.0);
    V3 ref = t.outward_ref;
    if (spec.surface == QBXG_SURF_TORUS) {
      const double uc = std::atan2(centroid[1], centroid[0]);
      ref = {2.0 * std::cos(uc), 2.0 * std::sin(uc), 0.0};
    }
    if (dot(n, sub(centroid, ref)) < 0) n = scl(n, -1.0);
    const double r = 0.5 * std::sqrt(area);
    tri_r[k] = r;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        const int64_t s = k * 16 + i * 4 + j;
        const double xi = kGLx[i], xj = kGLx[j];
        V3 x = add(add(t.a, scl(e1, xi)), scl(e2, xj * (1 - xi)));
        V3 pp = add(add(t.pa, scl(sub(t.pb, t.pa), xi)), scl(sub(t.pc, t.pa), xj * (1 - xi)));
        for (int d = 0; d < 3; ++d) {
          g.src_pos[3 * s + d] = x[d];
          g.src_normal[3 * s + d] = n[d];
          g.ctr_pos[3 * (2 * s) + d] = x[d] + r * n[d];
          g.ctr_pos[3 * (2 * s + 1) + d] = x[d] - r * n[d];
        }
        g.node_param[2 * s] = pp[0];
        g.node_param[2 * s + 1] = pp[1];
        g.qw[s] = 2.0 * area * kGLw[i] * kGLw[j] * (1 - xi);
        g.ctr_rad[2 * s] = r;
        g.ctr_rad[2 * s + 1] = r;
      }
  }

  // density (second in the draw order)
  switch (spec.density) {
    case QBXG_DENS_UNIFORM:
      g.density.resize(ns);
      for (int64_t s = 0; s < ns; ++s) g.density[s] = rng.uniform(-1.0, 1.0);
      break;
    case QBXG_DENS_ONES:
      g.density.assign(ns, 1.0);
      break;
    case QBXG_DENS_FOURIER8: {
      int a[8], b[8];
      double ph[8];
      for (int k = 0; k < 8; ++k) {
        a[k] = int(rng.uniform_int(-8, 8));
        b[k] = int(rng.uniform_int(-8, 8));
        ph[k] = rng.uniform(0.0, 2 * M_PI);
      }
      g.density.resize(ns);
#pragma omp parallel for schedule(static)
      for (int64_t s = 0; s < ns; ++s) {
        double u = g.node_param[2 * s], v = g.node_param[2 * s + 1], acc = 0;
        for (int k = 0; k < 8; ++k) acc += std::cos(a[k] * u + b[k] * v + ph[k]);
        g.density[s] = acc;
      }
      break;
    }
    case QBXG_DENS_COMPLEX_UNIFORM:
      g.density.resize(2 * ns);
      g.density_is_complex = 1;
      for (int64_t s = 0; s < ns; ++s) {
        g.density[2 * s] = rng.uniform(-1.0, 1.0);
        g.density[2 * s + 1] = rng.uniform(-1.0, 1.0);
      }
      break;
    default:
      throw InvalidArgument("geometry: unknown density kind");
  }

  // on-surface targets: node s evaluated through each of its two centres
  const int64_t nsurf = 2 * ns;
  g.tgt_pos.resize(3 * nsurf);
  g.assoc.resize(nsurf);
  for (int64_t s = 0; s < ns; ++s)
    for (int side = 0; side < 2; ++side) {
      for (int d = 0; d < 3; ++d) g.tgt_pos[3 * (2 * s + side) + d] = g.src_pos[3 * s + d];
      g.assoc[2 * s + side] = int32_t(2 * s + side);
    }

  // volume targets (third in the draw order), minus those within r(s) of a node s
  if (spec.n_volume_targets > 0) {
    const int64_t nv = spec.n_volume_targets;
    const double hw = spec.volume_halfwidth;
    std::vector<double> cand(3 * nv);
    for (int64_t i = 0; i < 3 * nv; ++i) cand[i] = rng.uniform(-hw, hw);
    g.n_volume_drawn = nv;
    // uniform grid over sources with cell >= max r
    double rmax = 0;
    for (double r : tri_r) rmax = std::max(rmax, r);
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int64_t s = 0; s < ns; ++s)
      for (int d = 0; d < 3; ++d) {
        lo[d] = std::min(lo[d], g.src_pos[3 * s + d]);
        hi[d] = std::max(hi[d], g.src_pos[3 * s + d]);
      }
    const double cell = std::max(rmax, 1e-12);
    int dims[3];
    for (int d = 0; d < 3; ++d) dims[d] = std::max(1, int((hi[d] - lo[d]) / cell) + 1);
    auto cell_of = [&](const double* x, int* c) {
      for (int d = 0; d < 3; ++d) c[d] = int(std::floor((x[d] - lo[d]) / cell));
    };
    std::unordered_map<int64_t, std::vector<int64_t>> grid;
    auto key = [&](int a, int b, int c) { return (int64_t(a) * dims[1] + b) * dims[2] + c; };
    for (int64_t s = 0; s < ns; ++s) {
      int c[3];
      cell_of(&g.src_pos[3 * s], c);
      grid[key(c[0], c[1], c[2])].push_back(s);
    }
    std::vector<uint8_t> keep(nv, 1);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < nv; ++i) {
      const double* x = &cand[3 * i];
      int c[3];
      cell_of(x, c);
      for (int a = c[0] - 1; a <= c[0] + 1 && keep[i]; ++a)
        for (int b = c[1] - 1; b <= c[1] + 1 && keep[i]; ++b)
          for (int e = c[2] - 1; e <= c[2] + 1 && keep[i]; ++e) {
            if (a < 0 || b < 0 || e < 0 || a >= dims[0] || b >= dims[1] || e >= dims[2]) continue;
            auto it = grid.find(key(a, b, e));
            if (it == grid.end()) continue;
            for (int64_t s : it->second) {
              const double dx = x[0] - g.src_pos[3 * s], dy = x[1] - g.src_pos[3 * s + 1],
                           dz = x[2] - g.src_pos[3 * s + 2];
              const double rs = tri_r[s / 16];
              if (dx * dx + dy * dy + dz * dz < rs * rs) {
                keep[i] = 0;
                break;
              }
            }
          }
    }
    for (int64_t i = 0; i < nv; ++i)
      if (keep[i]) {
        for (int d = 0; d < 3; ++d) g.tgt_pos.push_back(cand[3 * i + d]);
        g.assoc.push_back(-1);
      }
  }
}

}  // namespace qbxg

struct qbxg_generated {
  qbxg::Generated g;
};

extern "C" {

int qbxg_geometry_spec_for_config(int32_t config_id, int32_t variant, uint64_t seed,
                                  qbxg_geometry_spec* out) {
  return qbxg::guarded([&] {
    if (!out) throw qbxg::InvalidArgument("spec_for_config: null output");
    qbxg_geometry_spec s;
    std::memset(&s, 0, sizeof(s));
    s.seed = seed;
    s.spacing = 3.0;
    s.volume_halfwidth = 1.5;
    switch (config_id) {
      case 0:
        s.surface = QBXG_SURF_ICOSPHERE; s.level = 2;
        s.density = variant == 1 ? QBXG_DENS_ONES : QBXG_DENS_UNIFORM;
        break;
      case 1:
        s.surface = QBXG_SURF_TORUS; s.nu = 256; s.nv = 128; s.density = QBXG_DENS_FOURIER8;
        break;
      case 2:
        s.surface = QBXG_SURF_URCHIN; s.level = 5; s.density = QBXG_DENS_UNIFORM;
        s.n_volume_targets = 1000000;
        break;
      case 3:
        s.surface = QBXG_SURF_ICOSPHERE; s.level = 6; s.density = QBXG_DENS_COMPLEX_UNIFORM;
        break;
      case 4: {
        s.surface = QBXG_SURF_URCHIN_ARRAY; s.level = 5; s.density = QBXG_DENS_UNIFORM;
        int n = variant == 0 ? 64 : variant;
        if (n == 8) { s.nx = 2; s.ny = 2; s.nz = 2; }
        else if (n == 16) { s.nx = 2; s.ny = 2; s.nz = 4; }
        else if (n == 32) { s.nx = 2; s.ny = 4; s.nz = 4; }
        else if (n == 64) { s.nx = 4; s.ny = 4; s.nz = 4; }
        else throw qbxg::InvalidArgument("config 4 variant must be 8, 16, 32 or 64 urchins");
        break;
      }
      default:
        throw qbxg::InvalidArgument("unknown config id");
    }
    *out = s;
  });
}

int qbxg_geometry_generate(const qbxg_geometry_spec* spec, qbxg_generated** out) {
  return qbxg::guarded([&] {
    if (!spec || !out) throw qbxg::InvalidArgument("geometry_generate: null argument");
    auto* g = new qbxg_generated;
    try {
      qbxg::generate(*spec, g->g);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int qbxg_geometry_view(const qbxg_generated* gp, qbxg_generated_view* v) {
  return qbxg::guarded([&] {
    if (!gp || !v) throw qbxg::InvalidArgument("geometry_view: null argument");
    const auto& g = gp->g;
    v->n_triangles = g.n_triangles;
    v->n_sources = int64_t(g.qw.size());
    v->source_pos = g.src_pos.data();
    v->source_normal = g.src_normal.data();
    v->quad_weight = g.qw.data();
    v->density = g.density.data();
    v->density_is_complex = g.density_is_complex;
    v->n_centers = int64_t(g.ctr_rad.size());
    v->center_pos = g.ctr_pos.data();
    v->center_radius = g.ctr_rad.data();
    v->n_targets = int64_t(g.assoc.size());
    v->target_pos = g.tgt_pos.data();
    v->association = g.assoc.data();
    v->n_volume_drawn = g.n_volume_drawn;
  });
}

void qbxg_geometry_destroy(qbxg_generated* g) { delete g; }

}  // extern "C"
