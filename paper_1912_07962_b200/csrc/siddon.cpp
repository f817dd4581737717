// siddon.cpp -- host-side parallel-beam projector blocks (problem setup,
// not the hot path).  Restates the reference's exact-intersection ray
// tracer and per-view block builders:
//   _trace_ray        tomo.py:219-256
//   _view_block_2d    tomo.py:259-273
//   _detector_basis   tomo.py:276-282
//   _view_block_3d    tomo.py:285-301
// with the same floating-point operation order (compiled with
// -ffp-contract=off so no multiply-add is fused) and the same CSR
// canonicalisation scipy applies (columns sorted, duplicates summed).
// Two-phase API: call with col/val == NULL to get the row pointer (nnz
// counts), then again with buffers of rowptr[rows] entries.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <utility>
#include <vector>

#include "slimb200.h"

namespace {

struct Seg {
  int64_t cell;
  double len;
};

// returns the cells (C-order flat index, x fastest) and lengths of one ray
void trace_ray(const double* p0, const double* d, int dim, int64_t n, std::vector<Seg>& out,
               std::vector<double>& ts) {
  out.clear();
  const double lo = -0.5 * (double)n, hi = 0.5 * (double)n;
  double t_enter = -std::numeric_limits<double>::infinity();
  double t_exit = std::numeric_limits<double>::infinity();
  for (int a = 0; a < dim; ++a) {
    if (d[a] != 0.0) {
      const double t0 = (lo - p0[a]) / d[a];
      const double t1 = (hi - p0[a]) / d[a];
      t_enter = std::max(t_enter, std::min(t0, t1));
      t_exit = std::min(t_exit, std::max(t0, t1));
    } else if (!(lo < p0[a] && p0[a] < hi)) {
      return;
    }
  }
  if (!(t_enter < t_exit)) return;
  ts.clear();
  ts.push_back(t_enter);
  ts.push_back(t_exit);
  for (int a = 0; a < dim; ++a) {
    if (d[a] == 0.0) continue;
    for (int64_t k = 0; k <= n; ++k) {
      const double t = ((lo + (double)k) - p0[a]) / d[a];
      if (t > t_enter && t < t_exit) ts.push_back(t);
    }
  }
  std::sort(ts.begin(), ts.end());
  ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
  // np.linalg.norm(d) = sqrt(d . d)
  double dd = 0.0;
  for (int a = 0; a < dim; ++a) dd = dd + d[a] * d[a];
  const double nd = std::sqrt(dd);
  for (size_t q = 0; q + 1 < ts.size(); ++q) {
    const double len = (ts[q + 1] - ts[q]) * nd;
    if (!(len > 1e-12)) continue;
    const double mid = 0.5 * (ts[q] + ts[q + 1]);
    int64_t flat = 0;
    for (int a = dim - 1; a >= 0; --a) {
      double v = std::floor((p0[a] + mid * d[a]) - lo);
      int64_t idx = (int64_t)v;
      if (idx < 0) idx = 0;
      if (idx > n - 1) idx = n - 1;
      flat = flat * n + idx;
    }
    out.push_back({flat, len});
  }
}

// scipy's COO -> CSR: sort by column (stable), sum duplicates
void canonical(std::vector<Seg>& segs) {
  std::stable_sort(segs.begin(), segs.end(), [](const Seg& x, const Seg& y) { return x.cell < y.cell; });
  size_t w = 0;
  for (size_t q = 0; q < segs.size(); ++q) {
    if (w > 0 && segs[w - 1].cell == segs[q].cell) segs[w - 1].len += segs[q].len;
    else segs[w++] = segs[q];
  }
  segs.resize(w);
}

template <typename RayFn>
int build_block(int64_t rays, int64_t* rowptr, int32_t* col, double* val, RayFn&& ray) {
  std::vector<Seg> segs;
  std::vector<double> ts;
  if (col == nullptr || val == nullptr) {
    rowptr[0] = 0;
    for (int64_t j = 0; j < rays; ++j) {
      ray(j, segs, ts);
      canonical(segs);
      rowptr[j + 1] = rowptr[j] + (int64_t)segs.size();
    }
    return SLIM_OK;
  }
  for (int64_t j = 0; j < rays; ++j) {
    ray(j, segs, ts);
    canonical(segs);
    int64_t e = rowptr[j];
    if ((int64_t)segs.size() != rowptr[j + 1] - rowptr[j]) return SLIM_ESTATE;
    for (const Seg& s : segs) {
      col[e] = (int32_t)s.cell;
      val[e] = s.len;
      ++e;
    }
  }
  return SLIM_OK;
}

}  // namespace

// per-view geometry, 9 doubles: d[3], then the 2D detector axis or the 3D
// basis e1[3], e2[3] (tomo.py:260-262 and 276-282); shared by the host
// builders below and the device projector (siddon.cu)
namespace slim {
void view_geometry_2d(double angle_deg, double* g) {
  // np.radians(x) = x * (pi / 180)
  const double theta = angle_deg * (M_PI / 180.0);
  for (int q = 0; q < 9; ++q) g[q] = 0.0;
  g[0] = -std::sin(theta);
  g[1] = std::cos(theta);
  g[3] = std::cos(theta);
  g[4] = std::sin(theta);
}
void view_geometry_3d(const double* dir, double* g) {
  const double d[3] = {dir[0], dir[1], dir[2]};
  // e1 = cross(d, z), fallback cross(d, x) for near-axial d; e2 = cross(d, e1)
  auto cross = [](const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
  };
  auto norm3 = [](const double* v) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); };
  const double z[3] = {0.0, 0.0, 1.0}, xa[3] = {1.0, 0.0, 0.0};
  double e1[3], e2[3];
  cross(d, z, e1);
  if (norm3(e1) < 1e-8) cross(d, xa, e1);
  const double ne = norm3(e1);
  for (int a = 0; a < 3; ++a) e1[a] = e1[a] / ne;
  cross(d, e1, e2);
  for (int a = 0; a < 3; ++a) g[a] = d[a], g[3 + a] = e1[a], g[6 + a] = e2[a];
}
}  // namespace slim

extern "C" int slim_siddon2d_view(double angle_deg, int64_t grid, int64_t rays, double spacing,
                                  int64_t* rowptr, int32_t* col, double* val) {
  if (grid < 1 || rays < 1 || !rowptr || !(spacing > 0)) return SLIM_EINVAL;
  if (grid * grid > 0x7fffffffLL) return SLIM_EINVAL;
  double g[9];
  slim::view_geometry_2d(angle_deg, g);
  const double d[2] = {g[0], g[1]};
  const double axis[2] = {g[3], g[4]};
  auto ray = [&](int64_t j, std::vector<Seg>& segs, std::vector<double>& ts) {
    const double offset = ((double)j - (double)(rays - 1) / 2.0) * spacing;
    const double p0[2] = {offset * axis[0], offset * axis[1]};
    trace_ray(p0, d, 2, grid, segs, ts);
  };
  return build_block(rays, rowptr, col, val, ray);
}

extern "C" int slim_siddon3d_view(const double* dir, int64_t grid, int64_t side, double spacing,
                                  int64_t* rowptr, int32_t* col, double* val) {
  if (!dir || grid < 1 || side < 1 || !rowptr || !(spacing > 0)) return SLIM_EINVAL;
  if (grid * grid * grid > 0x7fffffffLL) return SLIM_EINVAL;
  double g[9];
  slim::view_geometry_3d(dir, g);
  const double d[3] = {g[0], g[1], g[2]};
  const double e1[3] = {g[3], g[4], g[5]}, e2[3] = {g[6], g[7], g[8]};
  auto ray = [&](int64_t j, std::vector<Seg>& segs, std::vector<double>& ts) {
    const int64_t u = j / side, v = j - u * side;
    const double off_u = ((double)u - (double)(side - 1) / 2.0) * spacing;
    const double off_v = ((double)v - (double)(side - 1) / 2.0) * spacing;
    const double p0[3] = {off_u * e1[0] + off_v * e2[0], off_u * e1[1] + off_v * e2[1],
                          off_u * e1[2] + off_v * e2[2]};
    trace_ray(p0, d, 3, grid, segs, ts);
  };
  return build_block(side * side, rowptr, col, val, ray);
}
