// siddon.cu -- device parallel-beam projector: the CSR
// blocks of the tomography configurations are traced on the GPU straight
// into the context's operator arrays, so the matrix never crosses PCIe.
//
// Same algorithm and the same floating-point operations, in the same order,
// as the reference ray tracer (tomo.py:219-256, _trace_ray) and the view
// builders (tomo.py:259-273 2D, 276-301 3D), i.e. as the host restatement
// csrc/siddon.cpp: every product and sum is an explicitly rounded
// __dmul_rn / __dadd_rn (no fused multiply-add), divisions and sqrt are the
// IEEE-rounded ones, the view geometry (sin/cos, detector basis) comes from
// the host. The blocks are therefore bit-identical to the host projector's.
//
// One thread per ray:
//  * the plane crossings of each axis are an increasing sequence in t, so
//    np.unique(concatenate(...)) is a k-way merge of dim sequences (exact
//    equal values dropped), walked without storing t;
//  * a segment's cell index along every axis is a monotone function of its
//    midpoint (every operation on the way is monotone), so the cells of a
//    ray change monotonically per axis, equal cells are consecutive in t
//    (scipy's stable sort sums duplicates in t order: the same sum here),
//    and sorting by the flat index (C order, x fastest) is a nested
//    reversal of the t-ordered runs: outer axis first, then the groups of
//    equal outer index. The result is checked for strict order; a violation
//    sets the error flag (never observed; it would make the host raise).
// Two passes: count (nnz per row -> row pointers by a device scan), fill.
#include <math_constants.h>

#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "siddon.h"

namespace slim {

struct RayGeom {
  int dims;            // 2 or 3
  int n;               // grid side
  int64_t rpv;         // rows per view: rays (2D) or side^2 (3D)
  int side;            // 3D detector side
  double spacing;
  const double* views; // 9 doubles per view: d[3], u[3], v[3] (2D: u = detector axis)
  const int* ray_of_row;  // within-view ray of each row, or null (identity)
  int64_t m;
};

struct RayState {
  double p0[3], d[3];
};

__device__ __forceinline__ bool ray_setup(const RayGeom& G, int64_t row, RayState& R) {
  const int64_t view = row / G.rpv;
  const int64_t j = G.ray_of_row ? (int64_t)G.ray_of_row[row] : row - view * G.rpv;
  const double* v = G.views + 9 * view;
  if (G.dims == 2) {
    // offset = (j - (rays - 1) / 2.0) * spacing; p0 = offset * axis
    const double off = __dmul_rn(__dsub_rn((double)j, (double)(G.rpv - 1) / 2.0), G.spacing);
    R.p0[0] = __dmul_rn(off, v[3]);
    R.p0[1] = __dmul_rn(off, v[4]);
    R.p0[2] = 0.0;
    R.d[0] = v[0], R.d[1] = v[1], R.d[2] = 0.0;
  } else {
    const int64_t u = j / G.side, w = j - u * G.side;
    const double half = (double)(G.side - 1) / 2.0;
    const double ou = __dmul_rn(__dsub_rn((double)u, half), G.spacing);
    const double ow = __dmul_rn(__dsub_rn((double)w, half), G.spacing);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      R.p0[a] = __dadd_rn(__dmul_rn(ou, v[3 + a]), __dmul_rn(ow, v[6 + a]));
      R.d[a] = v[a];
    }
  }
  return true;
}

// walk the segments of one ray in t order, consecutive equal cells merged;
// emit(flat, len) once per run
template <int DIM, typename Emit>
__device__ __forceinline__ void trace(const RayState& R, int n, Emit&& emit) {
  const double lo = -0.5 * (double)n, hi = 0.5 * (double)n;
  double t_enter = -CUDART_INF, t_exit = CUDART_INF;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    if (R.d[a] != 0.0) {
      const double t0 = __ddiv_rn(__dsub_rn(lo, R.p0[a]), R.d[a]);
      const double t1 = __ddiv_rn(__dsub_rn(hi, R.p0[a]), R.d[a]);
      const double mn = (t1 < t0) ? t1 : t0;  // std::min(t0, t1)
      const double mx = (t0 < t1) ? t1 : t0;  // std::max(t0, t1)
      t_enter = (t_enter < mn) ? mn : t_enter;
      t_exit = (mx < t_exit) ? mx : t_exit;
    } else if (!(lo < R.p0[a] && R.p0[a] < hi)) {
      return;
    }
  }
  if (!(t_enter < t_exit)) return;
  double dd = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) dd = __dadd_rn(dd, __dmul_rn(R.d[a], R.d[a]));
  const double nd = __dsqrt_rn(dd);
  // per axis: position i in ascending-t order, plane k(i) = i (d > 0) or n - i
  int pos[DIM];
  double tn[DIM];
  auto plane_t = [&](int a, int i) {
    const int k = R.d[a] > 0.0 ? i : n - i;
    return __ddiv_rn(__dsub_rn(__dadd_rn(lo, (double)k), R.p0[a]), R.d[a]);
  };
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    tn[a] = CUDART_INF;
    pos[a] = n + 1;
    if (R.d[a] == 0.0) continue;
    int l = 0, h = n + 1;  // smallest i with t(i) > t_enter
    while (l < h) {
      const int mid = (l + h) >> 1;
      if (plane_t(a, mid) > t_enter) h = mid;
      else l = mid + 1;
    }
    pos[a] = l;
    if (l <= n) {
      const double t = plane_t(a, l);
      if (t < t_exit) tn[a] = t;
    }
  }
  double tprev = t_enter;
  int64_t run_flat = -1;
  double run_len = 0.0;
  while (true) {
    double tmin = t_exit;
#pragma unroll
    for (int a = 0; a < DIM; ++a) tmin = tn[a] < tmin ? tn[a] : tmin;
    const double len = __dmul_rn(__dsub_rn(tmin, tprev), nd);
    if (len > 1e-12) {
      const double mid = __dmul_rn(0.5, __dadd_rn(tprev, tmin));
      int64_t flat = 0;
#pragma unroll
      for (int a = DIM - 1; a >= 0; --a) {
        const double v = floor(__dsub_rn(__dadd_rn(R.p0[a], __dmul_rn(mid, R.d[a])), lo));
        int64_t idx = (int64_t)v;
        idx = idx < 0 ? 0 : (idx > n - 1 ? n - 1 : idx);
        flat = flat * n + idx;
      }
      if (flat == run_flat) {
        run_len = __dadd_rn(run_len, len);
      } else {
        if (run_flat >= 0) emit(run_flat, run_len);
        run_flat = flat;
        run_len = len;
      }
    }
    if (!(tmin < t_exit)) break;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      if (tn[a] == tmin) {  // exact duplicates across axes are one crossing
        const int i = ++pos[a];
        tn[a] = CUDART_INF;
        if (i <= n) {
          const double t = plane_t(a, i);
          if (t < t_exit) tn[a] = t;
        }
      }
    }
    tprev = tmin;
  }
  if (run_flat >= 0) emit(run_flat, run_len);
}

template <int DIM>
__global__ void __launch_bounds__(256) k_siddon_count(RayGeom G, int64_t* __restrict__ cnt) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= G.m) return;
  RayState R;
  ray_setup(G, row, R);
  int64_t c = 0;
  trace<DIM>(R, G.n, [&](int64_t, double) { ++c; });
  cnt[row] = c;
}

template <typename T>
__device__ __forceinline__ void reverse_range(int* col, T* val, int64_t a, int64_t b) {
  for (--b; a < b; ++a, --b) {
    const int c = col[a];
    col[a] = col[b];
    col[b] = c;
    const T v = val[a];
    val[a] = val[b];
    val[b] = v;
  }
}

// reverse every maximal run of equal col / div
template <typename T>
__device__ __forceinline__ void reverse_groups(int* col, T* val, int64_t lo, int64_t hi,
                                               int64_t div) {
  int64_t g = lo;
  while (g < hi) {
    const int64_t key = col[g] / div;
    int64_t e = g + 1;
    while (e < hi && col[e] / div == key) ++e;
    reverse_range(col, val, g, e);
    g = e;
  }
}

template <int DIM, typename T>
__global__ void __launch_bounds__(256) k_siddon_fill(RayGeom G, const int64_t* __restrict__ rowptr,
                                                     int* __restrict__ col, T* __restrict__ val,
                                                     int* __restrict__ err) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= G.m) return;
  RayState R;
  ray_setup(G, row, R);
  const int64_t lo = rowptr[row], hi = rowptr[row + 1];
  const int n = G.n;
  if (DIM == 2 || R.d[2] == 0.0) {
    // At most two varying axes (2D, or 3D with the ray in a z plane): the
    // row is written straight into its sorted place -- mirrored when the
    // outer axis runs backwards -- and each group of equal outer index is
    // reversed as soon as it is complete (its entries are still in L2)
    // when the inner axis runs backwards in the written order. The
    // monotonicity that makes this the sorted order is checked per run.
    const bool mirror = R.d[1] < 0.0;
    const bool grev = (R.d[0] < 0.0) != mirror;
    int64_t q = 0, gkey = -1, gstart = 0, last = 0;
    int px = -1, py = -1, pz = -1;
    bool bad = false;
    trace<DIM>(R, n, [&](int64_t flat, double len) {
      const int ix = (int)(flat % n), iy = (int)((flat / n) % n), iz = (int)(flat / ((int64_t)n * n));
      if (px >= 0) {
        bad |= R.d[0] > 0.0 ? ix < px : (R.d[0] < 0.0 ? ix > px : ix != px);
        bad |= R.d[1] > 0.0 ? iy < py : (R.d[1] < 0.0 ? iy > py : iy != py);
        bad |= iz != pz;
      }
      px = ix, py = iy, pz = iz;
      const int64_t pos = mirror ? hi - 1 - q : lo + q;
      const int64_t key = flat / n;
      if (key != gkey) {
        if (grev && gkey >= 0) {
          if (mirror) reverse_range(col, val, last, gstart + 1);
          else reverse_range(col, val, gstart, last + 1);
        }
        gkey = key;
        gstart = pos;
      }
      if (pos >= lo && pos < hi) col[pos] = (int)flat, val[pos] = (T)len;
      last = pos;
      ++q;
    });
    if (q != hi - lo) {
      atomicOr(err, 1);
      return;
    }
    if (grev && gkey >= 0) {
      if (mirror) reverse_range(col, val, last, gstart + 1);
      else reverse_range(col, val, gstart, last + 1);
    }
    if (bad) atomicOr(err, 2);
    return;
  }
  int64_t e = lo;
  trace<DIM>(R, G.n, [&](int64_t flat, double len) {
    if (e < hi) col[e] = (int)flat, val[e] = (T)len;
    ++e;
  });
  if (e != hi) {
    atomicOr(err, 1);
    return;
  }
  // general 3D direction: sort by flat index in passes, the outermost axis
  // first, then within its groups
  int flip = 1;
  {
    const int a = DIM - 1;
    const int sg = R.d[a] < 0.0 ? -1 : 1;
    if (sg < 0) reverse_range(col, val, lo, hi), flip = -1;
  }
  if (DIM == 3) {
    const int sg = (R.d[1] < 0.0 ? -1 : 1) * flip;
    if (sg < 0) reverse_groups(col, val, lo, hi, (int64_t)n * n), flip = -flip;
  }
  {
    const int sg = (R.d[0] < 0.0 ? -1 : 1) * flip;
    if (sg < 0) reverse_groups(col, val, lo, hi, (int64_t)n);
  }
  for (int64_t q = lo + 1; q < hi; ++q)
    if (!(col[q - 1] < col[q])) {
      atomicOr(err, 2);
      break;
    }
}

template <typename T>
__global__ void k_csr_spmv(const int64_t* __restrict__ rowptr, const int* __restrict__ col,
                           const T* __restrict__ val, const double* __restrict__ x,
                           double* __restrict__ y, int64_t m) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  double s = 0.0;
  for (int64_t e = rowptr[row] + lane; e < rowptr[row + 1]; e += 32) s += (double)val[e] * x[col[e]];
  s = warp_sum(s);
  if (lane == 0) y[row] = s;
}

// ---- host launchers ---------------------------------------------------------

static RayGeom make_geom(const SiddonSpec& S) {
  RayGeom G{};
  G.dims = S.dims;
  G.n = (int)S.grid;
  G.rpv = S.rows_per_view;
  G.side = (int)S.side;
  G.spacing = S.spacing;
  G.views = S.views;
  G.ray_of_row = S.ray_of_row;
  G.m = S.m;
  return G;
}

cudaError_t siddon_count(const SiddonSpec& S, int64_t* rowptr, cudaStream_t s) {
  RayGeom G = make_geom(S);
  cudaMemsetAsync(rowptr, 0, sizeof(int64_t), s);
  const unsigned grid = (unsigned)((S.m + 255) / 256);
  int64_t* cnt = nullptr;
  cudaError_t e = cudaMallocAsync(&cnt, sizeof(int64_t) * (size_t)S.m, s);
  if (e != cudaSuccess) return e;
  if (S.dims == 2) k_siddon_count<2><<<grid, 256, 0, s>>>(G, cnt);
  else k_siddon_count<3><<<grid, 256, 0, s>>>(G, cnt);
  size_t tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, rowptr + 1, S.m, s);
  void* d_tmp = nullptr;
  e = cudaMallocAsync(&d_tmp, tmp, s);
  if (e != cudaSuccess) return e;
  cub::DeviceScan::InclusiveSum(d_tmp, tmp, cnt, rowptr + 1, S.m, s);
  cudaFreeAsync(d_tmp, s);
  cudaFreeAsync(cnt, s);
  return cudaGetLastError();
}

cudaError_t siddon_fill(const SiddonSpec& S, const int64_t* rowptr, int* col, void* val, bool f64,
                        int* err, cudaStream_t s) {
  RayGeom G = make_geom(S);
  const unsigned grid = (unsigned)((S.m + 255) / 256);
  if (S.dims == 2) {
    if (f64) k_siddon_fill<2, double><<<grid, 256, 0, s>>>(G, rowptr, col, (double*)val, err);
    else k_siddon_fill<2, float><<<grid, 256, 0, s>>>(G, rowptr, col, (float*)val, err);
  } else {
    if (f64) k_siddon_fill<3, double><<<grid, 256, 0, s>>>(G, rowptr, col, (double*)val, err);
    else k_siddon_fill<3, float><<<grid, 256, 0, s>>>(G, rowptr, col, (float*)val, err);
  }
  return cudaGetLastError();
}

cudaError_t csr_spmv(const int64_t* rowptr, const int* col, const void* val, bool f64,
                     const double* x, double* y, int64_t m, cudaStream_t s) {
  const unsigned grid = (unsigned)((m + 7) / 8);
  if (f64) k_csr_spmv<double><<<grid, 256, 0, s>>>(rowptr, col, (const double*)val, x, y, m);
  else k_csr_spmv<float><<<grid, 256, 0, s>>>(rowptr, col, (const float*)val, x, y, m);
  return cudaGetLastError();
}

}  // namespace slim
