// ops.cu -- streaming kernels of one slimLS step (everything but the
// factorization / triangular solves, which live in chol.cu).
//
//   residual   r = A_k x - b_k, ||r||              solvers.py:180-183
//   gram       new column panel A_k M_k^T          innersolve.py:298-302
//              (incremental: only the new block's products are formed;
//               the reference recomputes the full M M^T every step)
//   mtw        s = alpha M_k^T w                   innersolve.py:321
//   finish     x <- x - s, ||x||^2 divergence,     solvers.py:169-177
//              history row at record steps         solvers.py:543-554
//
// Every reduction has a fixed order, so a run is bit-reproducible
// (reference determinism contract, test_solvers.py:555-571).
#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "ops.h"

namespace slim {

// ---------------------------------------------------------------------------
// residual
// ---------------------------------------------------------------------------

// Row dots of one sampled block, split over column chunks so the whole GPU
// streams the block (one warp per row leaves most SMs idle):
//   residual:  r[row] = A[row0 + row, :] . x - b[brow0 + row]
//   diagonal:  out[row * ld + row] = A[row, :] . A[row, :]     (SQUARE)
// CTA (chunk, group) covers RD_ROWS rows of one column chunk: every thread
// loads its x values once (16-byte loads) and streams the group's rows with
// RD_ROWS independent 16-byte loads in flight, so x costs 1/RD_ROWS of the A
// traffic. Each CTA writes one partial per row; the last CTA of a group
// (counter) adds the partials in chunk order, so the result is deterministic.
template <typename T, bool SQUARE, int RD_ROWS>
__global__ void __launch_bounds__(256) k_rowdot(const T* __restrict__ A, int64_t lda, int64_t row0,
                                                int n, int ell, const double* __restrict__ x,
                                                RowSplit rs, double* __restrict__ out,
                                                int64_t ld_out, const double* __restrict__ b,
                                                int64_t brow0, const Ctl* ctl) {
  if (ctl != nullptr && ctl->diverged_at != 0) return;
  constexpr int V = 16 / sizeof(T);
  const int chunk = blockIdx.x, grp = blockIdx.y, tid = threadIdx.x;
  const int r0 = grp * RD_ROWS, nr = min(RD_ROWS, ell - r0);
  const int nch = rs.nch;
  const int csz = ((n + nch - 1) / nch + V - 1) / V * V;
  const int c0 = chunk * csz, c1 = min(n, c0 + csz);
  const T* a = A + (row0 + r0) * lda;
  double acc[RD_ROWS];
#pragma unroll
  for (int q = 0; q < RD_ROWS; ++q) acc[q] = 0.0;
  if (rs.vec) {
#pragma unroll(RD_ROWS == 1 ? 4 : 1)
    for (int c = c0 + V * tid; c < c1; c += V * 256) {
      double xv[V];
      if (!SQUARE) {
#pragma unroll
        for (int e = 0; e < V; e += 2) {
          const double2 t = __ldg(reinterpret_cast<const double2*>(x + c + e));
          xv[e] = t.x, xv[e + 1] = t.y;
        }
      }
      T v[RD_ROWS][V];
#pragma unroll
      for (int q = 0; q < RD_ROWS; ++q)
        if (q < nr)
          *reinterpret_cast<uint4*>(v[q]) =
              __ldcs(reinterpret_cast<const uint4*>(a + (int64_t)q * lda + c));
#pragma unroll
      for (int q = 0; q < RD_ROWS; ++q)
        if (q < nr) {
#pragma unroll
          for (int e = 0; e < V; ++e) {
            const double ve = to_f64(v[q][e]);
            acc[q] = fma(ve, SQUARE ? ve : xv[e], acc[q]);
          }
        }
    }
  } else {
    for (int c = c0 + tid; c < c1; c += 256) {
      const double xc = SQUARE ? 0.0 : x[c];
#pragma unroll
      for (int q = 0; q < RD_ROWS; ++q)
        if (q < nr) {
          const double ve = to_f64(a[(int64_t)q * lda + c]);
          acc[q] = fma(ve, SQUARE ? ve : xc, acc[q]);
        }
    }
  }
  __shared__ double ws[8][RD_ROWS];
  __shared__ bool last;
#pragma unroll
  for (int q = 0; q < RD_ROWS; ++q) {
    const double v = warp_sum(acc[q]);
    if ((tid & 31) == 0) ws[tid >> 5][q] = v;
  }
  __syncthreads();
  if (tid < nr) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += ws[w][tid];
    rs.part[(int64_t)(r0 + tid) * nch + chunk] = t;
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) last = atomicAdd(&rs.cnt[grp], 1) == nch - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    if (tid < nr) {
      const int row = r0 + tid;
      double tot = 0.0;
      for (int z = 0; z < nch; ++z) tot += __ldcg(&rs.part[(int64_t)row * nch + z]);
      if (SQUARE) out[(int64_t)row * ld_out + row] = tot;
      else out[row] = tot - b[brow0 + row];
    }
    if (tid == 0) rs.cnt[grp] = 0;  // ready for the next launch (stream-ordered)
  }
}

// rows per CTA: 8 when the blocks are wide enough to give every SM several
// (chunk, group) CTAs, else 1 (narrow dense blocks, configs[0])
int rowdot_rows(int ell, int64_t n) {
  const int64_t ctas8 = (int64_t)((ell + 7) / 8) * std::min<int64_t>(64, std::max<int64_t>(1, n / 2048));
  return ctas8 >= 2 * 148 ? 8 : 1;
}
int rowdot_chunks(int ell, int64_t n) {
  const int R = rowdot_rows(ell, n);
  const int groups = (ell + R - 1) / R;
  // R = 8: one full wave (3 resident CTAs of 256 threads per SM at ~80
  // registers), so no second partial wave; R = 1: 4 CTAs per SM
  int nch = R == 8 ? std::max(1, 3 * 148 / groups) : (int)((4 * 148 + groups - 1) / groups);
  if (const char* e = getenv("SLIM_RD_NCH")) nch = std::max(1, atoi(e));  // tuning knob
  nch = (int)std::min<int64_t>(nch, std::max<int64_t>(1, n / 2048));
  return std::max(1, std::min(nch, 64));
}

// ---------------------------------------------------------------------------
// configs[4] generator: A[i, j] = fp32((2u - 1) / sqrt(n)),
// u = (splitmix64(seed ^ (i n + j)) >> 11) 2^-53, evaluated in fp64.
// ---------------------------------------------------------------------------

__device__ __forceinline__ float gen_elem(uint64_t seed, uint64_t i, uint64_t j, uint64_t n_total,
                                         double sqrt_n) {
  const uint64_t z = splitmix64(seed ^ (i * n_total + j));
  const double u = (double)(z >> 11) * 0x1.0p-53;
  return (float)((2.0 * u - 1.0) / sqrt_n);
}

// one sampled block (ell rows from global row row0) into dst (ell x n_local);
// with hi/lo non-null also the 3xTF32 operand split for the tensor-core Gram
__global__ void __launch_bounds__(256) k_gen_block(float* __restrict__ dst, float* __restrict__ hi,
                                                   float* __restrict__ lo, uint64_t seed,
                                                   int64_t row0, int ell, int n_local,
                                                   int64_t n_total, int64_t col0) {
  const double sq = sqrt((double)n_total);
  const int64_t total = (int64_t)ell * n_local;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e / n_local, c = e - a * n_local;
    const float v =
        gen_elem(seed, (uint64_t)(row0 + a), (uint64_t)(col0 + c), (uint64_t)n_total, sq);
    dst[e] = v;
    if (hi != nullptr) {
      float h, l;
      split_tf32(v, h, l);
      hi[e] = h;
      lo[e] = l;
    }
  }
}

// out[i] = sum_j A[i, j] x[j] over all m rows (problem setup: clean data)
__global__ void __launch_bounds__(256) k_gen_apply(double* __restrict__ out, uint64_t seed,
                                                   int64_t m, int n_local, int64_t n_total,
                                                   int64_t col0, const double* __restrict__ x) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const double sq = sqrt((double)n_total);
  double s = 0.0;
  for (int c = lane; c < n_local; c += 32)
    s += (double)gen_elem(seed, (uint64_t)row, (uint64_t)(col0 + c), (uint64_t)n_total, sq) * x[c];
  s = warp_sum(s);
  if (lane == 0) out[row] = s;
}

// one CTA (RES_THREADS) per row, four interleaved partial sums per thread
// added in a fixed order (deterministic).  Rows of up to RES_PRE * RES_THREADS
// nonzeros (every ray of the tomography configs) load ALL their (column,
// value) pairs first and then gather x for all of them, so a row costs three
// dependent memory latencies (row pointer, entries, x) instead of two per
// group of four; the sums are formed in exactly the order of the loop below,
// which longer rows still take.
constexpr int RES_THREADS = 128;
constexpr int RES_PRE = 12;
template <typename T>
__global__ void __launch_bounds__(RES_THREADS) k_residual_csr(double* r, const int64_t* __restrict__ rowptr,
                                                      const int* __restrict__ col,
                                                      const T* __restrict__ val, int64_t row0,
                                                      int64_t brow0, int ell,
                                                      const double* __restrict__ x,
                                                      const double* __restrict__ b,
                                                      const Ctl* ctl) {
  const int row = blockIdx.x, tid = threadIdx.x;
  const int64_t lo = rowptr[row0 + row], hi = rowptr[row0 + row + 1];
  const double bv = b[brow0 + row];
  if (ctl->diverged_at != 0) return;
  constexpr int S = RES_THREADS;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (hi - lo <= (int64_t)RES_PRE * S) {
    const int64_t e0 = lo + tid;
    int k[RES_PRE];
    T v[RES_PRE];
    double xv[RES_PRE];
#pragma unroll
    for (int u = 0; u < RES_PRE; ++u) {
      const bool ok = e0 + u * S < hi;
      k[u] = ok ? __ldcs(col + e0 + u * S) : 0;
      v[u] = ok ? __ldcs(val + e0 + u * S) : T(0);
    }
#ifdef SLIM_BOUNDS
#pragma unroll
    for (int u = 0; u < RES_PRE; ++u)
      if ((unsigned)k[u] > 0x3fffffu) {
        printf("SLIM_BOUNDS k_residual_csr: row %d (global %lld) entry %lld col %d\n", row,
               (long long)(row0 + row), (long long)(e0 + u * S), k[u]);
        k[u] = 0;
      }
#endif
#pragma unroll
    for (int u = 0; u < RES_PRE; ++u) xv[u] = (e0 + u * S < hi) ? __ldg(x + k[u]) : 0.0;
    // whole groups of four go to s0..s3, the remaining entries to s0
    int done = 0;
#pragma unroll
    for (int g = 0; g < RES_PRE / 4; ++g)
      if (done == 4 * g && e0 + (4 * g + 3) * S < hi) {
        s0 = fma(to_f64(v[4 * g]), xv[4 * g], s0);
        s1 = fma(to_f64(v[4 * g + 1]), xv[4 * g + 1], s1);
        s2 = fma(to_f64(v[4 * g + 2]), xv[4 * g + 2], s2);
        s3 = fma(to_f64(v[4 * g + 3]), xv[4 * g + 3], s3);
        done = 4 * g + 4;
      }
#pragma unroll
    for (int u = 0; u < RES_PRE; ++u)
      if (u >= done && e0 + u * S < hi) s0 = fma(to_f64(v[u]), xv[u], s0);
  } else {
    int64_t e = lo + tid;
    for (; e + 3 * S < hi; e += 4 * S) {
      const int k0 = __ldcs(col + e), k1 = __ldcs(col + e + S), k2 = __ldcs(col + e + 2 * S),
                k3 = __ldcs(col + e + 3 * S);
      const double v0 = to_f64(__ldcs(val + e)), v1 = to_f64(__ldcs(val + e + S)),
                   v2 = to_f64(__ldcs(val + e + 2 * S)), v3 = to_f64(__ldcs(val + e + 3 * S));
      s0 = fma(v0, __ldg(x + k0), s0);
      s1 = fma(v1, __ldg(x + k1), s1);
      s2 = fma(v2, __ldg(x + k2), s2);
      s3 = fma(v3, __ldg(x + k3), s3);
    }
    for (; e < hi; e += S) s0 = fma(to_f64(val[e]), x[col[e]], s0);
  }
  const double sv = warp_sum((s0 + s1) + (s2 + s3));
  __shared__ double ws[S / 32];
  if ((tid & 31) == 0) ws[tid >> 5] = sv;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < S / 32; ++w) t += ws[w];
    r[row] = t - bv;
  }
}

// ---------------------------------------------------------------------------
// Gram panel of the newest block: panel[(slot(P) ell + a) ell + j] =
// A_P[a] . A_k[j] for every window row (P, a) and new row j.
// ---------------------------------------------------------------------------

// CSR: one warp per window row.  Each nonzero (c, v) of the row looks up
// column c of the new block's CSC (<= a few entries for ray geometry) and
// contributes v * u to acc[j].  Lanes that hit the same j in one round are
// grouped with match_any and summed by the group leader in lane order, so
// the accumulation order is a pure function of the data.
template <typename T>
__global__ void __launch_bounds__(128) k_gram_csr(double* __restrict__ panel, Window W,
                                                  const int64_t* __restrict__ rowptr,
                                                  const int* __restrict__ col,
                                                  const T* __restrict__ val,
                                                  const int* __restrict__ colptr_new,
                                                  const int* __restrict__ cscrow,
                                                  const T* __restrict__ cscval, int64_t base_new) {
  extern __shared__ __align__(16) double gacc[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ell = W.ell;
  // one window row per CTA; its nonzeros are split in 4 contiguous quarters
  // (one per warp: 4x shorter chains of dependent CSC lookups), the four
  // partial rows are added in warp order (deterministic)
  const int grow_w = blockIdx.x;
  const int P = grow_w / ell, a = grow_w - P * ell;
  double* acc = gacc + (size_t)warp * ell;
  for (int j = lane; j < ell; j += 32) acc[j] = 0.0;
  __syncwarp();
  const int64_t grow = (int64_t)W.blk[P] * ell + a;
  const int64_t rlo = rowptr[grow], rhi = rowptr[grow + 1];
  const int64_t q4 = (rhi - rlo + 3) / 4;
  const int64_t lo = rlo + warp * q4, hi = min(rhi, lo + q4);
  const unsigned full = 0xffffffffu;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = lo; base < hi; base += 32) {
    const int64_t e = base + lane;
    int cs = 0, cnt = 0;
    double v = 0.0;
    if (e < hi) {
      int c = col[e];
#ifdef SLIM_BOUNDS
      if ((unsigned)c > 0x3fffffu) {
        printf("SLIM_BOUNDS k_gram_csr: window row %d entry %lld col %d\n", grow_w, (long long)e, c);
        c = 0;
      }
#endif
      v = to_f64(val[e]);
      cs = colptr_new[c];
      cnt = colptr_new[c + 1] - cs;
#ifdef SLIM_BOUNDS
      if (cs < 0 || cnt < 0 || cnt > ell) {
        printf("SLIM_BOUNDS k_gram_csr: new block column %d range [%d, +%d)\n", c, cs, cnt);
        cnt = 0;
      }
#endif
    }
    int maxcnt = cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxcnt = max(maxcnt, __shfl_xor_sync(full, maxcnt, o));
    for (int s = 0; s < maxcnt; ++s) {
      const bool has = s < cnt;
      int j = -1 - lane;
      double prod = 0.0;
      if (has) {
        const int64_t q = base_new + cs + s;
        j = cscrow[q];
        prod = v * to_f64(cscval[q]);
      }
      const unsigned mask = __match_any_sync(full, j);
      const bool leader = has && ((mask & lt) == 0u);
      int gsz = __popc(mask);
      int maxg = has ? gsz : 1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxg = max(maxg, __shfl_xor_sync(full, maxg, o));
      double sum = prod;
      unsigned m = mask;
      for (int q = 1; q < maxg; ++q) {
        m &= (m - 1u);
        const int src = m ? (__ffs(m) - 1) : lane;
        const double pv = __shfl_sync(full, prod, src);
        if (m) sum += pv;
      }
      if (leader) acc[j] += sum;
      __syncwarp();
    }
  }
  __syncthreads();
  double* out = panel + ((int64_t)P * ell + a) * ell;  // panels are indexed by window position
  for (int j = threadIdx.x; j < ell; j += 128)
    out[j] = (gacc[j] + gacc[ell + j]) + (gacc[2 * ell + j] + gacc[3 * ell + j]);
}

// ---------------------------------------------------------------------------
// CSR Gram, round 2: per-column records + exact fixed-point accumulation.
//
// ncu of k_gram_csr: 10 warp instructions per nonzero, warps stalled on the
// match_any / shuffle / shared-memory chain that keeps the sums in a fixed
// order (short scoreboard 4.3, wait 2.5 per issue), not on memory.  Two
// changes:
//
// * k_gram_lut packs every column of the new block into ONE record (entry
//   count, the rows of its first two entries in 16 bits each, their values),
//   so a nonzero of a window row costs one gather instead of the chain
//   column pointer -> row index / value.  Ray geometry never has more than
//   two entries per column and view; longer columns fall back to the CSC
//   arrays for the entries past the second.
//
// * Products are accumulated as 64-bit integers.  With 2^ea >= 2 ||A_P[a]||_2
//   (computed by the CTA from the row it just loaded) and 2^ej >= 2 ||A_k[j]||_2
//   (k_gram_rowexp; the record values are pre-scaled by 2^-ej, exactly), every
//   partial sum of a panel entry is below 2^60 quanta of 2^(ea + ej - 62) by
//   Cauchy-Schwarz.  Integer addition is associative, so the result does not
//   depend on the order in which threads add -- no grouping, no per-warp
//   copies of the row -- and it is deterministic like the rest of the path.
//   Each product is rounded once to 2^-62 of ||a|| ||b||, below the
//   gamma_n |a|.|b| error bound of an fp64 dot product of the same rows.
// ---------------------------------------------------------------------------
template <typename T>
struct GramRec;
template <>
struct __align__(16) GramRec<float> {
  int cnt;
  unsigned j01;  // row of entry 0 | row of entry 1 << 16
  float v0, v1;  // values scaled by 2^-e(row)
};
template <>
struct __align__(32) GramRec<double> {
  int cnt;
  unsigned j01;
  double v0, v1;
  double pad;
};
__device__ __forceinline__ float scale_pow2(float v, int e) { return ldexpf(v, e); }
__device__ __forceinline__ double scale_pow2(double v, int e) { return ldexp(v, e); }
// exponent e with 2^e >= 2 sqrt(ss) (0 for an empty row): with b = floor(log2 ss) from
// the exponent field, sqrt(ss) < 2^ceil((b + 1) / 2)
__device__ __forceinline__ int norm_exp(double ss) {
  if (!(ss > 0.0)) return 0;
  const int bexp = (__double2hiint(ss) >> 20) & 0x7ff;
  const int b = bexp ? bexp - 1023 : ilogb(ss);  // subnormal sums take the slow path
  return ((b + 2) >> 1) + 1;
}

// one warp per row of the new block: rowexp[j] = norm_exp(||A_k[j]||^2)
template <typename T>
__global__ void __launch_bounds__(256) k_gram_rowexp(int* __restrict__ rowexp,
                                                     const int64_t* __restrict__ rowptr,
                                                     const T* __restrict__ val, int64_t row0,
                                                     int ell) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= ell) return;
  const int64_t lo = rowptr[row0 + j], hi = rowptr[row0 + j + 1];
  double ss = 0.0;
  for (int64_t e = lo + lane; e < hi; e += 32) {
    const double v = to_f64(__ldg(val + e));
    ss = fma(v, v, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) rowexp[j] = norm_exp(ss);
}

template <typename T>
__global__ void __launch_bounds__(256) k_gram_lut(GramRec<T>* __restrict__ lut,
                                                  const int* __restrict__ rowexp,
                                                  const int* __restrict__ colptr_new,
                                                  const int* __restrict__ cscrow,
                                                  const T* __restrict__ cscval, int64_t base_new,
                                                  int n) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int cs = colptr_new[c], cnt = colptr_new[c + 1] - cs;
  GramRec<T> rec{};
  rec.cnt = cnt;
  if (cnt > 0) {
    const int j = cscrow[base_new + cs];
    rec.j01 = (unsigned)j;
    rec.v0 = scale_pow2(cscval[base_new + cs], -rowexp[j]);
  }
  if (cnt > 1) {
    const int j = cscrow[base_new + cs + 1];
    rec.j01 |= (unsigned)j << 16;
    rec.v1 = scale_pow2(cscval[base_new + cs + 1], -rowexp[j]);
  }
  lut[c] = rec;
}

__device__ __forceinline__ GramRec<float> ld_rec(const GramRec<float>* p) {
  const int4 q = __ldg(reinterpret_cast<const int4*>(p));
  GramRec<float> r;
  r.cnt = q.x;
  r.j01 = (unsigned)q.y;
  r.v0 = __int_as_float(q.z);
  r.v1 = __int_as_float(q.w);
  return r;
}
__device__ __forceinline__ GramRec<double> ld_rec(const GramRec<double>* p) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  GramRec<double> r;
  r.cnt = a.x;
  r.j01 = (unsigned)a.y;
  r.v0 = __hiloint2double(a.w, a.z);
  r.v1 = b.x;
  return r;
}

constexpr int GFX_THREADS = 256;
constexpr int GFX_K = 6;  // nonzeros per thread and chunk (rows of <= 1536 nonzeros: one chunk)

// acc[j] += d for a 64-bit two's-complement d, with the accumulator held as
// two 32-bit words: shared memory has native 32-bit integer atomics only
// (a 64-bit atomicAdd compiles to a compare-and-swap spin loop, ~70 shared
// memory wavefronts per warp-level add under ncu).  The low word's add returns
// the old value, which tells THIS add's carry; carries are added to the high
// word with the addend's own high part.  The total is sum(d) mod 2^64 in any
// order of arrival.
__device__ __forceinline__ void fx_add(unsigned* lo, unsigned* hi, int j, long long d) {
  const unsigned dl = (unsigned)(unsigned long long)d, dh = (unsigned)((unsigned long long)d >> 32);
  const unsigned old = atomicAdd(lo + j, dl);
  const unsigned carry = (old + dl < old) ? 1u : 0u;
  if (dh + carry != 0u) atomicAdd(hi + j, dh + carry);
}

// 2^e as a double for any e in the normal range (callers keep it there)
__device__ __forceinline__ double pow2_double(int e) { return __hiloint2double((1023 + e) << 20, 0); }
__device__ __forceinline__ double pow2_any(int e) {
  return (e > -1000 && e < 1000) ? pow2_double(e) : ldexp(1.0, e);
}

// Persistent CTAs, each taking window rows blockIdx.x, + gridDim.x, ...; acc[j]
// (64-bit integers as two words) in shared memory.  A thread takes GFX_K
// ADJACENT nonzeros of the row: neighbours along a ray meet the same ray of
// the new view, so their products are first merged in registers (integer
// adds, any grouping gives the same total) and roughly half the shared-memory
// atomics go away.  While a row is processed, the row pointer of the CTA's
// next row is fetched and its (column, value) lines are prefetched into L2.
template <typename T>
__global__ void __launch_bounds__(GFX_THREADS, 4) k_gram_csr_fx(double* __restrict__ panel, Window W,
                                                                const int64_t* __restrict__ rowptr,
                                                                const int* __restrict__ col,
                                                                const T* __restrict__ val,
                                                                const GramRec<T>* __restrict__ lut,
                                                                const int* __restrict__ rowexp,
                                                                const int* __restrict__ colptr_new,
                                                                const int* __restrict__ cscrow,
                                                                const T* __restrict__ cscval,
                                                                int64_t base_new) {
  extern __shared__ __align__(16) unsigned facc[];
  __shared__ double red[2][GFX_THREADS / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ell = W.ell, nrows = W.nw * ell;
  unsigned* flo = facc;
  unsigned* fhi = facc + ell;
  constexpr int S = GFX_THREADS, CH = GFX_K * GFX_THREADS;
  auto global_row = [&](int r) {
    const int P = r / ell;
    return (int64_t)W.blk[P] * ell + (r - P * ell);
  };
  int r = blockIdx.x;
  if (r >= nrows) return;
  int64_t rlo, rhi;
  {
    const int64_t g = global_row(r);
    rlo = rowptr[g];
    rhi = rowptr[g + 1];
  }
  for (int it = 0; r < nrows; r += gridDim.x, ++it) {
    // next row of this CTA: row pointer now, its lines into L2
    const int rn = r + gridDim.x;
    int64_t nlo = 0, nhi = 0;
    if (rn < nrows) {
      const int64_t g = global_row(rn);
      nlo = rowptr[g];
      nhi = rowptr[g + 1];
    }
    int cc[GFX_K];
    T vv[GFX_K];
    {
      const int64_t e0 = rlo + (int64_t)tid * GFX_K;
#pragma unroll
      for (int u = 0; u < GFX_K; ++u) {
        cc[u] = -1;
        vv[u] = T(0);
        if (e0 + u < rhi) {
          cc[u] = __ldcs(col + e0 + u);
          vv[u] = __ldcs(val + e0 + u);
        }
      }
    }
    {  // 2 ell words, 16 bytes at a time (ell even is the common case)
      uint4* z = reinterpret_cast<uint4*>(facc);
      const int n4 = (2 * ell) >> 2;
      for (int j = tid; j < n4; j += S) z[j] = make_uint4(0u, 0u, 0u, 0u);
      for (int j = 4 * n4 + tid; j < 2 * ell; j += S) facc[j] = 0u;
    }
    if (rn < nrows) {
      // 128-byte lines of col[nlo, nhi) and val[nlo, nhi)
      const char* c0 = reinterpret_cast<const char*>(col + nlo);
      const char* c1 = reinterpret_cast<const char*>(col + nhi);
      for (const char* p = c0 + (size_t)tid * 128; p < c1; p += (size_t)S * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
      const char* v0 = reinterpret_cast<const char*>(val + nlo);
      const char* v1 = reinterpret_cast<const char*>(val + nhi);
      for (const char* p = v0 + (size_t)tid * 128; p < v1; p += (size_t)S * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
    }
    // ||row||^2 in a fixed order: per thread, warp shuffle tree, warps in order
    double ss = 0.0;
#pragma unroll
    for (int u = 0; u < GFX_K; ++u) ss = fma(to_f64(vv[u]), to_f64(vv[u]), ss);
    for (int64_t e = rlo + CH + tid; e < rhi; e += S) {
      const double v = to_f64(__ldg(val + e));
      ss = fma(v, v, ss);
    }
    ss = warp_sum(ss);
    if (lane == 0) red[it & 1][warp] = ss;
    __syncthreads();  // also: acc zeroed, and the previous row's output loop is done
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < S / 32; ++w) tot += red[it & 1][w];
    const int ea = norm_exp(tot);
    const double scale = pow2_any(62 - ea);
    for (int64_t base = rlo; base < rhi; base += CH) {
      if (base != rlo) {
        const int64_t e0 = base + (int64_t)tid * GFX_K;
#pragma unroll
        for (int u = 0; u < GFX_K; ++u) {
          cc[u] = -1;
          vv[u] = T(0);
          if (e0 + u < rhi) {
            cc[u] = __ldcs(col + e0 + u);
            vv[u] = __ldcs(val + e0 + u);
          }
        }
      }
      GramRec<T> rec[GFX_K];
#pragma unroll
      for (int u = 0; u < GFX_K; ++u) {
        rec[u].cnt = 0;
        if (cc[u] >= 0) rec[u] = ld_rec(lut + cc[u]);
      }
      // entries 0 and 1 of each column: runs of equal rows merged in registers
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        int curj = -1;
        long long cur = 0;
#pragma unroll
        for (int u = 0; u < GFX_K; ++u)
          if (rec[u].cnt > sl) {
            const int j = sl == 0 ? (int)(rec[u].j01 & 0xffffu) : (int)(rec[u].j01 >> 16);
            const double uv = to_f64(sl == 0 ? rec[u].v0 : rec[u].v1);
            const long long d = __double2ll_rn(to_f64(vv[u]) * scale * uv);
            if (j == curj) {
              cur += d;
            } else {
              if (curj >= 0) fx_add(flo, fhi, curj, cur);
              curj = j;
              cur = d;
            }
          }
        if (curj >= 0) fx_add(flo, fhi, curj, cur);
      }
#pragma unroll
      for (int u = 0; u < GFX_K; ++u)
        if (rec[u].cnt > 2) {  // a column with more than two entries: the CSC arrays
          const int64_t q0 = base_new + colptr_new[cc[u]];
          for (int t = 2; t < rec[u].cnt; ++t) {
            const int j = cscrow[q0 + t];
            const double uv = ldexp(to_f64(cscval[q0 + t]), -rowexp[j]);
            fx_add(flo, fhi, j, __double2ll_rn(to_f64(vv[u]) * scale * uv));
          }
        }
    }
    __syncthreads();
    const int P = r / ell;
    double* out = panel + ((int64_t)P * ell + (r - P * ell)) * ell;  // indexed by window position
    for (int j = tid; j < ell; j += S) {
      // (int)hi 2^32 + lo, rounded once: the correctly rounded 64-bit integer
      const double qd = fma((double)(int)fhi[j], 4294967296.0, (double)flo[j]);
      const int e = ea + __ldg(rowexp + j) - 62;
      out[j] = (e > -1000 && e < 1000) ? qd * pow2_double(e) : ldexp(qd, e);
    }
    __syncthreads();  // acc is zeroed again at the top
    rlo = nlo;
    rhi = nhi;
  }
}

// Dense: DMMA tile GEMM, 64 window rows x 64 new rows per CTA, split-K over
// blockIdx.z into fp64 partials reduced in a fixed order by k_gram_reduce.
constexpr int GK = 32, GS = 36;  // K chunk and smem stride (doubles)

template <typename T>
__global__ void __launch_bounds__(256) k_gram_dense(double* __restrict__ part, Window W,
                                                    const T* __restrict__ A, int64_t lda,
                                                    int64_t newrow0, int n, int klen) {
  __shared__ __align__(16) double As[64 * GS];
  __shared__ __align__(16) double Bs[64 * GS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ell = W.ell, N = W.nw * ell;
  const int p0 = blockIdx.x * 64, j0 = blockIdx.y * 64;
  const int kbeg = blockIdx.z * klen, kend = min(n, kbeg + klen);
  // row pointers this thread loads (8 rows x 4 lanes per 32-wide row)
  double acc[8][2];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
  for (int kc = kbeg; kc < kend; kc += GK) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int idx = tid + it * 256;
      const int rr = idx >> 5, cc = idx & 31;
      const int k = kc + cc;
      const int p = p0 + rr;
      double va = 0.0, vb = 0.0;
      if (p < N && k < kend) {
        const int P = p / ell;
        va = to_f64(A[((int64_t)W.blk[P] * ell + (p - P * ell)) * lda + k]);
      }
      const int jr = j0 + rr;
      if (jr < ell && k < kend) vb = to_f64(A[(newrow0 + jr) * lda + k]);
      As[rr * GS + cc] = va;
      Bs[rr * GS + cc] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < GK / 4; ++k4) {
      const double a = As[(warp * 8 + (lane >> 2)) * GS + 4 * k4 + (lane & 3)];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const double b = Bs[(nt * 8 + (lane >> 2)) * GS + 4 * k4 + (lane & 3)];
        dmma8x8x4(acc[nt], a, b);
      }
    }
    __syncthreads();
  }
  const int p = p0 + warp * 8 + (lane >> 2);
  if (p < N) {
    double* out = part + (int64_t)blockIdx.z * N * ell + (int64_t)p * ell;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int j = j0 + nt * 8 + 2 * (lane & 3);
      if (j < ell) out[j] = acc[nt][0];
      if (j + 1 < ell) out[j + 1] = acc[nt][1];
    }
  }
}

__global__ void k_gram_reduce(double* __restrict__ panel, Window W, const double* __restrict__ part,
                              int nsplit) {
  const int ell = W.ell, N = W.nw * ell;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)N * ell) return;
  const int p = (int)(idx / ell), j = (int)(idx - (int64_t)p * ell);
  double s = 0.0;
  for (int z = 0; z < nsplit; ++z) s += part[(int64_t)z * N * ell + idx];
  const int P = p / ell, a = p - P * ell;
  panel[((int64_t)P * ell + a) * ell + j] = s;
}

// ---------------------------------------------------------------------------
// s = M^T w (alpha applied in k_finish)
// ---------------------------------------------------------------------------

// part[y, c] = sum over the window rows of split y of A[row, c] w[row]:
// each thread owns V = 16 / sizeof(T) adjacent columns (one 16-byte load
// per row), rows unrolled so several loads are in flight per thread
template <typename T, int V>
__global__ void __launch_bounds__(256) k_mtw_dense(double* __restrict__ part, Window W,
                                                   const T* __restrict__ A, int64_t lda, int n,
                                                   const double* __restrict__ w, int rows_per_split,
                                                   const Ctl* ctl) {
  if (ctl->diverged_at != 0) return;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * V;
  if (c >= n) return;
  const int ell = W.ell, N = W.nw * ell;
  const int pbeg = blockIdx.y * rows_per_split, pend = min(N, pbeg + rows_per_split);
  double s[V];
#pragma unroll
  for (int e = 0; e < V; ++e) s[e] = 0.0;
  for (int p = pbeg; p < pend;) {
    const int P = p / ell;
    const int a0 = p - P * ell;
    const int cnt = min(ell - a0, pend - p);
    const T* base = A + ((int64_t)W.blk[P] * ell + a0) * lda + c;
#pragma unroll 4
    for (int q = 0; q < cnt; ++q) {
      T v[V];
      if (V > 1) *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(base + (int64_t)q * lda);
      else v[0] = base[(int64_t)q * lda];
      const double wq = w[p + q];
#pragma unroll
      for (int e = 0; e < V; ++e) s[e] = fma(to_f64(v[e]), wq, s[e]);
    }
    p += cnt;
  }
#pragma unroll
  for (int e = 0; e < V; ++e) part[(int64_t)blockIdx.y * n + c + e] = s[e];
}

// one thread per column; the window's blocks are taken MTW_GROUP at a time
// with every block's column range and first nonzero loaded before any is
// used, so a thread waits on ~3 dependent loads per group instead of per
// block (the kernel was latency-bound at 3 chains x r + 1 blocks). The
// accumulation order (block, then nonzero) is unchanged.
template <typename T, int MTW_GROUP>
__device__ __forceinline__ double mtw_csc_col(int c, const Window& W, const int* __restrict__ colptr,
                                              int n, const int* __restrict__ cscrow,
                                              const T* __restrict__ cscval,
                                              const int64_t* __restrict__ blkbase,
                                              const double* __restrict__ w) {
  const int ell = W.ell;
  double s = 0.0;
  for (int P0 = 0; P0 < W.nw; P0 += MTW_GROUP) {
    int lo[MTW_GROUP], hi[MTW_GROUP];
    int64_t base[MTW_GROUP];
#pragma unroll
    for (int q = 0; q < MTW_GROUP; ++q) {
      lo[q] = hi[q] = 0;
      base[q] = 0;
      if (P0 + q < W.nw) {
        const int bk = W.blk[P0 + q];
        const int* cp = colptr + (int64_t)bk * csc_stride(n);
        lo[q] = __ldcs(cp + c);
        hi[q] = __ldcs(cp + c + 1);
        base[q] = __ldg(blkbase + bk);
#ifdef SLIM_BOUNDS
        if (lo[q] < 0 || hi[q] < lo[q] || hi[q] - lo[q] > ell) {
          printf("SLIM_BOUNDS mtw_csc_col: block %d (position %d) column %d range [%d, %d)\n", bk, P0 + q,
                 c, lo[q], hi[q]);
          hi[q] = lo[q] = 0;
        }
#endif
      }
    }
    double v[MTW_GROUP], wv[MTW_GROUP];
#pragma unroll
    for (int q = 0; q < MTW_GROUP; ++q) {
      v[q] = 0.0, wv[q] = 0.0;
      if (lo[q] < hi[q]) {
        const int64_t e = base[q] + lo[q];
        v[q] = to_f64(__ldcs(cscval + e));
#ifdef SLIM_BOUNDS
        if ((unsigned)__ldcs(cscrow + e) >= (unsigned)ell) {
          printf("SLIM_BOUNDS mtw_csc_col: block at position %d column %d entry %lld row %d\n", P0 + q, c,
                 (long long)e, __ldcs(cscrow + e));
          lo[q] = hi[q] = 0;
          continue;
        }
#endif
        wv[q] = __ldg(w + (P0 + q) * ell + __ldcs(cscrow + e));
      }
    }
#pragma unroll
    for (int q = 0; q < MTW_GROUP; ++q) {
      if (lo[q] < hi[q]) {
        s += v[q] * wv[q];
        const double* wp = w + (P0 + q) * ell;
        for (int e = lo[q] + 1; e < hi[q]; ++e)
          s += to_f64(cscval[base[q] + e]) * wp[cscrow[base[q] + e]];
      }
    }
  }
  return s;
}
template <typename T, int MTW_GROUP>
__global__ void __launch_bounds__(256) k_mtw_csc(double* __restrict__ s_out, Window W,
                                                 const int* __restrict__ colptr, int n,
                                                 const int* __restrict__ cscrow,
                                                 const T* __restrict__ cscval,
                                                 const int64_t* __restrict__ blkbase,
                                                 const double* __restrict__ w, const Ctl* ctl) {
  if (ctl->diverged_at != 0) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  s_out[c] = mtw_csc_col<T, MTW_GROUP>(c, W, colptr, n, cscrow, cscval, blkbase, w);
}

// ---------------------------------------------------------------------------
// finish: x update, norms, divergence, history (last-block reduction)
// ---------------------------------------------------------------------------

// x[c] -= alpha sn for this thread's column, then the norms, divergence and
// history row by a last-block reduction (every thread of the grid calls it)
__device__ __forceinline__ void finish_reduce(const FinishParams& F, const double (&loc)[1 + MAX_REFS]);

__device__ __forceinline__ void finish_body(const FinishParams& F, int c, double sn) {
  double loc[1 + MAX_REFS];
#pragma unroll
  for (int q = 0; q < 1 + MAX_REFS; ++q) loc[q] = 0.0;
  if (c < F.n) {
    const double xn = F.x[c] - F.alpha * sn;
    F.x[c] = xn;
    loc[0] = xn * xn;
#pragma unroll
    for (int q = 0; q < MAX_REFS; ++q)
      if (q < F.nref) {
        const double d = xn - F.refs[q][c];
        loc[1 + q] = d * d;
      }
  }
  finish_reduce(F, loc);
}

// four consecutive columns c0 .. c0 + 3 per thread (n % 4 == 0): 16-byte
// loads and stores of x and the references
__device__ __forceinline__ void finish_body4(const FinishParams& F, int c0, const double (&sn)[4]) {
  double loc[1 + MAX_REFS];
#pragma unroll
  for (int q = 0; q < 1 + MAX_REFS; ++q) loc[q] = 0.0;
  if (c0 < F.n) {
    double2* xp = reinterpret_cast<double2*>(F.x + c0);
    const double2 xa = xp[0], xb = xp[1];
    const double x0 = xa.x - F.alpha * sn[0], x1 = xa.y - F.alpha * sn[1];
    const double x2 = xb.x - F.alpha * sn[2], x3 = xb.y - F.alpha * sn[3];
    xp[0] = make_double2(x0, x1);
    xp[1] = make_double2(x2, x3);
    loc[0] = (x0 * x0 + x1 * x1) + (x2 * x2 + x3 * x3);
#pragma unroll
    for (int q = 0; q < MAX_REFS; ++q)
      if (q < F.nref) {
        const double2* rp = reinterpret_cast<const double2*>(F.refs[q] + c0);
        const double2 ra = __ldg(rp), rb = __ldg(rp + 1);
        const double d0 = x0 - ra.x, d1 = x1 - ra.y, d2 = x2 - rb.x, d3 = x3 - rb.y;
        loc[1 + q] = (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
      }
  }
  finish_reduce(F, loc);
}

// per-thread partial norms -> block partials -> (last block) the totals,
// divergence test and history row, in a fixed order (deterministic)
__device__ __forceinline__ void finish_reduce(const FinishParams& F, const double (&loc)[1 + MAX_REFS]) {
  Ctl* ctl = F.ctl;
  const int tid = threadIdx.x;
  const int nq = 1 + F.nref;
  __shared__ double red[8][1 + MAX_REFS];
  __shared__ bool s_last;
  const int warp = tid >> 5, lane = tid & 31;
  for (int q = 0; q < nq; ++q) {
    const double v = warp_sum(loc[q]);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (tid < nq) {
    double v = 0.0;
    for (int wi = 0; wi < 8; ++wi) v += red[wi][tid];
    F.part[(int64_t)blockIdx.x * nq + tid] = v;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&ctl->done, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // deterministic final sums: warp q reduces quantity q over the blocks
  __shared__ double tot[1 + MAX_REFS];
  __shared__ double s_rn;
  if (warp < nq) {
    double v = 0.0;
    for (int bi = lane; bi < (int)gridDim.x; bi += 32) v += __ldcg(F.part + (int64_t)bi * nq + warp);
    v = warp_sum(v);
    if (lane == 0) tot[warp] = v;
  }
  if (warp == 7) {
    double v = 0.0;
    for (int jj = lane; jj < F.ell; jj += 32) {
      const double rv = __ldcg(F.r + jj);
      v += rv * rv;
    }
    v = warp_sum(v);
    if (lane == 0) s_rn = v;
  }
  __syncthreads();
  if (F.split) {
    if (tid < nq) F.norms[tid] = tot[tid];
    if (tid == 0) ctl->done = 0u;
    return;
  }
  if (tid == 0) {
    ctl->done = 0u;
    ctl->rnorm2 = s_rn;
    const double nsq = tot[0];
    const bool diverged = !(nsq <= ctl->div_limit_sq);
    if (diverged) ctl->diverged_at = F.k;
    if (F.record || diverged) {
      const int64_t row = ctl->nrows++;
      double* h = F.hist + row * (SLIM_HIST_FIXED_DEV + F.nref);
      h[0] = (double)F.k;
      h[1] = F.alpha;
      h[2] = sqrt(s_rn);
      h[3] = (double)(globaltimer_ns() - ctl->t_start_ns);
      h[4] = diverged ? 1.0 : 0.0;
      for (int q = 0; q < F.nref; ++q) h[SLIM_HIST_FIXED_DEV + q] = sqrt(tot[1 + q]);
    }
  }
}

__global__ void __launch_bounds__(256) k_finish(FinishParams F) {
  if (F.ctl->diverged_at != 0) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double sn = 0.0;
  if (c < F.n)
    for (int z = 0; z < F.nsplit; ++z) sn += F.s_parts[(int64_t)z * F.n + c];
  finish_body(F, c, sn);
}

// CSC M^T w fused with the finish: s stays in registers (bit-identical to
// k_mtw_csc + k_finish: the same sums, and 0 + s = s)
template <typename T>
__global__ void __launch_bounds__(256) k_mtw_finish_csc(FinishParams F, Window W,
                                                        const int* __restrict__ colptr,
                                                        const int* __restrict__ cscrow,
                                                        const T* __restrict__ cscval,
                                                        const int64_t* __restrict__ blkbase,
                                                        const double* __restrict__ w) {
  if (F.ctl->diverged_at != 0) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const double sn = c < F.n ? mtw_csc_col<T, 3>(c, W, colptr, F.n, cscrow, cscval, blkbase, w) : 0.0;
  finish_body(F, c, sn);
}

// Four columns per thread (c0 = 4 t, n % 4 == 0): one 16-byte load brings
// a block's four column pointers (the CSC arrays are padded to 16-byte
// aligned strides, csc_stride), the fifth comes from the next lane; the
// first E entries of G blocks are loaded before any is used, then their w
// gathers, so a thread keeps ~3 G E independent loads in flight instead of
// one dependent chain per block.  Per column the sums run block by block,
// entry by entry, like mtw_csc_col.
template <typename T, int G, int E>
__device__ __forceinline__ void mtw_csc_quad(int c0, bool valid, const Window& W,
                                             const int* __restrict__ colptr, int n,
                                             const int* __restrict__ cscrow,
                                             const T* __restrict__ cscval,
                                             const int64_t* __restrict__ blkbase,
                                             const double* __restrict__ w, double (&s)[4]) {
  const int64_t cps = csc_stride(n);
  const int ell = W.ell, lane = threadIdx.x & 31;
  for (int P0 = 0; P0 < W.nw; P0 += G) {
    int4 q[G];
    int hi[G];
    int64_t base[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      q[g] = make_int4(0, 0, 0, 0);
      base[g] = 0;
      if (P0 + g < W.nw) {
        const int bk = W.blk[P0 + g];
        q[g] = __ldcs(reinterpret_cast<const int4*>(colptr + (int64_t)bk * cps + c0));
        base[g] = __ldg(blkbase + bk);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      int nx = __shfl_down_sync(0xffffffffu, q[g].x, 1);
      if (lane == 31 && P0 + g < W.nw) nx = __ldcs(colptr + (int64_t)W.blk[P0 + g] * cps + c0 + 4);
      hi[g] = valid ? nx : q[g].x;
    }
    T v[G][E];
    int rw[G][E];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int idx = q[g].x + e;
        v[g][e] = T(0);
        rw[g][e] = 0;
        if (idx < hi[g]) {
          v[g][e] = __ldcs(cscval + base[g] + idx);
          rw[g][e] = __ldcs(cscrow + base[g] + idx);
        }
      }
    double wv[G][E];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int e = 0; e < E; ++e)
        wv[g][e] = (q[g].x + e < hi[g]) ? __ldg(w + (P0 + g) * ell + rw[g][e]) : 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double* wp = w + (P0 + g) * ell;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int idx = q[g].x + e;
        if (idx < hi[g]) {
          const int k = (idx >= q[g].y) + (idx >= q[g].z) + (idx >= q[g].w);
          const double pv = to_f64(v[g][e]);
          if (k == 0) s[0] = fma(pv, wv[g][e], s[0]);
          else if (k == 1) s[1] = fma(pv, wv[g][e], s[1]);
          else if (k == 2) s[2] = fma(pv, wv[g][e], s[2]);
          else s[3] = fma(pv, wv[g][e], s[3]);
        }
      }
      for (int idx = q[g].x + E; idx < hi[g]; ++idx) {  // long columns (rare)
        const int k = (idx >= q[g].y) + (idx >= q[g].z) + (idx >= q[g].w);
        const double pv = to_f64(__ldcs(cscval + base[g] + idx));
        const double wx = wp[__ldcs(cscrow + base[g] + idx)];
        if (k == 0) s[0] = fma(pv, wx, s[0]);
        else if (k == 1) s[1] = fma(pv, wx, s[1]);
        else if (k == 2) s[2] = fma(pv, wx, s[2]);
        else s[3] = fma(pv, wx, s[3]);
      }
    }
  }
}
template <typename T, int MTW4_G, int MTW4_E>
__global__ void __launch_bounds__(256) k_mtw_finish_csc4(FinishParams F, Window W,
                                                         const int* __restrict__ colptr,
                                                         const int* __restrict__ cscrow,
                                                         const T* __restrict__ cscval,
                                                         const int64_t* __restrict__ blkbase,
                                                         const double* __restrict__ w) {
  if (F.ctl->diverged_at != 0) return;
  const int c0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const bool valid = c0 < F.n;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  mtw_csc_quad<T, MTW4_G, MTW4_E>(valid ? c0 : F.n, valid, W, colptr, F.n, cscrow, cscval, blkbase,
                                  w, s);
  finish_body4(F, c0, s);
}
template <typename T, int MTW4_G, int MTW4_E>
__global__ void __launch_bounds__(256) k_mtw_csc4(double* __restrict__ s_out, Window W,
                                                  const int* __restrict__ colptr, int n,
                                                  const int* __restrict__ cscrow,
                                                  const T* __restrict__ cscval,
                                                  const int64_t* __restrict__ blkbase,
                                                  const double* __restrict__ w, const Ctl* ctl) {
  if (ctl->diverged_at != 0) return;
  const int c0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const bool valid = c0 < n;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  mtw_csc_quad<T, MTW4_G, MTW4_E>(valid ? c0 : n, valid, W, colptr, n, cscrow, cscval, blkbase, w,
                                  s);
  if (valid) {
    double2* o = reinterpret_cast<double2*>(s_out + c0);
    o[0] = make_double2(s[0], s[1]);
    o[1] = make_double2(s[2], s[3]);
  }
}

// ---------------------------------------------------------------------------
// M^T w with warp-staged, asynchronously prefetched entries (round 2, variant 6).
//
// ncu of the four-column kernel: 2.5 TB/s with the warps waiting on their own
// loads (long scoreboard) -- every byte in flight needs a destination
// register, and a lane walks its ~5 entries per block one dependent gather
// at a time.  Here a warp owns 128 consecutive columns (four per lane).  Per
// window block it reads their column pointers with one 16-byte load per lane.
// The warp's entries of that block are CONTIGUOUS in the block's CSC, so they
// are copied entry-parallel straight into shared memory with cp.async, two
// blocks ahead of the one being summed (the bytes in flight sit in shared
// memory, not registers).  When a block's entries have landed the lanes
// gather w[row] entry-parallel (neighbouring entries hit neighbouring rows)
// and each lane sums its four columns out of shared memory: two unrolled
// entries per column and a loop for longer ones.  A range longer than MS_CAP
// entries takes the direct global path for that block (warp-uniform).  Per
// column the sums still run block by block and entry by entry with the same
// fma chain, so s is bit-identical to the other variants.
// ---------------------------------------------------------------------------
constexpr int MS_CAP = 192;  // staged entries per warp and block
constexpr int MS_EPL = MS_CAP / 32;
constexpr int MS_NB = 3;     // entry buffers per warp (prefetch distance 2)
template <typename T>
constexpr size_t mtw_stage_smem() {
  return (size_t)8 * MS_CAP * (sizeof(double) + MS_NB * (sizeof(int) + sizeof(T)));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem));
}
__device__ __forceinline__ void cp_async_val(float* smem, const float* gmem) { cp_async4(smem, gmem); }
__device__ __forceinline__ void cp_async_val(double* smem, const double* gmem) { cp_async8(smem, gmem); }

// column pointers of one block for this lane's four columns
struct MtwCols {
  int4 q;
  int nx;        // lane 31: the pointer after its last column
  int64_t base;  // first entry of the block in cscrow / cscval
};

template <typename T>
__device__ __forceinline__ void mtw_csc_stage(int c0, bool valid, const Window& W,
                                              const int* __restrict__ colptr, int n,
                                              const int* __restrict__ cscrow,
                                              const T* __restrict__ cscval,
                                              const int64_t* __restrict__ blkbase,
                                              const double* __restrict__ w, double (&s)[4]) {
  extern __shared__ __align__(16) unsigned char ms_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  double* sw = reinterpret_cast<double*>(ms_raw) + warp * MS_CAP;
  T* svalb = reinterpret_cast<T*>(ms_raw + 8 * MS_CAP * sizeof(double)) + warp * MS_NB * MS_CAP;
  int* srowb = reinterpret_cast<int*>(ms_raw + 8 * MS_CAP * (sizeof(double) + MS_NB * sizeof(T))) +
               warp * MS_NB * MS_CAP;
  const int64_t cps = csc_stride(n);
  const int ell = W.ell, nw = W.nw;
  auto load_cols = [&](int P) {
    MtwCols m;
    m.q = make_int4(0, 0, 0, 0);
    m.nx = 0;
    m.base = 0;
    if (P < nw) {
      const int bk = W.blk[P];
      m.q = __ldcs(reinterpret_cast<const int4*>(colptr + (int64_t)bk * cps + c0));
      if (lane == 31) m.nx = __ldcs(colptr + (int64_t)bk * cps + c0 + (valid ? 4 : 0));
      m.base = __ldg(blkbase + bk);
    }
    return m;
  };
  // this lane's end pointer, the warp's first entry and entry count
  auto range = [&](const MtwCols& m, int& hi, int& s0, int& cnt) {
    hi = __shfl_down_sync(full, m.q.x, 1);
    if (lane == 31) hi = m.nx;
    if (!valid) hi = m.q.x;
    s0 = __shfl_sync(full, m.q.x, 0);
    cnt = __shfl_sync(full, hi, 31) - s0;
  };
  // start copying block P's entries into buffer P % MS_NB (one group per call)
  auto prefetch = [&](int P, const MtwCols& m) {
    if (P < nw) {
      int hi, s0, cnt;
      range(m, hi, s0, cnt);
      if (cnt > 0 && cnt <= MS_CAP) {
        int* sr = srowb + (P % MS_NB) * MS_CAP;
        T* sv = svalb + (P % MS_NB) * MS_CAP;
#pragma unroll
        for (int i = 0; i < MS_EPL; ++i) {
          const int idx = lane + 32 * i;
          if (idx < cnt) {
            cp_async4(sr + idx, cscrow + m.base + s0 + idx);
            cp_async_val(sv + idx, cscval + m.base + s0 + idx);
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  MtwCols m0 = load_cols(0), m1 = load_cols(1), m2 = load_cols(2);
  prefetch(0, m0);
  prefetch(1, m1);
  for (int P = 0; P < nw; ++P) {
    const MtwCols m3 = load_cols(P + 3);
    prefetch(P + 2, m2);
    asm volatile("cp.async.wait_group 2;" ::: "memory");
    __syncwarp();
    int hi, s0, cnt;
    range(m0, hi, s0, cnt);
    const int4 q = m0.q;
    const double* wp = w + (int64_t)P * ell;
    if (cnt > 0 && cnt <= MS_CAP) {
      const int* sr = srowb + (P % MS_NB) * MS_CAP;
      const T* sv = svalb + (P % MS_NB) * MS_CAP;
      int rw[MS_EPL];
#pragma unroll
      for (int i = 0; i < MS_EPL; ++i) rw[i] = (lane + 32 * i < cnt) ? sr[lane + 32 * i] : -1;
      double wv[MS_EPL];
#pragma unroll
      for (int i = 0; i < MS_EPL; ++i) wv[i] = rw[i] >= 0 ? __ldg(wp + rw[i]) : 0.0;
#pragma unroll
      for (int i = 0; i < MS_EPL; ++i)
        if (rw[i] >= 0) sw[lane + 32 * i] = wv[i];
      __syncwarp();
      const int st[5] = {q.x - s0, q.y - s0, q.z - s0, q.w - s0, hi - s0};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int a = st[k], b = st[k + 1];
        if (a < b) s[k] = fma(to_f64(sv[a]), sw[a], s[k]);
        if (a + 1 < b) s[k] = fma(to_f64(sv[a + 1]), sw[a + 1], s[k]);
        for (int idx = a + 2; idx < b; ++idx) s[k] = fma(to_f64(sv[idx]), sw[idx], s[k]);
      }
      __syncwarp();  // sw and this entry buffer are rewritten by later blocks
    } else if (cnt > 0) {
      for (int idx = q.x; idx < hi; ++idx) {
        const int k = (idx >= q.y) + (idx >= q.z) + (idx >= q.w);
        const double pv = to_f64(__ldcs(cscval + m0.base + idx));
        const double wx = wp[__ldcs(cscrow + m0.base + idx)];
        if (k == 0) s[0] = fma(pv, wx, s[0]);
        else if (k == 1) s[1] = fma(pv, wx, s[1]);
        else if (k == 2) s[2] = fma(pv, wx, s[2]);
        else s[3] = fma(pv, wx, s[3]);
      }
    }
    m0 = m1;
    m1 = m2;
    m2 = m3;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
template <typename T>
__global__ void __launch_bounds__(256) k_mtw_finish_stage(FinishParams F, Window W,
                                                          const int* __restrict__ colptr,
                                                          const int* __restrict__ cscrow,
                                                          const T* __restrict__ cscval,
                                                          const int64_t* __restrict__ blkbase,
                                                          const double* __restrict__ w) {
  if (F.ctl->diverged_at != 0) return;
  const int c0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const bool valid = c0 < F.n;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  mtw_csc_stage<T>(valid ? c0 : F.n, valid, W, colptr, F.n, cscrow, cscval, blkbase, w, s);
  finish_body4(F, c0, s);
}
template <typename T>
__global__ void __launch_bounds__(256) k_mtw_stage(double* __restrict__ s_out, Window W,
                                                   const int* __restrict__ colptr, int n,
                                                   const int* __restrict__ cscrow,
                                                   const T* __restrict__ cscval,
                                                   const int64_t* __restrict__ blkbase,
                                                   const double* __restrict__ w, const Ctl* ctl) {
  if (ctl->diverged_at != 0) return;
  const int c0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const bool valid = c0 < n;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  mtw_csc_stage<T>(valid ? c0 : n, valid, W, colptr, n, cscrow, cscval, blkbase, w, s);
  if (valid) {
    double2* o = reinterpret_cast<double2*>(s_out + c0);
    o[0] = make_double2(s[0], s[1]);
    o[1] = make_double2(s[2], s[3]);
  }
}

// ---------------------------------------------------------------------------
// Iterative refinement of w against the fp64 Gram ring (contexts whose
// factorization keeps six digits, chol_q6.cu): res = y - G w with
// G = I + alpha (ring) in slot order and y = r on the new block's rows.
// The ring holds the product of two window blocks in the panel of the newer
// one, at the older one's window position (see k_assemble), so for the rows
// of block X the columns of an older-or-equal block Y are read down the
// columns of X's own panel (threads along the rows of X: coalesced) and the
// columns of a newer block Y along the rows of Y's panel (a warp per row).
// One CTA per (64 rows of X, Y); the partial sums over Y are added in a fixed
// order by k_gram_apply_finish.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_gram_apply(GramApplyParams G) {
  if (G.ctl->diverged_at != 0) return;
  __shared__ double red[4][64];
  const int X = blockIdx.y, Y = blockIdx.z, a0 = blockIdx.x * 64;
  const int ell = G.ell, tid = threadIdx.x;
  const double* wy = G.w + (int64_t)Y * ell;
  double* out = G.part + (int64_t)Y * G.ldp + (int64_t)X * ell;
  if (G.age[Y] >= G.age[X]) {
    // G(X a, Y c) = pan_X[(Y ell + c) ell + a]: threads along a, four groups of rows c
    const double* pan = G.panels + (int64_t)G.slot[X] * G.panel_stride + (int64_t)Y * ell * ell;
    const int ag = tid & 63, cg = tid >> 6, a = a0 + ag;
    double s0 = 0.0, s1 = 0.0;
    if (a < ell) {
      int cidx = cg;
      for (; cidx + 4 < ell; cidx += 8) {
        s0 = fma(__ldcs(pan + (int64_t)cidx * ell + a), wy[cidx], s0);
        s1 = fma(__ldcs(pan + (int64_t)(cidx + 4) * ell + a), wy[cidx + 4], s1);
      }
      if (cidx < ell) s0 = fma(__ldcs(pan + (int64_t)cidx * ell + a), wy[cidx], s0);
    }
    red[cg][ag] = s0 + s1;
    __syncthreads();
    if (tid < 64 && a0 + tid < ell)
      out[a0 + tid] = (red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]);
  } else {
    // G(X a, Y c) = pan_Y[(X ell + a) ell + c]: a warp per row a, lanes along c
    const double* pan = G.panels + (int64_t)G.slot[Y] * G.panel_stride + (int64_t)X * ell * ell;
    const int warp = tid >> 5, lane = tid & 31;
    for (int q = warp; q < 64; q += 8) {
      const int a = a0 + q;
      if (a >= ell) break;
      const double* row = pan + (int64_t)a * ell;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int cidx = lane;
      for (; cidx + 96 < ell; cidx += 128) {
        s0 = fma(__ldcs(row + cidx), wy[cidx], s0);
        s1 = fma(__ldcs(row + cidx + 32), wy[cidx + 32], s1);
        s2 = fma(__ldcs(row + cidx + 64), wy[cidx + 64], s2);
        s3 = fma(__ldcs(row + cidx + 96), wy[cidx + 96], s3);
      }
      for (; cidx < ell; cidx += 32) s0 = fma(__ldcs(row + cidx), wy[cidx], s0);
      const double sv = warp_sum((s0 + s1) + (s2 + s3));
      if (lane == 0) out[a] = sv;
    }
  }
}

// res[p] = y[p] - (w[p] + alpha sum_Y part[Y][p]) for p < N, 0 on the padding rows
__global__ void __launch_bounds__(256) k_gram_apply_finish(GramApplyParams G) {
  if (G.ctl->diverged_at != 0) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= G.npad) return;
  const int N = G.nw * G.ell;
  double v = 0.0;
  if (p < N) {
    double sum = 0.0;
    for (int Y = 0; Y < G.nw; ++Y) sum += G.part[(int64_t)Y * G.ldp + p];
    const int q = p - G.newp * G.ell;
    const double y = (q >= 0 && q < G.ell) ? G.r[q] : 0.0;
    v = y - fma(G.alpha, sum, G.w[p]);
  }
  G.res[p] = v;
}

__global__ void __launch_bounds__(256) k_add_inplace(double* __restrict__ w, const double* __restrict__ dw,
                                                     int count, const Ctl* ctl) {
  if (ctl->diverged_at != 0) return;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < count) w[p] += dw[p];
}

void launch_gram_apply(const GramApplyParams& G, cudaStream_t s) {
  dim3 grid((unsigned)((G.ell + 63) / 64), G.nw, G.nw);
  k_gram_apply<<<grid, 256, 0, s>>>(G);
  k_gram_apply_finish<<<(unsigned)((G.npad + 255) / 256), 256, 0, s>>>(G);
}
void launch_add_inplace(double* w, const double* dw, int count, const Ctl* ctl, cudaStream_t s) {
  k_add_inplace<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(w, dw, count, ctl);
}

__global__ void k_stamp_start(Ctl* ctl) { ctl->t_start_ns = globaltimer_ns(); }

// sharded mode: divergence decision and history row from allreduced norms
__global__ void k_record(RecordParams R) {
  Ctl* ctl = R.ctl;
  if (ctl->diverged_at != 0) return;
  const int lane = threadIdx.x;
  double v = 0.0;
  for (int j = lane; j < R.ell; j += 32) {
    const double rv = R.r[j];
    v += rv * rv;
  }
  v = warp_sum(v);
  if (lane != 0) return;
  ctl->rnorm2 = v;
  const double nsq = R.norms[0];
  const bool diverged = !(nsq <= ctl->div_limit_sq);
  if (diverged) ctl->diverged_at = R.k;
  if (R.record || diverged) {
    const int64_t row = ctl->nrows++;
    double* h = R.hist + row * (SLIM_HIST_FIXED_DEV + R.nref);
    h[0] = (double)R.k;
    h[1] = R.alpha;
    h[2] = sqrt(v);
    h[3] = (double)(globaltimer_ns() - ctl->t_start_ns);
    h[4] = diverged ? 1.0 : 0.0;
    for (int q = 0; q < R.nref; ++q) h[SLIM_HIST_FIXED_DEV + q] = sqrt(R.norms[1 + q]);
  }
}

struct GroupIn {
  const double* p[8];
};

__global__ void k_group_sum(double* __restrict__ out, GroupIn in, int nin, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < nin; ++q) v += in.p[q][i];
    out[i] = v;
  }
}

// ---------------------------------------------------------------------------
// per-block CSC (built once per operator): column pointers relative to the
// block's first nonzero, rows 0-based within the block, rows sorted.
// ---------------------------------------------------------------------------

__global__ void k_csc_count(int* __restrict__ colptr, const int64_t* __restrict__ rowptr,
                            const int* __restrict__ col, int64_t row0, int64_t m, int ell, int n) {
  const int64_t row = row0 + (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const int64_t b = row / ell;
  int* cp = colptr + b * csc_stride(n);
  for (int64_t e = rowptr[row] + lane; e < rowptr[row + 1]; e += 32) atomicAdd(cp + col[e] + 1, 1);
}

__global__ void __launch_bounds__(256) k_csc_scan(int* __restrict__ colptr, int n) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  int* cp = colptr + (int64_t)blockIdx.x * csc_stride(n);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 1; base <= n; base += 256) {
    const int idx = base + threadIdx.x;
    int v = (idx <= n) ? cp[idx] : 0;
    int incl, agg;
    Scan(tmp).InclusiveSum(v, incl, agg);
    const int c0 = carry;
    if (idx <= n) cp[idx] = incl + c0;
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + agg;
    __syncthreads();
  }
}

template <typename T>
__global__ void k_csc_fill(int* __restrict__ colptr, const int64_t* __restrict__ rowptr,
                           const int* __restrict__ col, const T* __restrict__ val,
                           int* __restrict__ cscrow, T* __restrict__ cscval, int64_t row0,
                           int64_t m, int ell, int n) {
  const int64_t row = row0 + (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const int64_t b = row / ell;
  const int64_t base = rowptr[b * ell];
  int* cp = colptr + b * csc_stride(n);
  const int rloc = (int)(row - b * ell);
  for (int64_t e = rowptr[row] + lane; e < rowptr[row + 1]; e += 32) {
    const int pos = atomicAdd(cp + col[e], 1);
    cscrow[base + pos] = rloc;
    cscval[base + pos] = val[e];
  }
}

// after the fill, cp[c] holds the end of column c; shift right by one
__global__ void __launch_bounds__(256) k_csc_shift(int* __restrict__ colptr, int n) {
  int* cp = colptr + (int64_t)blockIdx.x * csc_stride(n);
  for (int hi = n + 1; hi > 0; hi -= 256) {
    const int c = hi - 256 + (int)threadIdx.x;  // writes positions [hi-256, hi)
    int v = 0;
    if (c >= 1) v = cp[c - 1];
    __syncthreads();
    if (c >= 1) cp[c] = v;
    else if (c == 0) cp[0] = 0;
    __syncthreads();
  }
}

template <typename T>
__global__ void k_csc_sort(const int* __restrict__ colptr, int* __restrict__ cscrow,
                           T* __restrict__ cscval, const int64_t* __restrict__ blkbase,
                           int64_t nblocks, int n) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nblocks * n) return;
  const int64_t b = gid / n;
  const int c = (int)(gid - b * n);
  const int* cp = colptr + b * csc_stride(n);
  const int64_t base = blkbase[b];
  const int lo = cp[c], hi = cp[c + 1];
  for (int e = lo + 1; e < hi; ++e) {
    const int rk = cscrow[base + e];
    const T vk = cscval[base + e];
    int q = e - 1;
    while (q >= lo && cscrow[base + q] > rk) {
      cscrow[base + q + 1] = cscrow[base + q];
      cscval[base + q + 1] = cscval[base + q];
      --q;
    }
    cscrow[base + q + 1] = rk;
    cscval[base + q + 1] = vk;
  }
}

// The same build for an arbitrary list of blocks (a streamed batch's
// first-use blocks): one launch per phase for the whole list.
template <typename T>
__global__ void k_csc_count_list(int* __restrict__ colptr, const int64_t* __restrict__ rowptr,
                                 const int* __restrict__ col, BlkList L, int ell, int n) {
  const int64_t lr = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (lr >= (int64_t)L.n * ell) return;
  const int64_t b = L.id[lr / ell];
  const int64_t row = b * ell + lr % ell;
  int* cp = colptr + b * csc_stride(n);
  for (int64_t e = rowptr[row] + lane; e < rowptr[row + 1]; e += 32) atomicAdd(cp + col[e] + 1, 1);
}
template <typename T>
__global__ void k_csc_fill_list(int* __restrict__ colptr, const int64_t* __restrict__ rowptr,
                                const int* __restrict__ col, const T* __restrict__ val,
                                int* __restrict__ cscrow, T* __restrict__ cscval, BlkList L, int ell,
                                int n) {
  const int64_t lr = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (lr >= (int64_t)L.n * ell) return;
  const int64_t b = L.id[lr / ell];
  const int rloc = (int)(lr % ell);
  const int64_t row = b * ell + rloc;
  const int64_t base = rowptr[b * ell];
  int* cp = colptr + b * csc_stride(n);
  for (int64_t e = rowptr[row] + lane; e < rowptr[row + 1]; e += 32) {
    const int pos = atomicAdd(cp + col[e], 1);
    cscrow[base + pos] = rloc;
    cscval[base + pos] = val[e];
  }
}
__global__ void __launch_bounds__(256) k_csc_scan_list(int* __restrict__ colptr, BlkList L, int n) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  int* cp = colptr + L.id[blockIdx.x] * csc_stride(n);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 1; base <= n; base += 256) {
    const int idx = base + threadIdx.x;
    int v = (idx <= n) ? cp[idx] : 0;
    int incl, agg;
    Scan(tmp).InclusiveSum(v, incl, agg);
    const int c0 = carry;
    if (idx <= n) cp[idx] = incl + c0;
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + agg;
    __syncthreads();
  }
}
__global__ void __launch_bounds__(256) k_csc_shift_list(int* __restrict__ colptr, BlkList L, int n) {
  int* cp = colptr + L.id[blockIdx.x] * csc_stride(n);
  for (int hi = n + 1; hi > 0; hi -= 256) {
    const int c = hi - 256 + (int)threadIdx.x;
    int v = 0;
    if (c >= 1) v = cp[c - 1];
    __syncthreads();
    if (c >= 1) cp[c] = v;
    else if (c == 0) cp[0] = 0;
    __syncthreads();
  }
}
template <typename T>
__global__ void k_csc_sort_list(const int* __restrict__ colptr, int* __restrict__ cscrow,
                                T* __restrict__ cscval, const int64_t* __restrict__ blkbase, BlkList L,
                                int n) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)L.n * n) return;
  const int64_t b = L.id[gid / n];
  const int c = (int)(gid % n);
  const int* cp = colptr + b * csc_stride(n);
  const int64_t base = blkbase[b];
  const int lo = cp[c], hi = cp[c + 1];
  for (int e = lo + 1; e < hi; ++e) {
    const int rk = cscrow[base + e];
    const T vk = cscval[base + e];
    int q = e - 1;
    while (q >= lo && cscrow[base + q] > rk) {
      cscrow[base + q + 1] = cscrow[base + q];
      cscval[base + q + 1] = cscval[base + q];
      --q;
    }
    cscrow[base + q + 1] = rk;
    cscval[base + q + 1] = vk;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

static inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

template <typename T>
void launch_residual_dense(double* r, const T* A, int64_t lda, int64_t row0, int64_t brow0,
                           int ell, int n, const double* x, const double* b, const Ctl* ctl,
                           RowSplit rs, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  rs.vec = (n % V == 0 && lda % V == 0) ? 1 : 0;
  if (rowdot_rows(ell, n) == 8)
    k_rowdot<T, false, 8><<<dim3(rs.nch, cdiv(ell, 8)), 256, 0, s>>>(A, lda, row0, n, ell, x, rs, r, 0,
                                                                     b, brow0, ctl);
  else
    k_rowdot<T, false, 1><<<dim3(rs.nch, ell), 256, 0, s>>>(A, lda, row0, n, ell, x, rs, r, 0, b,
                                                            brow0, ctl);
}
void launch_gen_block(float* dst, float* hi, float* lo, uint64_t seed, int64_t row0, int ell,
                      int n_local, int64_t n_total, int64_t col0, cudaStream_t s) {
  const int64_t total = (int64_t)ell * n_local;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), 148 * 16);
  k_gen_block<<<grid, 256, 0, s>>>(dst, hi, lo, seed, row0, ell, n_local, n_total, col0);
}
void launch_gen_apply(double* out, uint64_t seed, int64_t m, int n_local, int64_t n_total,
                      int64_t col0, const double* x, cudaStream_t s) {
  k_gen_apply<<<cdiv(m, 8), 256, 0, s>>>(out, seed, m, n_local, n_total, col0, x);
}
template <typename T>
void launch_residual_csr(double* r, const int64_t* rowptr, const int* col, const T* val,
                         int64_t row0, int64_t brow0, int ell, const double* x, const double* b,
                         const Ctl* ctl, cudaStream_t s) {
  k_residual_csr<T><<<ell, RES_THREADS, 0, s>>>(r, rowptr, col, val, row0, brow0, ell, x, b, ctl);
}
// CSR Gram kernel per operator: the fixed-point record kernel pays off once a
// block has enough nonzeros to amortise its two small preparation kernels
// (cold-L2 probe: configs[2], 1.3 M nonzeros per block: 195 vs 543 us;
// configs[3], 450 k: 126 vs 129 us; configs[1], 131 k: 56 vs 34 us);
// SLIM_GRAM_LUT=1/0 overrides
bool gram_csr_variant(double nnz_per_block) {
  if (const char* e = getenv("SLIM_GRAM_LUT")) return e[0] != '0';
  return nnz_per_block >= (double)(1 << 18);
}
// scratch of the fixed-point CSR Gram: n column records + ell row exponents
size_t gram_lut_bytes(int n, int ell) {
  return (size_t)n * sizeof(GramRec<double>) + (size_t)ell * sizeof(int);
}
template <typename T>
void launch_gram_csr(double* panel, const Window& W, const int64_t* rowptr, const int* col,
                     const T* val, const int* colptr_new, const int* cscrow, const T* cscval,
                     int64_t base_new, cudaStream_t s, void* lut, int n) {
  const unsigned grid = (unsigned)((int64_t)W.nw * W.ell);
  const size_t fx_smem = (size_t)W.ell * 2 * sizeof(unsigned);
  if (lut && W.ell <= 65536 && fx_smem <= 200 * 1024) {  // rows of the new block packed in 16 bits
    if (fx_smem > 48 * 1024) {
      static bool configured = false;
      if (!configured) {
        cudaFuncSetAttribute(k_gram_csr_fx<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = true;
      }
    }
    GramRec<T>* L = reinterpret_cast<GramRec<T>*>(lut);
    int* rowexp = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(lut) +
                                         (size_t)n * sizeof(GramRec<double>));
    const int64_t newrow0 = (int64_t)W.blk[W.newp] * W.ell;
    k_gram_rowexp<T><<<cdiv(W.ell, 8), 256, 0, s>>>(rowexp, rowptr, val, newrow0, W.ell);
    k_gram_lut<T><<<cdiv(n, 256), 256, 0, s>>>(L, rowexp, colptr_new, cscrow, cscval, base_new, n);
    const unsigned pgrid = std::min<unsigned>(grid, 148u * 4u);  // persistent: 4 CTAs per SM
    k_gram_csr_fx<T><<<pgrid, GFX_THREADS, fx_smem, s>>>(panel, W, rowptr, col, val, L, rowexp,
                                                         colptr_new, cscrow, cscval, base_new);
    return;
  }
  const size_t smem = (size_t)4 * W.ell * sizeof(double);
  if (smem > 48 * 1024) {
    static bool configured = false;  // one ell per process in practice; idempotent anyway
    if (!configured) {
      cudaFuncSetAttribute(k_gram_csr<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured = true;
    }
  }
  k_gram_csr<T><<<grid, 128, smem, s>>>(panel, W, rowptr, col, val, colptr_new, cscrow, cscval,
                                        base_new);
}
template <typename T>
void launch_gram_dense(double* panel, double* part, int nsplit, const Window& W, const T* A,
                       int64_t lda, int64_t newrow0, int n, cudaStream_t s) {
  const int N = W.nw * W.ell;
  int klen = (n + nsplit - 1) / nsplit;
  klen = ((klen + GK - 1) / GK) * GK;
  const int zs = (n + klen - 1) / klen;
  dim3 grid(cdiv(N, 64), cdiv(W.ell, 64), zs);
  k_gram_dense<T><<<grid, 256, 0, s>>>(part, W, A, lda, newrow0, n, klen);
  k_gram_reduce<<<cdiv((int64_t)N * W.ell, 256), 256, 0, s>>>(panel, W, part, zs);
}
// exact fp64 diagonal of A_k A_k^T (row sums of squares) into the panel: the
// tensor core accumulates in truncating fp32, which biases these large
// all-positive sums; every other entry has mixed signs and small partials
void launch_gram_diag_fp64(double* panel_diag, int64_t ld, const float* A, int ell, int n,
                           RowSplit rs, cudaStream_t s) {
  rs.vec = (n % 4 == 0) ? 1 : 0;
  if (rowdot_rows(ell, n) == 8)
    k_rowdot<float, true, 8><<<dim3(rs.nch, cdiv(ell, 8)), 256, 0, s>>>(
        A, n, 0, n, ell, nullptr, rs, panel_diag, ld, nullptr, 0, nullptr);
  else
    k_rowdot<float, true, 1><<<dim3(rs.nch, ell), 256, 0, s>>>(A, n, 0, n, ell, nullptr, rs, panel_diag,
                                                               ld, nullptr, 0, nullptr);
}

void launch_gram_reduce(double* panel, const Window& W, const double* part, int nsplit,
                        cudaStream_t s) {
  const int64_t cnt = (int64_t)W.nw * W.ell * W.ell;
  k_gram_reduce<<<cdiv(cnt, 256), 256, 0, s>>>(panel, W, part, nsplit);
}

template <typename T>
void launch_mtw_dense(double* part, int nsplit, const Window& W, const T* A, int64_t lda, int n,
                      const double* w, const Ctl* ctl, cudaStream_t s) {
  const int N = W.nw * W.ell;
  const int rps = (N + nsplit - 1) / nsplit;
  constexpr int V = 16 / sizeof(T);
  if (n % V == 0 && lda % V == 0) {
    dim3 grid(cdiv(n, 256 * V), nsplit);
    k_mtw_dense<T, V><<<grid, 256, 0, s>>>(part, W, A, lda, n, w, rps, ctl);
  } else {
    dim3 grid(cdiv(n, 256), nsplit);
    k_mtw_dense<T, 1><<<grid, 256, 0, s>>>(part, W, A, lda, n, w, rps, ctl);
  }
}
// variants 1..5 = four columns per thread with (G blocks, E entries)
// prefetched: (3,4) (2,6) (1,8) (3,2) (2,4); 6 = warp-staged entries with
// cp.async prefetch (k_mtw_stage).  Cold-L2 probe, round 2: configs[2] (1.25
// entries per column and block, n = 2^20) column kernel 67 us, (1,8) 53 us,
// staged 47 us; configs[3] (0.15 entries per column and block, n = 2^21)
// column kernel 45 us, staged 41 us; configs[1] (n = 2^16: n / 4 threads do
// not fill the GPU) column kernel 20 us = staged
int mtw_variant(int64_t n, double nnz_per_block) {
  if (const char* e = getenv("SLIM_MTW_QUAD")) return n % 4 == 0 ? atoi(e) : 0;
  (void)nnz_per_block;
  return (n % 4 == 0 && n >= (1 << 19)) ? 6 : 0;
}
static int mtw_quad(int n, int quad) { return n % 4 == 0 ? quad : 0; }
template <typename T>
static void mtw_stage_configure() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_mtw_stage<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)mtw_stage_smem<T>());
  cudaFuncSetAttribute(k_mtw_finish_stage<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)mtw_stage_smem<T>());
  done = true;
}
#define MTW4_DISPATCH(KERNEL, GRID, ...)                                   \
  switch (mtw_quad(n_, quad)) {                                                  \
    case 1: KERNEL<T, 3, 4><<<GRID, 256, 0, s>>>(__VA_ARGS__); break;      \
    case 2: KERNEL<T, 2, 6><<<GRID, 256, 0, s>>>(__VA_ARGS__); break;      \
    case 3: KERNEL<T, 1, 8><<<GRID, 256, 0, s>>>(__VA_ARGS__); break;      \
    case 4: KERNEL<T, 3, 2><<<GRID, 256, 0, s>>>(__VA_ARGS__); break;      \
    default: KERNEL<T, 2, 4><<<GRID, 256, 0, s>>>(__VA_ARGS__); break;     \
  }
template <typename T>
void launch_mtw_csc(double* s_out, const Window& W, const int* colptr, int n, const int* cscrow,
                    const T* cscval, const int64_t* blkbase, const double* w, const Ctl* ctl,
                    cudaStream_t s, int quad) {
  if (mtw_quad(n, quad) == 6) {
    mtw_stage_configure<T>();
    k_mtw_stage<T><<<cdiv(n / 4, 256), 256, mtw_stage_smem<T>(), s>>>(s_out, W, colptr, n, cscrow,
                                                                      cscval, blkbase, w, ctl);
    return;
  }
  if (mtw_quad(n, quad)) {
    const int n_ = n;
    MTW4_DISPATCH(k_mtw_csc4, cdiv(n / 4, 256), s_out, W, colptr, n, cscrow, cscval, blkbase, w, ctl);
    return;
  }
  static const int grp = getenv("SLIM_MTW_GROUP") ? atoi(getenv("SLIM_MTW_GROUP")) : 3;
  if (grp <= 1)
    k_mtw_csc<T, 1><<<cdiv(n, 256), 256, 0, s>>>(s_out, W, colptr, n, cscrow, cscval, blkbase, w, ctl);
  else if (grp == 2)
    k_mtw_csc<T, 2><<<cdiv(n, 256), 256, 0, s>>>(s_out, W, colptr, n, cscrow, cscval, blkbase, w, ctl);
  else if (grp <= 4)
    k_mtw_csc<T, 3><<<cdiv(n, 256), 256, 0, s>>>(s_out, W, colptr, n, cscrow, cscval, blkbase, w, ctl);
  else
    k_mtw_csc<T, 6><<<cdiv(n, 256), 256, 0, s>>>(s_out, W, colptr, n, cscrow, cscval, blkbase, w, ctl);
}
void launch_finish(const FinishParams& F, cudaStream_t s) {
  k_finish<<<cdiv(F.n, 256), 256, 0, s>>>(F);
}
template <typename T>
void launch_mtw_finish_csc(const FinishParams& F, const Window& W, const int* colptr,
                           const int* cscrow, const T* cscval, const int64_t* blkbase,
                           const double* w, cudaStream_t s, int quad) {
  const int n_ = F.n;
  if (mtw_quad(n_, quad) == 6) {
    mtw_stage_configure<T>();
    k_mtw_finish_stage<T><<<cdiv(F.n / 4, 256), 256, mtw_stage_smem<T>(), s>>>(F, W, colptr, cscrow,
                                                                              cscval, blkbase, w);
  } else if (mtw_quad(n_, quad)) {
    MTW4_DISPATCH(k_mtw_finish_csc4, cdiv(F.n / 4, 256), F, W, colptr, cscrow, cscval, blkbase, w);
  } else
    k_mtw_finish_csc<T><<<cdiv(F.n, 256), 256, 0, s>>>(F, W, colptr, cscrow, cscval, blkbase, w);
}
template void launch_mtw_finish_csc<double>(const FinishParams&, const Window&, const int*,
                                            const int*, const double*, const int64_t*,
                                            const double*, cudaStream_t, int);
template void launch_mtw_finish_csc<float>(const FinishParams&, const Window&, const int*,
                                           const int*, const float*, const int64_t*,
                                           const double*, cudaStream_t, int);
int finish_grid(int n) { return (int)cdiv(n, 256); }
// L2 flush by reading (the lines it leaves are clean, so the next kernel's
// DRAM bandwidth is not shared with write-backs)
__global__ void __launch_bounds__(256) k_flush_read(const uint4* __restrict__ p, int64_t count,
                                                    unsigned* sink) {
  unsigned acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u) *sink = acc;  // keeps the loads
}
void launch_flush_read(const void* buf, size_t bytes, unsigned* sink, cudaStream_t s) {
  k_flush_read<<<148 * 8, 256, 0, s>>>((const uint4*)buf, (int64_t)(bytes / 16), sink);
}
void launch_stamp_start(Ctl* ctl, cudaStream_t s) { k_stamp_start<<<1, 1, 0, s>>>(ctl); }
void launch_record(const RecordParams& R, cudaStream_t s) { k_record<<<1, 32, 0, s>>>(R); }
void launch_group_sum(double* out, const double* const* in, int nin, int64_t count,
                      cudaStream_t s) {
  GroupIn g{};
  for (int q = 0; q < nin && q < 8; ++q) g.p[q] = in[q];
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(count, 256), 148 * 8);
  k_group_sum<<<grid, 256, 0, s>>>(out, g, nin, count);
}

template <typename T>
void launch_build_csc(int* colptr, int* cscrow, T* cscval, const int64_t* rowptr, const int* col,
                      const T* val, const int64_t* blkbase, int64_t m, int ell, int n,
                      int64_t nblocks, cudaStream_t s, int64_t blk0, int64_t nblk) {
  if (nblk < 0) nblk = nblocks - blk0;
  if (nblk <= 0) return;
  int* cp = colptr + blk0 * csc_stride(n);
  const int64_t row0 = blk0 * ell, row1 = (blk0 + nblk) * (int64_t)ell;
  cudaMemsetAsync(cp, 0, sizeof(int) * (size_t)nblk * csc_stride(n), s);
  k_csc_count<<<cdiv(row1 - row0, 8), 256, 0, s>>>(colptr, rowptr, col, row0, row1, ell, n);
  k_csc_scan<<<(unsigned)nblk, 256, 0, s>>>(cp, n);
  k_csc_fill<T><<<cdiv(row1 - row0, 8), 256, 0, s>>>(colptr, rowptr, col, val, cscrow, cscval, row0,
                                                      row1, ell, n);
  k_csc_shift<<<(unsigned)nblk, 256, 0, s>>>(cp, n);
  k_csc_sort<T><<<cdiv(nblk * n, 256), 256, 0, s>>>(cp, cscrow, cscval, blkbase + blk0, nblk, n);
}

template <typename T>
void launch_build_csc_list(int* colptr, int* cscrow, T* cscval, const int64_t* rowptr, const int* col,
                           const T* val, const int64_t* blkbase, int ell, int n, const BlkList& L,
                           cudaStream_t s) {
  if (L.n <= 0) return;
  for (int q = 0; q < L.n; ++q)
    cudaMemsetAsync(colptr + (int64_t)L.id[q] * csc_stride(n), 0, sizeof(int) * (size_t)(n + 1), s);
  const int64_t rows = (int64_t)L.n * ell;
  k_csc_count_list<T><<<cdiv(rows, 8), 256, 0, s>>>(colptr, rowptr, col, L, ell, n);
  k_csc_scan_list<<<(unsigned)L.n, 256, 0, s>>>(colptr, L, n);
  k_csc_fill_list<T><<<cdiv(rows, 8), 256, 0, s>>>(colptr, rowptr, col, val, cscrow, cscval, L, ell, n);
  k_csc_shift_list<<<(unsigned)L.n, 256, 0, s>>>(colptr, L, n);
  k_csc_sort_list<T><<<cdiv((int64_t)L.n * n, 256), 256, 0, s>>>(colptr, cscrow, cscval, blkbase, L, n);
}

#define SLIM_INST(T)                                                                              \
  template void launch_residual_dense<T>(double*, const T*, int64_t, int64_t, int64_t, int, int, \
                                         const double*, const double*, const Ctl*, RowSplit,      \
                                         cudaStream_t);                                           \
  template void launch_residual_csr<T>(double*, const int64_t*, const int*, const T*, int64_t,    \
                                       int64_t, int, const double*, const double*, const Ctl*,   \
                                       cudaStream_t);                                            \
  template void launch_gram_csr<T>(double*, const Window&, const int64_t*, const int*, const T*,  \
                                   const int*, const int*, const T*, int64_t, cudaStream_t,       \
                                   void*, int);                                                  \
  template void launch_gram_dense<T>(double*, double*, int, const Window&, const T*, int64_t,     \
                                     int64_t, int, cudaStream_t);                                \
  template void launch_mtw_dense<T>(double*, int, const Window&, const T*, int64_t, int,          \
                                    const double*, const Ctl*, cudaStream_t);                    \
  template void launch_mtw_csc<T>(double*, const Window&, const int*, int, const int*, const T*,  \
                                  const int64_t*, const double*, const Ctl*, cudaStream_t, int); \
  template void launch_build_csc<T>(int*, int*, T*, const int64_t*, const int*, const T*,         \
                                    const int64_t*, int64_t, int, int, int64_t, cudaStream_t,     \
                                    int64_t, int64_t);                                            \
  template void launch_build_csc_list<T>(int*, int*, T*, const int64_t*, const int*, const T*,    \
                                         const int64_t*, int, int, const BlkList&, cudaStream_t);

SLIM_INST(double)
SLIM_INST(float)

}  // namespace slim
