// trsv.cu -- the triangular solves of the slimLS x-chain,
//     t = L^{-1} y,   w = L^{-T} t       (w = G^{-1} y, innersolve.py:320)
// with y = r on the new block's rows and zero elsewhere, plus the inverses
// of the 64x64 diagonal tiles of L they use.
//
// Design (B200): the solve is a dependent chain over tile rows, so its cost
// is the latency of one hop (segment t_k known -> segment t_{k+1} known)
// times the number of tile rows.  One thread-block cluster (C <= 16 CTAs)
// runs the whole solve; tile row i belongs to CTA i mod C.  A segment is
// published by writing it into the owner's shared memory and setting a
// flag in every CTA of the cluster (st.release.cluster over DSMEM, ~0.1 us,
// instead of a global flag round trip through L2).  When segment k lands,
// the owner of row k + 1 runs the critical step first -- one 64x64 product
// with the tile it staged in advance, one 64x64 product with the
// precomputed inverse of L_{k+1,k+1} -- and publishes; only then does every
// CTA stream the segment's contributions into its other rows.  The solve
// occupies C SMs for its duration, so it does not starve the factorization
// batch running beside it.
#include "common.cuh"
#include "kernels.h"

namespace slim {

// ---- cluster / DSMEM helpers ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t map_to_cta(uint32_t a, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
__device__ __forceinline__ double ld_remote_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_remote_release(uint32_t a, int v) {
  asm volatile("st.release.cluster.shared::cluster.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_local_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void stage_tile(double* s, const double* g, int tid) {
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int c = tid + it * 256;  // 2048 16-byte chunks
    const int row = c >> 5, cc = (c & 31) * 2;
    cp_async16(s + row * TS + cc, g + row * TB + cc);
  }
}

// v[a] -= sum_b M[a][b] x[b]   (M in shared memory, row stride TS)
__device__ __forceinline__ void gemv_sub_smem(double* v, const double* M, const double* x, int tid) {
  const int a = tid >> 2, q = tid & 3;
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < 16; ++m) s = fma(M[a * TS + q + 4 * m], x[q + 4 * m], s);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (q == 0) v[a] -= s;
}
// out[a] = sum_b M[a][b] x[b]
__device__ __forceinline__ void gemv_smem(double* out, const double* M, const double* x, int tid) {
  const int a = tid >> 2, q = tid & 3;
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < 16; ++m) s = fma(M[a * TS + q + 4 * m], x[q + 4 * m], s);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  if (q == 0) out[a] = s;
}
// out[a] (=|-=) sum_b M[b][a] x[b]; part: 4 x 64 scratch; ends with a barrier
template <bool SUB>
__device__ __forceinline__ void gemvT_smem(double* out, const double* M, const double* x, double* part,
                                           int tid) {
  const int a = tid & 63, g = tid >> 6;
  double s = 0.0;
#pragma unroll
  for (int b = 0; b < 16; ++b) s = fma(M[(16 * g + b) * TS + a], x[16 * g + b], s);
  part[g * TB + a] = s;
  __syncthreads();
  if (tid < TB) {
    const double t = (part[tid] + part[TB + tid]) + (part[2 * TB + tid] + part[3 * TB + tid]);
    out[tid] = SUB ? out[tid] - t : t;
  }
  __syncthreads();
}
// ---- bulk-copy ring of the non-critical tiles ----
constexpr int RS_MAX = 4;  // 32 KB slots (P.rs in use)
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
// one 32 KB tile (contiguous, tile-major) global -> shared, completing on b
__device__ __forceinline__ void bulk_tile(double* dst, const double* src, uint64_t* b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
               "r"(TB * TB * 8)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(TB * TB * 8), "r"(smem_addr(b))
      : "memory");
}

// The non-critical tiles a CTA consumes, in consumption order:
// forward  k = i0 .. last - 1, own rows ip >= k + 2 ascending: tile (ip, k);
// backward k = T - 1 .. me + 1, own rows ip <= k - 2 ascending: tile (k, ip).
struct TileSeq {
  int dir, k, ip;
};
struct SeqCtx {
  int me, C, T, i0, last;
  bool has_fwd;
  __device__ int first_own_ge(int v) const { return v <= me ? me : me + ((v - me + C - 1) / C) * C; }
  // move s to the next valid position (itself if valid); false when exhausted
  __device__ bool norm(TileSeq& s) const {
    while (true) {
      if (s.dir == 0) {
        if (!has_fwd || s.k >= last) {
          s.dir = 1;
          s.k = T - 1;
          s.ip = me;
          continue;
        }
        if (s.ip <= last) return true;
        ++s.k;
        s.ip = first_own_ge(s.k + 2);
      } else {
        if (s.k <= me) return false;
        if (s.ip <= s.k - 2) return true;
        --s.k;
        s.ip = me;
      }
    }
  }
  __device__ const double* tile(const double* L, const TileSeq& s) const {
    return L + (s.dir == 0 ? tile_off(s.ip, s.k) : tile_off(s.k, s.ip));
  }
  __device__ void advance(TileSeq& s) const { s.ip += C; }
};

// v[8w + r] -= sum_b M[8w + r][b] x[b] for the 64x64 row-major (unpadded)
// tile M: warp w reads one 512-byte row per instruction (conflict-free) and
// a butterfly reduces its 8 row partials across the lanes in 9 shuffles
__device__ __forceinline__ void gemv_sub_ring(double* v, const double* M, const double* x, int tid) {
  const int w = tid >> 5, lane = tid & 31;
  const double2 xv = *reinterpret_cast<const double2*>(x + 2 * lane);
  double p[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const double2 l = *reinterpret_cast<const double2*>(M + (8 * w + r) * TB + 2 * lane);
    p[r] = fma(l.x, xv.x, l.y * xv.y);
  }
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double mine = h16 ? p[i + 4] : p[i];
    const double other = __shfl_xor_sync(0xffffffffu, h16 ? p[i] : p[i + 4], 16);
    p[i] = mine + other;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double mine = h8 ? p[i + 2] : p[i];
    const double other = __shfl_xor_sync(0xffffffffu, h8 ? p[i] : p[i + 2], 8);
    p[i] = mine + other;
  }
  {
    const double mine = h4 ? p[1] : p[0];
    const double other = __shfl_xor_sync(0xffffffffu, h4 ? p[0] : p[1], 4);
    p[0] = mine + other;
  }
  p[0] += __shfl_xor_sync(0xffffffffu, p[0], 2);
  p[0] += __shfl_xor_sync(0xffffffffu, p[0], 1);
  if ((lane & 3) == 0) v[8 * w + (h16 ? 4 : 0) + (h8 ? 2 : 0) + (h4 ? 1 : 0)] -= p[0];
}
// v[a] -= sum_b M[b][a] x[b] (unpadded tile, transposed); ends with a barrier
__device__ __forceinline__ void gemvT_sub_ring(double* v, const double* M, const double* x, double* part,
                                               int tid) {
  const int a = tid & 63, g = tid >> 6;
  double s = 0.0;
#pragma unroll
  for (int b = 0; b < 16; ++b) s = fma(M[(16 * g + b) * TB + a], x[16 * g + b], s);
  part[g * TB + a] = s;
  __syncthreads();
  if (tid < TB) v[tid] -= (part[tid] + part[TB + tid]) + (part[2 * TB + tid] + part[3 * TB + tid]);
  __syncthreads();
}

size_t trsv_smem_bytes(int T, int C, int rs) {
  const int nown = (T + C - 1) / C;
  return sizeof(double) * (size_t)(rs * TB * TB + 3 * nown * TB + 2 * TB * TS + TB + 4 * TB) +
         sizeof(int) * 2 * (size_t)T;
}

// shared-memory carve-up of one solve (dynamic part)
struct TrsvSmem {
  double *ring, *acc, *tv, *wv, *Lc, *Li, *seg, *part;
  int *ff, *bf;
};
__device__ __forceinline__ TrsvSmem trsv_carve(double* sm, int RS, int T, int C) {
  const int nown = (T + C - 1) / C;
  TrsvSmem S;
  S.ring = sm;                       // RS x 4096: streamed non-critical tiles
  S.acc = S.ring + RS * TB * TB;     // per own row: forward, then backward accumulator
  S.tv = S.acc + nown * TB;          // own forward segments t_i
  S.wv = S.tv + nown * TB;           // own backward segments w_i
  S.Lc = S.wv + nown * TB;           // staged critical tile
  S.Li = S.Lc + TB * TS;             // staged inverse of the critical diagonal tile
  S.seg = S.Li + TB * TS;            // the segment being applied
  S.part = S.seg + TB;               // 4 x 64 partial sums
  S.ff = reinterpret_cast<int*>(S.part + 4 * TB);  // forward segment flags (T)
  S.bf = S.ff + T;                                 // backward segment flags (T)
  return S;
}

// One solve w = L^{-T} L^{-1} y by the whole cluster (every CTA calls it).
// `full` are the ring's mbarriers and qbase the ring tiles consumed by
// earlier solves of the same launch (the barrier phases continue).  Starts
// with a cluster barrier (flags zeroed everywhere), ends with the CTA's own
// copies drained; the caller separates consecutive solves by a cluster barrier.
__device__ void trsv_body(const TrsvParams& P, const TrsvSmem& S, uint64_t* full, uint32_t& qbase,
                          int me, int tid) {
  const int RS = P.rs;
  const int C = P.C, T = P.T, i0 = P.i0;
  double* const ring = S.ring;
  double* const acc = S.acc;
  double* const tv = S.tv;
  double* const wv = S.wv;
  double* const Lc = S.Lc;
  double* const Li = S.Li;
  double* const seg = S.seg;
  double* const part = S.part;
  int* const ff = S.ff;
  int* const bf = S.bf;

  for (int e = tid; e < 2 * T; e += 256) ff[e] = 0;
  const int mine = me < T ? (T - 1 - me) / C + 1 : 0;  // own rows me, me + C, ...
  for (int e = tid; e < mine * TB; e += 256) {
    const int q = e >> 6, a = e & 63;
    const int p = (me + q * C) * TB + a;
    acc[e] = (p >= P.rstart && p < P.rend) ? P.r[p - P.rstart] : 0.0;
  }
  const int last = me + (mine - 1) * C;                                  // largest own row
  const int ffirst = me >= i0 ? me : me + ((i0 - me + C - 1) / C) * C;  // first own row >= i0
  const bool has_fwd = mine > 0 && ffirst <= last;
  const SeqCtx sc{me, C, T, i0, last, has_fwd};
  TileSeq prod{0, i0, sc.first_own_ge(i0 + 2)};
  bool prod_ok = false;
  if (tid == 0 && mine > 0) {
    // slots were last read (generic proxy) by the previous solve: order those
    // reads before the async-proxy refills
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    prod_ok = sc.norm(prod);
    for (int q = 0; q < RS && prod_ok; ++q) {  // the ring runs ahead from the start
      const uint32_t slot = (qbase + q) % RS;
      bulk_tile(ring + slot * TB * TB, sc.tile(P.L, prod), &full[slot]);
      sc.advance(prod);
      prod_ok = sc.norm(prod);
    }
  }
  cluster_barrier();  // every CTA's flags are zero before anyone publishes
  if (mine > 0) {
    uint32_t qc = 0;  // tiles consumed by this solve
    // consume the next ring tile (tile qbase + qc of the launch), then refill its slot
    auto consume = [&](double* v, bool transposed) {
      const uint32_t q = qbase + qc;
      const int slot = q % RS;
      mbar_wait(&full[slot], (q / RS) & 1);
      const double* M = ring + slot * TB * TB;
      if (transposed) gemvT_sub_ring(v, M, seg, part, tid);
      else gemv_sub_ring(v, M, seg, tid);
      __syncthreads();  // every warp is done with the slot
      if (tid == 0 && prod_ok) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads -> async write
        bulk_tile(ring + slot * TB * TB, sc.tile(P.L, prod), &full[slot]);
        sc.advance(prod);
        prod_ok = sc.norm(prod);
      }
      ++qc;
    };
    auto stage_fwd = [&](int i) {
      if (i > i0) stage_tile(Lc, P.L + tile_off(i, i - 1), tid);
      stage_tile(Li, P.Linv + (int64_t)i * TB * TB, tid);
      cp_async_commit();
    };
    auto stage_bwd = [&](int i, bool keep_inv) {
      if (i < T - 1) stage_tile(Lc, P.L + tile_off(i + 1, i), tid);
      if (!keep_inv) stage_tile(Li, P.Linv + (int64_t)i * TB * TB, tid);
      cp_async_commit();
    };
    auto publish = [&](int* flags, int i) {
      __syncthreads();
      if (tid < C) st_remote_release(map_to_cta(smem_addr(flags + i), (uint32_t)tid), 1);
    };
    auto fetch = [&](const int* flags, const double* own_store, int k) {
      while (ld_local_acquire(flags + k) == 0) {
      }
      const int owner = k % C;
      if (tid < TB) {
        const double* src = own_store + (k / C) * TB + tid;
        seg[tid] = owner == me ? *src : ld_remote_f64(map_to_cta(smem_addr(src), (uint32_t)owner));
      }
      __syncthreads();
    };
    if (has_fwd) stage_fwd(ffirst);
    else stage_bwd(last, false);

    // ---------------- forward: t = L^{-1} y ----------------
    if (has_fwd && ffirst == i0) {
      cp_async_wait_all();
      __syncthreads();
      gemv_smem(tv + (i0 / C) * TB, Li, acc + (i0 / C) * TB, tid);
      publish(ff, i0);
      if (i0 + C <= last) stage_fwd(i0 + C);
      else stage_bwd(last, true);
    }
    for (int k = i0; k < last && has_fwd; ++k) {
      fetch(ff, tv, k);
      const int i = k + 1;
      if (i % C == me) {  // critical: finish row k + 1
        double* a = acc + (i / C) * TB;
        cp_async_wait_all();
        __syncthreads();
        gemv_sub_smem(a, Lc, seg, tid);
        __syncthreads();
        gemv_smem(tv + (i / C) * TB, Li, a, tid);
        publish(ff, i);
        if (i + C <= last) stage_fwd(i + C);
        else stage_bwd(last, true);
      }
      // the segment's other contributions: own rows i' > k + 1, streamed
      for (int ip = sc.first_own_ge(k + 2); ip <= last; ip += C) consume(acc + (ip / C) * TB, false);
      __syncthreads();
    }
    // ---------------- backward: w = L^{-T} t ----------------
    for (int q = 0; q < mine; ++q) {
      const int i = me + q * C;
      for (int a = tid; a < TB; a += 256) acc[q * TB + a] = i >= i0 ? tv[q * TB + a] : 0.0;
    }
    __syncthreads();
    auto finish_bwd = [&](int i) {  // w_i = Linv_i^T acc_i, publish, stage the next
      double* w = wv + (i / C) * TB;
      gemvT_smem<false>(w, Li, acc + (i / C) * TB, part, tid);
      if (tid < TB) P.w[(int64_t)i * TB + tid] = w[tid];
      publish(bf, i);
      if (i - C >= 0) stage_bwd(i - C, false);
    };
    if (last == T - 1) {
      cp_async_wait_all();
      __syncthreads();
      finish_bwd(T - 1);
    }
    for (int k = T - 1; k > me; --k) {
      fetch(bf, wv, k);
      const int i = k - 1;
      if (i % C == me) {  // critical: finish row k - 1
        cp_async_wait_all();
        __syncthreads();
        gemvT_smem<true>(acc + (i / C) * TB, Lc, seg, part, tid);
        finish_bwd(i);
      }
      // other own rows i' < k - 1, streamed
      for (int ip = me; ip < k - 1; ip += C) consume(acc + (ip / C) * TB, true);
      __syncthreads();
    }
    qbase += qc;
  }
  cp_async_wait_all();
}

__global__ void __launch_bounds__(256, 1) k_trsv_cluster(TrsvParams P) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t full[RS_MAX];
  const int me = (int)cluster_rank();
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < P.rs; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool skip = P.ctl != nullptr && P.ctl->diverged_at != 0;  // uniform over the cluster
  if (!skip) {
    uint32_t qbase = 0;
    trsv_body(P, trsv_carve(sm, P.rs, P.T, P.C), full, qbase, me, tid);
  }
  cluster_barrier();  // no CTA leaves while its segments may still be read
}

// ---------------------------------------------------------------------------
// Inverses of the diagonal tiles (after the factorization of a batch): one
// CTA per (system, tile column j).  Warp q builds block column q of
// X = L_jj^{-1} by 8x8 blocked substitution from the diagonal-block inverses
// the POTRF stored (X_qq = Dinv_q, X_pq = -Dinv_p sum_{q<=m<p} L_pm X_mq).
// ---------------------------------------------------------------------------
constexpr size_t DIAG_INV_SMEM = sizeof(double) * (2 * TB * (TB + 1) + 512 + 512);

__global__ void __launch_bounds__(256) k_diag_inv(CholParams P) {
  extern __shared__ double dsm[];
  double (*Ls)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(dsm);
  double (*Xs)[TB + 1] = reinterpret_cast<double (*)[TB + 1]>(dsm + TB * (TB + 1));
  double* Dv = dsm + 2 * TB * (TB + 1);
  double (*Ss)[64] = reinterpret_cast<double (*)[64]>(Dv + 512);
  int b = 0, j = blockIdx.x;
  while (b + 1 < P.nb && j >= P.m[b].T) j -= P.m[b++].T;
  const CholMat& M = P.m[b];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* Lg = M.L + tile_off(j, j);
  for (int e = tid; e < TB * TB; e += 256) {
    Ls[e >> 6][e & 63] = __ldcg(Lg + e);
    Xs[e >> 6][e & 63] = 0.0;
  }
  for (int e = tid; e < 512; e += 256) Dv[e] = __ldcg(M.Dinv + (int64_t)j * 512 + e);
  __syncthreads();
  const int q = warp;
  const int rr = lane >> 2, cc = 2 * (lane & 3);  // this lane: entries (rr, cc), (rr, cc + 1)
  Xs[8 * q + rr][8 * q + cc] = Dv[q * 64 + rr * 8 + cc];
  Xs[8 * q + rr][8 * q + cc + 1] = Dv[q * 64 + rr * 8 + cc + 1];
  __syncwarp();
  for (int p = q + 1; p < 8; ++p) {
    double s0 = 0.0, s1 = 0.0;
    for (int m = q; m < p; ++m)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double l = Ls[8 * p + rr][8 * m + u];
        s0 = fma(l, Xs[8 * m + u][8 * q + cc], s0);
        s1 = fma(l, Xs[8 * m + u][8 * q + cc + 1], s1);
      }
    Ss[q][rr * 8 + cc] = s0;
    Ss[q][rr * 8 + cc + 1] = s1;
    __syncwarp();
    double x0 = 0.0, x1 = 0.0;
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double d = Dv[p * 64 + rr * 8 + v];
      x0 = fma(d, Ss[q][v * 8 + cc], x0);
      x1 = fma(d, Ss[q][v * 8 + cc + 1], x1);
    }
    Xs[8 * p + rr][8 * q + cc] = -x0;
    Xs[8 * p + rr][8 * q + cc + 1] = -x1;
    __syncwarp();
  }
  __syncthreads();
  double* dst = M.Linv + (int64_t)j * TB * TB;
  for (int e = tid; e < TB * TB; e += 256) dst[e] = Xs[e >> 6][e & 63];
}

void launch_diag_inv(const CholParams& P, cudaStream_t s) {
  int n = 0;
  for (int b = 0; b < P.nb; ++b) n += P.m[b].T;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_diag_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DIAG_INV_SMEM);
    configured = true;
  }
  k_diag_inv<<<n, 256, DIAG_INV_SMEM, s>>>(P);
}

int trsv_cluster_size(int T) {
  int C = 1;
  while (C * 2 <= T && C * 2 <= 16) C *= 2;
  return C;
}

cudaError_t launch_trsv(const TrsvParams& P, cudaStream_t s) {
  static int max_dyn = 0;
  if (max_dyn == 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_trsv_cluster);
    max_dyn = optin - (int)fa.sharedSizeBytes;
    cudaFuncSetAttribute(k_trsv_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaFuncSetAttribute(k_trsv_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
    if (e != cudaSuccess) {
      max_dyn = 0;
      return e;
    }
  }
  if ((int)trsv_smem_bytes(P.T, P.C, P.rs) > max_dyn) return cudaErrorInvalidValue;  // T beyond ~576 tiles
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.C, 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.dynamicSmemBytes = trsv_smem_bytes(P.T, P.C, P.rs);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_trsv_cluster, P);
}

}  // namespace slim
