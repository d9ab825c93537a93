// reduce.cuh -- plane reductions and the numpy-pairwise combine.
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace; the host engine instantiates the templates).
#pragma once

// ------------------------------------------------------------------
// plain per-plane reductions (norm / dot) without a sweep
// block = TY warps, grid = (tiles, planes); same tile partition and summation
// order as the sweep's fused partials.
// ------------------------------------------------------------------
template <bool DOT>
__global__ void __launch_bounds__(32 * TY)
    k_planesum(const double* __restrict__ f1, const double* __restrict__ s1p,
               const double* __restrict__ f2, const double* __restrict__ s2p, double* part, int q,
               int n, int pitch, long long plane_stride, int planes, int tiles_k, int tiles,
               int z_lo) {
  __shared__ double lsum[TY][32];
  const int tile = blockIdx.x;
  const int p = z_lo + blockIdx.y;
  const int tj = tile / tiles_k, tk = tile - tj * tiles_k;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = 1 + tj * TY + w;
  const int k = 1 + tk * TX + 2 * lane;
  const bool ok0 = (j <= n) && (k <= n);
  const bool ok1 = (j <= n) && (k + 1 <= n);
  const double sc1 = *s1p;
  const double sc2 = DOT ? *s2p : 0.0;
  double r = 0.0;
  if (j <= n) {
    const long long base = (long long)p * plane_stride + (long long)j * pitch + k + COL_OFF;
    double a0 = ok0 ? __dmul_rn(f1[base], sc1) : 0.0;
    double a1 = ok1 ? __dmul_rn(f1[base + 1], sc1) : 0.0;
    double b0 = a0, b1 = a1;
    if (DOT) {
      b0 = ok0 ? __dmul_rn(f2[base], sc2) : 0.0;
      b1 = ok1 ? __dmul_rn(f2[base + 1], sc2) : 0.0;
    }
    r = __dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1));
  }
  // same order as the sweep's fused NORM partials: per lane the rows in
  // ascending order, then the xor butterfly over lanes
  lsum[w][lane] = r;
  __syncthreads();
  if (w == 0) {
    double acc = lsum[0][lane];
    for (int i = 1; i < TY; ++i) acc = __dadd_rn(acc, lsum[i][lane]);
    acc = warp_sum(acc);
    if (lane == 0) part[((size_t)q * planes + p) * tiles + tile] = acc;
  }
}

// ------------------------------------------------------------------
// numpy pairwise sum replica (numpy _core/src/umath/loops_utils.h.src,
// DOUBLE_pairwise_sum; np.sum = 0.0 + pairwise(a, n))
// ------------------------------------------------------------------
constexpr int PW_SMEM = 4096;        // plane sums staged in shared memory up to this length
constexpr int PW_MAX_LEAVES = 512;   // leaves are >= ~60 long -> n <= ~30000
constexpr int PW_MAX_N = 16384;

__device__ double pw_leaf(const double* a, int n) {
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = a[q];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], a[i + q]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// enumerate the leaves of the recursion in left-to-right order
__device__ int pw_leaves(int off, int n, int* lo, int* len, int cnt) {
  if (n <= 128) {
    lo[cnt] = off;
    len[cnt] = n;
    return cnt + 1;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  cnt = pw_leaves(off, n2, lo, len, cnt);
  return pw_leaves(off + n2, n - n2, lo, len, cnt);
}

__device__ double pw_tree(int n, const double* leafv, int* idx) {
  if (n <= 128) return leafv[(*idx)++];
  int n2 = n / 2;
  n2 -= n2 % 8;
  const double l = pw_tree(n2, leafv, idx);
  const double r = pw_tree(n - n2, leafv, idx);
  return __dadd_rn(l, r);
}

struct CombineSmem {
  double buf[PW_SMEM];
  double leafv[PW_MAX_LEAVES];
  int lo[PW_MAX_LEAVES];
  int len[PW_MAX_LEAVES];
  int nleaves;
  int last;
};

// block-wide pairwise sum of a[0..n); result valid in thread 0
__device__ double block_pairwise(const double* a, int n, CombineSmem& sm) {
  if (threadIdx.x == 0) sm.nleaves = pw_leaves(0, n, sm.lo, sm.len, 0);
  __syncthreads();
  const int L = sm.nleaves;
  for (int t = threadIdx.x; t < L; t += blockDim.x) sm.leafv[t] = pw_leaf(a + sm.lo[t], sm.len[t]);
  __syncthreads();
  double res = 0.0;
  if (threadIdx.x == 0) {
    int idx = 0;
    res = __dadd_rn(0.0, pw_tree(n, sm.leafv, &idx));
  }
  __syncthreads();
  return res;
}

// scal: [0..3] totals, [4] E, [5] norm2, [6] r_rms, [7] n2, [8] factor, [9] status,
//       [11] one
constexpr int S_E = 4, S_NORM2 = 5, S_RRMS = 6, S_N2 = 7, S_FACTOR = 8, S_STATUS = 9, S_ONE = 11;
constexpr int NSCAL = 16;

__device__ void combine_scalars(const double* tot, unsigned qmask, double a3, double* scal,
                                double* hist_rec, const int* bad);

// cross-plane combine exactly like observables.combine_plane_sums (np.sum) and
// the scalars of evolve._record_from_sums / SweepBuffers.renormalize
__device__ void combine_body(const double* plane_sums, int n, unsigned qmask, double a3,
                             double* scal, double* hist_rec, const int* bad, CombineSmem& sm) {
  double tot[NQ] = {0.0, 0.0, 0.0, 0.0};
  for (int q = 0; q < NQ; ++q) {
    if (!(qmask & (1u << q))) continue;
    const double* src = plane_sums + (size_t)q * n;
    const double* a = src;
    if (n <= PW_SMEM) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) sm.buf[i] = __ldcg(src + i);
      __syncthreads();
      a = sm.buf;
    }
    tot[q] = block_pairwise(a, n, sm);
  }
  if (threadIdx.x == 0) combine_scalars(tot, qmask, a3, scal, hist_rec, bad);
  // copy the measured plane sums into the history record
  if (hist_rec && (qmask & 7u) == 7u) {
    for (int i = threadIdx.x; i < 3 * n; i += blockDim.x) hist_rec[2 + i] = __ldcg(plane_sums + i);
  }
}

// the scalars of evolve._record_from_sums / SweepBuffers.renormalize from the
// totals (thread 0 of the combining block)
__device__ void combine_scalars(const double* tot, unsigned qmask, double a3, double* scal,
                                double* hist_rec, const int* bad) {
  {
    for (int q = 0; q < NQ; ++q)
      if (qmask & (1u << q)) scal[q] = tot[q];
    double status = scal[S_STATUS];
    if (qmask & (1u << PSG_Q_DEN)) {
      const double den = tot[PSG_Q_DEN];
      scal[S_E] = __ddiv_rn(tot[PSG_Q_NUM], den);
      scal[S_NORM2] = __dmul_rn(den, a3);
      scal[S_RRMS] = __dsqrt_rn(__ddiv_rn(tot[PSG_Q_R2], den));
      const bool zero = (den == 0.0 || !finite_d(den));
      if (zero && status == 0.0) status = 3.0;
      if (hist_rec) hist_rec[1] = zero ? 3.0 : 0.0;
    }
    if (qmask & (1u << PSG_Q_NORM)) {
      const double n2 = __dmul_rn(tot[PSG_Q_NORM], a3);
      scal[S_N2] = n2;
      if (n2 == 0.0) {
        if (status == 0.0) status = 3.0;
        scal[S_FACTOR] = 1.0;
      } else if (!finite_d(n2)) {
        if (status == 0.0) status = 4.0;
        scal[S_FACTOR] = 1.0;
      } else {
        scal[S_FACTOR] = __ddiv_rn(1.0, __dsqrt_rn(n2));
      }
    }
    if (bad && __ldcg(bad) && status == 0.0) status = 4.0;
    scal[S_STATUS] = status;
  }
}

// tile partials [q][plane][tiles] (q at qstride) -> plane sums: one warp per
// plane, lane l sums tiles l, l+32, ...
// sequentially, then the fixed xor butterfly; with `combine`, the last block to
// finish runs the cross-plane combine
constexpr int RED_WARPS = 8;
__global__ void __launch_bounds__(32 * RED_WARPS)
    k_plane_reduce(const double* __restrict__ part, double* plane_sums, unsigned qmask,
                   long long qstride, int tiles, int z_lo, int z_hi, int x_off, int n, int* counter,
                   int combine, double a3, double* scal, double* hist_rec, const int* bad) {
  __shared__ CombineSmem sm;
  // launched as a programmatic dependent of the sweep: wait for its partials
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int p = z_lo + blockIdx.x * RED_WARPS + (threadIdx.x >> 5);
  if (p <= z_hi) {
    const int gplane = x_off + p - 1;  // 0-based interior index of this plane
    for (int q = 0; q < NQ; ++q) {
      if (!(qmask & (1u << q))) continue;
      const double* src = part + (size_t)q * qstride + (size_t)p * tiles;
      double acc = 0.0;
      for (int t = lane; t < tiles; t += 32) acc = __dadd_rn(acc, src[t]);
      acc = warp_sum(acc);
      if (lane == 0 && gplane >= 0 && gplane < n) plane_sums[(size_t)q * n + gplane] = acc;
    }
  }
  if (!combine) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sm.last = (atomicAdd(counter, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  combine_body(plane_sums, n, qmask, a3, scal, hist_rec, bad, sm);
  if (threadIdx.x == 0) *counter = 0;
}

__global__ void __launch_bounds__(256)
    k_combine(const double* plane_sums, int n, unsigned qmask, double a3, double* scal,
              double* hist_rec, const int* bad) {
  __shared__ CombineSmem sm;
  pdl_launch_dependents();
  pdl_wait();
  combine_body(plane_sums, n, qmask, a3, scal, hist_rec, bad, sm);
}

// Total of a renormalising pass's NORM slots (one per step-2 warp and launch)
// in a fixed order -- per thread a strided sequential sum, then a fixed
// shared-memory tree -- and the factor / status the combine would form
// (scal[S_N2], scal[S_FACTOR], scal[S_STATUS]).  One block.
constexpr int NT_THREADS = 512;
__global__ void __launch_bounds__(NT_THREADS)
    k_norm_total(const double* __restrict__ slots, long long count, double a3, double* scal,
                 const int* bad) {
  __shared__ double red[NT_THREADS];
  pdl_launch_dependents();
  pdl_wait();
  double acc = 0.0;
  for (long long i = threadIdx.x; i < count; i += NT_THREADS) acc = __dadd_rn(acc, slots[i]);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = NT_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double status = scal[S_STATUS];
    const double n2 = __dmul_rn(red[0], a3);
    scal[S_N2] = n2;
    if (n2 == 0.0) {
      if (status == 0.0) status = 3.0;
      scal[S_FACTOR] = 1.0;
    } else if (!finite_d(n2)) {
      if (status == 0.0) status = 4.0;
      scal[S_FACTOR] = 1.0;
    } else {
      scal[S_FACTOR] = __ddiv_rn(1.0, __dsqrt_rn(n2));
    }
    if (bad && __ldcg(bad) && status == 0.0) status = 4.0;
    scal[S_STATUS] = status;
  }
}

// Small whole lattices (n <= 128): tile partials -> plane sums -> combine in ONE
// block (no cross-block counter, no recursion): warp w reduces planes w, w+8,
// ... exactly like k_plane_reduce, then warp q's lane 0 forms quantity q's
// np.sum (0.0 + one pairwise leaf, numpy's order for n <= 128) -- bitwise the
// multi-block path.  Measured: the multi-block reduce + combine takes 9-13 us
// at 64^3 (profiles/ncu_r02_c1_small.json), most of a norm / measure step.
constexpr int RS_MAX_N = 128;
constexpr int RS_WARPS = 32;
__global__ void __launch_bounds__(32 * RS_WARPS)
    k_reduce_small(const double* __restrict__ part, double* plane_sums, unsigned qmask,
                   long long qstride, int tiles, int z_lo, int z_hi, int x_off, int n, double a3,
                   double* scal, double* hist_rec, const int* bad) {
  __shared__ double ps[NQ][RS_MAX_N];
  __shared__ double tot[NQ];
  pdl_launch_dependents();
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // (quantity, plane) pairs spread over all 32 warps
  int qs[NQ], nq = 0;
  for (int q = 0; q < NQ; ++q)
    if (qmask & (1u << q)) qs[nq++] = q;
  const int np = z_hi - z_lo + 1;
  for (int w = warp; w < nq * np; w += RS_WARPS) {
    const int q = qs[w / np];
    const int p = z_lo + w % np;
    const int gplane = x_off + p - 1;
    const double* src = part + (size_t)q * qstride + (size_t)p * tiles;
    double acc = 0.0;
    for (int t = lane; t < tiles; t += 32) acc = __dadd_rn(acc, src[t]);
    acc = warp_sum(acc);
    if (lane == 0 && gplane >= 0 && gplane < n) {
      plane_sums[(size_t)q * n + gplane] = acc;
      ps[q][gplane] = acc;
    }
  }
  __syncthreads();
  if (lane == 0 && warp < NQ && (qmask & (1u << warp))) tot[warp] = __dadd_rn(0.0, pw_leaf(ps[warp], n));
  __syncthreads();
  if (threadIdx.x == 0) combine_scalars(tot, qmask, a3, scal, hist_rec, bad);
  if (hist_rec && (qmask & 7u) == 7u) {
    for (int q = 0; q < 3; ++q)
      for (int i = threadIdx.x; i < n; i += blockDim.x) hist_rec[2 + q * n + i] = ps[q][i];
  }
}
