// fieldops.cuh -- elementwise field kernels (scale, impose, resample, checks).
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace; the host engine instantiates the templates).
#pragma once

// ------------------------------------------------------------------
// elementwise kernels
// ------------------------------------------------------------------
__global__ void k_scale(double* f, long long count, const double* sp, double factor) {
  const double s = sp ? *sp : factor;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    f[i] = __dmul_rn(f[i], s);
}

// first site (host C order) with 1 + (0.5 dtau) V == 0 (potential._coefficients,
// potential.py:103-110), over count uploaded planes of the full padded extent
__global__ void k_singular(const double* __restrict__ v, double h, int ext, int pitch,
                           long long plane_stride, int first, int count, long long gfirst,
                           unsigned long long* first_bad, unsigned* wide) {
  // grid: x over rows of all uploaded planes, threads over columns.  Also
  // flags any d outside [0.25, 4), where the sweeps' shared-reciprocal
  // coefficients need their checked path.
  bool w = false;
  for (long long r = blockIdx.x; r < (long long)count * ext; r += gridDim.x) {
    const int p = (int)(r / ext);
    const int j = (int)(r - (long long)p * ext);
    const double* row = v + (long long)(first + p) * plane_stride + (long long)j * pitch + COL_OFF;
    for (int k = threadIdx.x; k < ext; k += blockDim.x) {
      const double d = __dadd_rn(1.0, __dmul_rn(h, row[k]));
      if (d == 0.0) atomicMin(first_bad, (unsigned long long)(((gfirst + p) * ext + j) * ext + k));
      w |= !(d >= 0.25 && d < 4.0);
    }
  }
  if (__syncthreads_or(w) && threadIdx.x == 0) atomicOr(wide, 1u);
}

// f1 <- f1*s1 - c*(f2*s2)  (states._project_inplace: values -= c * b.values, states.py:92-99)
__global__ void k_axpy(double* f1, const double* s1p, const double* __restrict__ f2,
                       const double* s2p, double c, long long count) {
  const double s1 = *s1p, s2 = *s2p;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    f1[i] = __dsub_rn(__dmul_rn(f1[i], s1), __dmul_rn(c, __dmul_rn(f2[i], s2)));
}

// parity (states.impose_inplace, states.py:70-82, and the projector start):
// out = copy / projector of in (scaled by *sp) along `axis`, full padded
// extent.  Every lane owns mirror pairs (c, n+1-c) along the axis and reads
// both sites before writing either (so out may alias in: the single-buffer
// slabs' in-place imposition), 16 B of traffic per site instead of 24 for a
// separate mirror read.  One warp per row, lanes along k, four pairs in
// flight per lane: axis 0 -> rows (c, j) for c <= (n+1)/2; axis 1 -> rows
// (i, c); axis 2 -> rows (i, j), lanes along c <= (n+1)/2 (the mirror read
// is the same row backwards).  The only integer divisions are per row.
__device__ __forceinline__ double impose_val(int ci, double self, double mir, double sign,
                                             int mode, int first_target, int n,
                                             bool zero_center, int center) {
  if (mode != 0) return __dmul_rn(__dadd_rn(self, __dmul_rn(sign, mir)), 0.5);
  if (ci >= first_target && ci <= n) return __dmul_rn(sign, mir);
  if (zero_center && ci == center) return 0.0;
  return self;
}

constexpr int IMP_UNROLL = 4;
__global__ void __launch_bounds__(256)
    k_impose(const double* in, double* out, const double* sp, int axis, double sign, int mode,
             int n, int pitch, long long plane_stride, int planes) {
  const int ext = n + 2;
  const int hext = (n + 1) / 2 + 1;   // c = 0 .. (n+1)/2 (the centre pairs with itself for odd n)
  const double sc = *sp;
  const int first_target = n - n / 2 + 1;
  const bool zero_center = (n % 2 == 1) && sign < 0.0;
  const int center = (n + 1) / 2;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  // axis 0 pairs planes: the field's planes must be the whole padded lattice
  const int rows = axis == 2 ? planes * ext : (axis == 1 ? planes * hext : hext * ext);
  const int inner = axis == 2 ? hext : ext;
  const int div = axis == 1 ? hext : ext;
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    const int r0 = row / div;            // axis 0: c; axis 1: i; axis 2: i
    const int r1 = row - r0 * div;       // axis 0: j; axis 1: c (< hext); axis 2: j
    long long bc, bm;   // row bases of the pair (axis 2: one row)
    int cr = 0;         // the pair's coordinate along the axis (axes 0, 1)
    if (axis == 0) {
      cr = r0;
      bc = (long long)r0 * plane_stride + (long long)r1 * pitch + COL_OFF;
      bm = (long long)(n + 1 - r0) * plane_stride + (long long)r1 * pitch + COL_OFF;
    } else if (axis == 1) {
      cr = r1;
      bc = (long long)r0 * plane_stride + (long long)r1 * pitch + COL_OFF;
      bm = (long long)r0 * plane_stride + (long long)(n + 1 - r1) * pitch + COL_OFF;
    } else {
      bc = bm = (long long)r0 * plane_stride + (long long)r1 * pitch + COL_OFF;
    }
    for (int t0 = lane; t0 < inner; t0 += 32 * IMP_UNROLL) {
      double xc[IMP_UNROLL], xm[IMP_UNROLL];
#pragma unroll
      for (int u = 0; u < IMP_UNROLL; ++u) {
        const int t = t0 + 32 * u;
        if (t < inner) {
          const long long pc = axis == 2 ? bc + t : bc + t;
          const long long pm = axis == 2 ? bm + (n + 1 - t) : bm + t;
          xc[u] = __dmul_rn(in[pc], sc);
          xm[u] = __dmul_rn(in[pm], sc);
        }
      }
#pragma unroll
      for (int u = 0; u < IMP_UNROLL; ++u) {
        const int t = t0 + 32 * u;
        if (t < inner) {
          const int c = axis == 2 ? t : cr;
          const int m = n + 1 - c;
          const long long pc = bc + t;
          const long long pm = axis == 2 ? bm + (n + 1 - t) : bm + t;
          out[pc] = impose_val(c, xc[u], xm[u], sign, mode, first_target, n, zero_center, center);
          if (m != c) out[pm] = impose_val(m, xm[u], xc[u], sign, mode, first_target, n, zero_center, center);
        }
      }
    }
  }
}

// trilinear resample, bitwise replica of multires._axis_interp applied along
// axis 0, then 1, then 2 (multires.py:116-154): each lerp is lo + f*(hi - lo).
// One warp per fine row (a, b), lanes along c: the fine row is written
// coalesced; the four coarse rows (ia|ia+1, ib|ib+1) it reads are fixed per row
// and their segments are shared by neighbouring lanes (L1).
__global__ void k_resample(const double* __restrict__ coarse, const double* csp, int nc,
                           int cpitch, long long cplane, double* __restrict__ fine, int nf,
                           int fpitch, long long fplane, const int* __restrict__ i0,
                           const double* __restrict__ fr) {
  (void)nc;
  const double sc = *csp;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int rows = nf * nf;
  auto lerp = [](double lo, double hi, double f) {
    return __dadd_rn(lo, __dmul_rn(f, __dsub_rn(hi, lo)));
  };
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    const int a = row / nf;
    const int b = row - a * nf;
    const int ia = __ldg(i0 + a), ib = __ldg(i0 + b);
    const double fa = __ldg(fr + a), fb = __ldg(fr + b);
    const double* r00 = coarse + (long long)ia * cplane + (long long)ib * cpitch + COL_OFF;
    const double* r10 = r00 + cplane;
    const double* r01 = r00 + cpitch;
    const double* r11 = r10 + cpitch;
    double* dst = fine + (long long)(a + 1) * fplane + (long long)(b + 1) * fpitch + 1 + COL_OFF;
    // two output sites per lane in flight (16 independent coarse loads)
    for (int c0 = lane; c0 < nf; c0 += 64) {
      double g[2][8];
      int cc[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        cc[u] = c0 + 32 * u;
        if (cc[u] < nf) {
          const int ic = __ldg(i0 + cc[u]);
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) {
            g[u][4 * dk + 0] = r00[ic + dk];
            g[u][4 * dk + 1] = r10[ic + dk];
            g[u][4 * dk + 2] = r01[ic + dk];
            g[u][4 * dk + 3] = r11[ic + dk];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (cc[u] < nf) {
          const double fc = __ldg(fr + cc[u]);
          double t1[2];
#pragma unroll
          for (int dk = 0; dk < 2; ++dk) {
            const double t0lo = lerp(__dmul_rn(g[u][4 * dk + 0], sc), __dmul_rn(g[u][4 * dk + 1], sc), fa);
            const double t0hi = lerp(__dmul_rn(g[u][4 * dk + 2], sc), __dmul_rn(g[u][4 * dk + 3], sc), fa);
            t1[dk] = lerp(t0lo, t0hi, fb);
          }
          dst[cc[u]] = lerp(t1[0], t1[1], fc);
        }
      }
    }
  }
}
