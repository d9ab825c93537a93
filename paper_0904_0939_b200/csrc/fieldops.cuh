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
// extent.  One warp per row (i, j), lanes along k: every access is a
// coalesced row segment (the mirror row too; along axis 2 it is the same row
// read backwards), and the only integer division is one per row.
__device__ __forceinline__ double impose_val(int ci, double self, double mir, double sign,
                                             int mode, int first_target, int n,
                                             bool zero_center, int center) {
  if (mode != 0) return __dmul_rn(__dadd_rn(self, __dmul_rn(sign, mir)), 0.5);
  if (ci >= first_target && ci <= n) return __dmul_rn(sign, mir);
  if (zero_center && ci == center) return 0.0;
  return self;
}

__global__ void k_impose(const double* __restrict__ in, double* __restrict__ out,
                         const double* sp, int axis, double sign, int mode, int n, int pitch,
                         long long plane_stride, int planes) {
  const int ext = n + 2;
  const double sc = *sp;
  const int first_target = n - n / 2 + 1;
  const bool zero_center = (n % 2 == 1) && sign < 0.0;
  const int center = (n + 1) / 2;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int rows = planes * ext;
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    const int i = row / ext;
    const int j = row - i * ext;
    const long long base = (long long)i * plane_stride + (long long)j * pitch + COL_OFF;
    long long mbase = base;   // mirror row (axes 0, 1)
    if (axis == 0) mbase = (long long)(n + 1 - i) * plane_stride + (long long)j * pitch + COL_OFF;
    else if (axis == 1) mbase = (long long)i * plane_stride + (long long)(n + 1 - j) * pitch + COL_OFF;
    const int cr = axis == 0 ? i : j;   // coordinate along the axis (row-uniform unless axis 2)
    for (int k = lane; k < ext; k += 32) {
      const double self = __dmul_rn(in[base + k], sc);
      const double mir = __dmul_rn(in[axis == 2 ? base + (n + 1 - k) : mbase + k], sc);
      out[base + k] = impose_val(axis == 2 ? k : cr, self, mir, sign, mode, first_target, n,
                                 zero_center, center);
    }
  }
}

// k_impose in place (single-buffer slabs): each lane owns a mirror pair
// (c, n+1-c) along `axis` and reads both sites before writing either, so the
// values are those of k_impose (same operations per site).  Rows as in
// k_impose: axis 0 -> rows (c, j) for c <= (n+1)/2, lanes along k; axis 1 ->
// rows (i, c); axis 2 -> rows (i, j), lanes along c <= (n+1)/2.
__global__ void k_impose_pairs(double* f, const double* sp, int axis, double sign, int mode, int n,
                               int pitch, long long plane_stride) {
  const int ext = n + 2;
  const int hext = (n + 1) / 2 + 1;   // c = 0 .. (n+1)/2 (the centre pairs with itself for odd n)
  const double sc = *sp;
  const int first_target = n - n / 2 + 1;
  const bool zero_center = (n % 2 == 1) && sign < 0.0;
  const int center = (n + 1) / 2;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int rows = axis == 2 ? ext * ext : hext * ext;
  const int inner = axis == 2 ? hext : ext;
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    const int div = axis == 1 ? hext : ext;
    const int r0 = row / div;            // axis 0: c; axis 1: i; axis 2: i
    const int r1 = row - r0 * div;       // axis 0: j; axis 1: c (< hext); axis 2: j
    for (int t = lane; t < inner; t += 32) {
      long long pc, pm;
      int c;
      if (axis == 0) {
        c = r0;
        pc = (long long)c * plane_stride + (long long)r1 * pitch + t + COL_OFF;
        pm = (long long)(n + 1 - c) * plane_stride + (long long)r1 * pitch + t + COL_OFF;
      } else if (axis == 1) {
        c = r1;
        pc = (long long)r0 * plane_stride + (long long)c * pitch + t + COL_OFF;
        pm = (long long)r0 * plane_stride + (long long)(n + 1 - c) * pitch + t + COL_OFF;
      } else {
        c = t;
        const long long b = (long long)r0 * plane_stride + (long long)r1 * pitch + COL_OFF;
        pc = b + c;
        pm = b + (n + 1 - c);
      }
      const int m = n + 1 - c;
      const double xc = __dmul_rn(f[pc], sc);
      const double xm = __dmul_rn(f[pm], sc);
      f[pc] = impose_val(c, xc, xm, sign, mode, first_target, n, zero_center, center);
      if (m != c) f[pm] = impose_val(m, xm, xc, sign, mode, first_target, n, zero_center, center);
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
    for (int c = lane; c < nf; c += 32) {
      const int ic = __ldg(i0 + c);
      const double fc = __ldg(fr + c);
      double t1[2];
#pragma unroll
      for (int dk = 0; dk < 2; ++dk) {
        const double t0lo = lerp(__dmul_rn(r00[ic + dk], sc), __dmul_rn(r10[ic + dk], sc), fa);
        const double t0hi = lerp(__dmul_rn(r01[ic + dk], sc), __dmul_rn(r11[ic + dk], sc), fa);
        t1[dk] = lerp(t0lo, t0hi, fb);
      }
      dst[c] = lerp(t1[0], t1[1], fc);
    }
  }
}
