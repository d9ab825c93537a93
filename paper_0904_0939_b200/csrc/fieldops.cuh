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

// parity: out = copy / projector of in (scaled by *sp) along `axis`, full padded extent
__global__ void k_impose(const double* __restrict__ in, double* __restrict__ out,
                         const double* sp, int axis, double sign, int mode, int n, int pitch,
                         long long plane_stride, int planes) {
  const int ext = n + 2;
  const long long total = (long long)planes * ext * ext;
  const double sc = *sp;
  const int half = n / 2;
  const int first_target = n - half + 1;
  const bool zero_center = (n % 2 == 1) && sign < 0.0;
  const int center = (n + 1) / 2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % ext);
    const long long r = t / ext;
    const int j = (int)(r % ext);
    const int i = (int)(r / ext);
    int c[3] = {i, j, k};
    const long long dst = (long long)i * plane_stride + (long long)j * pitch + k + COL_OFF;
    const double self = __dmul_rn(in[dst], sc);
    int m[3] = {i, j, k};
    m[axis] = n + 1 - c[axis];
    const long long src = (long long)m[0] * plane_stride + (long long)m[1] * pitch + m[2] + COL_OFF;
    const double mir = __dmul_rn(in[src], sc);
    double val;
    if (mode == 0) {
      const int ci = c[axis];
      if (ci >= first_target && ci <= n) val = __dmul_rn(sign, mir);
      else if (zero_center && ci == center) val = 0.0;
      else val = self;
    } else {
      val = __dmul_rn(__dadd_rn(self, __dmul_rn(sign, mir)), 0.5);
    }
    out[dst] = val;
  }
}

// k_impose in place (single-buffer slabs): one thread per mirror pair
// (c, n+1-c) along `axis` reads both sites before writing either, so the
// values are those of k_impose (same operations per site)
__global__ void k_impose_pairs(double* f, const double* sp, int axis, double sign, int mode, int n,
                               int pitch, long long plane_stride) {
  const int ext = n + 2;
  const int hext = (n + 1) / 2 + 1;   // c = 0 .. (n+1)/2 (the centre pairs with itself for odd n)
  const long long total = (long long)hext * ext * ext;
  const double sc = *sp;
  const int half = n / 2;
  const int first_target = n - half + 1;
  const bool zero_center = (n % 2 == 1) && sign < 0.0;
  const int center = (n + 1) / 2;
  const long long st[3] = {plane_stride, (long long)pitch, 1};
  auto val = [&](int ci, double self, double mir) {
    if (mode != 0) return __dmul_rn(__dadd_rn(self, __dmul_rn(sign, mir)), 0.5);
    if (ci >= first_target && ci <= n) return __dmul_rn(sign, mir);
    if (zero_center && ci == center) return 0.0;
    return self;
  };
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    // t enumerates (c, u, v): c along `axis`, u, v the other two axes in order
    const int v = (int)(t % ext);
    const long long r = t / ext;
    const int u = (int)(r % ext);
    const int c = (int)(r / ext);
    const int m = n + 1 - c;
    int ax[3], q = 0;
    for (int d = 0; d < 3; ++d) ax[d] = d == axis ? -1 : (q++ == 0 ? u : v);
    long long base = COL_OFF;
    for (int d = 0; d < 3; ++d)
      if (d != axis) base += (long long)ax[d] * st[d];
    const long long pc = base + (long long)c * st[axis];
    const long long pm = base + (long long)m * st[axis];
    const double xc = __dmul_rn(f[pc], sc);
    const double xm = __dmul_rn(f[pm], sc);
    f[pc] = val(c, xc, xm);
    if (m != c) f[pm] = val(m, xm, xc);
  }
}

// trilinear resample, bitwise replica of multires._axis_interp applied along
// axis 0, then 1, then 2: each lerp is lo + f*(hi - lo)
__global__ void k_resample(const double* __restrict__ coarse, const double* csp, int nc,
                           int cpitch, long long cplane, double* __restrict__ fine, int nf,
                           int fpitch, long long fplane, const int* __restrict__ i0,
                           const double* __restrict__ fr) {
  const long long total = (long long)nf * nf * nf;
  const double sc = *csp;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(t % nf);
    const long long r = t / nf;
    const int b = (int)(r % nf);
    const int a = (int)(r / nf);
    const int ia = i0[a], ib = i0[b], ic = i0[c];
    const double fa = fr[a], fb = fr[b], fc = fr[c];
    auto at = [&](int i, int j, int k) {
      return __dmul_rn(coarse[(long long)i * cplane + (long long)j * cpitch + k + COL_OFF], sc);
    };
    auto lerp = [](double lo, double hi, double f) {
      return __dadd_rn(lo, __dmul_rn(f, __dsub_rn(hi, lo)));
    };
    double t1[2];
#pragma unroll
    for (int dk = 0; dk < 2; ++dk) {
      const double t0lo = lerp(at(ia, ib, ic + dk), at(ia + 1, ib, ic + dk), fa);
      const double t0hi = lerp(at(ia, ib + 1, ic + dk), at(ia + 1, ib + 1, ic + dk), fa);
      t1[dk] = lerp(t0lo, t0hi, fb);
    }
    fine[(long long)(a + 1) * fplane + (long long)(b + 1) * fpitch + (c + 1) + COL_OFF] =
        lerp(t1[0], t1[1], fc);
  }
}
