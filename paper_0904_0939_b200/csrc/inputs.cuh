// inputs.cuh -- device-side inputs: Philox uniform start, BASELINE potentials, potential checks.
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace, after the slab object it operates on).
#pragma once

// ------------------------------------------------------------------
// device-side inputs: the seeded uniform start and the
// BASELINE potentials generated in HBM, so a 2048^3 run needs no host copy of
// either field.  Bitwise the host recipes (workloads.py) except the wells'
// exp (CUDA's exp vs the host libm: <= 1 ulp per well term).
// ------------------------------------------------------------------
// Philox4x64-10 (Salmon et al., SC'11; the numpy.random.Philox bit generator):
// 10 rounds of two 64x64->128 multiplies with the key bumped by the Weyl
// constants between rounds.
__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
  }
}

// plane gi (1..n) of the uniform start: numpy Philox(key=seed) advanced by
// (gi-1)*ceil(n^2/4) blocks, one 64-bit word per site in (j, k) order, each
// block's counter incremented before use; u = ((raw >> 11) + 0.5) 2^-53 - 0.5
// (lattice.uniform_plane).  One thread per block of 4 words.
__global__ void k_fill_uniform(double* __restrict__ psi, uint64_t k0, uint64_t k1, int n,
                               int pitch, long long plane_stride, int planes, int x_off) {
  const long long bpp = ((long long)n * n + 3) / 4;
  const long long total = (long long)planes * bpp;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(t / bpp);
    const long long b = t - (long long)p * bpp;
    const int gi = x_off + p;
    if (gi < 1 || gi > n) continue;
    uint64_t c[4] = {(uint64_t)((long long)(gi - 1) * bpp + b + 1), 0, 0, 0};
    philox4x64_10(c, k0, k1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long w = 4 * b + q;
      if (w >= (long long)n * n) break;
      const int j = 1 + (int)(w / n);
      const int k = 1 + (int)(w - (long long)(j - 1) * n);
      const double u = __dmul_rn(__dadd_rn((double)(c[q] >> 11), 0.5), 0x1.0p-53);
      psi[(long long)p * plane_stride + (long long)j * pitch + k + COL_OFF] = __dsub_rn(u, 0.5);
    }
  }
}

constexpr int POT_HARMONIC = 0, POT_COULOMB = 1, POT_CORNELL = 2, POT_WELLS = 3,
              POT_COULOMB_SHIFTED = 4, POT_DODECAHEDRON = 5;
struct PotParams {
  double p[48];   // cornell: alpha, sigma; wells: centres[8][3], depths[8], widths[8];
                  // dodecahedron: normals[12][3], limit, depth
};

// V on every local plane (padding zero), the workloads.py / potential.py expressions:
// off = (i - center) a, r = sqrt((dx^2 + dy^2) + dz^2)
__global__ void k_fill_potential(double* __restrict__ v, int kind, const PotParams prm, int n,
                                 int pitch, long long plane_stride, int planes, int x_off,
                                 double a, double center) {
  const int ext = n + 2;
  const long long total = (long long)planes * ext * ext;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(t / ((long long)ext * ext));
    const long long r2 = t - (long long)p * ext * ext;
    const int j = (int)(r2 / ext);
    const int k = (int)(r2 - (long long)j * ext);
    const int gi = x_off + p;
    double val = 0.0;
    if (gi >= 1 && gi <= n && j >= 1 && j <= n && k >= 1 && k <= n) {
      const double ox = __dmul_rn(__dsub_rn((double)gi, center), a);
      const double oy = __dmul_rn(__dsub_rn((double)j, center), a);
      const double oz = __dmul_rn(__dsub_rn((double)k, center), a);
      const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(ox, ox), __dmul_rn(oy, oy)),
                                            __dmul_rn(oz, oz)));
      const double half_a = __dmul_rn(0.5, a);
      if (kind == POT_HARMONIC) {
        val = __dmul_rn(__dmul_rn(0.5, r), r);
      } else if (kind == POT_COULOMB) {
        val = __ddiv_rn(-1.0, fmax(r, half_a));
      } else if (kind == POT_COULOMB_SHIFTED) {
        // potential.py:126-136: 0 for r < a, -1/r + 1/a beyond
        val = r >= a ? __dadd_rn(__ddiv_rn(-1.0, r), __ddiv_rn(1.0, a)) : 0.0;
      } else if (kind == POT_DODECAHEDRON) {
        // potential.py:165-183: u = (2i - n - 1)/(n - 1) per axis; inside iff every face
        // normal's (nx ux + ny uy) + nz uz <= limit
        const double dn = (double)n, dm = __dsub_rn(dn, 1.0);
        const double ux = __ddiv_rn(__dsub_rn(__dsub_rn(__dmul_rn(2.0, (double)gi), dn), 1.0), dm);
        const double uy = __ddiv_rn(__dsub_rn(__dsub_rn(__dmul_rn(2.0, (double)j), dn), 1.0), dm);
        const double uz = __ddiv_rn(__dsub_rn(__dsub_rn(__dmul_rn(2.0, (double)k), dn), 1.0), dm);
        bool inside = true;
        for (int f = 0; f < 12; ++f) {
          const double dot = __dadd_rn(__dadd_rn(__dmul_rn(prm.p[3 * f], ux),
                                                 __dmul_rn(prm.p[3 * f + 1], uy)),
                                       __dmul_rn(prm.p[3 * f + 2], uz));
          inside = inside && dot <= prm.p[36];
        }
        val = inside ? prm.p[37] : 0.0;
      } else if (kind == POT_CORNELL) {
        const double rf = fmax(r, half_a);
        val = __dadd_rn(__ddiv_rn(-prm.p[0], rf), __dmul_rn(prm.p[1], rf));
      } else {
        val = __dmul_rn(__dmul_rn(0.5, r), r);
        for (int w = 0; w < 8; ++w) {
          const double dx = __dsub_rn(ox, prm.p[3 * w]);
          const double dy = __dsub_rn(oy, prm.p[3 * w + 1]);
          const double dz = __dsub_rn(oz, prm.p[3 * w + 2]);
          const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                      __dmul_rn(dz, dz));
          const double wd = prm.p[32 + w];
          const double den = __dmul_rn(__dmul_rn(2.0, wd), wd);
          val = __dsub_rn(val, __dmul_rn(prm.p[24 + w], exp(__ddiv_rn(-d2, den))));
        }
      }
    }
    v[(long long)p * plane_stride + (long long)j * pitch + k + COL_OFF] = val;
  }
}
