// small.cuh -- k_small: many plain sweeps of a small lattice in ONE persistent
// cooperative launch (N <= 64; BASELINE config 1 is 64^3).
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace; the host engine launches it from run_loop).
//
// At N = 64 the whole lattice is 2 MB: one launch per sweep (or per two-sweep
// pass) is latency-bound -- prologue, pipeline fill and drain of a kernel
// whose 148 blocks each hold a few planes of a 4-tile plane.
// Here every block owns an 8 x 16 x 16 brick of the lattice for the whole run
// (128 bricks at 64^3, one block per SM, co-resident by cooperative launch):
//   * the brick and its one-site halo live in shared memory, each thread's
//     column of 8 sites along axis 0 in registers, and A, C of its 8 sites are
//     formed once from V (the reference's coefficient arithmetic);
//   * a sweep updates the brick from shared memory (the reference's per-site
//     order, upd()), then publishes its six faces to a global face buffer
//     (two sweep parities), every value tagged with its sweep number;
//   * its halo for the next sweep is read from the <= 6 neighbours' faces,
//     each value awaited by its tag (data-carried synchronisation: no flag,
//     no fence, no grid barrier; a tagged 64-bit word is single-copy atomic).
// No grid-wide barrier and no launch per sweep; every site's value is bitwise
// k_sweep's (same upd(), same coefficients).  Plain steps only: runs with a
// norm / measure / impose step between them are cut by run_loop, which sends
// those steps through k_sweep as before.
#pragma once

constexpr int SB_I = 8, SB_J = 16, SB_K = 16;   // brick: planes x rows x columns
constexpr int SB_THREADS = SB_J * SB_K;          // one thread per (row, column): a column of SB_I sites
constexpr int SB_FACE = 2 * SB_J * SB_K + 4 * SB_I * SB_K;   // doubles per brick and parity (SB_J == SB_K)

struct SmallArgs {
  const double* in;        // current field (device layout)
  double* out;             // result field (the other buffer)
  const double* v;         // potential
  unsigned long long* faces;   // [2 parities][bricks][SB_FACE][2 words]: tagged face values
  unsigned long long base;     // tag of the sweep before this launch's first (monotonic)
  long long plane_stride;
  int n, pitch, steps;
  int nbi, nbj, nbk;       // bricks per axis
  double h, c0;
};

// A face value travels as two 64-bit words {32 bits of the double, 32-bit
// sweep tag}: each word is single-copy atomic, so a reader that sees both
// tags equal to the sweep it waits for holds that sweep's value -- the data
// carries its own synchronisation (no flag, no fence, no grid barrier).
__device__ __forceinline__ void put_tagged(unsigned long long* p, double v, uint32_t tag) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = (bits << 32) | tag;
  const unsigned long long w1 = (bits & 0xffffffff00000000ull) | tag;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ double get_tagged(const unsigned long long* p, uint32_t tag) {
  unsigned long long w0, w1;
  unsigned spins = 0;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
    if ((uint32_t)w0 == tag && (uint32_t)w1 == tag) break;
    if (++spins > (1u << 30)) __trap();
  }
  return __longlong_as_double((long long)((w1 & 0xffffffff00000000ull) | (w0 >> 32)));
}

template <bool FASTC>
__global__ void __launch_bounds__(SB_THREADS, 1) k_small(const SmallArgs a) {
  __shared__ double sp[SB_I][SB_J + 2][SB_K + 2];   // brick + halo rows / columns
  __shared__ double sh[2][SB_J][SB_K];              // halo planes below / above the brick
  const int b = blockIdx.x;
  const int bk = b % a.nbk;
  const int bj = (b / a.nbk) % a.nbj;
  const int bi = b / (a.nbk * a.nbj);
  const int tk = threadIdx.x % SB_K, tj = threadIdx.x / SB_K;
  const int i0 = 1 + bi * SB_I, j0 = 1 + bj * SB_J, k0 = 1 + bk * SB_K;
  const long long ps = a.plane_stride;
  auto at = [&](int i, int j, int k) { return (long long)i * ps + (long long)j * a.pitch + k + COL_OFF; };
  pdl_wait();   // the predecessor's output is this launch's input
  // brick + halo ring from the input field (lattice padding reads zeros)
  for (int t = threadIdx.x; t < SB_I * (SB_J + 2) * (SB_K + 2); t += SB_THREADS) {
    const int kk = t % (SB_K + 2), r = t / (SB_K + 2);
    const int jj = r % (SB_J + 2), ii = r / (SB_J + 2);
    sp[ii][jj][kk] = a.in[at(i0 + ii, j0 - 1 + jj, k0 - 1 + kk)];
  }
  sh[0][tj][tk] = a.in[at(i0 - 1, j0 + tj, k0 + tk)];
  sh[1][tj][tk] = a.in[at(i0 + SB_I, j0 + tj, k0 + tk)];
  double A[SB_I], C[SB_I], c[SB_I];
#pragma unroll
  for (int i = 0; i < SB_I; ++i) coef1<FASTC>(a.v[at(i0 + i, j0 + tj, k0 + tk)], a.h, a.c0, A[i], C[i]);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SB_I; ++i) c[i] = sp[i][tj + 1][tk + 1];
  // neighbours (-1: lattice boundary, its halo stays the padding's zeros)
  const int nb_ilo = bi > 0 ? b - a.nbk * a.nbj : -1, nb_ihi = bi + 1 < a.nbi ? b + a.nbk * a.nbj : -1;
  const int nb_jlo = bj > 0 ? b - a.nbk : -1, nb_jhi = bj + 1 < a.nbj ? b + a.nbk : -1;
  const int nb_klo = bk > 0 ? b - 1 : -1, nb_khi = bk + 1 < a.nbk ? b + 1 : -1;
  const int nbs = a.nbi * a.nbj * a.nbk;
  // face offsets in a brick's record (values; two words each)
  constexpr int F_ILO = 0, F_IHI = SB_J * SB_K, F_JLO = 2 * SB_J * SB_K;
  constexpr int F_JHI = F_JLO + SB_I * SB_K, F_KLO = F_JHI + SB_I * SB_K, F_KHI = F_KLO + SB_I * SB_J;
  const int t = threadIdx.x;
  for (int s = 1; s <= a.steps; ++s) {
    double nv[SB_I];
#pragma unroll
    for (int i = 0; i < SB_I; ++i) {
      const double im = i == 0 ? sh[0][tj][tk] : c[i - 1];
      const double ip = i == SB_I - 1 ? sh[1][tj][tk] : c[i + 1];
      nv[i] = upd(A[i], C[i], c[i], im, ip, sp[i][tj][tk + 1], sp[i][tj + 2][tk + 1],
                  sp[i][tj + 1][tk], sp[i][tj + 1][tk + 2]);
    }
    __syncthreads();   // every read of the old brick and halo is done
#pragma unroll
    for (int i = 0; i < SB_I; ++i) {
      c[i] = nv[i];
      sp[i][tj + 1][tk + 1] = nv[i];
    }
    if (s == a.steps) break;
    const uint32_t tag = (uint32_t)(a.base + (unsigned long long)s);
    // publish the six faces of sweep s (parity s & 1: a neighbour overwrites
    // a parity only after it has read our faces of the sweep in between)
    unsigned long long* f = a.faces + ((size_t)(s & 1) * nbs + b) * (2 * SB_FACE);
    put_tagged(f + 2 * (F_ILO + tj * SB_K + tk), c[0], tag);
    put_tagged(f + 2 * (F_IHI + tj * SB_K + tk), c[SB_I - 1], tag);
#pragma unroll
    for (int i = 0; i < SB_I; ++i) {
      if (tj == 0) put_tagged(f + 2 * (F_JLO + i * SB_K + tk), c[i], tag);
      if (tj == SB_J - 1) put_tagged(f + 2 * (F_JHI + i * SB_K + tk), c[i], tag);
      if (tk == 0) put_tagged(f + 2 * (F_KLO + i * SB_J + tj), c[i], tag);
      if (tk == SB_K - 1) put_tagged(f + 2 * (F_KHI + i * SB_J + tj), c[i], tag);
    }
    // halos of sweep s: the neighbours' faces, each value awaited by its tag
    const unsigned long long* fs = a.faces + (size_t)(s & 1) * nbs * (2 * SB_FACE);
    auto face = [&](int q, int off) { return fs + (size_t)q * (2 * SB_FACE) + 2 * off; };
    if (nb_ilo >= 0) sh[0][tj][tk] = get_tagged(face(nb_ilo, F_IHI + tj * SB_K + tk), tag);
    if (nb_ihi >= 0) sh[1][tj][tk] = get_tagged(face(nb_ihi, F_ILO + tj * SB_K + tk), tag);
    if (t < SB_I * SB_K) {   // rows j0-1 and j0+SB_J: (i, k) = (t / SB_K, t % SB_K)
      const int i = t / SB_K, k = t % SB_K;
      if (nb_jlo >= 0) sp[i][0][k + 1] = get_tagged(face(nb_jlo, F_JHI + i * SB_K + k), tag);
      if (nb_jhi >= 0) sp[i][SB_J + 1][k + 1] = get_tagged(face(nb_jhi, F_JLO + i * SB_K + k), tag);
    } else {                 // columns k0-1 and k0+SB_K: (i, j)
      const int u = t - SB_I * SB_K, i = u / SB_J, j = u % SB_J;
      if (nb_klo >= 0) sp[i][j + 1][0] = get_tagged(face(nb_klo, F_KHI + i * SB_J + j), tag);
      if (nb_khi >= 0) sp[i][j + 1][SB_K + 1] = get_tagged(face(nb_khi, F_KLO + i * SB_J + j), tag);
    }
    __syncthreads();
  }
  pdl_launch_dependents();
#pragma unroll
  for (int i = 0; i < SB_I; ++i) a.out[at(i0 + i, j0 + tj, k0 + tk)] = c[i];
}
