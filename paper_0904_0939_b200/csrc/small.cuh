// small.cuh -- k_small2: a whole run of sweeps of a small lattice in ONE
// persistent cooperative launch (N <= 64, N % 16 == 0; BASELINE config 1 is 64^3).
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace, after reduce.cuh; the host engine launches it from run_loop).
//
// At N = 64 the whole lattice is 2 MB: one launch per sweep (or per two-sweep
// pass) is latency-bound -- prologue, pipeline fill and drain of a kernel
// whose 148 blocks each hold a few planes of a 4-tile plane.
// Here every block owns an 8 x 16 x 16 brick of the lattice for the whole run
// (128 bricks at 64^3, one block per SM, co-resident by cooperative launch):
//   * each thread's column of 8 sites along axis 0 and their A, C live in
//     registers (A, C formed once from V with the reference's coefficient
//     arithmetic), the brick with a TWO-deep halo in shared memory;
//   * per pair of sweeps the brick and its face ring are updated from the halo
//     (the reference's per-site order, upd()), then the block publishes its
//     faces two layers deep to a global face buffer and reads its neighbours'
//     faces and edge lines, every value carrying its sweep number as a tag
//     (data-carried synchronisation: no flag, no fence, no grid barrier; a
//     tagged 64-bit word is single-copy atomic);
//   * k_small2<_, true> also runs the run's norm and measurement steps inside
//     the launch (tagged all-gather of NORM brick partials; observables as
//     brick partials, combined after the launch by k_small_meas).
// Every site's value is bitwise k_sweep's between norm / measure steps.
#pragma once

constexpr int SB_I = 8, SB_J = 16, SB_K = 16;   // brick: planes x rows x columns
constexpr int SB_THREADS = SB_J * SB_K;          // one thread per (row, column): a column of SB_I sites

struct SmallArgs {
  const double* in;        // current field (device layout)
  double* out;             // result field (the other buffer)
  const double* v;         // potential
  unsigned long long* faces;   // [2 parities][bricks][SB2_FACE][2 words]: tagged face values
  unsigned long long base;     // tag of the sweep before this launch's first (monotonic)
  long long plane_stride;
  int n, pitch, steps;
  int nbi, nbj, nbk;       // bricks per axis
  double h, c0;
  // in-kernel checks (k_small2<_, true>): the run's norm / measure steps inside
  // the launch.  State g (global sweep count) is normalised when
  // norm_every > 0 && g % norm_every == 0 and measured (observables of the
  // state entering sweep g + 1) when g > 0 && g % measure_every == 0, at most
  // max_meas times -- run_loop's schedule (evolve.py:249-270).
  long long g0;            // global index of the state entering the launch
  long long norm_every, measure_every;
  int max_meas;
  int linear;              // PSG_RUN_LINEAR_NORM with norm_every == 1: pairs, one normalisation per pair
  const double* fac0;      // factor pending on the input field (&scal[S_ONE] or &scal[S_FACTOR])
  unsigned long long* nparts;  // [2 parities][bricks][SB_I][2 words]: tagged NORM brick partials
  double* mparts;          // [max_meas][3][n][nbj * nbk]: observables' brick partials
  double* scal;
  const int* bad;
  double a3, kin, a, center;
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

// ---------------------------------------------------------------------------
// k_small2: the same bricks with TWO-deep halos -- one face exchange per two
// sweeps (the exchange, ~2 us through L2, is what k_small's sweeps cost; its
// compute is 0.5 us).  Per pair: sweep A on the brick and its face ring (the
// sites one step outside the brick along one axis), sweep B on the brick from
// sweep A's values.  Sweep A at a face-ring site reads the halo two deep along
// its axis and the EDGE sites one step out along two axes, which belong to the
// 12 diagonal bricks; they are read from those bricks' published faces (an
// edge line lies in a face layer).  A run of odd length ends with one sweep
// from the one-deep halo.  Bitwise k_sweep's per-site arithmetic.
constexpr int SB2_FACE = 4 * SB_J * SB_K + 8 * SB_I * SB_K;   // two layers per face
constexpr int S2_E = SB_I + 4, S2_J = SB_J + 4, S2_K = SB_K + 4;   // S0 box (halo 2)
constexpr int SA_E = SB_I + 2, SA_J = SB_J + 2, SA_K = SB_K + 2;   // sweep-A box (halo 1)
constexpr int SB2_RING = 2 * SB_J * SB_K + 4 * SB_I * SB_K;       // face-ring sites
constexpr int SB2_SMEM = (S2_E * S2_J * S2_K + SA_E * SA_J * SA_K + 2 * SB2_RING) * 8;
// in-kernel checks: gathered NORM partials of every brick (N <= 64: at most 128
// bricks), plane sums, per-warp partials of the norm (8 planes) and of the
// observables (3 quantities x 8 planes), the factor
constexpr int SB_MAXB = 128;
constexpr int SB_WARPS = SB_THREADS / 32;
constexpr int SB2_CHK_DOUBLES =
    SB_MAXB * SB_I + 64 + SB_WARPS * SB_I + SB_WARPS * 3 * SB_I + 2 + SB_I * SB_J * SB_K;
constexpr int SB2_SMEM_CHK = SB2_SMEM + SB2_CHK_DOUBLES * 8;


// ---- in-kernel checks of k_small2<_, true>: out of line (called ~once per
// hundred sweeps; keeps the sweep loop's registers those of the plain kernel).
// Both read the brick's current state from S0 (site (i,j,k) of the brick at
// S0[((i+2)*S2_J + j+2)*S2_K + k+2]).
struct SmallChk {
  double* S0;
  double* NG;   // [bricks][SB_I] gathered NORM partials
  double* PS;   // [64] plane sums
  double* NR;   // [warps][SB_I]
  double* MR;   // [warps][3][SB_I]
  double* FS;   // [0] the factor
  double* VB;   // [SB_I][SB_J][SB_K] the brick's V
};

// observables of the current state (the brick + one-deep halo): the
// reference's energy_plane_sums / radius2_plane_sums terms per site
// (kernels.py:52-100); brick partials per plane (xor butterfly per warp, the
// warps in ascending order) to dst[q][plane][brick in plane]
__device__ __noinline__ void small_measure(const SmallChk& k, double* dst, int n, int nbjk, int bjk,
                                           int i0, int j0, int k0, double kin, double a, double center) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tk = t % SB_K, tj = t / SB_K;
  auto s0 = [&](int i, int j, int kk) { return k.S0[((i + 2) * S2_J + (j + 2)) * S2_K + (kk + 2)]; };
  const double dy = __dmul_rn(__dsub_rn((double)(j0 + tj), center), a);
  const double dz = __dmul_rn(__dsub_rn((double)(k0 + tk), center), a);
  const double dy2 = __dmul_rn(dy, dy), dz2 = __dmul_rn(dz, dz);
  // the brick's V, staged in shared memory at kernel start ([SB_I][SB_J][SB_K])
  double val[32];   // [q][i] slots of this lane, 24 used
#pragma unroll
  for (int i = 0; i < SB_I; ++i) {
    const double p = s0(i, tj, tk);
    double sl = __dadd_rn(s0(i - 1, tj, tk), s0(i + 1, tj, tk));
    sl = __dadd_rn(sl, s0(i, tj - 1, tk));
    sl = __dadd_rn(sl, s0(i, tj + 1, tk));
    sl = __dadd_rn(sl, s0(i, tj, tk - 1));
    sl = __dadd_rn(sl, s0(i, tj, tk + 1));
    sl = __dsub_rn(sl, __dmul_rn(6.0, p));
    const double hp = __dsub_rn(__dmul_rn(k.VB[(i * SB_J + tj) * SB_K + tk], p), __dmul_rn(kin, sl));
    const double dx = __dmul_rn(__dsub_rn((double)(i0 + i), center), a);
    const double rr = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), dy2), dz2);
    const double w = __dmul_rn(p, p);
    val[0 * SB_I + i] = __dmul_rn(p, hp);
    val[1 * SB_I + i] = w;
    val[2 * SB_I + i] = __dmul_rn(w, rr);
  }
#pragma unroll
  for (int e = 3 * SB_I; e < 32; ++e) val[e] = 0.0;
  // reduce-scatter over the warp (31 shuffles for the 24 sums): at the step
  // with offset o a lane keeps the half of its slots selected by bit o of its
  // lane index and adds its partner's copy of that half; lane l ends with the
  // warp sum of slot l (a fixed order: deterministic)
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int e = 0; e < o; ++e) {
      const double send = up ? val[e] : val[e + o];
      const double keep = up ? val[e + o] : val[e];
      val[e] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
  if (lane < 3 * SB_I) k.MR[warp * 3 * SB_I + lane] = val[0];   // slot lane = q * SB_I + i
  __syncthreads();
  if (t < 3 * SB_I) {
    double acc = k.MR[t];
    for (int w2 = 1; w2 < SB_WARPS; ++w2) acc = __dadd_rn(acc, k.MR[w2 * 3 * SB_I + t]);
    const int q = t / SB_I, i = t % SB_I;
    dst[((size_t)q * n + (i0 - 1 + i)) * nbjk + bjk] = acc;
  }
  __syncthreads();   // MR free again
}

// the normalisation factor of the current state: NORM brick partials per
// plane, a tagged all-gather of every brick's partials, plane sums over the
// bricks ((bj, bk) ascending), numpy's pairwise total, 1/sqrt(n2) with
// n2 = total * a^3 (SweepBuffers.renormalize, evolve.py:171-181) -- every
// block forms the same factor from the same values in the same order.  Block
// 0 writes the combine's scalars (k_norm_total).  Returns the factor.
__device__ __noinline__ double small_normalise(const SmallChk& k, unsigned long long* np, uint32_t tag,
                                               int b, int nbs, int n, int nbjk, double a3, double* scal,
                                               const int* bad) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int tk = t % SB_K, tj = t / SB_K;
#pragma unroll
  for (int i = 0; i < SB_I; ++i) {
    const double c = k.S0[((i + 2) * S2_J + (tj + 2)) * S2_K + (tk + 2)];
    const double q = warp_sum(__dmul_rn(c, c));
    if (lane == 0) k.NR[warp * SB_I + i] = q;
  }
  __syncthreads();
  if (t < SB_I) {
    double acc = k.NR[t];
    for (int w2 = 1; w2 < SB_WARPS; ++w2) acc = __dadd_rn(acc, k.NR[w2 * SB_I + t]);
    put_tagged(np + 2 * ((size_t)b * SB_I + t), acc, tag);
  }
  constexpr int PER = SB_MAXB * SB_I / SB_THREADS;   // values per thread (at most)
  const int cnt = nbs * SB_I;
  unsigned pend = 0;
#pragma unroll
  for (int r = 0; r < PER; ++r)
    if (t + r * SB_THREADS < cnt) pend |= 1u << r;
  unsigned spins = 0;
  while (pend) {
    unsigned long long w0[PER], w1[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r)
      if (pend & (1u << r))
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                     : "=l"(w0[r]), "=l"(w1[r]) : "l"(np + 2 * (size_t)(t + r * SB_THREADS)) : "memory");
#pragma unroll
    for (int r = 0; r < PER; ++r)
      if ((pend & (1u << r)) && (uint32_t)w0[r] == tag && (uint32_t)w1[r] == tag) {
        k.NG[t + r * SB_THREADS] =
            __longlong_as_double((long long)((w1[r] & 0xffffffff00000000ull) | (w0[r] >> 32)));
        pend &= ~(1u << r);
      }
    if (++spins > (1u << 30)) __trap();
  }
  __syncthreads();
  if (t < n) {   // plane t (0-based): brick row t / SB_I, local plane t % SB_I
    const double* src = k.NG + (size_t)(t / SB_I) * nbjk * SB_I + (t % SB_I);
    double acc = src[0];
    for (int q = 1; q < nbjk; ++q) acc = __dadd_rn(acc, src[(size_t)q * SB_I]);
    k.PS[t] = acc;
  }
  __syncthreads();
  if (t == 0) {
    const double n2 = __dmul_rn(__dadd_rn(0.0, pw_leaf(k.PS, n)), a3);
    double f = 1.0;
    int st = 0;
    if (n2 == 0.0)
      st = 3;
    else if (!finite_d(n2))
      st = 4;
    else
      f = __ddiv_rn(1.0, __dsqrt_rn(n2));
    k.FS[0] = f;
    if (b == 0) {   // the combine's scalars (k_norm_total, combine_scalars)
      scal[S_N2] = n2;
      scal[S_FACTOR] = f;
      double status = scal[S_STATUS];
      if (st && status == 0.0) status = (double)st;
      if (bad && __ldcg(bad) && status == 0.0) status = 4.0;
      scal[S_STATUS] = status;
    }
  }
  __syncthreads();
  const double f = k.FS[0];
  __syncthreads();   // FS free again
  return f;
}

template <bool FASTC, bool CHK>
__global__ void __launch_bounds__(SB_THREADS, 1) k_small2(const SmallArgs a) {
  extern __shared__ __align__(16) double sm2[];
  double* S0 = sm2;                                   // [S2_E][S2_J][S2_K], site (i,j,k) at (i+2, j+2, k+2)
  double* SA = S0 + S2_E * S2_J * S2_K;               // [SA_E][SA_J][SA_K], site at (i+1, j+1, k+1)
  double* RA = SA + SA_E * SA_J * SA_K;               // face-ring A coefficients [SB2_RING]
  double* RC = RA + SB2_RING;                         // face-ring C coefficients
  auto s0 = [&](int i, int j, int k) -> double& { return S0[((i + 2) * S2_J + (j + 2)) * S2_K + (k + 2)]; };
  auto sa = [&](int i, int j, int k) -> double& { return SA[((i + 1) * SA_J + (j + 1)) * SA_K + (k + 1)]; };
  const int b = blockIdx.x;
  const int bk = b % a.nbk;
  const int bj = (b / a.nbk) % a.nbj;
  const int bi = b / (a.nbk * a.nbj);
  const int t = threadIdx.x;
  const int tk = t % SB_K, tj = t / SB_K;
  const int i0 = 1 + bi * SB_I, j0 = 1 + bj * SB_J, k0 = 1 + bk * SB_K;
  const int n = a.n;
  const long long ps = a.plane_stride;
  auto at = [&](int i, int j, int k) { return (long long)i * ps + (long long)j * a.pitch + k + COL_OFF; };
  auto inlat = [&](int gi, int gj, int gk) {
    return ((unsigned)(gi - 1) < (unsigned)n) & ((unsigned)(gj - 1) < (unsigned)n) &
           ((unsigned)(gk - 1) < (unsigned)n);
  };
  pdl_wait();
  const double f0 = CHK ? *a.fac0 : 1.0;
  // check scratch (CHK): after the ring coefficients
  SmallChk ck;
  ck.S0 = sm2;
  ck.NG = sm2 + (S2_E * S2_J * S2_K + SA_E * SA_J * SA_K + 2 * SB2_RING);
  ck.PS = ck.NG + SB_MAXB * SB_I;
  ck.NR = ck.PS + 64;
  ck.MR = ck.NR + SB_WARPS * SB_I;
  ck.FS = ck.MR + SB_WARPS * 3 * SB_I;
  ck.VB = ck.FS + 2;
  // S0: the brick with a two-deep halo box from the input field (outside the
  // lattice: padding zeros, or beyond the allocation's planes: zero)
  for (int q = t; q < S2_E * S2_J * S2_K; q += SB_THREADS) {
    const int kk = q % S2_K, r = q / S2_K;
    const int jj = r % S2_J, ii = r / S2_J;
    const int gi = i0 - 2 + ii, gj = j0 - 2 + jj, gk = k0 - 2 + kk;
    const bool in_box = (gi >= 0) & (gi <= n + 1) & (gj >= 0) & (gj <= n + 1) & (gk >= 0) & (gk <= n + 1);
    const double x = in_box ? a.in[at(gi, gj, gk)] : 0.0;
    // a pending normalisation factor: round(psi * f) is the reference's stored psi *= f
    S0[q] = CHK ? __dmul_rn(x, f0) : x;
  }
  // face-ring site q of this thread's four (two i-face sites, one j-face, one k-face)
  // -> local coordinates; ring index layout: i-lo 0..255, i-hi 256.., j-lo 512, j-hi 640,
  // k-lo 768, k-hi 896
  int ri[4], rj[4], rk[4], rx[4];
  {
    ri[0] = -1; rj[0] = tj; rk[0] = tk; rx[0] = t;
    ri[1] = SB_I; rj[1] = tj; rk[1] = tk; rx[1] = 256 + t;
    const int u = t & 127, hi = t >> 7;
    ri[2] = u / SB_K; rj[2] = hi ? SB_J : -1; rk[2] = u % SB_K; rx[2] = 512 + 128 * hi + u;
    ri[3] = u / SB_J; rj[3] = u % SB_J; rk[3] = hi ? SB_K : -1; rx[3] = 768 + 128 * hi + u;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int gi = i0 + ri[q], gj = j0 + rj[q], gk = k0 + rk[q];
    double A = 0.0, C = 0.0;
    if (inlat(gi, gj, gk)) coef_pair(a.v[at(gi, gj, gk)], a.h, a.c0, A, C);
    RA[rx[q]] = A;
    RC[rx[q]] = C;
  }
  double A[SB_I], C[SB_I], c[SB_I];
#pragma unroll
  for (int i = 0; i < SB_I; ++i) {
    const double vi = a.v[at(i0 + i, j0 + tj, k0 + tk)];
    coef1<FASTC>(vi, a.h, a.c0, A[i], C[i]);
    if (CHK) ck.VB[(i * SB_J + tj) * SB_K + tk] = vi;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SB_I; ++i) c[i] = s0(i, tj, tk);
  bool rin[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) rin[q] = inlat(i0 + ri[q], j0 + rj[q], k0 + rk[q]);
  const int nbs = a.nbi * a.nbj * a.nbk;
  auto bid = [&](int di, int dj, int dk) {   // neighbour brick or -1
    const int xi = bi + di, xj = bj + dj, xk = bk + dk;
    if (xi < 0 || xi >= a.nbi || xj < 0 || xj >= a.nbj || xk < 0 || xk >= a.nbk) return -1;
    return (xi * a.nbj + xj) * a.nbk + xk;
  };
  // face record of a brick (two layers per face): i-lo layers (0,1) [2][J][K],
  // i-hi layers (I-2, I-1), j-lo (0,1) [2][I][K], j-hi, k-lo (0,1) [2][I][J], k-hi
  constexpr int F_ILO = 0, F_IHI = 2 * SB_J * SB_K, F_JLO = 4 * SB_J * SB_K;
  constexpr int F_JHI = F_JLO + 2 * SB_I * SB_K, F_KLO = F_JHI + 2 * SB_I * SB_K;
  constexpr int F_KHI = F_KLO + 2 * SB_I * SB_J;
  static_assert(SB_J == 16 && SB_K == 16 && SB_I == 8, "face publishing assumes 8 x 16 x 16 bricks");
  // countdowns instead of per-pair 64-bit modulos: dn sweeps to the next
  // normalised state, dm sweeps to the next measured one (0: the current)
  // (32-bit: a launch runs at most 2^30 sweeps, so a countdown clamped to
  // 2^30 + 2 never reaches 0 or 1 when the event lies beyond the launch)
  constexpr long long CLAMP = (1ll << 30) + 2;
  int dn = -1, dm = -1, me = 0, nev = 0;
  if constexpr (CHK) {
    if (a.norm_every > 0) {
      dn = (int)min(a.norm_every - a.g0 % a.norm_every, CLAMP);
      nev = (int)min(a.norm_every, CLAMP);
    }
    if (a.measure_every > 0) {
      const long long lo = a.g0 > 0 ? a.g0 : 1;
      dm = (int)min((lo + a.measure_every - 1) / a.measure_every * a.measure_every - a.g0, CLAMP);
      me = (int)min(a.measure_every, CLAMP);
    }
  }
  int s = 0, ex = 0, ne = 0, nm = 0;
  while (s < a.steps) {
    bool pair = a.steps - s >= 2;
    if constexpr (CHK) {
      if (dm == 0) {
        if (nm < a.max_meas) {
          small_measure(ck, a.mparts + (size_t)nm * 3 * n * (a.nbj * a.nbk), n, a.nbj * a.nbk,
                        bj * a.nbk + bk, i0, j0, k0, a.kin, a.a, a.center);
          ++nm;
        }
        dm = me;
      }
      // the state after one sweep is normalised or measured: a single sweep --
      // unless it is a linear pair (every state normalised: the pair's
      // normalisation subsumes its first sweep's, S(f psi) = f S(psi))
      if ((dn == 1 && !a.linear) || (dm == 1 && nm < a.max_meas)) pair = false;
    }
    if (pair) {
      // ---- sweep A: brick (registers) and face ring ----
      double av[SB_I];
#pragma unroll
      for (int i = 0; i < SB_I; ++i) {
        const double im = i == 0 ? s0(-1, tj, tk) : c[i - 1];
        const double ip = i == SB_I - 1 ? s0(SB_I, tj, tk) : c[i + 1];
        av[i] = upd(A[i], C[i], c[i], im, ip, s0(i, tj - 1, tk), s0(i, tj + 1, tk),
                    s0(i, tj, tk - 1), s0(i, tj, tk + 1));
        sa(i, tj, tk) = av[i];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = ri[q], j = rj[q], k = rk[q];
        const double cv = s0(i, j, k);
        const double u = upd(RA[rx[q]], RC[rx[q]], cv, s0(i - 1, j, k), s0(i + 1, j, k),
                             s0(i, j - 1, k), s0(i, j + 1, k), s0(i, j, k - 1), s0(i, j, k + 1));
        sa(i, j, k) = rin[q] ? u : cv;
      }
      __syncthreads();
      // ---- sweep B: the brick ----
#pragma unroll
      for (int i = 0; i < SB_I; ++i) {
        const double im = i == 0 ? sa(-1, tj, tk) : av[i - 1];
        const double ip = i == SB_I - 1 ? sa(SB_I, tj, tk) : av[i + 1];
        c[i] = upd(A[i], C[i], av[i], im, ip, sa(i, tj - 1, tk), sa(i, tj + 1, tk),
                   sa(i, tj, tk - 1), sa(i, tj, tk + 1));
      }
      s += 2;
    } else {
      // ---- one sweep from the one-deep halo (the last of an odd run) ----
      double nv[SB_I];
#pragma unroll
      for (int i = 0; i < SB_I; ++i) {
        const double im = i == 0 ? s0(-1, tj, tk) : c[i - 1];
        const double ip = i == SB_I - 1 ? s0(SB_I, tj, tk) : c[i + 1];
        nv[i] = upd(A[i], C[i], c[i], im, ip, s0(i, tj - 1, tk), s0(i, tj + 1, tk),
                    s0(i, tj, tk - 1), s0(i, tj, tk + 1));
      }
#pragma unroll
      for (int i = 0; i < SB_I; ++i) c[i] = nv[i];
      s += 1;
    }
    const uint32_t tag = (uint32_t)(a.base + (unsigned long long)s);
    if constexpr (CHK) {
      const int k = pair ? 2 : 1;
      dm -= k;
      dn -= k;
      if (nev > 0 && dn <= 0) {   // (< 0: a linear pair passed two normalised states)
        __syncthreads();   // every read of S0 / SA for this sweep is done
#pragma unroll
        for (int i = 0; i < SB_I; ++i) s0(i, tj, tk) = c[i];
        const double f = small_normalise(ck, a.nparts + (size_t)(ne & 1) * nbs * (2 * SB_I), tag, b, nbs, n,
                                         a.nbj * a.nbk, a.a3, a.scal, a.bad);
        ++ne;
#pragma unroll
        for (int i = 0; i < SB_I; ++i) c[i] = __dmul_rn(c[i], f);
        dn = nev;
      }
    }
    if (s >= a.steps) break;
    __syncthreads();   // every read of S0 / SA for this pair is done
#pragma unroll
    for (int i = 0; i < SB_I; ++i) s0(i, tj, tk) = c[i];
    // ---- publish the two-layer faces of the new state (parity by exchange:
    // a block rewrites a parity only after every neighbour published the
    // exchange in between, which it did after reading this one) ----
    const int par = ex & 1;
    ++ex;
    unsigned long long* f = a.faces + ((size_t)par * nbs + b) * (2 * SB2_FACE);
    put_tagged(f + 2 * (F_ILO + (0 * SB_J + tj) * SB_K + tk), c[0], tag);
    put_tagged(f + 2 * (F_ILO + (1 * SB_J + tj) * SB_K + tk), c[1], tag);
    put_tagged(f + 2 * (F_IHI + (0 * SB_J + tj) * SB_K + tk), c[SB_I - 2], tag);
    put_tagged(f + 2 * (F_IHI + (1 * SB_J + tj) * SB_K + tk), c[SB_I - 1], tag);
    // j / k faces (1024 values) from the new brick in S0, four per thread,
    // each warp storing 32 consecutive record slots: from the owners'
    // registers they were 8 scattered stores on 4 lanes of every warp (a
    // store-queue stall) or per-site divergent branches
    __syncthreads();   // the brick in S0
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = t + SB_THREADS * r;           // [kind j|k][side lo|hi][layer][i][x]
      const int side = (e >> 8) & 1, layer = (e >> 7) & 1, i = (e >> 4) & 7, x = e & 15;
      const int w = side ? SB_J - 2 + layer : layer;   // SB_J == SB_K
      const double val = r < 2 ? s0(i, w, x) : s0(i, x, w);
      const int off = (r < 2 ? (side ? F_JHI : F_JLO) : (side ? F_KHI : F_KLO)) + (layer * SB_I + i) * 16 + x;
      put_tagged(f + 2 * off, val, tag);
    }
    // ---- read the halo: faces two deep, the 12 edge lines one deep ----
    // every load of this thread is issued before any tag is checked (one L2
    // round trip for all of them), then only the values not yet tagged with
    // this pair's sweep are loaded again
    const unsigned long long* fs = a.faces + (size_t)par * nbs * (2 * SB2_FACE);
    auto rec = [&](int q, int off) { return fs + (size_t)q * (2 * SB2_FACE) + 2 * off; };
    // fixed slots (registers, no local memory): 0-3 i-faces, 4-5 j-faces,
    // 6-7 k-faces, 8 an edge value
    constexpr int MAXG = 9;
    const unsigned long long* src[MAXG];
    int dst[MAXG];
    unsigned pend = 0;
#pragma unroll
    for (int g2 = 0; g2 < MAXG; ++g2) {
      src[g2] = fs;
      dst[g2] = 0;
    }
    auto want = [&](auto slot, int q, int off, int i, int j, int k) {
      constexpr int G2 = decltype(slot)::value;
      src[G2] = rec(q, off);
      dst[G2] = ((i + 2) * S2_J + (j + 2)) * S2_K + (k + 2);
      pend |= 1u << G2;
    };
    using Z0 = std::integral_constant<int, 0>;
    using Z1 = std::integral_constant<int, 1>;
    using Z2 = std::integral_constant<int, 2>;
    using Z3 = std::integral_constant<int, 3>;
    using Z4 = std::integral_constant<int, 4>;
    using Z5 = std::integral_constant<int, 5>;
    using Z6 = std::integral_constant<int, 6>;
    using Z7 = std::integral_constant<int, 7>;
    using Z8 = std::integral_constant<int, 8>;
    {
      const int qlo = bid(-1, 0, 0), qhi = bid(1, 0, 0);
      if (qlo >= 0) {   // its layers I-2, I-1 -> my i = -2, -1
        want(Z0{}, qlo, F_IHI + (0 * SB_J + tj) * SB_K + tk, -2, tj, tk);
        want(Z1{}, qlo, F_IHI + (1 * SB_J + tj) * SB_K + tk, -1, tj, tk);
      }
      if (qhi >= 0) {   // its layers 0, 1 -> my i = I, I+1
        want(Z2{}, qhi, F_ILO + (0 * SB_J + tj) * SB_K + tk, SB_I, tj, tk);
        want(Z3{}, qhi, F_ILO + (1 * SB_J + tj) * SB_K + tk, SB_I + 1, tj, tk);
      }
    }
    {
      const int layer = t >> 7, u = t & 127, i = u / SB_K, k = u % SB_K;
      const int qlo = bid(0, -1, 0), qhi = bid(0, 1, 0);
      if (qlo >= 0) want(Z4{}, qlo, F_JHI + (layer * SB_I + i) * SB_K + k, i, layer - 2, k);
      if (qhi >= 0) want(Z5{}, qhi, F_JLO + (layer * SB_I + i) * SB_K + k, i, SB_J + layer, k);
      const int j = u % SB_J, ik = u / SB_J;
      const int plo = bid(0, 0, -1), phi = bid(0, 0, 1);
      if (plo >= 0) want(Z6{}, plo, F_KHI + (layer * SB_I + ik) * SB_J + j, ik, j, layer - 2);
      if (phi >= 0) want(Z7{}, phi, F_KLO + (layer * SB_I + ik) * SB_J + j, ik, j, SB_K + layer);
    }
    if (t < 4 * SB_K) {   // edge lines along k: (i, j) corners
      const int e = t / SB_K, k = t % SB_K;
      const int di = (e & 1) ? 1 : -1, dj = (e & 2) ? 1 : -1;
      const int q = bid(di, dj, 0);
      if (q >= 0)   // neighbour's site (I-1 | 0, J-1 | 0, k): in its i-face layer
        want(Z8{}, q, (di < 0 ? F_IHI + (1 * SB_J + (dj < 0 ? SB_J - 1 : 0)) * SB_K
                        : F_ILO + (0 * SB_J + (dj < 0 ? SB_J - 1 : 0)) * SB_K) + k,
             di < 0 ? -1 : SB_I, dj < 0 ? -1 : SB_J, k);
    } else if (t < 8 * SB_K) {   // along j: (i, k) corners
      const int u = t - 4 * SB_K, e = u / SB_J, j = u % SB_J;
      const int di = (e & 1) ? 1 : -1, dk = (e & 2) ? 1 : -1;
      const int q = bid(di, 0, dk);
      if (q >= 0)
        want(Z8{}, q, (di < 0 ? F_IHI + (1 * SB_J + j) * SB_K : F_ILO + (0 * SB_J + j) * SB_K) +
                    (dk < 0 ? SB_K - 1 : 0),
             di < 0 ? -1 : SB_I, j, dk < 0 ? -1 : SB_K);
    } else if (t < 8 * SB_K + 4 * SB_I) {   // along i: (j, k) corners
      const int u = t - 8 * SB_K, e = u / SB_I, i = u % SB_I;
      const int dj = (e & 1) ? 1 : -1, dk = (e & 2) ? 1 : -1;
      const int q = bid(0, dj, dk);
      if (q >= 0)   // neighbour's site (i, J-1 | 0, K-1 | 0): in its j-face layer
        want(Z8{}, q, dj < 0 ? F_JHI + (1 * SB_I + i) * SB_K + (dk < 0 ? SB_K - 1 : 0)
                       : F_JLO + (0 * SB_I + i) * SB_K + (dk < 0 ? SB_K - 1 : 0),
             i, dj < 0 ? -1 : SB_J, dk < 0 ? -1 : SB_K);
    }
    unsigned spins = 0;
    while (pend) {
      unsigned long long w0[MAXG], w1[MAXG];
#pragma unroll
      for (int g2 = 0; g2 < MAXG; ++g2)
        if (pend & (1u << g2))
          asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                       : "=l"(w0[g2]), "=l"(w1[g2]) : "l"(src[g2]) : "memory");
#pragma unroll
      for (int g2 = 0; g2 < MAXG; ++g2)
        if ((pend & (1u << g2)) && (uint32_t)w0[g2] == tag && (uint32_t)w1[g2] == tag) {
          S0[dst[g2]] = __longlong_as_double((long long)((w1[g2] & 0xffffffff00000000ull) | (w0[g2] >> 32)));
          pend &= ~(1u << g2);
        }
      if (++spins > (1u << 30)) __trap();
    }
    __syncthreads();
  }
  pdl_launch_dependents();
#pragma unroll
  for (int i = 0; i < SB_I; ++i) a.out[at(i0 + i, j0 + tj, k0 + tk)] = c[i];
}

// The checks of a k_small2<_, true> launch: per record, plane sums over the
// bricks ((bj, bk) ascending) of each observable, numpy's pairwise totals,
// the scalars and the history record exactly as k_reduce_small forms them
// (combine_scalars, in record order); the last record's plane sums also to
// plane_sums.  One block; warp w forms records w, w + 32, ...
constexpr int SMQ_WARPS = 32;
constexpr int SMALL_MEAS_MAX = 256;   // records per launch (do_small_chk's cap)
__global__ void __launch_bounds__(32 * SMQ_WARPS)
    k_small_meas(const double* __restrict__ mparts, int count, int n, int nbjk, double a3, double* scal,
                 double* hist, long long rec, double* plane_sums, const int* bad) {
  __shared__ double tot[SMALL_MEAS_MAX][NQ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int m = warp; m < count; m += SMQ_WARPS) {
    double* hr = hist + (size_t)m * rec;
    for (int e = lane; e < 3 * n; e += 32) {
      const double* src = mparts + ((size_t)m * 3 * n + e) * nbjk;
      double acc = src[0];
      for (int q = 1; q < nbjk; ++q) acc = __dadd_rn(acc, src[q]);
      hr[2 + e] = acc;
    }
    __syncwarp();
    if (lane < 3) tot[m][lane] = __dadd_rn(0.0, pw_leaf(hr + 2 + lane * n, n));
    if (lane == 3) tot[m][3] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int m = 0; m < count; ++m) combine_scalars(tot[m], 7u, a3, scal, hist + (size_t)m * rec, bad);
  if (count > 0)
    for (int e = threadIdx.x; e < 3 * n; e += blockDim.x) plane_sums[e] = hist[(size_t)(count - 1) * rec + 2 + e];
}
