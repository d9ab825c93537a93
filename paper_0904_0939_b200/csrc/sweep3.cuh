// sweep3.cuh -- k_sweep3: THREE sweeps per HBM pass (temporal blocking, depth 3).
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace, after sweep2.cuh whose helpers it uses).
//
// Plain steps s, s+1, s+2 of the update in one z-march: HBM sees one read of
// psi and V and one write of psi for three site-updates (8 B per update
// instead of the two-sweep pass's 12).  Under the board's power cap the memory
// system is half of the dynamic power at full streaming (a device copy at
// 6.55 TB/s draws 683 W against 195 W idle; scripts/power_probe.py), so bytes
// per update are energy per update.
//
// Tile: TB rows x 64 columns of output.  Regions, with k0 / j0 the tile origin:
//   step 1 (psi')   rows j0-2 .. j0+TB+1, columns k0-2 .. k0+65
//   step 2 (psi'')  rows j0-1 .. j0+TB,   columns k0-1 .. k0+64
//   step 3 (output) rows j0   .. j0+TB-1, columns k0   .. k0+63
// Warps: TB+4 row warps (row j0-2+w, two sites per lane in columns k0..k0+63;
// steps 2 and 3 on the rows of their regions), ring warps for the four side
// columns k0-2, k0-1, k0+64, k0+65 (one site per lane; step 2 on k0-1 and
// k0+64), one TMA producer warp.  psi' and psi'' planes go through two rings
// of 4 shared-memory slots, both written in iteration g (slot g % 4) and read
// in iteration g+1; ONE per-slot mbarrier covers both: a warp arrives at the
// end of iteration g (psi'(p) and psi''(p-1) stored) and waits, before its
// steps 2 and 3 of iteration g+1, for everyone's iteration-g arrival.  A slot
// is rewritten at g+4, after its writer has waited on the iteration-(g+2)
// barrier, i.e. after every warp finished iteration g+2 (its reads were in
// g+1).  One barrier round per plane, like k_sweep2b (a first version with a
// round per ring issued at 37 %).
// A and C are formed once per site in step 1 and kept in registers for
// steps 2 and 3 (three rotating sets).  Per-site arithmetic is k_sweep's, so
// the result is bitwise three k_sweep launches (tests/test_gpu_core.py).
// Whole-lattice slabs only (two-buffer or single-buffer): a slab of a
// decomposed lattice would need three halo planes per face.
#pragma once

template <int TB>
struct T3Geo {
  static constexpr int RW = 72;                          // shared row width: columns k0-4 .. k0+67
  static constexpr int ROWW = TB + 4;                    // row warps
  static constexpr int RSITES = 4 * (TB + 4);            // ring sites
  static constexpr int RINGW = (RSITES + 31) / 32;       // ring warps
  static constexpr int CW = ROWW + RINGW;                // consumer warps
  static constexpr int THREADS = 32 * (CW + 1);
  static constexpr int PSI_H = TB + 6;                   // psi rows j0-3 .. j0+TB+2
  static constexpr int PSI_BYTES = RW * PSI_H * 8;
  static constexpr int PSI_STRIDE = (PSI_BYTES + 127) / 128 * 128;
  static constexpr int VH = TB + 4;                      // V rows j0-2 .. j0+TB+1
  static constexpr int V_BYTES = RW * VH * 8;
  static constexpr int V_STRIDE = (V_BYTES + 127) / 128 * 128;
  static constexpr int STAGE = PSI_STRIDE + V_STRIDE;
  static constexpr int R1 = RW * (TB + 4) * 8;           // psi' slot: rows j0-2 .. j0+TB+1
  static constexpr int R2 = RW * (TB + 2) * 8;           // psi'' slot: rows j0-1 .. j0+TB
};
template <int NST, int TB>
struct T3Cfg {
  using G = T3Geo<TB>;
  static constexpr int R1_OFF = NST * G::STAGE;
  static constexpr int R2_OFF = R1_OFF + 4 * G::R1;
  static constexpr int BAR_OFF = R2_OFF + 4 * G::R2;    // full[NST], empty[NST], ring[4]
  static constexpr int SMEM = BAR_OFF + (2 * NST + 4) * 8;
};

template <int TB>
__device__ __forceinline__ T2Item t3_item(const SweepArgs& a, int item) {
  int chunk = item / a.tiles;
  const int tile = item - chunk * a.tiles;
  const int tj = tile / a.tiles_k;
  const int tk = tile - tj * a.tiles_k;
  if (a.reverse) chunk = a.nchunks - 1 - chunk;
  T2Item r;
  r.idx = item;
  chunk_range(a, chunk, r.z0, r.z1);
  r.j = 1 + tj * TB;
  r.k = 1 + tk * TX;
  return r;
}

// the whole step-1 region (planes z0-2 .. z1+2, rows j0-2 .. j0+TB+1, columns
// k0-2 .. k0+65) inside the lattice: no site masks
template <int TB>
__device__ __forceinline__ bool t3_interior(const T2Item& I, int n) {
  return (I.j >= 3) & (I.j + TB + 1 <= n) & (I.k >= 3) & (I.k + TX + 1 <= n) & (I.z0 >= 3) &
         (I.z1 + 2 <= n);
}

// barrier cursor of the TMA stages + both rings, shared by all consumer roles
template <int S, int TB>
struct T3Sync {
  using G = T3Geo<TB>;
  using C = T3Cfg<S, TB>;
  uint32_t fb;       // full[0]
  uint32_t sb;       // stage slot byte offset (of the stage holding plane i+1 after next())
  uint32_t sbar;     // full barrier of that stage
  uint32_t sph;      // its phase parity
  __device__ __forceinline__ void next() {
    sb += G::STAGE;
    sbar += 8;
    if (sbar == fb + S * 8) {
      sb = 0;
      sbar = fb;
      sph ^= 1u;
    }
  }
};

// one row warp's work item.  S2 / S3: this row takes part in step 2 / 3;
// MASK: sites outside the lattice keep their input (Dirichlet zero)
template <int S, int TB, bool S2, bool S3, bool FASTC, bool MASK>
__device__ __forceinline__ void t3_rows_item(const SweepArgs& args, const T2Item& I, uint32_t sm0,
                                             int w, int lane, T3Sync<S, TB>& sy, uint32_t& g) {
  using G = T3Geo<TB>;
  using C = T3Cfg<S, TB>;
  constexpr uint32_t RW8 = G::RW * 8;
  const int n = args.n;
  const double h = args.h, c0 = args.c0;
  const int j = I.j - 2 + w;
  const int k = I.k + 2 * lane;
  const uint32_t col = (uint32_t)(2 * lane + 4) * 8;           // byte column of site k
  const uint32_t psi_row = (uint32_t)(w + 1) * RW8 + col;      // row j in the psi box
  const uint32_t v_row = G::PSI_STRIDE + (uint32_t)w * RW8 + col;
  const uint32_t r1_row = C::R1_OFF + (uint32_t)w * RW8 + col;
  const uint32_t r2_row = C::R2_OFF + (uint32_t)(w - 1) * RW8 + col;   // w >= 1 for S2
  const uint32_t r1bar = sm0 + C::BAR_OFF + 2 * S * 8;
  const bool in_j = (unsigned)(j - 1) < (unsigned)n;
  const bool in0 = in_j & (k <= n);
  const bool in1 = in_j & (k + 1 <= n);
  // output offset of plane z0, row j, column k (32-bit: fields < 2^32 elements)
  uint32_t doff = (uint32_t)((long long)(I.z0 - args.z_base) * args.plane_stride +
                             (long long)j * args.pitch + (k + COL_OFF));
  const uint32_t pstride = (uint32_t)args.plane_stride;
  // psi(z0-3), psi(z0-2): the first two stages
  double2 c[3], q[3], r[3], av[3], fv[3];
  mbar_wait_u(sy.sbar, sy.sph);
  c[0] = lds2_u(sm0 + sy.sb + psi_row);
  mbar_arrive_u(sy.sbar + S * 8);
  sy.next();
  mbar_wait_u(sy.sbar, sy.sph);
  c[1] = lds2_u(sm0 + sy.sb + psi_row);
  uint32_t cur_sb = sy.sb, cur_bar = sy.sbar;
  sy.next();
  q[0] = q[1] = q[2] = r[0] = r[1] = r[2] = av[0] = av[1] = av[2] = fv[0] = fv[1] = fv[2] =
      make_double2(0.0, 0.0);
  int p = I.z0 - 2;   // step-1 plane of this iteration
  const int pend = I.z1 + 3;
  // one iteration: step 1 on plane p, step 2 on p-1, step 3 on p-2.  PH = p mod 3
  // relative to the item start (register rotation); D2 / D3: steps 2 / 3 run.
  auto iter = [&](auto ph, auto d2, auto d3) {
    constexpr int P0 = decltype(ph)::value;          // slot of plane p
    constexpr int PM = (P0 + 2) % 3, PN = (P0 + 1) % 3;   // p-1 (and p-2 == p+1 mod 3), p+1
    constexpr bool DO2 = S2 && decltype(d2)::value;
    constexpr bool DO3 = S3 && decltype(d3)::value;
    // barriers probed early (test_wait), blocking waits only where a probe
    // failed: the barrier latency overlaps the shared loads and arithmetic
    const uint32_t sr = ((g - 1) & 3u);
    const uint32_t rph = ((g - 1) >> 2) & 1u;
    const bool okf = mbar_test_u(sy.sbar, sy.sph);
    const bool ok1 = mbar_test_u(r1bar + sr * 8, rph);
    // next plane's psi (own column) and this plane's neighbours
    mbar_wait_if(okf, sy.sbar, sy.sph);
    c[PN] = lds2_u(sm0 + sy.sb + psi_row);
    const uint32_t st = sm0 + cur_sb;
    const double2 jm = lds2_u(st + psi_row - RW8);
    const double2 jp = lds2_u(st + psi_row + RW8);
    const double km = lds1_u(st + psi_row - 8);
    const double kp = lds1_u(st + psi_row + 16);
    const double2 v = lds2_u(st + v_row);
    coef2<FASTC>(v, h, c0, av[P0].x, fv[P0].x, av[P0].y, fv[P0].y);
    const double2 cc = c[P0], cp = c[PM];
    const double u0 = upd(av[P0].x, fv[P0].x, cc.x, cp.x, c[PN].x, jm.x, jp.x, km, cc.y);
    const double u1 = upd(av[P0].y, fv[P0].y, cc.y, cp.y, c[PN].y, jm.y, jp.y, cc.x, kp);
    if (MASK) {
      const bool pin = (unsigned)(p - 1) < (unsigned)n;
      q[P0].x = (pin & in0) ? u0 : cc.x;
      q[P0].y = (pin & in1) ? u1 : cc.y;
    } else {
      q[P0] = make_double2(u0, u1);
    }
    const uint32_t s1 = (g & 3u);
    sts2_u(sm0 + r1_row + s1 * G::R1, q[P0]);
    mbar_arrive_u(cur_bar + S * 8);     // stage of plane p consumed
    cur_sb = sy.sb;
    cur_bar = sy.sbar;
    sy.next();
    // steps 2 and 3 read what every warp published in iteration g-1:
    // psi'(p-1) (ring 1) and psi''(p-2) (ring 2) -- one barrier round per plane
    mbar_wait_if(ok1, r1bar + sr * 8, rph);
    if (DO2) {
      const uint32_t rq = sm0 + r1_row + sr * G::R1;
      const double2 rjm = lds2_u(rq - RW8);
      const double2 rjp = lds2_u(rq + RW8);
      const double rkm = lds1_u(rq - 8);
      const double rkp = lds1_u(rq + 16);
      const double2 qc = q[PM];
      const double o0 = upd(av[PM].x, fv[PM].x, qc.x, q[PN].x, q[P0].x, rjm.x, rjp.x, rkm, qc.y);
      const double o1 = upd(av[PM].y, fv[PM].y, qc.y, q[PN].y, q[P0].y, rjm.y, rjp.y, qc.x, rkp);
      if (MASK) {
        const bool pin = (unsigned)(p - 2) < (unsigned)n;
        r[PM].x = (pin & in0) ? o0 : qc.x;
        r[PM].y = (pin & in1) ? o1 : qc.y;
      } else {
        r[PM] = make_double2(o0, o1);
      }
      sts2_u(sm0 + r2_row + s1 * G::R2, r[PM]);
    }
    // step 3 on plane p-2 from psi''(p-2) (published in iteration g-1)
    if (DO3) {
      const uint32_t rr = sm0 + r2_row + sr * G::R2;
      const double2 sjm = lds2_u(rr - RW8);
      const double2 sjp = lds2_u(rr + RW8);
      const double skm = lds1_u(rr - 8);
      const double skp = lds1_u(rr + 16);
      const double2 rc = r[PN];   // psi''(p-2): slot (p-2) mod 3 == (p+1) mod 3
      const double o0 = upd(av[PN].x, fv[PN].x, rc.x, r[P0].x, r[PM].x, sjm.x, sjp.x, skm, rc.y);
      const double o1 = upd(av[PN].y, fv[PN].y, rc.y, r[P0].y, r[PM].y, sjm.y, sjp.y, rc.x, skp);
      double* dst = args.out + doff;
      if (!MASK || ((unsigned)(p - 3) < (unsigned)n && in1)) {
        *reinterpret_cast<double2*>(dst) = make_double2(o0, o1);
      } else if ((unsigned)(p - 3) < (unsigned)n && in0) {
        *dst = o0;
      }
      doff += pstride;
    }
    mbar_arrive_u(r1bar + s1 * 8);      // psi'(p) and psi''(p-1) published
    ++g;
    ++p;
  };
  using F = std::false_type;
  using T = std::true_type;
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  // planes z0-2, z0-1: step 1 only; z0, z0+1: steps 1, 2; then all three
  // (an item has z1 - z0 + 5 >= 5 iterations).  Register slots rotate with p.
  iter(I1{}, F{}, F{});   // p = z0-2 (slot 1: c[0] = psi(z0-3), c[1] = psi(z0-2))
  iter(I2{}, F{}, F{});
  iter(I0{}, T{}, F{});
  iter(I1{}, T{}, F{});
  for (;;) {
    iter(I2{}, T{}, T{});
    if (p == pend) break;
    iter(I0{}, T{}, T{});
    if (p == pend) break;
    iter(I1{}, T{}, T{});
    if (p == pend) break;
  }
  mbar_arrive_u(cur_bar + S * 8);   // the stage of plane z1+3 (read as the last own-column plane)
}

// one ring warp's work item: lane site (column k0-2 | k0-1 | k0+64 | k0+65, row
// j0-2 .. j0+TB+1); step 2 on the k0-1 / k0+64 columns of rows j0-1 .. j0+TB
template <int S, int TB, bool FASTC, bool MASK>
__device__ __forceinline__ void t3_ring_item(const SweepArgs& args, const T2Item& I, uint32_t sm0,
                                             int idx, T3Sync<S, TB>& sy, uint32_t& g) {
  using G = T3Geo<TB>;
  using C = T3Cfg<S, TB>;
  constexpr uint32_t RW8 = G::RW * 8;
  const int n = args.n;
  const double h = args.h, c0 = args.c0;
  const bool active = idx < G::RSITES;
  // lanes interleave the four columns (lane & 3), so a half-warp touches 4
  // rows x 4 columns instead of 16 rows of one column (8-way bank conflicts
  // at the 576-byte row stride)
  const int csel = active ? idx & 3 : 0;
  const int rr0 = active ? idx >> 2 : 0;                 // row j0-2+rr0
  const int ccol = csel == 0 ? 2 : csel == 1 ? 3 : csel == 2 ? 68 : 69;   // shared column
  const int j = I.j - 2 + rr0;
  const int k = I.k - 4 + ccol;
  const bool do2 = active & (csel == 1 || csel == 2) & (rr0 >= 1) & (rr0 <= TB + 2);
  const uint32_t colb = (uint32_t)ccol * 8;
  const uint32_t psi_row = (uint32_t)(rr0 + 1) * RW8 + colb;
  const uint32_t v_row = G::PSI_STRIDE + (uint32_t)rr0 * RW8 + colb;
  const uint32_t r1_row = C::R1_OFF + (uint32_t)rr0 * RW8 + colb;
  const uint32_t r2_row = C::R2_OFF + (uint32_t)(rr0 > 0 ? rr0 - 1 : 0) * RW8 + colb;
  const uint32_t r1bar = sm0 + C::BAR_OFF + 2 * S * 8;
  const bool in_jk = active & ((unsigned)(j - 1) < (unsigned)n) & ((unsigned)(k - 1) < (unsigned)n);
  double c[3], q[3], av[3], fv[3];
  mbar_wait_u(sy.sbar, sy.sph);
  c[0] = lds1_u(sm0 + sy.sb + psi_row);
  mbar_arrive_u(sy.sbar + S * 8);
  sy.next();
  mbar_wait_u(sy.sbar, sy.sph);
  c[1] = lds1_u(sm0 + sy.sb + psi_row);
  uint32_t cur_sb = sy.sb, cur_bar = sy.sbar;
  sy.next();
  q[0] = q[1] = q[2] = av[0] = av[1] = av[2] = fv[0] = fv[1] = fv[2] = 0.0;
  int p = I.z0 - 2;
  const int pend = I.z1 + 3;
  auto iter = [&](auto ph, auto d2) {
    constexpr int P0 = decltype(ph)::value;
    constexpr int PM = (P0 + 2) % 3, PN = (P0 + 1) % 3;
    constexpr bool D2 = decltype(d2)::value;
    const uint32_t sr = ((g - 1) & 3u);
    const uint32_t rph = ((g - 1) >> 2) & 1u;
    const bool okf = mbar_test_u(sy.sbar, sy.sph);
    const bool ok1 = mbar_test_u(r1bar + sr * 8, rph);
    mbar_wait_if(okf, sy.sbar, sy.sph);
    c[PN] = lds1_u(sm0 + sy.sb + psi_row);
    const uint32_t st = sm0 + cur_sb;
    const double jm = lds1_u(st + psi_row - RW8);
    const double jp = lds1_u(st + psi_row + RW8);
    const double km = lds1_u(st + psi_row - 8);
    const double kp = lds1_u(st + psi_row + 8);
    const double v = lds1_u(st + v_row);
    coef1<FASTC>(v, h, c0, av[P0], fv[P0]);
    const double u = upd(av[P0], fv[P0], c[P0], c[PM], c[PN], jm, jp, km, kp);
    q[P0] = u;
    if (MASK) q[P0] = (((unsigned)(p - 1) < (unsigned)n) & in_jk) ? u : c[P0];
    const uint32_t s1 = (g & 3u);
    if (active) sts1_u(sm0 + r1_row + s1 * G::R1, q[P0]);
    mbar_arrive_u(cur_bar + S * 8);
    cur_sb = sy.sb;
    cur_bar = sy.sbar;
    sy.next();
    mbar_wait_if(ok1, r1bar + sr * 8, rph);
    if (D2 && do2) {
      const uint32_t rq = sm0 + r1_row + sr * G::R1;
      const double rjm = lds1_u(rq - RW8);
      const double rjp = lds1_u(rq + RW8);
      const double rkm = lds1_u(rq - 8);
      const double rkp = lds1_u(rq + 8);
      const double o = upd(av[PM], fv[PM], q[PM], q[PN], q[P0], rjm, rjp, rkm, rkp);
      double ov = o;
      if (MASK) ov = (((unsigned)(p - 2) < (unsigned)n) & in_jk) ? o : q[PM];
      sts1_u(sm0 + r2_row + s1 * G::R2, ov);
    }
    mbar_arrive_u(r1bar + s1 * 8);      // psi'(p) and psi''(p-1) published
    ++g;
    ++p;
  };
  using F = std::false_type;
  using T = std::true_type;
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  iter(I1{}, F{});
  iter(I2{}, F{});
  for (;;) {
    iter(I0{}, T{});
    if (p == pend) break;
    iter(I1{}, T{});
    if (p == pend) break;
    iter(I2{}, T{});
    if (p == pend) break;
  }
  mbar_arrive_u(cur_bar + S * 8);
}

template <int NST, int TB, bool FASTC>
__global__ void __launch_bounds__(T3Geo<TB>::THREADS, 1)
    k_sweep3(const __grid_constant__ CUtensorMap tm_psi, const __grid_constant__ CUtensorMap tm_v,
             const SweepArgs args) {
  using G = T3Geo<TB>;
  using C = T3Cfg<NST, TB>;
  constexpr int S = NST;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + S;
  uint64_t* r1 = empty + S;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::CW * 32);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&r1[i], G::CW * 32);
    fence_barrier_init();
  }
  __syncthreads();
  // both rings count iterations from 4: every consumer lane completes phase 0
  // of each slot once, so the first iterations' waits are already satisfied
  if (warp < G::CW) {
    for (int i = 0; i < 4; ++i) mbar_arrive(&r1[i]);
  }
  pdl_launch_dependents();
  pdl_wait();
  const int nitems = args.nitems;
  if (warp == G::CW) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_psi);
      tma_prefetch_desc(&tm_v);
      int it = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        const T2Item I = t3_item<TB>(args, item);
        const int kc = I.k + COL_OFF;
        for (int p = I.z0 - 3; p <= I.z1 + 3; ++p, ++it) {
          const int slot = it % S;
          if (it >= S) mbar_wait_sleep(&empty[slot], ((it / S) - 1) & 1);
          const bool hasv = (p >= I.z0 - 2) && (p <= I.z1 + 2);
          unsigned char* st = smem + slot * G::STAGE;
          mbar_arrive_expect_tx(&full[slot], G::PSI_BYTES + (hasv ? G::V_BYTES : 0));
          tma_load_3d(st, &tm_psi, kc - 4, I.j - 3, p + 1, &full[slot]);   // deep-halo map: plane + 1
          if (hasv) tma_load_3d(st + G::PSI_STRIDE, &tm_v, kc - 4, I.j - 2, p, &full[slot]);
        }
      }
    }
    return;
  }
  const uint32_t sm0 = smem_u32(smem);
  T3Sync<S, TB> sy;
  sy.fb = sm0 + C::BAR_OFF;
  sy.sb = 0;
  sy.sbar = sy.fb;
  sy.sph = 0;
  uint32_t g = 4;
  const int n = args.n;
  if (warp >= G::ROWW) {
    const int idx = (warp - G::ROWW) * 32 + lane;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      const T2Item I = t3_item<TB>(args, item);
      if (t3_interior<TB>(I, n)) t3_ring_item<S, TB, FASTC, false>(args, I, sm0, idx, sy, g);
      else t3_ring_item<S, TB, FASTC, true>(args, I, sm0, idx, sy, g);
    }
    return;
  }
  // row warps: the roles split at entry (straight-line loops per role)
  auto rows = [&](auto s2, auto s3) {
    constexpr bool R2 = decltype(s2)::value, R3 = decltype(s3)::value;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      const T2Item I = t3_item<TB>(args, item);
      if (t3_interior<TB>(I, n)) t3_rows_item<S, TB, R2, R3, FASTC, false>(args, I, sm0, warp, lane, sy, g);
      else t3_rows_item<S, TB, R2, R3, FASTC, true>(args, I, sm0, warp, lane, sy, g);
    }
  };
  if (warp == 0 || warp == TB + 3) rows(std::false_type{}, std::false_type{});
  else if (warp == 1 || warp == TB + 2) rows(std::true_type{}, std::false_type{});
  else rows(std::true_type{}, std::true_type{});
}
