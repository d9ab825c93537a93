// sweep2p.cuh -- k_sweep2p: the two-sweep pass with two tile rows per warp.
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace, after sweep2.cuh whose tile geometry, stage pipeline,
// psi' ring and barrier helpers it shares).
#pragma once

// Same work items, 16 x 64 tiles, TMA stages, 4-slot psi' ring and barriers
// as k_sweep2b; what changes is the warp-to-row map:
//   warp 0      the y-halo rows j0-1 and j0+16 (step 1 only)
//   warps 1..8  tile rows j0+2(w-1) and j0+2(w-1)+1 (steps 1 and 2)
//   warp 9      the ring columns k0-1 / k0+64 (k_sweep2b's ring warp)
//   warp 10     the TMA producer
// A lane holds 4 sites (2 rows x 2 columns).  The two rows of a tile warp are
// each other's j-neighbours, so step 1 takes psi of row a+1 / a from the
// centre registers and step 2 takes psi' of row a+1 / a from the registers
// of the previous plane instead of shared memory, and every per-plane cost
// that does not scale with the sites (barrier probes and arrivals, the stage
// cursor, ring and output addressing) is paid once per 4 sites.  Per-site
// arithmetic is k_sweep's: results are bitwise those of k_sweep2b.

struct T2PGeo {
  static constexpr int TB = 16;
  static constexpr int CW = 10;                 // consumer warps
  static constexpr int THREADS = 32 * (CW + 1);
};

// a lane's sites: row a (.a) and row b (.b), two columns each
struct D4 {
  double2 a, b;
};

// rows ja = I.j - 1 + ea and jb = I.j - 1 + eb inside the lattice, the
// columns k0 .. k0+63 too, and the item's step-1 planes: no site masks
__device__ __forceinline__ bool t2p_rows_interior(const T2Item& I, int ea, int eb, int n,
                                                  int x_off) {
  const int ja = I.j - 1 + ea, jb = I.j - 1 + eb;
  return (ja >= 1) & (ja <= n) & (jb >= 1) & (jb <= n) & (I.k + TX - 1 <= n) &
         t2b_z_interior(I, n, x_off);
}

// one work item of a row-pair warp.  TILE: rows a, b = a+1 are tile rows
// (step 2 stored); else the two y-halo rows (step 1 only, not adjacent).
template <int S, bool TILE, bool FASTC, bool MASK>
__device__ __forceinline__ void t2p_rows_item(const SweepArgs& args, const T2Item& I,
                                              uint32_t fb, uint32_t base, uint32_t boff, int ea,
                                              int eb, int lane, StageCursor<S>& nx, uint32_t& g) {
  using G = T2BGeo<16>;
  using C = T2BCfg<S, 16>;
  constexpr uint32_t RW = BOXW * 8;                    // one shared-memory row
  constexpr uint32_t VOFF = G::PSI_STRIDE - RW;        // V box starts one row lower
  constexpr uint32_t ROFF = C::RING_OFF - RW;          // ring holds E rows
  const int n = args.n;
  const double h = args.h, c0 = args.c0;
  const int ja = I.j - 1 + ea, jb = I.j - 1 + eb;
  const int k = I.k + 2 * lane;
  const bool ina = (unsigned)(ja - 1) < (unsigned)n, inb = (unsigned)(jb - 1) < (unsigned)n;
  const bool ina0 = ina & (k <= n), ina1 = ina & (k + 1 <= n);
  const bool inb0 = inb & (k <= n), inb1 = inb & (k + 1 <= n);
  const bool oka0 = (ja <= n) & (k <= n), oka1 = (ja <= n) & (k + 1 <= n);
  const bool okb0 = (jb <= n) & (k <= n), okb1 = (jb <= n) & (k + 1 <= n);
  // element offset of row a's output pair (row b: + pitch)
  uint32_t doff = (uint32_t)((long long)(I.z0 - 2 - args.z_base) * args.plane_stride + (long long)ja * args.pitch +
                             (k + COL_OFF));
  const uint32_t pstride = (uint32_t)args.plane_stride;
  const uint32_t pitch = (uint32_t)args.pitch;
  uint32_t rw = (g & 3u) * G::RING, rr = ((g - 1) & 3u) * G::RING;
  constexpr uint32_t RB_END = 4 * G::RING;
  mbar_wait_u(fb + nx.slot * 8, nx.ph);
  D4 c_a, c_b, c_c;
  {
    const uint32_t s0 = base + nx.slot * G::STAGE;
    c_a.a = lds2_u(s0);
    c_a.b = lds2_u(s0 + boff);
  }
  mbar_arrive_u(fb + (S + nx.slot) * 8);
  nx.next();
  mbar_wait_u(fb + nx.slot * 8, nx.ph);
  {
    const uint32_t s0 = base + nx.slot * G::STAGE;
    c_b.a = lds2_u(s0);
    c_b.b = lds2_u(s0 + boff);
  }
  int cur = nx.slot;
  nx.next();
  bool okf = mbar_test_u(fb + nx.slot * 8, nx.ph);
  const double2 z2 = make_double2(0.0, 0.0);
  D4 q0{z2, z2}, q1 = q0, q2 = q0, a0 = q0, a1 = q0, a2 = q0, f0 = q0, f1 = q0, f2 = q0;
  const int pend = I.z1 + 2;
  int p = I.z0 - 1;
  auto plane = [&](const D4& cp, const D4& cc, D4& cn, D4& qw, const D4& qm, const D4& qmm,
                   D4& aw, D4& fw, const D4& am, const D4& fm) {
    mbar_wait_if(okf, fb + nx.slot * 8, nx.ph);
    const uint32_t gp = g - 1;
    const uint32_t rbar = fb + (2 * S + (gp & 3u)) * 8, rph = (gp >> 2) & 1u;
    const bool okr = mbar_test_u(rbar, rph);
    const uint32_t sn = base + nx.slot * G::STAGE;
    cn.a = lds2_u(sn);
    cn.b = lds2_u(sn + boff);
    const uint32_t sc = base + cur * G::STAGE;
    const double2 jma = lds2_u(sc - RW);
    const double2 jpb = lds2_u(sc + boff + RW);
    double2 jpa, jmb;
    if (TILE) {
      jpa = cc.b;
      jmb = cc.a;
    } else {
      jpa = lds2_u(sc + RW);
      jmb = lds2_u(sc + boff - RW);
    }
    const double kma = lds1_u(sc - 8);
    const double kpa = lds1_u(sc + 16);
    const double kmb = lds1_u(sc + boff - 8);
    const double kpb = lds1_u(sc + boff + 16);
    const double2 va = lds2_u(sc + VOFF);
    const double2 vb = lds2_u(sc + boff + VOFF);
    coef2<FASTC>(va, h, c0, aw.a.x, fw.a.x, aw.a.y, fw.a.y);
    coef2<FASTC>(vb, h, c0, aw.b.x, fw.b.x, aw.b.y, fw.b.y);
    const double ua0 = upd(aw.a.x, fw.a.x, cc.a.x, cp.a.x, cn.a.x, jma.x, jpa.x, kma, cc.a.y);
    const double ua1 = upd(aw.a.y, fw.a.y, cc.a.y, cp.a.y, cn.a.y, jma.y, jpa.y, cc.a.x, kpa);
    const double ub0 = upd(aw.b.x, fw.b.x, cc.b.x, cp.b.x, cn.b.x, jmb.x, jpb.x, kmb, cc.b.y);
    const double ub1 = upd(aw.b.y, fw.b.y, cc.b.y, cp.b.y, cn.b.y, jmb.y, jpb.y, cc.b.x, kpb);
    if (MASK) {
      const bool pin = (unsigned)(args.x_off + p - 1) < (unsigned)n;   // global plane
      qw.a.x = (pin & ina0) ? ua0 : cc.a.x;
      qw.a.y = (pin & ina1) ? ua1 : cc.a.y;
      qw.b.x = (pin & inb0) ? ub0 : cc.b.x;
      qw.b.y = (pin & inb1) ? ub1 : cc.b.y;
    } else {
      qw.a = make_double2(ua0, ua1);
      qw.b = make_double2(ub0, ub1);
    }
    const uint32_t rq_w = base + ROFF + rw;
    sts2_u(rq_w, qw.a);
    sts2_u(rq_w + boff, qw.b);
    mbar_arrive_u(fb + (S + cur) * 8);
    mbar_arrive_u(fb + (2 * S + (g & 3u)) * 8);
    cur = nx.slot;
    nx.next();
    okf = mbar_test_u(fb + nx.slot * 8, nx.ph);
    mbar_wait_if(okr, rbar, rph);
    if (TILE && p > I.z0) {   // plane p-1 >= z0: an output plane of this item
      const uint32_t rq = base + ROFF + rr;
      const double2 rjma = lds2_u(rq - RW);
      const double2 rjpb = lds2_u(rq + boff + RW);
      const double rkma = lds1_u(rq - 8);
      const double rkpa = lds1_u(rq + 16);
      const double rkmb = lds1_u(rq + boff - 8);
      const double rkpb = lds1_u(rq + boff + 16);
      const double oa0 = upd(am.a.x, fm.a.x, qm.a.x, qmm.a.x, qw.a.x, rjma.x, qm.b.x, rkma, qm.a.y);
      const double oa1 = upd(am.a.y, fm.a.y, qm.a.y, qmm.a.y, qw.a.y, rjma.y, qm.b.y, qm.a.x, rkpa);
      const double ob0 = upd(am.b.x, fm.b.x, qm.b.x, qmm.b.x, qw.b.x, qm.a.x, rjpb.x, rkmb, qm.b.y);
      const double ob1 = upd(am.b.y, fm.b.y, qm.b.y, qmm.b.y, qw.b.y, qm.a.y, rjpb.y, qm.b.x, rkpb);
      double* dst = args.out + doff;
      if (!MASK || oka1) {
        *reinterpret_cast<double2*>(dst) = make_double2(oa0, oa1);
      } else if (oka0) {
        *dst = oa0;
      }
      if (!MASK || okb1) {
        *reinterpret_cast<double2*>(dst + pitch) = make_double2(ob0, ob1);
      } else if (okb0) {
        dst[pitch] = ob0;
      }
    }
    if (TILE) doff += pstride;
    rr = rw;
    rw = rw + G::RING == RB_END ? 0u : rw + G::RING;
    ++p;
    ++g;
  };
  for (;;) {
    plane(c_a, c_b, c_c, q0, q2, q1, a0, f0, a2, f2);
    if (p == pend) break;
    plane(c_b, c_c, c_a, q1, q0, q2, a1, f1, a0, f0);
    if (p == pend) break;
    plane(c_c, c_a, c_b, q2, q1, q0, a2, f2, a1, f1);
    if (p == pend) break;
  }
  mbar_arrive_u(fb + (S + cur) * 8);
  if (TILE && I.idx < args.sig_items) {
    // an edge item's planes are stored: make them visible, then count this
    // warp done (the exchange waits for the count on its own stream)
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(args.sig, 1ull);
  }
}

template <int S, bool TILE, bool FASTC>
__device__ __forceinline__ void t2p_rows(const SweepArgs& args, uint32_t sm0, int ea, int eb,
                                         int lane) {
  using C = T2BCfg<S, 16>;
  const uint32_t fb = sm0 + C::BAR_OFF;               // full[S], empty[S], rfull[4]
  const uint32_t base = sm0 + (uint32_t)(((ea + 1) * BOXW + 2 * lane + 2) * 8);
  const uint32_t boff = (uint32_t)((eb - ea) * BOXW * 8);
  StageCursor<S> nx;
  uint32_t g = 4;   // ring plane counter (runs across items; 0..3 are the pre-completed phases)
  t2b_for_items<16>(args, [&](const T2Item& I) {
    if (t2p_rows_interior(I, ea, eb, args.n, args.x_off))
      t2p_rows_item<S, TILE, FASTC, false>(args, I, fb, base, boff, ea, eb, lane, nx, g);
    else
      t2p_rows_item<S, TILE, FASTC, true>(args, I, fb, base, boff, ea, eb, lane, nx, g);
  });
}

template <int NST, bool FASTC>
__global__ void __launch_bounds__(T2PGeo::THREADS, 1)
    k_sweep2p(const __grid_constant__ CUtensorMap tm_psi, const __grid_constant__ CUtensorMap tm_v,
              const SweepArgs args) {
  using G = T2BGeo<16>;
  constexpr int RS = T2B_RS;
  using C = T2BCfg<NST, 16, RS>;
  constexpr int S = NST;
  constexpr int CW = T2PGeo::CW;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + S;
  uint64_t* rfull = empty + S;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW * 32);   // per-lane arrivals of the consumer warps
    }
    for (int r = 0; r < RS; ++r) mbar_init(&rfull[r], CW * 32);
    fence_barrier_init();
  }
  __syncthreads();
  if (warp < CW) {
    for (int r = 0; r < RS; ++r) mbar_arrive(&rfull[r]);   // phase 0 of every ring slot
  }
  pdl_launch_dependents();
  pdl_wait();
  if (warp == CW) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_psi);
      tma_prefetch_desc(&tm_v);
      int it = 0;
      t2b_for_items<16>(args, [&](const T2Item& I) {
        const int kc = I.k + COL_OFF;
        for (int p = I.z0 - 2; p <= I.z1 + 2; ++p, ++it) {
          const int slot = it % S;
          if (it >= S) mbar_wait_sleep(&empty[slot], ((it / S) - 1) & 1);
          const bool hasv = (p >= I.z0 - 1) && (p <= I.z1 + 1);
          unsigned char* st = smem + slot * G::STAGE;
          mbar_arrive_expect_tx(&full[slot], G::PSI_BYTES + (hasv ? G::V_BYTES : 0));
          tma_load_3d(st, &tm_psi, kc - 2, I.j - 2, p + 1, &full[slot]);   // deep-halo map: plane + 1
          if (hasv) tma_load_3d(st + G::PSI_STRIDE, &tm_v, kc - 2, I.j - 1, p, &full[slot]);
        }
      });
    }
    return;
  }
  const uint32_t sm0 = smem_u32(smem);
  if (warp == CW - 1) {
    t2b_ringw<S, 16, FASTC>(args, sm0, lane);
  } else if (warp == 0) {
    t2p_rows<S, false, FASTC>(args, sm0, 0, 17, lane);
  } else {
    t2p_rows<S, true, FASTC>(args, sm0, 2 * warp - 1, 2 * warp, lane);
  }
}
