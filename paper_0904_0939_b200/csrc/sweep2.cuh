// sweep2.cuh -- k_sweep2b: two sweeps per HBM pass (temporal blocking).
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace; the host engine instantiates the templates).
#pragma once
#include <type_traits>

// ------------------------------------------------------------------
// two sweeps per pass (temporal blocking, k_sweep2b): plain steps s, s+1 of
// the update in one march over z, so HBM sees one read of psi and V and one
// write of psi for two site-updates.  Step 1 runs on the tile plus a one-site
// ring (tile rows +-1 and the columns either side) into a shared-memory ring
// of psi' planes; step 2 updates the tile from it one plane behind, with A and
// C formed once per site in step 1 and kept in registers.  Per-site
// arithmetic is k_sweep's: results are bitwise those of two k_sweep launches.
// The kernel is issue-bound rather than DRAM-bound, so the code is written
// for instruction count: warp roles are split at block entry into straight-
// line loops, the plane loop is unrolled by three so the centre / psi' / A / C
// registers rotate by renaming, shared memory is addressed by 32-bit offsets
// with immediates and the output pointer advances by one plane stride.
// ------------------------------------------------------------------
// one site of the update from explicit neighbours, the reference's order
// (kernels.py:33-37): left-to-right sum of the six neighbours, minus 6 psi,
// A psi + C s
__device__ __forceinline__ double upd(double A, double C, double c, double im, double ip, double jm,
                                      double jp, double km, double kp) {
  double s = __dadd_rn(im, ip);
  s = __dadd_rn(s, jm);
  s = __dadd_rn(s, jp);
  s = __dadd_rn(s, km);
  s = __dadd_rn(s, kp);
  s = __dsub_rn(s, __dmul_rn(6.0, c));
  return __dadd_rn(__dmul_rn(A, c), __dmul_rn(C, s));
}

__device__ __forceinline__ double2 lds2_u(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double lds1_u(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts2_u(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void sts1_u(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ bool mbar_try_u(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// non-blocking probe (test_wait): issued well before its result is needed,
// so the ~150-cycle barrier latency overlaps other work instead of sitting
// between the wait and the shared loads it guards
__device__ __forceinline__ bool mbar_test_u(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// wait for a phase unless a probe already saw it complete: one asm block
// (the retry loop and its watchdog inside), so the compiler emits no
// reconvergence region or call around it
__device__ __forceinline__ void mbar_wait_if(bool done, uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1, P2;\n\t.reg .u32 C;\n\t"
      "setp.ne.u32 P1, %0, 0;\n\t"
      "@P1 bra DONE;\n\t"
      "mov.u32 C, 0;\n"
      "WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P2, [%1], %2;\n\t"
      "@P2 bra DONE;\n\t"
      "add.u32 C, C, 1;\n\t"
      "setp.gt.u32 P1, C, 16777216;\n\t"
      "@P1 trap;\n\t"
      "bra WAIT;\n"
      "DONE:\n}"
      :
      : "r"((uint32_t)done), "r"(bar), "r"(parity)
      : "memory");
}
// the retry loop (with the watchdog) out of line: the hot path is one
// try_wait and a branch
__device__ __noinline__ void mbar_wait_slow(uint32_t bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try_u(bar, parity)) {
    if (++spins > (1u << 24)) __trap();
  }
}
__device__ __forceinline__ void mbar_wait_u(uint32_t bar, uint32_t parity) {
  if (!mbar_try_u(bar, parity)) mbar_wait_slow(bar, parity);
}
__device__ __forceinline__ void mbar_arrive_u(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}


// pipeline cursor over the TMA stages (consumer side)
template <int S>
struct StageCursor {
  int slot = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++slot == S) {
      slot = 0;
      ph ^= 1u;
    }
  }
};

// consumer cursor over the TMA stages that rotates the lane's shared-memory
// address in the stage and the stage's full barrier by adds (no slot
// multiplies in the plane loop); persists across work items
template <int S, uint32_t STAGE>
struct StageRot {
  uint32_t addr, bar, ph;
  __device__ __forceinline__ StageRot(uint32_t base, uint32_t fb) : addr(base), bar(fb), ph(0) {}
  __device__ __forceinline__ void next(uint32_t base, uint32_t fb) {
    addr += STAGE;
    bar += 8;
    if (bar == fb + S * 8) {
      addr = base;
      bar = fb;
      ph ^= 1u;
    }
  }
};

// psi' ring slots of plane g (write) and g-1 (read): byte offsets, rfull
// barriers and the read phase parity, rotating mod 4 inside an item
template <uint32_t RING>
struct RingRot {
  uint32_t rw, rr, bw, br, rph;
  __device__ __forceinline__ RingRot(uint32_t g, uint32_t rf0) {
    rw = (g & 3u) * RING;
    rr = ((g - 1) & 3u) * RING;
    bw = rf0 + (g & 3u) * 8;
    br = rf0 + ((g - 1) & 3u) * 8;
    rph = ((g - 1) >> 2) & 1u;
  }
  __device__ __forceinline__ void next(uint32_t rf0) {
    rr = rw;
    br = bw;
    const bool wrap = rw == 3 * RING;
    rw = wrap ? 0u : rw + RING;
    bw = wrap ? rf0 : bw + 8;
    rph ^= br == rf0 ? 1u : 0u;   // plane g-1 starts a new lap of the 4 slots
  }
};

struct T2Item {
  int z0, z1, j, k, idx;
};

// Tile of TB rows (8 or 16) x 64 columns.  Consumer warp w < TB+2 owns E row
// w (psi' rows j0-1 .. j0+TB; columns k0+2l, k0+2l+1); warps 1..TB (STEP2)
// also update their two tile sites one plane behind; warp TB+2 computes the
// ring columns k0-1 / k0+64 of rows j0 .. j0+TB-1 (lane l < 2 TB: one site).
// The psi' planes go through a ring of 4 slots: warp w publishes plane g with
// an arrive on rfull[g % 4] and, before step 2 of plane g-1, waits for
// rfull[(g-1) % 4], so warps drift by up to one plane instead of meeting at a
// block barrier.  Slot g % 4 is rewritten at g+4, after the writer has seen
// rfull(g+2), i.e. after every warp finished the step 2 that read plane g.
constexpr int T2B_RS = 4;
template <int TB>
struct T2BGeo {
  static constexpr int CW = TB + 3;                     // consumer warps
  static constexpr int THREADS = 32 * (CW + 1);
  static constexpr int MINB = TB <= 8 ? 2 : 1;
  static constexpr int PSI_H = TB + 4;                  // psi rows j0-2 .. j0+TB+1
  static constexpr int PSI_BYTES = BOXW * PSI_H * 8;
  static constexpr int PSI_STRIDE = (PSI_BYTES + 127) / 128 * 128;
  static constexpr int VH = TB + 2;                     // V rows j0-1 .. j0+TB
  static constexpr int V_BYTES = BOXW * VH * 8;
  static constexpr int V_STRIDE = (V_BYTES + 127) / 128 * 128;
  static constexpr int STAGE = PSI_STRIDE + V_STRIDE;
  static constexpr int RING = BOXW * VH * 8;            // bytes per psi' plane
};
template <int NST, int TB, int RS = T2B_RS>
struct T2BCfg {
  using G = T2BGeo<TB>;
  static constexpr int RING_OFF = NST * G::STAGE;
  static constexpr int BAR_OFF = RING_OFF + RS * G::RING;
  static constexpr int SMEM = BAR_OFF + (2 * NST + RS) * 8;
};

template <int TB>
__device__ __forceinline__ T2Item t2b_item(const SweepArgs& a, int item) {
  int chunk = item / a.tiles;
  const int tile = item - chunk * a.tiles;
  const int tj = tile / a.tiles_k;
  const int tk = tile - tj * a.tiles_k;
  T2Item r;
  r.idx = item;
  if (a.corder > 0) {
    // edges first: 0, nch-1 (, nch-2), then 1, 2, ...
    const int nch = a.nchunks;
    if (chunk == 1) chunk = nch - 1;
    else if (chunk == 2 && a.corder == 3) chunk = nch - 2;
    else if (chunk > 0) chunk = chunk - (a.corder - 1);
  } else if (a.reverse) {
    chunk = a.nchunks - 1 - chunk;
  }
  chunk_range(a, chunk, r.z0, r.z1);
  r.j = 1 + tj * TB;
  r.k = 1 + tk * TX;
  return r;
}

// The items of this block, in order.  Chunk mode: items blockIdx.x,
// blockIdx.x + gridDim.x, ... of the chunk-major list.  Segment mode
// (args.seg): block b owns the range [b T / G, (b+1) T / G) of the sequence
// of T = tiles x planes (tile, plane) pairs, tiles row-band major, split at
// tile boundaries.  With G a multiple of the tile rows, the block holding
// (tile, z) and the one holding its j-neighbour (tile +- tiles_k, z) are
// exactly G / tiles_j blocks apart and reach z at the same time, so the
// psi halo rows they share are read once from DRAM; every block marches
// about T / G planes with at most two z-halo restarts.
template <int TB, typename F>
__device__ __forceinline__ void t2b_for_items(const SweepArgs& a, F&& f) {
  // two loops (the body is inlined in each; only one runs per launch): a
  // shared loop with the mode test per item measured 3 % slower at 128^3
  if (!a.seg) {
    for (int item = blockIdx.x; item < a.nitems; item += gridDim.x) f(t2b_item<TB>(a, item));
    return;
  }
  const int np = a.z_hi - a.z_lo + 1;
  const long long total = (long long)a.tiles * np;
  long long pos = total * blockIdx.x / gridDim.x;
  const long long end = total * (blockIdx.x + 1) / gridDim.x;
  while (pos < end) {
    const int tile = (int)(pos / np);
    const int zz = (int)(pos - (long long)tile * np);
    const int len = (int)min((long long)(np - zz), end - pos);
    const int tj = tile / a.tiles_k;
    T2Item r;
    r.idx = 0x7fffffff;   // no signalled items in segment mode
    r.z0 = a.z_lo + zz;
    r.z1 = r.z0 + len - 1;
    r.j = 1 + tj * TB;
    r.k = 1 + (tile - tj * a.tiles_k) * TX;
    f(r);
    pos += len;
  }
}

// a work item whose step-1 region (tile rows j0-1 .. j0+TB, columns k0-1 ..
// k0+64, global planes x_off+z0-1 .. x_off+z1+1) lies inside the lattice
// needs no site masks
template <int TB>
__device__ __forceinline__ bool t2b_interior(const T2Item& I, int n, int x_off) {
  return (I.j >= 2) & (I.j + TB <= n) & (I.k >= 2) & (I.k + TX <= n) & (x_off + I.z0 >= 2) &
         (x_off + I.z1 < n);
}
// per warp role: E row j = I.j - 1 + w (columns k0 .. k0+63) and the ring
// columns k0-1, k0+64 of rows j0 .. j0+TB-1.  Tile rows never leave the
// lattice when N is a multiple of TB (nor columns when it is one of 64), so
// the tile-row warps run masked only on the first and last z-chunks.
__device__ __forceinline__ bool t2b_z_interior(const T2Item& I, int n, int x_off) {
  return (x_off + I.z0 >= 2) & (x_off + I.z1 < n);
}
__device__ __forceinline__ bool t2b_row_interior(const T2Item& I, int w, int n, int x_off) {
  const int j = I.j - 1 + w;
  return (j >= 1) & (j <= n) & (I.k + TX - 1 <= n) & t2b_z_interior(I, n, x_off);
}
template <int TB>
__device__ __forceinline__ bool t2b_ring_interior(const T2Item& I, int n, int x_off) {
  return (I.k >= 2) & (I.k + TX <= n) & (I.j + TB - 1 <= n) & t2b_z_interior(I, n, x_off);
}


// one work item of an E-row warp (MASK: item touches the lattice boundary;
// PEER: the slab's edge output planes are also stored into the neighbour
// slabs' halo planes, peer memory over NVLink -- the fused halo exchange)
// NRM (linear renormalisation pairs): the output is scaled by the pending
// factor of the input (fnorm; by linearity S(f psi) = f S(psi) up to rounding)
// and every step-2 lane accumulates the squares of its outputs over the whole
// launch (qacc, in a fixed order); one xor butterfly per warp at the end
// writes args.part[nslot + block * TB + warp - 1] for k_norm_total.  No
// per-plane sums: a whole-lattice slab needs only the total (per-plane
// butterflies cost +31 % instructions, measured).
template <int S, int TB, bool STEP2, bool FASTC, bool MASK, bool PEER = false, bool NRM = false,
          bool MS = false>
__device__ __forceinline__ void t2b_rows_item(const SweepArgs& args, const T2Item& I,
                                              uint32_t fb, uint32_t base, int w, int lane,
                                              StageRot<S, T2BGeo<TB>::STAGE>& nx, uint32_t& g,
                                              double fnorm = 1.0, double* qacc = nullptr,
                                              bool peer_edge = false) {
  using G = T2BGeo<TB>;
  using C = T2BCfg<S, TB>;
  constexpr uint32_t VOFF = G::PSI_STRIDE - BOXW * 8;  // V box starts one row lower
  constexpr uint32_t ROFF = C::RING_OFF - BOXW * 8;    // ring holds E rows
  const uint32_t rf0 = fb + 2 * S * 8;                 // rfull[0]
  const int n = args.n;
  const double h = args.h, c0 = args.c0;
  const int j = I.j - 1 + w;
  const int k = I.k + 2 * lane;
  const bool in_j = (unsigned)(j - 1) < (unsigned)n;
  const bool in0 = in_j & (k <= n);
  const bool in1 = in_j & (k + 1 <= n);
  const bool ok0 = (j <= n) & (k <= n);
  const bool ok1 = (j <= n) & (k + 1 <= n);
  // element offset of this lane's output pair (fields < 2^32 elements, checked
  // on the host): one 32-bit add per plane instead of 64-bit pointer math
  uint32_t doff = (uint32_t)((long long)(I.z0 - 2 - args.z_base) * args.plane_stride + (long long)j * args.pitch +
                             (k + COL_OFF));
  const uint32_t pstride = (uint32_t)args.plane_stride;
  RingRot<G::RING> rg(g, rf0);
  mbar_wait_u(nx.bar, nx.ph);
  double2 c_a = lds2_u(nx.addr);
  mbar_arrive_u(nx.bar + S * 8);   // every lane arrives on empty (count 32 per warp)
  nx.next(base, fb);
  mbar_wait_u(nx.bar, nx.ph);
  double2 c_b = lds2_u(nx.addr);
  uint32_t cur = nx.addr, cur_bar = nx.bar;
  nx.next(base, fb);
  bool okf = mbar_test_u(nx.bar, nx.ph);   // stage of the first loop plane
  double2 c_c;
  double2 q0 = make_double2(0.0, 0.0), q1 = q0, q2 = q0;
  double2 a0 = q0, a1 = q0, a2 = q0, f0 = q0, f1 = q0, f2 = q0;
  const int pend = I.z1 + 2;
  int p = I.z0 - 1;
  // DO2: step 2 runs on this plane (false for an item's first two planes,
  // which the loop below peels, so the steady loop carries no per-plane test)
  auto plane = [&](const double2& cp, const double2& cc, double2& cn, double2& qw,
                   const double2& qm, const double2& qmm, double2& aw, double2& fw,
                   const double2& am, const double2& fm, auto do2) {
    mbar_wait_if(okf, nx.bar, nx.ph);   // probed one plane earlier
    // all warps' psi' of plane g-1, needed by step 2 below: probe now (ahead
    // of the shared loads, which the compiler keeps in order)
    const bool okr = mbar_test_u(rg.br, rg.rph);
    cn = lds2_u(nx.addr);
    const uint32_t sc = cur;
    const double2 jm = lds2_u(sc - BOXW * 8);
    const double2 jp = lds2_u(sc + BOXW * 8);
    const double km = lds1_u(sc - 8);
    const double kp = lds1_u(sc + 16);
    const double2 v = lds2_u(sc + VOFF);
    coef2<FASTC>(v, h, c0, aw.x, fw.x, aw.y, fw.y);
    const double u0 = upd(aw.x, fw.x, cc.x, cp.x, cn.x, jm.x, jp.x, km, cc.y);
    const double u1 = upd(aw.y, fw.y, cc.y, cp.y, cn.y, jm.y, jp.y, cc.x, kp);
    if (MASK) {
      const bool pin = (unsigned)(args.x_off + p - 1) < (unsigned)n;   // global plane
      qw.x = (pin & in0) ? u0 : cc.x;
      qw.y = (pin & in1) ? u1 : cc.y;
    } else {
      qw = make_double2(u0, u1);
    }
    if constexpr (MS && STEP2) {
      if (p >= I.z0 && p <= I.z1) {   // this item's own planes (block-uniform)
        // observables of the pass's input state on this lane's two sites: the
        // reference's energy_plane_sums / radius2_plane_sums terms
        // (kernels.py:52-100) from step 1's operands; the input carries the
        // pending factor f, applied by linearity: sums x f^2
        double s0 = __dadd_rn(cp.x, cn.x);
        s0 = __dadd_rn(s0, jm.x);
        s0 = __dadd_rn(s0, jp.x);
        s0 = __dadd_rn(s0, km);
        s0 = __dadd_rn(s0, cc.y);
        s0 = __dsub_rn(s0, __dmul_rn(6.0, cc.x));
        double s1 = __dadd_rn(cp.y, cn.y);
        s1 = __dadd_rn(s1, jm.y);
        s1 = __dadd_rn(s1, jp.y);
        s1 = __dadd_rn(s1, cc.x);
        s1 = __dadd_rn(s1, kp);
        s1 = __dsub_rn(s1, __dmul_rn(6.0, cc.y));
        const double h0 = __dsub_rn(__dmul_rn(v.x, cc.x), __dmul_rn(args.kin, s0));
        const double h1 = __dsub_rn(__dmul_rn(v.y, cc.y), __dmul_rn(args.kin, s1));
        const double dx = __dmul_rn(__dsub_rn((double)(args.x_off + p), args.center), args.a);
        const double dy = __dmul_rn(__dsub_rn((double)j, args.center), args.a);
        const double dza = __dmul_rn(__dsub_rn((double)k, args.center), args.a);
        const double dzb = __dmul_rn(__dsub_rn((double)(k + 1), args.center), args.a);
        const double dxy = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
        const double w0 = __dmul_rn(cc.x, cc.x), w1 = __dmul_rn(cc.y, cc.y);
        double r_num = __dadd_rn(ok0 ? __dmul_rn(cc.x, h0) : 0.0, ok1 ? __dmul_rn(cc.y, h1) : 0.0);
        double r_den = __dadd_rn(ok0 ? w0 : 0.0, ok1 ? w1 : 0.0);
        double r_r2 = __dadd_rn(ok0 ? __dmul_rn(w0, __dadd_rn(dxy, __dmul_rn(dza, dza))) : 0.0,
                                ok1 ? __dmul_rn(w1, __dadd_rn(dxy, __dmul_rn(dzb, dzb))) : 0.0);
        r_num = warp_sum(r_num);
        r_den = warp_sum(r_den);
        r_r2 = warp_sum(r_r2);
        if (lane == 0) {   // [q][plane][tile row]: one slot per (tile, row) of the plane
          const long long tx = (long long)args.tiles * TB;
          const long long slot = (long long)p * tx +
                                 (long long)((I.j - 1) / TB * args.tiles_k + (I.k - 1) / TX) * TB + (w - 1);
          const long long qs = (long long)args.planes * tx;
          const double f2 = __dmul_rn(fnorm, fnorm);
          args.part[slot] = __dmul_rn(r_num, f2);
          args.part[qs + slot] = __dmul_rn(r_den, f2);
          args.part[2 * qs + slot] = __dmul_rn(r_r2, f2);
        }
      }
    }
    sts2_u(base + ROFF + rg.rw, qw);
    mbar_arrive_u(cur_bar + S * 8);
    mbar_arrive_u(rg.bw);
    cur = nx.addr;
    cur_bar = nx.bar;
    nx.next(base, fb);
    okf = mbar_test_u(nx.bar, nx.ph);   // the next plane's stage
    // (the kernel's first plane waits on a pre-completed phase; no item
    // stores or computes step 2 in its first two planes)
    mbar_wait_if(okr, rg.br, rg.rph);
    if (STEP2 && decltype(do2)::value) {   // plane p-1 >= z0: an output plane of this item
      const uint32_t rq = base + ROFF + rg.rr;
      const double2 rjm = lds2_u(rq - BOXW * 8);
      const double2 rjp = lds2_u(rq + BOXW * 8);
      const double rkm = lds1_u(rq - 8);
      const double rkp = lds1_u(rq + 16);
      double o0 = upd(am.x, fm.x, qm.x, qmm.x, qw.x, rjm.x, rjp.x, rkm, qm.y);
      double o1 = upd(am.y, fm.y, qm.y, qmm.y, qw.y, rjm.y, rjp.y, qm.x, rkp);
      if (NRM || MS) {   // the input's pending factor, applied at the store by linearity
        o0 = __dmul_rn(o0, fnorm);
        o1 = __dmul_rn(o1, fnorm);
      }
      double* dst = args.out + doff;
      if (!MASK || ok1) {
        *reinterpret_cast<double2*>(dst) = make_double2(o0, o1);
      } else if (ok0) {
        *dst = o0;
      }
      if (NRM) {   // this lane's share of the output's norm, summed over the launch
        if (!MASK || ok0) *qacc = __fma_rn(o0, o0, *qacc);
        if (!MASK || ok1) *qacc = __fma_rn(o1, o1, *qacc);
      }
    }
    if (STEP2) doff += pstride;
    rg.next(rf0);
    ++p;
  };
  using no2 = std::false_type;
  using yes2 = std::true_type;
  // planes z0-1 and z0 (step 1 only), then the steady 3-plane rotation from
  // its third phase; an item has z1 - z0 + 3 >= 3 planes
  plane(c_a, c_b, c_c, q0, q2, q1, a0, f0, a2, f2, no2{});
  plane(c_b, c_c, c_a, q1, q0, q2, a1, f1, a0, f0, no2{});
  for (;;) {
    plane(c_c, c_a, c_b, q2, q1, q0, a2, f2, a1, f1, yes2{});
    if (p == pend) break;
    plane(c_a, c_b, c_c, q0, q2, q1, a0, f0, a2, f2, yes2{});
    if (p == pend) break;
    plane(c_b, c_c, c_a, q1, q0, q2, a1, f1, a0, f0, yes2{});
    if (p == pend) break;
  }
  g += (uint32_t)(pend - (I.z0 - 1));
  mbar_arrive_u(cur_bar + S * 8);
  if (PEER && STEP2 && peer_edge) {
    // the fused exchange: this item's edge output planes (z <= pl_hi go to the
    // left neighbour's halo, z >= pr_lo to the right one's) copied after the
    // plane loop from the lane's own just-stored sites (same thread: program
    // order) -- inside the loop the peer stores and their 64-bit offsets cost
    // the loop its registers (312 B of stack at 96 registers, +47 % per pass)
    const long long base_off = (long long)j * args.pitch + (k + COL_OFF);
    auto copy_plane = [&](int z, long long dd) {
      const double* src = args.out + ((long long)(z - args.z_base) * args.plane_stride + base_off);
      if (!MASK || ok1) {
        *reinterpret_cast<double2*>(const_cast<double*>(src) + dd) = *reinterpret_cast<const double2*>(src);
      } else if (ok0) {
        const_cast<double*>(src)[dd] = src[0];
      }
    };
    for (int z = I.z0; z <= min(I.z1, args.pl_hi); ++z) copy_plane(z, args.dl);
    for (int z = max(I.z0, args.pr_lo); z <= I.z1; ++z) copy_plane(z, args.dr);
  }
  if (STEP2 && I.idx < args.sig_items) {
    // an edge item's planes are stored: make them visible, then count this
    // warp done (the exchange waits for the count on its own stream)
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(args.sig, 1ull);
  }
}

template <int S, int TB, bool STEP2, bool FASTC, bool PEER = false, bool NRM = false, bool MS = false>
__device__ __forceinline__ void t2b_rows(const SweepArgs& args, uint32_t sm0, int w, int lane,
                                         double fnorm = 1.0) {
  using C = T2BCfg<S, TB>;
  const uint32_t fb = sm0 + C::BAR_OFF;               // full[S], empty[S], rfull[4]
  const uint32_t base = sm0 + (uint32_t)(((w + 1) * BOXW + 2 * lane + 2) * 8);
  StageRot<S, T2BGeo<TB>::STAGE> nx(base, fb);
  uint32_t g = 4;   // ring plane counter (runs across items; 0..3 are the pre-completed phases)
  if constexpr (PEER && STEP2) {
    t2b_for_items<TB>(args, [&](const T2Item& I) {
      // only items holding an edge output plane take the peer-store variant
      const bool edge = I.z0 <= args.pl_hi || I.z1 >= args.pr_lo;
      // (a runtime flag, not two more inlined variants: the larger body was not
      // inlined, which put the kernel's parameters on the stack -- 312 B,
      // +47 % per pass at 512^2 x 256, profiles/fused_pass_r02.txt)
      if (t2b_row_interior(I, w, args.n, args.x_off))
        t2b_rows_item<S, TB, STEP2, FASTC, false, true>(args, I, fb, base, w, lane, nx, g, 1.0, nullptr, edge);
      else
        t2b_rows_item<S, TB, STEP2, FASTC, true, true>(args, I, fb, base, w, lane, nx, g, 1.0, nullptr, edge);
    });
    // no fence here: the peer stores are performed when this grid completes;
    // whoever reads them is ordered after that completion (an event, or the
    // IPC transport's post kernel, which fences at system scope and then
    // publishes its counter)
  } else {
    double qacc = 0.0;
    t2b_for_items<TB>(args, [&](const T2Item& I) {
      if (t2b_row_interior(I, w, args.n, args.x_off))
        t2b_rows_item<S, TB, STEP2, FASTC, false, false, NRM, MS>(args, I, fb, base, w, lane, nx, g, fnorm,
                                                                 &qacc);
      else
        t2b_rows_item<S, TB, STEP2, FASTC, true, false, NRM, MS>(args, I, fb, base, w, lane, nx, g, fnorm,
                                                                &qacc);
    });
    if constexpr (NRM && STEP2) {
      qacc = warp_sum(qacc);
      if (lane == 0) args.part[args.nslot + blockIdx.x * TB + (w - 1)] = qacc;
    }
  }
}

template <int S, int TB, bool FASTC, bool MASK>
__device__ __forceinline__ void t2b_ring_item(const SweepArgs& args, const T2Item& I, uint32_t fb,
                                              uint32_t base, int rrow, int rcol, bool active,
                                              int lane, StageRot<S, T2BGeo<TB>::STAGE>& nx,
                                              uint32_t& g) {
  using G = T2BGeo<TB>;
  using C = T2BCfg<S, TB>;
  constexpr uint32_t VOFF = G::PSI_STRIDE - BOXW * 8;
  constexpr uint32_t ROFF = C::RING_OFF - BOXW * 8;
  const uint32_t rf0 = fb + 2 * S * 8;
  const int n = args.n;
  const double h = args.h, c0 = args.c0;
  const int j = I.j - 1 + rrow;
  const int k = I.k - 2 + rcol;
  const bool in0 = active & (j <= n) & ((unsigned)(k - 1) < (unsigned)n);
  RingRot<G::RING> rg(g, rf0);
  mbar_wait_u(nx.bar, nx.ph);
  double c_a = lds1_u(nx.addr);
  mbar_arrive_u(nx.bar + S * 8);   // every lane arrives on empty (count 32 per warp)
  nx.next(base, fb);
  mbar_wait_u(nx.bar, nx.ph);
  double c_b = lds1_u(nx.addr);
  uint32_t cur = nx.addr, cur_bar = nx.bar;
  nx.next(base, fb);
  bool okf = mbar_test_u(nx.bar, nx.ph);
  double c_c;
  const int pend = I.z1 + 2;
  int p = I.z0 - 1;
  auto plane = [&](const double& cp, const double& cc, double& cn) {
    mbar_wait_if(okf, nx.bar, nx.ph);
    const bool okr = mbar_test_u(rg.br, rg.rph);
    cn = lds1_u(nx.addr);
    const uint32_t sc = cur;
    const double jm = lds1_u(sc - BOXW * 8);
    const double jp = lds1_u(sc + BOXW * 8);
    const double km = lds1_u(sc - 8);
    const double kp = lds1_u(sc + 8);
    const double v = lds1_u(sc + VOFF);
    double A, Cc;
    coef1<FASTC>(v, h, c0, A, Cc);
    const double u = upd(A, Cc, cc, cp, cn, jm, jp, km, kp);
    double qv = u;
    if (MASK) {
      const bool pin = (unsigned)(args.x_off + p - 1) < (unsigned)n;   // global plane
      qv = (pin & in0) ? u : cc;
    }
    if (active) sts1_u(base + ROFF + rg.rw, qv);
    mbar_arrive_u(cur_bar + S * 8);
    mbar_arrive_u(rg.bw);
    cur = nx.addr;
    cur_bar = nx.bar;
    nx.next(base, fb);
    okf = mbar_test_u(nx.bar, nx.ph);
    mbar_wait_if(okr, rg.br, rg.rph);
    rg.next(rf0);
    ++p;
  };
  for (;;) {
    plane(c_a, c_b, c_c);
    if (p == pend) break;
    plane(c_b, c_c, c_a);
    if (p == pend) break;
    plane(c_c, c_a, c_b);
    if (p == pend) break;
  }
  g += (uint32_t)(pend - (I.z0 - 1));
  mbar_arrive_u(cur_bar + S * 8);
}

template <int S, int TB, bool FASTC>
__device__ __forceinline__ void t2b_ringw(const SweepArgs& args, uint32_t sm0, int lane) {
  using C = T2BCfg<S, TB>;
  const uint32_t fb = sm0 + C::BAR_OFF;
  const int rrow = 1 + (lane % TB);
  const int rcol = lane < TB ? 1 : 66;
  const bool active = lane < 2 * TB;
  const uint32_t base = sm0 + (uint32_t)(((rrow + 1) * BOXW + rcol) * 8);
  StageRot<S, T2BGeo<TB>::STAGE> nx(base, fb);
  uint32_t g = 4;
  t2b_for_items<TB>(args, [&](const T2Item& I) {
    if (t2b_ring_interior<TB>(I, args.n, args.x_off))
      t2b_ring_item<S, TB, FASTC, false>(args, I, fb, base, rrow, rcol, active, lane, nx, g);
    else
      t2b_ring_item<S, TB, FASTC, true>(args, I, fb, base, rrow, rcol, active, lane, nx, g);
  });
}

template <int NST, int TB, bool FASTC, bool PEER = false, bool NRM = false, bool MS = false>
__global__ void __launch_bounds__(T2BGeo<TB>::THREADS, T2BGeo<TB>::MINB)
    k_sweep2b(const __grid_constant__ CUtensorMap tm_psi, const __grid_constant__ CUtensorMap tm_v,
              const SweepArgs args) {
  using G = T2BGeo<TB>;
  constexpr int RS = T2B_RS;
  using C = T2BCfg<NST, TB, RS>;
  constexpr int S = NST;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + S;
  uint64_t* rfull = empty + S;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::CW * 32);   // per-lane arrivals of the consumer warps
    }
    for (int r = 0; r < RS; ++r) mbar_init(&rfull[r], G::CW * 32);
    fence_barrier_init();
  }
  __syncthreads();
  // ring planes count from 4: every consumer lane completes phase 0 of each
  // slot once, so the first planes' waits need no g > 0 test
  if (warp < G::CW) {
    for (int r = 0; r < RS; ++r) mbar_arrive(&rfull[r]);
  }
  pdl_launch_dependents();
  pdl_wait();
  if (warp == G::CW) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_psi);
      tma_prefetch_desc(&tm_v);
      int it = 0;
      t2b_for_items<TB>(args, [&](const T2Item& I) {
        const int kc = I.k + COL_OFF;
        for (int p = I.z0 - 2; p <= I.z1 + 2; ++p, ++it) {
          const int slot = it % S;
          if (it >= S) mbar_wait_sleep(&empty[slot], ((it / S) - 1) & 1);
          const bool hasv = (p >= I.z0 - 1) && (p <= I.z1 + 1);
          unsigned char* st = smem + slot * G::STAGE;
          mbar_arrive_expect_tx(&full[slot], G::PSI_BYTES + (hasv ? G::V_BYTES : 0));
          tma_load_3d(st, &tm_psi, kc - 2, I.j - 2, p + 1, &full[slot]);   // deep-halo map: plane + 1
          // V without the evict-first hint here: neighbouring tiles re-read its halo
          // rows / columns from L2 (-4 % DRAM bytes, +1..2 % at 256^3..512^3)
          if (hasv) tma_load_3d(st + G::PSI_STRIDE, &tm_v, kc - 2, I.j - 1, p, &full[slot]);
        }
      });
    }
    return;
  }
  const uint32_t sm0 = smem_u32(smem);
  if (warp == TB + 2) {
    t2b_ringw<S, TB, FASTC>(args, sm0, lane);
  } else if (warp == 0 || warp == TB + 1) {
    t2b_rows<S, TB, false, FASTC>(args, sm0, warp, lane);
  } else {
    static_assert(!(PEER && NRM), "no fused exchange in the renormalising pass");
    static_assert(!(MS && (PEER || NRM)), "the measuring pass is a plain whole-lattice pass");
    const double fnorm = (NRM || MS) ? *args.scale : 1.0;   // after pdl_wait: the predecessor's factor
    t2b_rows<S, TB, true, FASTC, PEER, NRM, MS>(args, sm0, warp, lane, fnorm);
  }
}

// division self-test: compares coef_pair against IEEE division on random
// potentials h*V in [lo, hi) (psg_selftest_division)
__global__ void k_div_check(unsigned long long seed, long long count, double lo, double hi,
                            unsigned long long* mismatches, int variant) {
  unsigned long long bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned long long x = seed ^ (0x9E3779B97F4A7C15ull * (unsigned long long)(i + 1));
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
    const double u = (double)(x >> 11) * 0x1.0p-53;
    const double v = lo + u * (hi - lo);
    double A, Cc;
    if (variant) {
      double A1, C1;
      coef_pair2(make_double2(v, v), 1.0, 1.0, A, Cc, A1, C1);
    } else {
      coef_pair(v, 1.0, 1.0, A, Cc);
    }
    const double d = __dadd_rn(1.0, v);
    const double Aw = __ddiv_rn(__dsub_rn(1.0, v), d);
    const double Bw = __ddiv_rn(1.0, d);
    if (__double_as_longlong(A) != __double_as_longlong(Aw) ||
        __double_as_longlong(Cc) != __double_as_longlong(Bw))
      ++bad;
  }
  if (bad) atomicAdd(mismatches, bad);
}
