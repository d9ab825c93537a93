// march.cuh -- k_march: persistent multi-step sweep (kept as an option; slower).
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace; the host engine instantiates the templates).
#pragma once

// ------------------------------------------------------------------
// persistent multi-step sweep ("march"): steps step0 .. step0+nsteps-1 of the
// plain update (no scale, no reductions) in one cooperative launch.  Items are
// (step, chunk, tile) in step-major order; an item may start once the previous
// step has finished its own (chunk, tile) and the six stencil neighbours
// (chunk +-1, tile row +-1, tile column +-1): that covers both the data it
// reads (RAW) and the data the previous step still had to read from the
// buffer it overwrites (WAR).  done[chunk][tile] holds the last finished step
// (release by the consumers, acquire by the producer).  Blocks sweep across
// step boundaries without a grid-wide drain, so per-step tails and launch
// gaps disappear.
// ------------------------------------------------------------------
struct MarchArgs {
  double* out0;           // buffer 0 / 1 base
  double* out1;
  int* done;              // [nchunks][tiles]
  int* bad;
  long long plane_stride;
  int n, pitch, planes;
  int z_lo, z_hi, zc, nchunks, tiles_k, tiles, items_per_step, nitems;
  int step0;              // absolute march-step number of the first step
  int parity0;            // buffer read by the first step
  int variant;            // diagnostics: bit0 = fence in every thread, bit1 = skip waits (WRONG results)
  double h, c0;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_done(const int* p, int target) {
  uint32_t spins = 0;
  while (ld_acquire(p) < target) {
    __nanosleep(64);
    if (++spins > (1u << 26)) __trap();
  }
}

template <int NST>
__global__ void __launch_bounds__(NTHREADS, 2)
    k_march(const __grid_constant__ CUtensorMap tm_psi0, const __grid_constant__ CUtensorMap tm_psi1,
            const __grid_constant__ CUtensorMap tm_v, const MarchArgs args) {
  using C = SweepCfg<M_WRITE, NST>;
  constexpr int S = C::STAGES;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int tiles_k = args.tiles_k;
  const int tiles = args.tiles;
  const int ips = args.items_per_step;

  if (warp == NCW) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_psi0);
      tma_prefetch_desc(&tm_psi1);
      tma_prefetch_desc(&tm_v);
      const uint64_t pol_stream = policy_evict_first();
      int it = 0;
      for (int item = blockIdx.x; item < args.nitems; item += gridDim.x) {
        const int st = item / ips;
        const int rem = item - st * ips;
        const int chunk = rem / tiles;
        const int tile = rem - chunk * tiles;
        const int tj = tile / tiles_k;
        const int tk = tile - tj * tiles_k;
        if (st > 0 && !(args.variant & 2)) {
          const int target = args.step0 + st - 1;
          const int* row = args.done + (size_t)chunk * tiles;
          wait_done(row + tile, target);
          if (tk > 0) wait_done(row + tile - 1, target);
          if (tk + 1 < tiles_k) wait_done(row + tile + 1, target);
          if (tj > 0) wait_done(row + tile - tiles_k, target);
          if (tile + tiles_k < tiles) wait_done(row + tile + tiles_k, target);
          if (chunk > 0) wait_done(row - tiles + tile, target);
          if (chunk + 1 < args.nchunks) wait_done(row + tiles + tile, target);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        const CUtensorMap* tm = ((args.parity0 + st) & 1) ? &tm_psi1 : &tm_psi0;
        const int z0 = args.z_lo + chunk * args.zc;
        const int z1 = min(z0 + args.zc - 1, args.z_hi);
        const int kc = 1 + tk * TX + COL_OFF;
        const int j0 = 1 + tj * TY;
        for (int p = z0 - 1; p <= z1 + 1; ++p, ++it) {
          const int slot = it % S;
          if (it >= S) mbar_wait_sleep(&empty[slot], ((it / S) - 1) & 1);
          const bool outp = (p >= z0) && (p <= z1);
          unsigned char* stg = smem + slot * C::STAGE;
          mbar_arrive_expect_tx(&full[slot], PSI_BYTES + (outp ? CO_BYTES : 0));
          tma_load_3d(stg, tm, kc - 2, j0 - 1, p, &full[slot]);
          if (outp) tma_load_3d_hint(stg + C::V_OFF, &tm_v, kc, j0, p, &full[slot], pol_stream);
        }
      }
    }
    return;
  }

  const int w = warp;
  const int n = args.n;
  const int cidx = (w + 1) * BOXW + 2 * lane + 2;
  const int vidx = w * TX + 2 * lane;
  int it = 0;
  int any_bad = 0;
  for (int item = blockIdx.x; item < args.nitems; item += gridDim.x) {
    const int st = item / ips;
    const int rem = item - st * ips;
    const int chunk = rem / tiles;
    const int tile = rem - chunk * tiles;
    const int tj = tile / tiles_k;
    const int tk = tile - tj * tiles_k;
    double* out = ((args.parity0 + st + 1) & 1) ? args.out1 : args.out0;
    const int z0 = args.z_lo + chunk * args.zc;
    const int z1 = min(z0 + args.zc - 1, args.z_hi);
    const int j = 1 + tj * TY + w;
    const int k = 1 + tk * TX + 2 * lane;
    const bool ok0 = (j <= n) && (k <= n);
    const bool ok1 = (j <= n) && (k + 1 <= n);

    int slot = it % S;
    mbar_wait(&full[slot], (it / S) & 1);
    double2 cp = lds2(reinterpret_cast<const double*>(smem + slot * C::STAGE) + cidx);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    ++it;
    int slot_c = it % S;
    mbar_wait(&full[slot_c], (it / S) & 1);
    double2 cc = lds2(reinterpret_cast<const double*>(smem + slot_c * C::STAGE) + cidx);
    ++it;
    for (int p = z0; p <= z1; ++p, ++it) {
      const int slot_n = it % S;
      mbar_wait(&full[slot_n], (it / S) & 1);
      const double* bn = reinterpret_cast<const double*>(smem + slot_n * C::STAGE);
      const unsigned char* stc = smem + slot_c * C::STAGE;
      const double* bc = reinterpret_cast<const double*>(stc);
      const double2 cn = lds2(bn + cidx);
      const double2 jm = lds2(bc + cidx - BOXW);
      const double2 jp = lds2(bc + cidx + BOXW);
      const double km = bc[cidx - 1];
      const double kp = bc[cidx + 2];
      const double2 v = lds2(reinterpret_cast<const double*>(stc + C::V_OFF) + vidx);
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
      double A0, A1, C0, C1;
      coef_pair(v.x, args.h, args.c0, A0, C0);
      coef_pair(v.y, args.h, args.c0, A1, C1);
      const double o0 = __dadd_rn(__dmul_rn(A0, cc.x), __dmul_rn(C0, s0));
      const double o1 = __dadd_rn(__dmul_rn(A1, cc.y), __dmul_rn(C1, s1));
      double* dst = out + (long long)p * args.plane_stride + (long long)j * args.pitch + (k + COL_OFF);
      if (ok1) {
        *reinterpret_cast<double2*>(dst) = make_double2(o0, o1);
      } else if (ok0) {
        *dst = o0;
      }
      any_bad |= (ok0 && !finite_d(o0)) | (ok1 && !finite_d(o1));
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot_c]);
      cp = cc;
      cc = cn;
      slot_c = slot_n;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot_c]);
    // publish this item: the consumers' stores are ordered before the barrier;
    // thread 0's gpu-scope fence + release store is cumulative over them
    if (args.variant & 1) __threadfence();
    asm volatile("bar.sync 1, %0;" ::"n"(32 * NCW) : "memory");
    if (threadIdx.x == 0) {
      __threadfence();
      st_release(args.done + (size_t)chunk * tiles + tile, args.step0 + st);
    }
  }
  if (__any_sync(0xffffffffu, any_bad) && lane == 0) atomicOr(args.bad, 1);
}

// one site of the update from explicit neighbours (reference order)
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
