// transport.cuh -- slab transports (NCCL, peer copies) and the fused fixed-step run loop.
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace, after the slab object it operates on).
#pragma once

// ------------------------------------------------------------------
// slab transports.  A z-decomposed run moves halo planes between neighbouring
// slabs and sums the zero-padded plane-sum vectors; the loop below is the same
// for NCCL ranks (one slab per process) and for several slabs driven by one
// process (peer copies over NVLink, or plain copies on one device).
//   post(depth): enqueue the exchange of `depth` planes per face (after each
//                slab's previous work) on the slabs' communication streams
//   wait():      order each slab's main stream after its halo arrival
//   allreduce(): after every slab's reduce, every slab holds the global sums
// Every cross-stream dependency is an event; nothing spins on the device.
// ------------------------------------------------------------------
struct Transport {
  bool deep = false;   // two halo planes per face of every slab's current buffer are posted
  virtual ~Transport() {}
  virtual bool has_left(size_t r) const = 0;
  virtual bool has_right(size_t r) const = 0;
  virtual int post(int depth) = 0;
  // exchange of the OUTPUT buffers' edge planes of the pass just launched,
  // started on the device's signal that the slab's edge items are stored
  // (slab counter >= its sig_target) instead of after the whole pass
  virtual int post_signal(int depth) = 0;
  virtual int wait() = 0;
  virtual int allreduce() = 0;
  // fused exchange: two-sweep passes store their edge planes straight into the
  // neighbours' output-buffer halos (peer memory); after_fused() then orders
  // every slab's next work after its neighbours' passes (via wait())
  virtual bool fused() const { return false; }
  virtual int after_fused() { return PSG_OK; }
  // slab r's neighbour on `side` (0 left, 1 right): its OUTPUT buffer of the
  // pass about to run (local plane 0) and its W; nullptr when there is none
  virtual double* peer_out(size_t r, int side, int64_t* w) const {
    (void)r; (void)side; (void)w;
    return nullptr;
  }
};

struct NcclTransport : Transport {
  psg_slab* s;
  psg_comm* c;
  int left, right;
  bool posted = false;
  NcclTransport(psg_slab* s_, psg_comm* c_, int l, int r) : s(s_), c(c_), left(l), right(r) {}
  bool has_left(size_t) const override { return left >= 0; }
  bool has_right(size_t) const override { return right >= 0; }
  int post(int depth) override { return exchange(depth, false); }
  int post_signal(int depth) override { return exchange(depth, true); }
  int exchange(int depth, bool signal) {
    posted = false;
    if (left < 0 && right < 0) return PSG_OK;
    NcclApi* api = nccl();
    const size_t ps = (size_t)s->plane_stride;
    const size_t cnt = (size_t)depth * ps;
    double* cur = s->psi[signal ? 1 - s->cur : s->cur];
    const int64_t w = s->w;
    if (signal) {
      int rc = stream_wait_value(c->cstream, s->sig_dev, s->sig_target);
      if (rc) return rc;
    } else {
      CU_TRY(cudaEventRecord(c->ev_main, s->stream));
      CU_TRY(cudaStreamWaitEvent(c->cstream, c->ev_main, 0));
    }
    NCCL_TRY(api->GroupStart());
    if (left >= 0) {   // planes 1..depth -> left's W+1..; left's W-depth+1..W -> 1-depth..0
      NCCL_TRY(api->Send(cur + ps, cnt, ncclFloat64, left, c->comm, c->cstream));
      NCCL_TRY(api->Recv(cur + ps - cnt, cnt, ncclFloat64, left, c->comm, c->cstream));
    }
    if (right >= 0) {
      NCCL_TRY(api->Send(cur + (size_t)(w + 1) * ps - cnt, cnt, ncclFloat64, right, c->comm, c->cstream));
      NCCL_TRY(api->Recv(cur + (size_t)(w + 1) * ps, cnt, ncclFloat64, right, c->comm, c->cstream));
    }
    NCCL_TRY(api->GroupEnd());
    CU_TRY(cudaEventRecord(c->ev_comm, c->cstream));
    posted = true;
    return PSG_OK;
  }
  int wait() override {
    if (posted) CU_TRY(cudaStreamWaitEvent(s->stream, c->ev_comm, 0));
    return PSG_OK;
  }
  int allreduce() override {
    if (c->nranks > 1)
      NCCL_TRY(nccl()->AllReduce(s->plane_sums, s->plane_sums, (size_t)NQ * s->n, ncclFloat64,
                                 ncclSum, c->comm, s->stream));
    return PSG_OK;
  }
};

__global__ void k_add(double* __restrict__ out, const double* __restrict__ in, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = __dadd_rn(out[i], in[i]);
}

struct LocalTransport : Transport {
  std::vector<psg_slab*> sl;
  std::vector<cudaStream_t> cs;
  std::vector<cudaEvent_t> evm, evc, evr;
  double* tmp0 = nullptr;   // on slab 0's device: one incoming plane-sum vector
  ~LocalTransport() override {
    for (size_t r = 0; r < sl.size(); ++r) {
      cudaSetDevice(sl[r]->device);
      if (r < cs.size() && cs[r]) cudaStreamSynchronize(cs[r]);
      if (r < cs.size() && cs[r]) cudaStreamDestroy(cs[r]);
      if (r < evm.size() && evm[r]) cudaEventDestroy(evm[r]);
      if (r < evc.size() && evc[r]) cudaEventDestroy(evc[r]);
      if (r < evr.size() && evr[r]) cudaEventDestroy(evr[r]);
    }
    if (tmp0) {
      cudaSetDevice(sl[0]->device);
      cudaFree(tmp0);
    }
  }
  int init(psg_slab** slabs, int m) {
    sl.assign(slabs, slabs + m);
    cs.assign(m, nullptr);
    evm.assign(m, nullptr);
    evc.assign(m, nullptr);
    evr.assign(m, nullptr);
    for (int r = 0; r < m; ++r) {
      CU_TRY(cudaSetDevice(sl[r]->device));
      CU_TRY(cudaStreamCreateWithFlags(&cs[r], cudaStreamNonBlocking));
      CU_TRY(cudaEventCreateWithFlags(&evm[r], cudaEventDisableTiming));
      CU_TRY(cudaEventCreateWithFlags(&evc[r], cudaEventDisableTiming));
      CU_TRY(cudaEventCreateWithFlags(&evr[r], cudaEventDisableTiming));
    }
    CU_TRY(cudaSetDevice(sl[0]->device));
    CU_TRY(cudaMalloc(&tmp0, (size_t)NQ * sl[0]->n * sizeof(double)));
    // fused exchange: every slab wide enough that no output plane goes both
    // ways (W >= 4), and neighbours on one device or with peer access
    fused_ok = m >= 2 && sl[0]->fused_halo;
    for (int r = 0; r < m && fused_ok; ++r) fused_ok = sl[r]->w >= 4;
    for (int r = 1; r < m && fused_ok; ++r) {
      const int d0 = sl[r - 1]->device, d1 = sl[r]->device;
      if (d0 == d1) continue;
      int a01 = 0, a10 = 0;
      CU_TRY(cudaDeviceCanAccessPeer(&a01, d0, d1));
      CU_TRY(cudaDeviceCanAccessPeer(&a10, d1, d0));
      if (!a01 || !a10) {
        fused_ok = false;
        break;
      }
      for (int pair = 0; pair < 2; ++pair) {
        CU_TRY(cudaSetDevice(pair ? d1 : d0));
        const cudaError_t e = cudaDeviceEnablePeerAccess(pair ? d0 : d1, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return fail(PSG_ERR_CUDA, "peer access between slab devices");
      }
    }
    return PSG_OK;
  }
  bool has_left(size_t r) const override { return r > 0; }
  bool has_right(size_t r) const override { return r + 1 < sl.size(); }
  bool fused_ok = false;
  bool fused() const override { return fused_ok; }
  double* peer_out(size_t r, int side, int64_t* w) const override {
    const size_t q = side ? r + 1 : r - 1;
    if ((side == 0 && r == 0) || q >= sl.size()) return nullptr;
    *w = sl[q]->w;
    return sl[q]->psi[1 - sl[q]->cur];
  }
  int after_fused() override {
    for (size_t r = 0; r < sl.size(); ++r) {
      CU_TRY(cudaSetDevice(sl[r]->device));
      CU_TRY(cudaEventRecord(evc[r], sl[r]->stream));
    }
    pushed = true;   // wait(): my halos were written by my neighbours' passes
    return PSG_OK;
  }
  bool pushed = false;   // last exchange pushed by the source slabs (post_signal)
  int post(int depth) override {
    const size_t m = sl.size();
    pushed = false;
    if (m < 2) return PSG_OK;
    for (size_t r = 0; r < m; ++r) {
      CU_TRY(cudaSetDevice(sl[r]->device));
      CU_TRY(cudaEventRecord(evm[r], sl[r]->stream));
    }
    for (size_t r = 0; r < m; ++r) {
      psg_slab* s = sl[r];
      CU_TRY(cudaSetDevice(s->device));
      const size_t ps = (size_t)s->plane_stride;
      const size_t bytes = (size_t)depth * ps * sizeof(double);
      double* cur = s->psi[s->cur];
      CU_TRY(cudaStreamWaitEvent(cs[r], evm[r], 0));
      if (r > 0) {   // left neighbour's last planes -> my planes 1-depth .. 0
        psg_slab* o = sl[r - 1];
        CU_TRY(cudaStreamWaitEvent(cs[r], evm[r - 1], 0));
        CU_TRY(cudaMemcpyPeerAsync(cur + ps - (size_t)depth * ps, s->device,
                                   o->psi[o->cur] + (size_t)(o->w + 1 - depth) * ps, o->device,
                                   bytes, cs[r]));
      }
      if (r + 1 < m) {   // right neighbour's first planes -> my planes W+1 .. W+depth
        psg_slab* o = sl[r + 1];
        CU_TRY(cudaStreamWaitEvent(cs[r], evm[r + 1], 0));
        CU_TRY(cudaMemcpyPeerAsync(cur + (size_t)(s->w + 1) * ps, s->device, o->psi[o->cur] + ps,
                                   o->device, bytes, cs[r]));
      }
      CU_TRY(cudaEventRecord(evc[r], cs[r]));
    }
    return PSG_OK;
  }
  // push model: when slab r's edge items are stored (its counter), copy its new
  // edge planes into the neighbours' output-buffer halos (copy engines: no SMs)
  int post_signal(int depth) override {
    const size_t m = sl.size();
    pushed = true;
    if (m < 2) return PSG_OK;
    for (size_t r = 0; r < m; ++r) {
      psg_slab* s = sl[r];
      CU_TRY(cudaSetDevice(s->device));
      const size_t ps = (size_t)s->plane_stride;
      const size_t bytes = (size_t)depth * ps * sizeof(double);
      const double* out = s->psi[1 - s->cur];
      int rc = stream_wait_value(cs[r], s->sig_dev, s->sig_target);
      if (rc) return rc;
      if (r > 0) {   // my planes 1..depth -> left's W+1 ..
        psg_slab* o = sl[r - 1];
        CU_TRY(cudaMemcpyPeerAsync(o->psi[1 - o->cur] + (size_t)(o->w + 1) * ps, o->device,
                                   out + ps, s->device, bytes, cs[r]));
      }
      if (r + 1 < m) {   // my planes W-depth+1..W -> right's 1-depth .. 0
        psg_slab* o = sl[r + 1];
        CU_TRY(cudaMemcpyPeerAsync(o->psi[1 - o->cur] + ps - (size_t)depth * ps, o->device,
                                   out + (size_t)(s->w + 1 - depth) * ps, s->device, bytes, cs[r]));
      }
      CU_TRY(cudaEventRecord(evc[r], cs[r]));
    }
    return PSG_OK;
  }
  int wait() override {
    const size_t m = sl.size();
    if (m < 2) return PSG_OK;
    for (size_t r = 0; r < m; ++r) {
      CU_TRY(cudaSetDevice(sl[r]->device));
      if (pushed) {   // my halos were written by my neighbours' streams
        if (r > 0) CU_TRY(cudaStreamWaitEvent(sl[r]->stream, evc[r - 1], 0));
        if (r + 1 < m) CU_TRY(cudaStreamWaitEvent(sl[r]->stream, evc[r + 1], 0));
      } else {
        CU_TRY(cudaStreamWaitEvent(sl[r]->stream, evc[r], 0));
      }
    }
    return PSG_OK;
  }
  int allreduce() override {
    const size_t m = sl.size();
    if (m < 2) return PSG_OK;
    psg_slab* s0 = sl[0];
    const size_t cnt = (size_t)NQ * s0->n;
    for (size_t r = 1; r < m; ++r) {
      CU_TRY(cudaSetDevice(sl[r]->device));
      CU_TRY(cudaEventRecord(evr[r], sl[r]->stream));
    }
    // slab 0 gathers (one non-zero contributor per slot: exact in any order)
    CU_TRY(cudaSetDevice(s0->device));
    for (size_t r = 1; r < m; ++r) {
      CU_TRY(cudaStreamWaitEvent(s0->stream, evr[r], 0));
      CU_TRY(cudaMemcpyPeerAsync(tmp0, s0->device, sl[r]->plane_sums, sl[r]->device,
                                 cnt * sizeof(double), s0->stream));
      k_add<<<std::min<int>(1024, (int)((cnt + 255) / 256)), 256, 0, s0->stream>>>(s0->plane_sums,
                                                                                 tmp0, (int)cnt);
      CU_TRY(cudaGetLastError());
    }
    CU_TRY(cudaEventRecord(evr[0], s0->stream));
    // and hands the total back
    for (size_t r = 1; r < m; ++r) {
      CU_TRY(cudaSetDevice(sl[r]->device));
      CU_TRY(cudaStreamWaitEvent(sl[r]->stream, evr[0], 0));
      CU_TRY(cudaMemcpyPeerAsync(sl[r]->plane_sums, sl[r]->device, s0->plane_sums, s0->device,
                                 cnt * sizeof(double), sl[r]->stream));
    }
    return PSG_OK;
  }
};

// edge / interior plane ranges of slab r for a halo depth (1: single sweep,
// 2: two-sweep pass)
inline void split_ranges(const psg_slab* s, bool l, bool r, int depth, int64_t& lo, int64_t& hi) {
  lo = l ? 1 + depth : 1;
  hi = r ? s->w - depth : s->w;
}


// one sweep of every slab: exchange one halo plane per face (overlapped with
// the interior planes; nothing to post if the deep halos of the current
// buffers are already in flight), then the edge planes
int multi_sweep(std::vector<psg_slab*>& sl, Transport* tr, unsigned flags, bool write) {
  int rc = PSG_OK;
  if (!tr->deep) {
    NvtxRange nv("psg:halo_post");
    rc = tr->post(1);
  }
  if (rc) return rc;
  for (size_t r = 0; r < sl.size(); ++r) {
    CU_TRY(cudaSetDevice(sl[r]->device));
    int64_t lo, hi;
    split_ranges(sl[r], tr->has_left(r), tr->has_right(r), 1, lo, hi);
    if (lo <= hi) rc = do_sweep(sl[r], lo, hi, flags, write);
    if (rc) return rc;
  }
  rc = tr->wait();
  if (rc) return rc;
  for (size_t r = 0; r < sl.size(); ++r) {
    psg_slab* s = sl[r];
    CU_TRY(cudaSetDevice(s->device));
    const bool l = tr->has_left(r), rr = tr->has_right(r);
    if (l) rc = do_sweep(s, 1, 1, flags, write);
    if (!rc && rr && (s->w > 1 || !l)) rc = do_sweep(s, s->w, s->w, flags, write);
    if (rc) return rc;
  }
  tr->deep = false;
  return PSG_OK;
}

// two sweeps of every slab in one pass each (k_sweep2b), pipelined so that
// the halo exchange hides behind the interior, all on the slab's stream:
//   the edge pairs 1..2 / W-1..W first (one launch), once the deep halos (two
//   planes per face: local -1, 0 / W+1, W+2) of the current state are in;
//   then the exchange for the NEXT pass is posted (it sends the edge planes
//   just written and lands in the output buffer's halos) and runs while
//   the interior planes 3..W-2 are updated.
// One exchange per two sweeps; cross-stream ordering by events only.
// two sweeps of every slab in one pass each (k_sweep2b): ONE launch per slab
// whose chunk order puts the edge planes (1..2, W-1..W) first; as the step-2
// warps of those items store, they count on the slab's device counter, and
// the exchange of the new edge planes (the next pass's deep halos) is queued
// on the communication stream behind a wait for that count
// (cuStreamWaitValue64), so it runs while the launch is still updating the
// interior.  One exchange per two sweeps; no host in the loop.
int multi_sweep2(std::vector<psg_slab*>& sl, Transport* tr) {
  int rc = PSG_OK;
  if (!tr->deep) {
    NvtxRange nv("psg:halo_post");
    rc = tr->post(2);
  }
  if (rc) return rc;
  rc = tr->wait();
  if (rc) return rc;
  if (tr->fused()) {
    // one launch per slab computes both sweeps AND delivers its new edge planes
    // into the neighbours' halos: a site of output plane z <= 2 is stored at
    // the same (j, k) of the left neighbour's plane W_L + z, z >= W - 1 at the
    // right neighbour's plane z - W (element offsets between the buffers)
    for (size_t r = 0; r < sl.size(); ++r) {
      psg_slab* s = sl[r];
      CU_TRY(cudaSetDevice(s->device));
      const long long ps = s->plane_stride;
      const double* out = s->psi[1 - s->cur];
      PeerStores pst;
      int64_t wl = 0, wr = 0;
      if (const double* lo = tr->peer_out(r, 0, &wl)) {
        pst.dl = (long long)((intptr_t)(lo + wl * ps) - (intptr_t)out) / 8;
        pst.pl_hi = 2;
      }
      if (const double* ro = tr->peer_out(r, 1, &wr)) {
        pst.dr = (long long)((intptr_t)(ro - s->w * ps) - (intptr_t)out) / 8;
        pst.pr_lo = (int)s->w - 1;
      }
      rc = pass2(s, 1, s->w, false, &pst);
      if (rc) return rc;
      s->fused_passes++;
    }
    rc = tr->after_fused();
    if (rc) return rc;
    tr->deep = true;
    for (psg_slab* s : sl) s->cur = 1 - s->cur;
    return PSG_OK;
  }
  for (psg_slab* s : sl) {
    CU_TRY(cudaSetDevice(s->device));
    if (!s->sig_dev) {
      // plain device allocation: stream memory operations do not accept pool memory
      if (cudaMalloc((void**)&s->sig_dev, sizeof(unsigned long long)) != cudaSuccess)
        return fail(PSG_ERR_CUDA, "signal counter allocation failed");
      CU_TRY(cudaMemsetAsync(s->sig_dev, 0, sizeof(unsigned long long), s->stream));
      s->sig_target = 0;
    }
    rc = pass2(s, 1, s->w, true);
    if (rc) return rc;
  }
  rc = tr->post_signal(2);
  if (rc) return rc;
  tr->deep = true;
  for (psg_slab* s : sl) s->cur = 1 - s->cur;
  return PSG_OK;
}

int ensure_hist(psg_slab* s, int64_t want) {
  const int64_t rec = 3 * s->n + 2;
  if (want > s->hist_cap) {
    dev_free(s->hist_dev, s->stream);
    s->hist_dev = nullptr;
    if (dev_alloc((void**)&s->hist_dev, (size_t)want * rec * sizeof(double), s->stream))
      return fail(PSG_ERR_CUDA, "history allocation failed");
    s->hist_cap = want;
  }
  return PSG_OK;
}

// observables of the current state of every slab (halo exchange, measuring
// pass, global sums, combine); slab 0's record (3n+2 doubles) to rec
int measure_loop(std::vector<psg_slab*>& sl, Transport* tr, double* rec) {
  int rc = PSG_OK;
  for (psg_slab* s : sl) {
    CU_TRY(cudaSetDevice(s->device));
    rc = ensure_hist(s, 1);
    if (rc) return rc;
  }
  rc = multi_sweep(sl, tr, PSG_F_MEASURE, false);
  if (rc) return rc;
  const unsigned q = qmask_of(PSG_F_MEASURE);
  for (psg_slab* s : sl) {
    CU_TRY(cudaSetDevice(s->device));
    CU_TRY(cudaMemsetAsync(s->plane_sums, 0, (size_t)NQ * s->n * sizeof(double), s->stream));
    rc = do_reduce(s, 1, s->w, q, false, nullptr);
    if (rc) return rc;
  }
  rc = tr->allreduce();
  if (rc) return rc;
  for (psg_slab* s : sl) {
    CU_TRY(cudaSetDevice(s->device));
    rc = do_combine(s, q, s->hist_dev);
    if (rc) return rc;
  }
  psg_slab* s0 = sl[0];
  CU_TRY(cudaSetDevice(s0->device));
  CU_TRY(cudaMemcpyAsync(rec, s0->hist_dev, (size_t)(3 * s0->n + 2) * sizeof(double),
                         cudaMemcpyDeviceToHost, s0->stream));
  for (psg_slab* s : sl) {
    CU_TRY(cudaSetDevice(s->device));
    CU_TRY(cudaStreamSynchronize(s->stream));
  }
  return PSG_OK;
}

// the fused fixed-step loop of psg_run / psg_run_dist / psg_run_multi
// (evolve.py:249-270, parallel.py:413-485): sweeps with their fused
// reductions, the combine (after the sum of the zero-padded plane-sum vectors
// for slabs), the factor folded into the next sweep, re-imposition; pairs of
// plain steps go through the two-sweep pass.  No host round trip until the
// end.  tr == nullptr: one whole-lattice slab.
int run_loop(std::vector<psg_slab*>& sl, Transport* tr, const psg_run_params* p, double* hist,
             int64_t max_checks, int64_t* n_checks) {
  int rc = PSG_OK;
  if (!p || p->steps < 0) return fail(PSG_ERR_CONFIG, "bad run parameters");
  psg_slab* s0 = sl[0];
  const int64_t rec = 3 * s0->n + 2;
  int64_t want = 0;
  if (p->measure_every > 0) want = p->steps / p->measure_every + 1;
  want = std::min(want, max_checks);
  for (psg_slab* s : sl) {
    CU_TRY(cudaSetDevice(s->device));
    rc = ensure_hist(s, want);
    if (rc) return rc;
  }
  int64_t nc = 0;
  std::vector<double> steps_of;
  auto plain = [&](int64_t t) {  // step t is a bare update (no measure / norm / re-impose)
    const int64_t sidx = p->step_offset + t;
    const bool meas = p->measure_every > 0 && sidx - 1 > 0 && (sidx - 1) % p->measure_every == 0;
    const bool norm = p->norm_every > 0 && sidx % p->norm_every == 0;
    const bool reimp = p->reimpose_every > 0 && p->n_impose > 0 && sidx % p->reimpose_every == 0;
    return !meas && !norm && !reimp;
  };
  // two-sweep passes: a whole-lattice slab, or slabs of W >= 2 (two halo
  // planes per face); the march only for a whole lattice
  bool t2_ok = true;
  for (psg_slab* s : sl)
    t2_ok = t2_ok && s->use_t2 && !s->use_ac && (!tr || s->w >= 2);
  const bool whole = !tr;
  auto set_all = [&](auto&& f) {
    for (psg_slab* s : sl) {
      CU_TRY(cudaSetDevice(s->device));
      const int r = f(s);
      if (r) return r;
    }
    return (int)PSG_OK;
  };
  if (tr) tr->deep = false;
  // linear renormalisation pairs (whole lattice): steps t, t+1 renormalised
  // after t+1 run as one renormalising two-sweep pass (do_sweep2_nrm) when
  // neither state inside the pair is measured nor re-imposed
  const bool lin = whole && t2_ok && (p->flags & PSG_RUN_LINEAR_NORM) != 0;
  auto meas_at = [&](int64_t t) {   // observables on the state entering sweep t
    const int64_t state_idx = p->step_offset + t - 1;
    return p->measure_every > 0 && state_idx > 0 && state_idx % p->measure_every == 0;
  };
  auto reimp_at = [&](int64_t t) {  // re-imposition after sweep t
    const int64_t sidx = p->step_offset + t;
    return p->reimpose_every > 0 && p->n_impose > 0 && sidx % p->reimpose_every == 0;
  };
  // a small whole lattice without re-imposition: the whole run, its norm and
  // measure steps included, in persistent k_small launches (do_small_chk)
  bool done_small = false;
  if (whole && s0->small_chk && !(p->flags & PSG_RUN_EXACT) && !(p->reimpose_every > 0 && p->n_impose > 0) &&
      p->steps >= SMALL_MIN_RUN && small_ok(s0)) {
    int64_t t = 1;
    while (t <= p->steps) {
      const int64_t g0 = p->step_offset + t - 1;
      int64_t len = std::min<int64_t>(p->steps - t + 1, int64_t(1) << 30);
      const int64_t room = want - nc;
      const int64_t me = p->measure_every;
      if (me > 0 && room > SMALL_MEAS_CAP && small_meas_count(g0, len, me) > SMALL_MEAS_CAP)
        len = small_first_meas(g0, me) + (int64_t)SMALL_MEAS_CAP * me - g0;   // stop before the next one
      int nm = 0;
      {
        NvtxRange nv("psg:small_run_checks");
        rc = do_small_chk(s0, len, g0, p->norm_every, me, (int)std::min<int64_t>(room, SMALL_MEAS_CAP),
                          (p->flags & PSG_RUN_LINEAR_NORM) != 0, s0->hist_dev + nc * rec, &nm);
      }
      if (rc) return rc;
      for (int k = 0; k < nm; ++k) steps_of.push_back((double)(small_first_meas(g0, me) + k * me));
      nc += nm;
      t += len;
    }
    done_small = true;
  }
  // norm / measure steps of a whole lattice inside two-sweep passes (option
  // 16; PSG_RUN_EXACT opts out): a pair ending on a normalisation runs as a
  // renormalising pass (the norm of its output, no factor to subsume), a pair
  // starting on a measured state as a measuring pass -- instead of two single
  // sweeps per check (each costs about a pass: 24 B per site for one update)
  const bool fast = whole && t2_ok && s0->fast_checks && !(p->flags & PSG_RUN_EXACT);
  auto norm_at = [&](int64_t t) { return p->norm_every > 0 && (p->step_offset + t) % p->norm_every == 0; };
  for (int64_t t = done_small ? p->steps + 1 : 1; t <= p->steps; ++t) {
    if (fast && t + 1 <= p->steps && p->norm_every >= 2 && norm_at(t + 1) && !norm_at(t) &&
        !meas_at(t) && !meas_at(t + 1) && !reimp_at(t) && s0->pending == s0->scal + S_ONE) {
      { NvtxRange nv("psg:pass2_norm"); rc = do_sweep2_nrm(s0); }
      if (rc) return rc;
      ++t;
      if (reimp_at(t)) {
        for (int k = 0; k < p->n_impose && k < 3; ++k) {
          rc = psg_impose(s0, p->impose_axis[k], p->impose_sign[k], 0);
          if (rc) return rc;
        }
      }
      continue;
    }
    if (fast && t + 1 <= p->steps && meas_at(t) && nc < want && !norm_at(t) && !norm_at(t + 1) &&
        !meas_at(t + 1) && !reimp_at(t)) {
      { NvtxRange nv("psg:pass2_measure"); rc = do_sweep2_ms(s0, s0->hist_dev + nc * rec); }
      if (rc) return rc;
      steps_of.push_back((double)(p->step_offset + t - 1));
      ++nc;
      ++t;
      if (reimp_at(t)) {
        for (int k = 0; k < p->n_impose && k < 3; ++k) {
          rc = psg_impose(s0, p->impose_axis[k], p->impose_sign[k], 0);
          if (rc) return rc;
        }
      }
      continue;
    }
    if (lin && t + 1 <= p->steps && p->norm_every > 0 &&
        (p->step_offset + t + 1) % p->norm_every == 0 && !meas_at(t) && !reimp_at(t) &&
        !meas_at(t + 1)) {
      { NvtxRange nv("psg:pass2_renorm"); rc = do_sweep2_nrm(s0); }
      if (rc) return rc;
      ++t;
      if (reimp_at(t)) {
        for (int k = 0; k < p->n_impose && k < 3; ++k) {
          rc = psg_impose(s0, p->impose_axis[k], p->impose_sign[k], 0);
          if (rc) return rc;
        }
      }
      continue;
    }
    if (t2_ok && s0->pending == s0->scal + S_ONE && plain(t)) {
      int64_t run = 1;
      while (t + run <= p->steps && plain(t + run)) ++run;
      if (whole && run >= SMALL_MIN_RUN && small_ok(s0)) {
        // a small lattice: the whole run of plain sweeps in one persistent launch
        { NvtxRange nv("psg:small_run"); rc = do_small(s0, run); }
        if (rc) return rc;
        t += run - 1;
        continue;
      }
      if (whole && run >= 3 && t3_ok(s0)) {
        // triples of plain steps: three sweeps per pass over HBM (the rest as a pair / single)
        const int64_t triples = run / 3;
        for (int64_t q = 0; q < triples; ++q) {
          NvtxRange nv("psg:pass3");
          rc = do_sweep3(s0);
          if (rc) return rc;
        }
        t += 3 * triples - 1;
        continue;
      }
      if (run >= 2) {
        // pairs of plain steps: two sweeps per pass over HBM
        const int64_t pairs = run / 2;
        for (int64_t q = 0; q < pairs; ++q) {
          NvtxRange nv("psg:pass2");
          rc = tr ? multi_sweep2(sl, tr) : do_sweep2(s0);
          if (rc) return rc;
        }
        t += 2 * pairs - 1;
        continue;
      }
    }
    const int64_t sidx = p->step_offset + t;   // global sweep number
    const int64_t state_idx = sidx - 1;
    unsigned flags = PSG_F_WRITE;
    const bool meas = p->measure_every > 0 && state_idx > 0 && state_idx % p->measure_every == 0 &&
                      nc < want;
    const bool norm = p->norm_every > 0 && sidx % p->norm_every == 0;
    if (meas) flags |= PSG_F_MEASURE;
    if (norm) flags |= PSG_F_NORM;
    {
      NvtxRange nv(flags & PSG_F_MEASURE ? "psg:sweep_measure" : "psg:sweep");
      rc = tr ? multi_sweep(sl, tr, flags, true) : do_sweep(s0, 1, s0->w, flags, true);
    }
    if (rc) return rc;
    const unsigned q = qmask_of(flags);
    if (q) {
      if (tr) {
        // zero-padded global plane-sum vectors: one non-zero contributor per
        // slot, so the sum is exact and the combine M-invariant
        rc = set_all([&](psg_slab* s) {
          CU_TRY(cudaMemsetAsync(s->plane_sums, 0, (size_t)NQ * s->n * sizeof(double), s->stream));
          return do_reduce(s, 1, s->w, q, false, nullptr);
        });
        if (rc) return rc;
        {
          NvtxRange nv("psg:allreduce");
          rc = tr->allreduce();
        }
        if (rc) return rc;
        rc = set_all([&](psg_slab* s) { return do_combine(s, q, meas ? s->hist_dev + nc * rec : nullptr); });
      } else {
        rc = do_reduce(s0, 1, s0->n, q, true, meas ? s0->hist_dev + nc * rec : nullptr);
      }
      if (rc) return rc;
      if (meas) {
        steps_of.push_back((double)state_idx);
        ++nc;
      }
    }
    for (psg_slab* s : sl) {
      s->cur = 1 - s->cur;
      s->pending = norm ? s->scal + S_FACTOR : s->scal + S_ONE;
    }
    if (p->reimpose_every > 0 && sidx % p->reimpose_every == 0) {
      for (int k = 0; k < p->n_impose && k < 3; ++k) {
        rc = set_all([&](psg_slab* s) { return psg_impose(s, p->impose_axis[k], p->impose_sign[k], 0); });
        if (rc) return rc;
      }
      if (tr) tr->deep = false;
    }
  }
  CU_TRY(cudaSetDevice(s0->device));
  if (hist && nc > 0) {
    CU_TRY(cudaMemcpyAsync(hist, s0->hist_dev, (size_t)nc * rec * sizeof(double),
                           cudaMemcpyDeviceToHost, s0->stream));
  }
  rc = set_all([&](psg_slab* s) {
    CU_TRY(cudaStreamSynchronize(s->stream));
    return (int)PSG_OK;
  });
  if (rc) return rc;
  if (hist)
    for (int64_t k = 0; k < nc; ++k) hist[k * rec] = steps_of[k];
  if (n_checks) *n_checks = nc;
  return PSG_OK;
}
