// ipc.cuh -- NCCL-free transport for one slab per process: peer memory through
// CUDA IPC mappings, cross-process ordering by device counters.
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace, after transport.cuh).
//
// Every rank maps its neighbours' psi buffers and every rank's "link block"
// (counters + all-reduce mailboxes).  Then:
//   * two-sweep passes deliver their edge planes themselves: k_sweep2b<PEER>
//     stores them into the neighbours' output-buffer halos (the fused
//     exchange of the in-process engine, here across processes);
//   * single sweeps pull the neighbours' edge planes (P2P copies);
//   * the plane-sum all-reduce writes each rank's zero-padded vector into
//     every rank's mailbox and sums the slots in rank order (exact: one
//     non-zero contributor per element, so bitwise M-invariant);
//   * ordering is a neighbour barrier: a rank posts an epoch into its
//     neighbours' counters (st.release.sys after a system fence, from a
//     one-warp kernel behind its previous work) and its stream waits for
//     theirs (cuStreamWaitValue64).  No kernel ever waits for another rank.
// Lock-step argument: every rank runs the same sequence of barrier() /
// allreduce() calls; a rank passes barrier e only after both neighbours
// finished all work issued before their barrier e, so a neighbour is at most
// one operation ahead -- it may write its own other buffer and our other
// buffer's halos, never the planes we are reading.
#pragma once

constexpr int IPC_MAX_RANKS = 64;

struct IpcExport {
  cudaIpcMemHandle_t blk, psi0, psi1;
  int64_t w, x_lo, n;
  int32_t rank, nranks;
};
static_assert(sizeof(IpcExport) <= PSG_IPC_HANDLE_BYTES, "IPC handle too large");

struct IpcPost {
  unsigned long long* p[IPC_MAX_RANKS];
  int n;
  unsigned long long v;
};

// make all prior writes of this device visible system-wide, then publish
// the epoch in each target counter (peer memory)
__global__ void k_ipc_post(const IpcPost a) {
  __threadfence_system();
  for (int i = threadIdx.x; i < a.n; i += blockDim.x)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.p[i]), "l"(a.v) : "memory");
}

}  // namespace

struct psg_ipc {
  psg_slab* s = nullptr;
  int rank = 0, nranks = 0;
  char* blk = nullptr;            // local link block: counters, then the mailboxes
  size_t blk_bytes = 0;
  std::vector<char*> rblk;        // every rank's link block (self: blk)
  double* npsi[2][2] = {};        // [left / right][buffer] neighbour psi, local plane 0
  int64_t nw[2] = {0, 0};
  uint64_t bar_epoch = 0, red_epoch = 0;
  bool connected = false;
  int64_t mbox_elems = 0;         // NQ * n per slot
  // layout: ctr_bar[nranks], ctr_red[nranks] (u64, padded to 256 B), then
  // mailboxes [2 parities][nranks][NQ * n] doubles
  uint64_t* ctr(int which, char* base) const {
    return reinterpret_cast<uint64_t*>(base) + (size_t)which * nranks;
  }
  double* mbox(char* base, int parity, int slot) const {
    const size_t off = ((size_t)2 * nranks * 8 + 255) / 256 * 256;
    return reinterpret_cast<double*>(base + off) + ((size_t)parity * nranks + slot) * mbox_elems;
  }
};

namespace {

struct IpcTransport : Transport {
  psg_ipc* c;
  psg_slab* s;
  explicit IpcTransport(psg_ipc* c_) : c(c_), s(c_->s) {}
  bool has_left(size_t) const override { return c->rank > 0; }
  bool has_right(size_t) const override { return c->rank + 1 < c->nranks; }
  bool fused() const override { return true; }

  int post_to(int which, const std::vector<int>& ranks, uint64_t v) {
    IpcPost a{};
    for (int q : ranks) a.p[a.n++] = (unsigned long long*)(c->ctr(which, c->rblk[q]) + c->rank);
    a.v = v;
    if (a.n == 0) return PSG_OK;
    k_ipc_post<<<1, 32, 0, s->stream>>>(a);
    CU_TRY(cudaGetLastError());
    return PSG_OK;
  }
  int wait_for(int which, const std::vector<int>& ranks, uint64_t v) {
    for (int q : ranks) {
      const int rc = stream_wait_value(s->stream, (const unsigned long long*)(c->ctr(which, c->blk) + q), v);
      if (rc) return rc;
    }
    return PSG_OK;
  }
  std::vector<int> neighbours() const {
    std::vector<int> r;
    if (c->rank > 0) r.push_back(c->rank - 1);
    if (c->rank + 1 < c->nranks) r.push_back(c->rank + 1);
    return r;
  }
  // both neighbours have finished everything issued before their matching call
  int barrier() {
    const uint64_t e = ++c->bar_epoch;
    const std::vector<int> nb = neighbours();
    int rc = post_to(0, nb, e);
    return rc ? rc : wait_for(0, nb, e);
  }
  // pull the neighbours' current edge planes into this slab's current halos
  int post(int depth) override {
    int rc = barrier();
    if (rc) return rc;
    const size_t ps = (size_t)s->plane_stride;
    const size_t bytes = (size_t)depth * ps * sizeof(double);
    double* cur = s->psi[s->cur];
    if (c->rank > 0)   // left's planes W_L-depth+1 .. W_L -> my 1-depth .. 0
      CU_TRY(cudaMemcpyAsync(cur + ps - (size_t)depth * ps,
                             c->npsi[0][s->cur] + (size_t)(c->nw[0] + 1 - depth) * ps, bytes,
                             cudaMemcpyDeviceToDevice, s->stream));
    if (c->rank + 1 < c->nranks)   // right's planes 1 .. depth -> my W+1 ..
      CU_TRY(cudaMemcpyAsync(cur + (size_t)(s->w + 1) * ps, c->npsi[1][s->cur] + ps, bytes,
                             cudaMemcpyDeviceToDevice, s->stream));
    return PSG_OK;
  }
  int post_signal(int) override { return fail(PSG_ERR_CONFIG, "IPC transport: no signalled passes"); }
  int wait() override { return PSG_OK; }   // pulls run on the slab's own stream
  int after_fused() override { return barrier(); }
  int allreduce() override {
    if (c->nranks < 2) return PSG_OK;
    const uint64_t e = ++c->red_epoch;
    const int par = (int)(e & 1);
    const size_t bytes = (size_t)c->mbox_elems * sizeof(double);
    std::vector<int> others;
    for (int q = 0; q < c->nranks; ++q)
      if (q != c->rank) {
        others.push_back(q);
        CU_TRY(cudaMemcpyAsync(c->mbox(c->rblk[q], par, c->rank), s->plane_sums, bytes,
                               cudaMemcpyDeviceToDevice, s->stream));
      }
    int rc = post_to(1, others, e);
    if (!rc) rc = wait_for(1, others, e);
    if (rc) return rc;
    const int cnt = (int)c->mbox_elems;
    for (int q : others)   // rank order; exact (one non-zero contributor per slot)
      k_add<<<std::min<int>(1024, (cnt + 255) / 256), 256, 0, s->stream>>>(
          s->plane_sums, c->mbox(c->blk, par, q), cnt);
    CU_TRY(cudaGetLastError());
    return PSG_OK;
  }
  double* peer_out(size_t, int side, int64_t* w) const override {
    const bool has = side ? c->rank + 1 < c->nranks : c->rank > 0;
    if (!has) return nullptr;
    *w = c->nw[side];
    return c->npsi[side][1 - s->cur];
  }
};
