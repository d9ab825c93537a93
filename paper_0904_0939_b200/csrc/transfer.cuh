// transfer.cuh -- host <-> device transfers of dense planes (chunked DMA, re-pitch kernel, pinned staging).
// Part of the single translation unit csrc/psigpu.cu (included there, inside its
// anonymous namespace, after the slab object it operates on).
#pragma once

// ------------------------------------------------------------------
// host <-> device transfers of dense (planes, ext, ext) host arrays to the
// pitched device layout: whole 32 MiB chunks move by contiguous DMA into a
// device scratch buffer and are re-pitched by a kernel (row-by-row 2D DMA of
// 2 KiB rows runs at a third of the link rate).  Pageable host memory goes
// through pinned staging buffers, copied by a host thread pool while the DMA
// of the neighbouring chunk runs.
// ------------------------------------------------------------------
__global__ void k_pitch(const double* __restrict__ src, double* __restrict__ dst, long long rows,
                        int ext, int pitch, int to_device) {
  // row r of the dense chunk <-> device row r after the chunk's first row;
  // the device-side pointer is the start of that first row
  // (device rows of consecutive planes are pitch apart too: plane stride = ext * pitch)
  for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
    const long long drow = r * pitch + COL_OFF;
    for (int c = threadIdx.x; c < ext; c += blockDim.x) {
      if (to_device)
        dst[drow + c] = src[r * ext + c];
      else
        dst[r * ext + c] = src[drow + c];
    }
  }
}

class HostPool {
 public:
  explicit HostPool(int n) : n_(n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  int size() const { return n_; }
  // run f(worker) on every worker, return when all finished
  void run(const std::function<void(int)>& f) {
    std::unique_lock<std::mutex> lk(m_);
    job_ = &f;
    pending_ = n_;
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int i) {
    unsigned seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      const std::function<void(int)>* f = job_;
      lk.unlock();
      (*f)(i);
      lk.lock();
      if (--pending_ == 0) done_.notify_all();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int pending_ = 0;
  unsigned gen_ = 0;
};

HostPool& host_pool() {
  // leaked on purpose: workers block in a condition wait at process exit;
  // PSG_HOST_THREADS overrides the size (default: three quarters of the
  // hardware threads, 2 .. 12; scripts/xfer_probe.py on the 16-thread GPU
  // hosts: staged downloads 40-53 GB/s with 8 threads, a steady 53 with 12)
  static HostPool* p = [] {
    int n = (int)std::max(2u, std::min(12u, std::thread::hardware_concurrency() * 3 / 4));
    if (const char* e = std::getenv("PSG_HOST_THREADS")) n = std::max(1, std::min(64, std::atoi(e)));
    return new HostPool(n);
  }();
  return *p;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  HostPool& hp = host_pool();
  const size_t nt = (size_t)hp.size();
  if (bytes < (4u << 20)) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t piece = ((bytes + nt - 1) / nt + 4095) & ~size_t(4095);
  hp.run([&](int i) {
    const size_t lo = (size_t)i * piece;
    if (lo >= bytes) return;
    std::memcpy((char*)dst + lo, (const char*)src + lo, std::min(piece, bytes - lo));
  });
}

constexpr size_t XFER_CHUNK = 32u << 20;   // bytes per chunk

struct XferBufs {
  double* dscratch[2] = {nullptr, nullptr};   // device, per slab stream use
  double* hstage[2] = {nullptr, nullptr};     // pinned host
  cudaEvent_t ev[2] = {nullptr, nullptr};
};

// per-device transfer buffers, created on first use and kept for the process
XferBufs* xfer_bufs(int dev) {
  static XferBufs* bufs[64] = {};
  static std::mutex m;
  std::lock_guard<std::mutex> lk(m);
  XferBufs*& b = bufs[dev & 63];
  if (b) return b;
  XferBufs* x = new XferBufs();
  for (int i = 0; i < 2; ++i) {
    if (cudaMalloc(&x->dscratch[i], XFER_CHUNK) != cudaSuccess ||
        cudaHostAlloc(&x->hstage[i], XFER_CHUNK, cudaHostAllocPortable) != cudaSuccess ||
        cudaEventCreateWithFlags(&x->ev[i], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
  }
  b = x;
  return b;
}

bool host_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

std::mutex& xfer_mutex() {
  static std::mutex m;
  return m;
}

// dense host planes [count][ext][ext] <-> device planes first.. (pitched)
int transfer_planes(psg_slab* s, double* dev, double* host, int64_t first, int64_t count,
                    bool to_device) {
  if (first < 0 || first + count > s->planes || count < 0)
    return fail(PSG_ERR_CONFIG, "plane range outside the slab");
  if (count == 0) return PSG_OK;
  {
    // dense planes already in device memory: one re-pitch kernel, no copies
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, host) == cudaSuccess &&
        (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged)) {
      if (at.type == cudaMemoryTypeDevice && at.device != s->device)
        return fail(PSG_ERR_CONFIG, "dense device planes must be on the slab's device");
      const int64_t rows = count * s->ext;
      double* drow0 = dev + first * s->plane_stride;
      const int grid = (int)std::min<int64_t>(rows, (int64_t)s->sm_count * 16);
      if (to_device)
        k_pitch<<<grid, 256, 0, s->stream>>>(host, drow0, rows, (int)s->ext, (int)s->pitch, 1);
      else
        k_pitch<<<grid, 256, 0, s->stream>>>(drow0, host, rows, (int)s->ext, (int)s->pitch, 0);
      CU_TRY(cudaGetLastError());
      CU_TRY(cudaStreamSynchronize(s->stream));
      return PSG_OK;
    }
    cudaGetLastError();
  }
  std::lock_guard<std::mutex> lk(xfer_mutex());   // one user of the shared buffers at a time
  XferBufs* x = xfer_bufs(s->device);
  if (!x) return fail(PSG_ERR_CUDA, "transfer buffers: allocation failed");
  const int64_t ext = s->ext;
  const int64_t rows_total = count * ext;
  const int64_t rows_chunk = std::max<int64_t>(1, (int64_t)(XFER_CHUNK / (ext * 8)));
  const bool pinned = host_pinned(host);
  double* dbase = dev + first * s->plane_stride;
  const int64_t nchunk = (rows_total + rows_chunk - 1) / rows_chunk;
  auto rows_of = [&](int64_t c) { return std::min(rows_chunk, rows_total - c * rows_chunk); };
  auto pitch_launch = [&](int64_t c, double* dsc) {
    const int64_t r0 = c * rows_chunk;
    const int64_t nr = rows_of(c);
    // device rows of the chunk start at plane r0 / ext, row r0 % ext; rows
    // are consecutive in (plane, row) order, so offset by whole rows
    const int64_t p0 = r0 / ext, j0 = r0 % ext;
    double* drow0 = dbase + p0 * s->plane_stride + j0 * s->pitch;
    const int grid = (int)std::min<int64_t>(nr, (int64_t)s->sm_count * 16);
    if (to_device)
      k_pitch<<<grid, 256, 0, s->stream>>>(dsc, drow0, nr, (int)ext, (int)s->pitch, 1);
    else
      k_pitch<<<grid, 256, 0, s->stream>>>(drow0, dsc, nr, (int)ext, (int)s->pitch, 0);
  };
  if (to_device) {
    for (int64_t c = 0; c < nchunk; ++c) {
      const int b = (int)(c & 1);
      const size_t bytes = (size_t)rows_of(c) * ext * 8;
      const double* src = host + c * rows_chunk * ext;
      if (pinned) {
        CU_TRY(cudaMemcpyAsync(x->dscratch[b], src, bytes, cudaMemcpyHostToDevice, s->stream));
      } else {
        CU_TRY(cudaEventSynchronize(x->ev[b]));   // staging buffer b free again
        par_memcpy(x->hstage[b], src, bytes);
        CU_TRY(cudaMemcpyAsync(x->dscratch[b], x->hstage[b], bytes, cudaMemcpyHostToDevice, s->stream));
        CU_TRY(cudaEventRecord(x->ev[b], s->stream));
      }
      pitch_launch(c, x->dscratch[b]);
      CU_TRY(cudaGetLastError());
    }
  } else {
    for (int64_t c = 0; c <= nchunk; ++c) {
      if (c < nchunk) {
        const int b = (int)(c & 1);
        const size_t bytes = (size_t)rows_of(c) * ext * 8;
        pitch_launch(c, x->dscratch[b]);
        CU_TRY(cudaGetLastError());
        if (pinned) {
          CU_TRY(cudaMemcpyAsync(host + c * rows_chunk * ext, x->dscratch[b], bytes,
                                 cudaMemcpyDeviceToHost, s->stream));
        } else {
          CU_TRY(cudaMemcpyAsync(x->hstage[b], x->dscratch[b], bytes, cudaMemcpyDeviceToHost,
                                 s->stream));
          CU_TRY(cudaEventRecord(x->ev[b], s->stream));
        }
      }
      if (!pinned && c >= 1) {   // host copy of the previous chunk while this one moves
        const int64_t pc = c - 1;
        const int pb = (int)(pc & 1);
        CU_TRY(cudaEventSynchronize(x->ev[pb]));
        par_memcpy(host + pc * rows_chunk * ext, x->hstage[pb], (size_t)rows_of(pc) * ext * 8);
      }
    }
  }
  CU_TRY(cudaStreamSynchronize(s->stream));
  return PSG_OK;
}

// contiguous device <-> host copy through the staging engine (pageable host
// memory at full link rate); dev on `device`
int copy_host(int device, void* dev, void* host, size_t bytes, bool to_device) {
  if (bytes == 0) return PSG_OK;
  CU_TRY(cudaSetDevice(device));
  if (host_pinned(host)) {
    CU_TRY(cudaMemcpy(to_device ? dev : host, to_device ? host : dev, bytes,
                      to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost));
    return PSG_OK;
  }
  std::lock_guard<std::mutex> lk(xfer_mutex());
  XferBufs* x = xfer_bufs(device);
  if (!x) return fail(PSG_ERR_CUDA, "transfer buffers: allocation failed");
  cudaStream_t st = nullptr;
  CU_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const size_t nchunk = (bytes + XFER_CHUNK - 1) / XFER_CHUNK;
  auto len = [&](size_t c) { return std::min(XFER_CHUNK, bytes - c * XFER_CHUNK); };
  int rc = PSG_OK;
  for (size_t c = 0; c <= nchunk && !rc; ++c) {
    if (c < nchunk) {
      const int b = (int)(c & 1);
      char* d = (char*)dev + c * XFER_CHUNK;
      if (to_device) {
        if (cudaEventSynchronize(x->ev[b]) != cudaSuccess) rc = PSG_ERR_CUDA;
        par_memcpy(x->hstage[b], (char*)host + c * XFER_CHUNK, len(c));
        if (cudaMemcpyAsync(d, x->hstage[b], len(c), cudaMemcpyHostToDevice, st) != cudaSuccess)
          rc = PSG_ERR_CUDA;
      } else if (cudaMemcpyAsync(x->hstage[b], d, len(c), cudaMemcpyDeviceToHost, st) != cudaSuccess) {
        rc = PSG_ERR_CUDA;
      }
      if (!rc && cudaEventRecord(x->ev[b], st) != cudaSuccess) rc = PSG_ERR_CUDA;
    }
    if (!to_device && c >= 1 && !rc) {
      const size_t pc = c - 1;
      const int pb = (int)(pc & 1);
      if (cudaEventSynchronize(x->ev[pb]) != cudaSuccess) rc = PSG_ERR_CUDA;
      par_memcpy((char*)host + pc * XFER_CHUNK, x->hstage[pb], len(pc));
    }
  }
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = PSG_ERR_CUDA;
  cudaStreamDestroy(st);
  if (rc) return fail(PSG_ERR_CUDA, "staged copy failed");
  return PSG_OK;
}

int upload_planes(psg_slab* s, double* dev, const double* host, int64_t first, int64_t count) {
  return transfer_planes(s, dev, const_cast<double*>(host), first, count, true);
}

// singularity check of uploaded potential planes on the device (first site
// in C order like np.argwhere) and the coefficient range flag
int check_potential(psg_slab* s, int64_t first, int64_t count, int64_t* bad_site) {
  unsigned long long* d = nullptr;
  CU_TRY(cudaMallocAsync((void**)&d, 2 * sizeof(unsigned long long), s->stream));
  CU_TRY(cudaMemsetAsync(d, 0xff, sizeof(unsigned long long), s->stream));
  CU_TRY(cudaMemsetAsync(d + 1, 0, sizeof(unsigned long long), s->stream));
  k_singular<<<s->sm_count * 8, 256, 0, s->stream>>>(s->v, 0.5 * s->dtau, (int)s->ext,
                                                     (int)s->pitch, s->plane_stride, (int)first,
                                                     (int)count, s->x_lo - 1 + first, d,
                                                     reinterpret_cast<unsigned*>(d + 1));
  CU_TRY(cudaGetLastError());
  unsigned long long res[2] = {0, 0};
  CU_TRY(cudaMemcpyAsync(res, d, sizeof(res), cudaMemcpyDeviceToHost, s->stream));
  CU_TRY(cudaFreeAsync(d, s->stream));
  CU_TRY(cudaStreamSynchronize(s->stream));
  const unsigned long long bad = res[0];
  // sticky until a whole-slab upload: a partial upload keeps earlier planes
  if (first == 0 && count == s->planes) s->v_wide = res[1] != 0;
  else s->v_wide = s->v_wide || res[1] != 0;
  if (bad != ~0ull) {
    const long long e = s->ext;
    if (bad_site) {
      bad_site[0] = (int64_t)(bad / (e * e));
      bad_site[1] = (int64_t)((bad / e) % e);
      bad_site[2] = (int64_t)(bad % e);
    }
    return fail(PSG_ERR_SINGULAR, "1 + (dtau/2) V = 0");
  }
  return PSG_OK;
}
