/*
 * psigpu.h — C-ABI of the B200 (sm_100a) imaginary-time FDTD hot path.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `psibox` (/root/reference/pkg/src/psibox).  Plain pointers, sizes and int
 * status codes only; no torch or CUDA types appear in the signatures
 * (streams and device pointers travel as `void*` / `double*`).
 *
 * Two layers:
 *
 *  1. Operator layer (psg_kernel_*): one entry point per numba kernel of
 *     kernels.py.  Same argument meaning as the reference (host numpy
 *     arrays of shape (planes, ext, ext), C order, inclusive local plane
 *     range x_lo..x_hi, outputs written into caller-supplied arrays,
 *     padding never written).  Each call uploads, runs the CUDA kernel and
 *     downloads; it is the literal replacement a ctypes binding of
 *     `psibox.kernels` would make.
 *
 *  2. Engine layer (psg_*): a device-resident slab (one GPU, local planes
 *     0..W+1 of a lattice of N^3 interior sites) that keeps psi, V and the
 *     reduction scratch in HBM and runs sweeps, fused norm/observable
 *     reductions, parity imposition and trilinear resampling without
 *     host round trips.  It replaces the per-sweep body of
 *     evolve.SweepBuffers / evolve_to_convergence (evolve.py:160-272) and of
 *     parallel._worker_loop (parallel.py:393-506).
 *
 * Status codes map onto psibox.errors (errors.py:1-45) in the Python host:
 *   PSG_OK               0
 *   PSG_ERR_CONFIG       1  -> ConfigError
 *   PSG_ERR_CUDA         2  -> RuntimeError (CUDA failure; message in psg_last_error)
 *   PSG_ERR_ZERO_NORM    3  -> ZeroNormError
 *   PSG_ERR_DIVERGED     4  -> DivergenceError
 *   PSG_ERR_SINGULAR     5  -> SingularCoefficientError
 *   PSG_ERR_NO_DEVICE    6  -> RuntimeError (no CUDA device: there is no CPU fallback)
 */
#ifndef PSIGPU_H
#define PSIGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSG_OK 0
#define PSG_ERR_CONFIG 1
#define PSG_ERR_CUDA 2
#define PSG_ERR_ZERO_NORM 3
#define PSG_ERR_DIVERGED 4
#define PSG_ERR_SINGULAR 5
#define PSG_ERR_NO_DEVICE 6

/* sweep / reduction flags */
#define PSG_F_WRITE 1u   /* update psi (stencil_update) */
#define PSG_F_NORM 2u    /* per-plane sum of out^2 (norm_plane_sums on the output) */
#define PSG_F_MEASURE 4u /* per-plane num/den/r2 on the input (energy_ + radius2_plane_sums) */
#define PSG_F_CHECK 8u   /* flag non-finite outputs (evolve.step's isfinite check, evolve.py:49-52) */

/* reduction quantity slots in the plane-sum vectors */
#define PSG_Q_NUM 0
#define PSG_Q_DEN 1
#define PSG_Q_R2 2
#define PSG_Q_NORM 3

/* ------------------------------------------------------------------ */
/* misc                                                                 */
/* ------------------------------------------------------------------ */

/* ABI version of this header (bumped on any signature change). */
int psg_abi_version(void);
/* Thread-local message of the last failing call ("" when none). */
const char* psg_last_error(void);
/* Number of visible CUDA devices (0 on a machine without a GPU). */
int psg_device_count(void);

/* Device layout of a slab: [planes][ext][pitch] doubles, column of site k
 * at k + 3 so that interior rows start 32-byte aligned.  Returns the row
 * pitch (doubles) for a lattice of n interior sites per axis. */
int64_t psg_row_pitch(int64_t n);

/* Slab fields come from the device's stream-ordered memory pool and go back
 * to it on psg_destroy (cached for the next slab of the process); this
 * returns the cached memory of `device` to the driver. */
int psg_trim_memory(int device);

/* Contiguous copies between device memory (on `device`) and host memory at
 * link rate also for pageable host memory (pinned staging, host threads). */
int psg_copy_to_host(int device, void* host, const void* dev, int64_t bytes);
/* Page-locked host buffers, cached by size after release (downloads into them
 * run at link rate); NULL on failure. */
void* psg_host_alloc(int64_t bytes);
void psg_host_free(void* p, int64_t bytes);
int psg_copy_to_device(int device, void* dev, const void* host, int64_t bytes);

/* numpy.sum replica (pairwise, 8 accumulators, 128 blocks) on the device:
 * replaces observables.combine_plane_sums (observables.py:32-34) where the
 * combine must happen without a host round trip.  out[0] = sum(a[0..n)). */
int psg_pairwise_sum_device(const double* host_a, int64_t n, double* out);

/* Self-test of the sweep's shared-reciprocal coefficient division: compares
 * A = (1-hv)/(1+hv) and B = 1/(1+hv) against IEEE division for `count`
 * pseudo-random hv in [lo, hi); *mismatches = number of differing sites. */
int psg_selftest_division(int64_t count, uint64_t seed, double lo, double hi,
                          uint64_t* mismatches);

/* ------------------------------------------------------------------ */
/* 1. operator layer: kernels.py entry points on host arrays             */
/* ------------------------------------------------------------------ */

/* kernels.stencil_update(psi, coef_a, coef_c, out, x_lo, x_hi)  kernels.py:22-37
 * arrays are (planes, ext, ext) C-order fp64, ext = N+2. */
int psg_kernel_stencil_update(const double* psi, const double* coef_a, const double* coef_c,
                              double* out, int64_t planes, int64_t ext, int64_t x_lo,
                              int64_t x_hi);

/* Same update with A and C synthesised from V in-kernel (potential._coefficients
 * order, potential.py:102-115): 24 B/site instead of 32. */
int psg_kernel_stencil_update_v(const double* psi, const double* v, double dtau, double m,
                                double a, double* out, int64_t planes, int64_t ext,
                                int64_t x_lo, int64_t x_hi);

/* kernels.norm_plane_sums(psi, x_lo, x_hi, out)  kernels.py:40-49 */
int psg_kernel_norm_plane_sums(const double* psi, int64_t planes, int64_t ext, int64_t x_lo,
                               int64_t x_hi, double* out);

/* kernels.energy_plane_sums(psi, v, kin, x_lo, x_hi, num_out, den_out)  kernels.py:52-74 */
int psg_kernel_energy_plane_sums(const double* psi, const double* v, double kin, int64_t planes,
                                 int64_t ext, int64_t x_lo, int64_t x_hi, double* num_out,
                                 double* den_out);

/* kernels.radius2_plane_sums(psi, x_global0, center, a, x_lo, x_hi, r2_out, den_out)
 * kernels.py:77-100 */
int psg_kernel_radius2_plane_sums(const double* psi, int64_t x_global0, double center, double a,
                                  int64_t planes, int64_t ext, int64_t x_lo, int64_t x_hi,
                                  double* r2_out, double* den_out);

/* kernels.dot_plane_sums(psi1, psi2, x_lo, x_hi, out)  kernels.py:103-112 */
int psg_kernel_dot_plane_sums(const double* psi1, const double* psi2, int64_t planes,
                              int64_t ext, int64_t x_lo, int64_t x_hi, double* out);

/* ------------------------------------------------------------------ */
/* 2. engine layer: device-resident slab                                 */
/* ------------------------------------------------------------------ */

typedef struct psg_slab psg_slab;
typedef struct psg_comm psg_comm;

/* Create a slab on `device` for a lattice (N=n, a, m, dtau) owning the
 * global interior planes x_lo..x_lo+w-1 (1-based; w=n for one GPU).
 * Allocates psi (2 buffers), V and reduction scratch in HBM, all zeroed
 * (Dirichlet padding).  Mirrors evolve.SweepBuffers (evolve.py:160-166)
 * and parallel.Worker (parallel.py:125-176). */
int psg_create(int device, int64_t n, int64_t w, int64_t x_lo, double a, double m, double dtau,
               psg_slab** out);

/* psg_create with options.  PSG_CREATE_SINGLE_BUFFER (whole lattice only,
 * w == n): both psi "buffers" share one allocation of w + 4 + chunk + 2
 * planes instead of 2 (w + 4), the second shifted `chunk + 2` planes below
 * the first; every sweep / two-sweep pass runs as launches over `chunk`-plane
 * pieces, ascending into the lower buffer and descending into the upper one,
 * so no piece overwrites a plane a later piece still reads.  Results are
 * bitwise those of psg_create.  chunk = 0: ceil(w / 8).  A 2048^3 lattice
 * (psi 73.6 GB + V 69.1 GB) then fits one B200.  Not for psg_run_dist /
 * multi-slab runs (there each GPU holds a slab with its own halos).  Extends evolve.SweepBuffers (evolve.py:160-166), whose
 * two full buffers are the reference's memory layout. */
#define PSG_CREATE_SINGLE_BUFFER 1u
/* PSG_CREATE_IPC: psi buffers from cudaMalloc, exportable to the neighbouring
 * ranks' processes (psg_ipc_create). */
#define PSG_CREATE_IPC 2u
int psg_create_ex(int device, int64_t n, int64_t w, int64_t x_lo, double a, double m, double dtau,
                  unsigned flags, int64_t chunk, psg_slab** out);
int psg_destroy(psg_slab* s);

/* Device memory a new slab can use: free bytes plus the bytes the slabs'
 * memory pool holds unused; total = the device's memory. */
int psg_mem_info(int device, int64_t* avail, int64_t* total);

/* Host-side singular-coefficient scan (no GPU needed): *first_bad = the first
 * flat C-order index with 1 + h*v == 0 (h = dtau/2), or -1.  Replaces the
 * numpy scan of potential._coefficients (potential.py:102-110) at
 * PotentialGrid construction: multithreaded, no full-size temporaries. */
int psg_host_find_singular(const double* v, int64_t count, double h, int64_t* first_bad);

/* Device bytes held by the slab's psi buffers and V (fields only). */
int64_t psg_field_bytes(psg_slab* s);

/* The slab's CUDA stream (cudaStream_t as void*). */
void* psg_stream(psg_slab* s);
int psg_sync(psg_slab* s);

/* Geometry: pitch (doubles per row), plane stride (doubles), local planes (w+2). */
int psg_geometry(psg_slab* s, int64_t* pitch, int64_t* plane_stride, int64_t* planes);

/* Device pointer of local plane `p` (0..w+1) of the current psi buffer
 * (which=0) or the other buffer (which=1); plane is `plane_stride`
 * contiguous doubles.  Used by the host for halo exchange (NCCL). */
double* psg_plane_ptr(psg_slab* s, int which, int64_t p);

/* Upload `count` planes of a dense host field (ext x ext doubles each,
 * C order) into local planes first..first+count-1 of BOTH psi buffers and
 * reset the pending normalisation scale to 1.  Padding rows/cols are
 * copied as given (evolve.step carries padding over, evolve.py:45-53).
 * The dense planes (here and in psg_get_field / psg_set_potential) may also
 * be device memory on the slab's device: then no host copy is made. */
int psg_set_field(psg_slab* s, const double* host, int64_t first, int64_t count);

/* Download local planes first..first+count-1 of the current state,
 * materialised (pending normalisation applied, exactly psi *= f of
 * evolve.py:180). */
int psg_get_field(psg_slab* s, double* host, int64_t first, int64_t count);

/* Device-side inputs (no host copy of the field; 2048^3 runs):
 * psg_fill_uniform: the seeded U(-0.5, 0.5) start of every interior site of
 * the slab's planes, bitwise lattice.uniform_plane (numpy Philox4x64 keyed by
 * seed, plane i at counter block (i-1)*ceil(N^2/4)); padding zero; pending
 * normalisation reset.
 * psg_fill_potential: V on the slab's planes, kind 0 harmonic (0.5 r) r,
 * 1 Coulomb -1/max(r, a/2), 2 Cornell -alpha/max(r,a/2) + sigma max(r,a/2)
 * (params alpha, sigma), 3 harmonic plus 8 Gaussian wells (params: centres
 * [8][3] by storage axis, depths[8], widths[8]), 4 psibox coulomb (0 for
 * r < a, -1/r + 1/a beyond; potential.py:126-136), 5 psibox dodecahedron
 * (params: face normals[12][3], limit, depth; potential.py:165-183); r from
 * the lattice centre as in workloads.py / potential.py (bitwise, except the
 * wells' exp: <= 1 ulp per term), then
 * the same checks as psg_set_potential. */
int psg_fill_uniform(psg_slab* s, uint64_t seed);
/* Download potential planes (dense, like psg_get_field). */
int psg_get_potential(psg_slab* s, double* host, int64_t first, int64_t count);
int psg_fill_potential(psg_slab* s, int kind, const double* params, int nparams,
                       int64_t* bad_site);

/* Upload the potential for local planes first..first+count-1 (dense host
 * planes, ext x ext).  Returns PSG_ERR_SINGULAR and the offending global
 * site in bad_site[3] when 1 + (dtau/2) V == 0 (potential.py:103-110). */
int psg_set_potential(psg_slab* s, const double* host_v, int64_t first, int64_t count,
                      int64_t* bad_site);

/* Use streamed A/C coefficient arrays (psibox PotentialGrid.coef_a/coef_c)
 * instead of synthesising them from V (32 B/site path, kernels.py:37). */
int psg_set_coefficients(psg_slab* s, const double* host_a, const double* host_c, int64_t first,
                         int64_t count);

/* One sweep of local planes z_lo..z_hi (inclusive) from the current buffer
 * into the other one, with the fused reductions selected by flags
 * (PSG_F_WRITE | PSG_F_NORM | PSG_F_MEASURE).  Does not swap. */
int psg_sweep(psg_slab* s, int64_t z_lo, int64_t z_hi, unsigned flags);

/* Swap current/other buffers (SweepBuffers.sweep's swap, evolve.py:169).
 * `renorm`: the sweep just finished carried PSG_F_NORM and the next state
 * must be read through the factor produced by psg_reduce. */
int psg_swap(psg_slab* s, int renorm);

/* Reduce the tile partials of the last sweep (or psg_measure) for local
 * planes z_lo..z_hi into the global plane-sum vectors (slots PSG_Q_*, each
 * n doubles, zero outside the slab).  combine != 0 also runs the numpy
 * pairwise combine on the device and produces the scalars (totals, E,
 * norm2, r_rms, next normalisation factor). */
int psg_reduce(psg_slab* s, int64_t z_lo, int64_t z_hi, unsigned flags, int combine);

/* Device pointer of the plane-sum vectors [4][n] (for an all-reduce of
 * the zero-padded vectors across slabs). */
double* psg_plane_sums_ptr(psg_slab* s);

/* Zero the plane-sum vectors (before a slab's reduce + all-reduce). */
int psg_zero_sums(psg_slab* s);

/* Combine only (after an external all-reduce of the plane sums). */
int psg_combine(psg_slab* s, unsigned flags);

/* Copy the plane sums [4][n] and the scalars to the host:
 * scal[0..3] = totals (num, den, r2, norm), scal[4] = E, scal[5] = norm2
 * (den*a^3), scal[6] = r_rms, scal[7] = n2 (norm*a^3), scal[8] = next
 * factor 1/sqrt(n2), scal[9] = status (0 ok, 3 zero norm, 4 non-finite),
 * scal[12] = non-finite-output flag of the sweeps since psg_set_field. */
int psg_read_sums(psg_slab* s, double* plane_sums, double* scal);

/* Observables of the current state without updating it (energy_plane_sums +
 * radius2_plane_sums, observables.py:73-97), leaves partials for psg_reduce. */
int psg_measure(psg_slab* s, int64_t z_lo, int64_t z_hi);

/* Dot-product partials of the current state with a second slab's current
 * state (dot_plane_sums, kernels.py:103-112), into PSG_Q_NUM. */
int psg_dot(psg_slab* s, psg_slab* other, int64_t z_lo, int64_t z_hi);

/* Norm partials (sum psi^2 per tile, PSG_Q_NORM) of the current state
 * (norm_plane_sums, kernels.py:40-49), for psg_reduce(PSG_F_NORM). */
int psg_norm_partials(psg_slab* s, int64_t z_lo, int64_t z_hi);

/* Read the current state through the factor of the last combine from now on
 * (SweepBuffers.renormalize's psi *= 1/sqrt(n2), folded into the next read). */
int psg_use_factor(psg_slab* s);

/* Read the current state through an explicit factor (slab engine: the factor
 * is combined from all slabs' plane sums). */
int psg_set_factor(psg_slab* s, double factor);

/* psi_s <- psi_s - c * psi_o (both materialised), states._project_inplace
 * (states.py:92-99). */
int psg_axpy(psg_slab* s, psg_slab* o, double c);

/* Copy one local plane between slabs (same or peer device), ordered on the
 * destination stream after the source stream's pending work: the halo
 * exchange of the single-process slab engine (parallel.halo_step,
 * parallel.py:179-217). which: 0 current buffer, 1 other. */
int psg_copy_plane(psg_slab* dst, int dst_which, int64_t dst_plane, psg_slab* src, int src_which,
                   int64_t src_plane);

/* Apply the pending normalisation to the stored state (psi *= f). */
int psg_materialize(psg_slab* s);

/* Scale the stored state by an explicit factor (renormalize(), evolve.py:56-64). */
int psg_scale(psg_slab* s, double factor);

/* Reflection-parity imposition (axis 0 needs the whole lattice on the slab,
 * w == n; axes 1 and 2 act within every plane of any slab): mode 0 = copy (states.impose_inplace, states.py:70-82),
 * mode 1 = projector psi <- (psi + sign * R psi) * 0.5.  axis 0/1/2 is the
 * storage axis, sign = +1 / -1.  The pending scale is applied on the fly. */
int psg_impose(psg_slab* s, int axis, int sign, int mode);

/* Trilinear resampling (multires.resample, multires.py:116-154) of the
 * coarse slab's state into the fine slab's interior: per-axis coarse
 * padded indices i0 (lo = i0, hi = i0+1) and fractions for each fine site
 * (length fine n), computed by the host exactly as multires does.  The
 * fine slab must hold the whole fine lattice.  No renormalisation. */
int psg_resample(psg_slab* coarse, psg_slab* fine, const int64_t* i0, const double* frac);

/* Run parameters of the fused fixed-step driver (one GPU, w == n). */
typedef struct psg_run_params {
  int64_t steps;          /* sweeps to run */
  int64_t measure_every;  /* observables on the state entering sweep s when (s-1) % m == 0, s>1; 0 = never */
  int64_t norm_every;     /* renormalise after sweep s when s % k == 0; 0 = never */
  int64_t reimpose_every; /* impose the constraints after sweep s when s % r == 0; 0 = never */
  int64_t step_offset;    /* sweeps already done before this call (s counts from step_offset+1) */
  int32_t n_impose;       /* number of parity constraints (0..3), applied in order */
  int32_t impose_axis[3]; /* storage axis of each constraint */
  int32_t impose_sign[3]; /* +1 symmetric / -1 antisymmetric */
  int32_t flags;          /* PSG_RUN_* */
} psg_run_params;

/* psg_run flag: linear renormalisation pairs.  Two sweeps whose second is a
 * renormalisation step (and whose inner state is neither measured nor
 * re-imposed) run as one two-sweep HBM pass that applies the pending factor
 * at the store (S(f psi) = f S(psi) up to rounding) and fuses the NORM
 * partials of its output; the normalisation after the first sweep is
 * subsumed by the one after the second.  evolve_to_convergence's default
 * (renormalise every sweep, evolve.py:171-181) within roundoff, not bitwise
 * (whole-lattice slabs; ignored by the multi-slab drivers). */
#define PSG_RUN_LINEAR_NORM 1

/* psg_run flag: exact.  Every norm / measure step through the per-step path
 * (single sweeps; plane sums over the sweep's tiles: bitwise the same run on
 * any number of slabs).  Without it, a whole-lattice slab runs its norm /
 * measure steps inside the persistent brick kernel when N <= 64, N % 16 == 0
 * and nothing is re-imposed (option 15), else inside two-sweep passes
 * (option 16) -- within roundoff (1e-13 max|psi|) of the per-step path. */
#define PSG_RUN_EXACT 2

/* Fused fixed-step driver: runs the evolve_to_convergence loop body
 * (evolve.py:249-270) for `steps` sweeps without host round trips.
 * Measurement records go to hist (host, may be NULL): per check c,
 * hist[c*(3n+2)+0..] = step index, status, then 3n plane sums
 * (num | den | r2).  max_checks bounds the history. */
int psg_run(psg_slab* s, const psg_run_params* p, double* hist, int64_t max_checks,
            int64_t* n_checks);

/* --- multi-GPU (z-slabs, one process per GPU; parallel.py:413-485) ------
 * NCCL is loaded at run time (libnccl.so.2; the one PyTorch loaded when
 * present).  The 128-byte unique id of rank 0 reaches the other ranks through
 * the caller's own channel (torch.distributed broadcast). */
int psg_nccl_available(void);
int psg_nccl_unique_id(void* out128);
int psg_comm_create(int device, int nranks, int rank, const void* unique_id128, psg_comm** out);
int psg_comm_destroy(psg_comm* c);
/* planes sent by this rank so far (the reference's halo message counter) */
int64_t psg_comm_halo_messages(psg_comm* c);

/* psg_run for one slab of a z-decomposed lattice (the slab worker loop of
 * parallel.py:413-485 without host round trips): every sweep posts the
 * edge-plane send/recv to the neighbour ranks (left / right, -1 = lattice
 * boundary) on a communication stream, sweeps the interior planes meanwhile,
 * then the edge planes; reductions go into the zero-padded global plane-sum
 * vector, NCCL all-reduce (exact: one non-zero contributor per slot), combine
 * on the device; the factor is folded into the next sweep.  Bitwise equal to
 * the single-slab run for any slab count.  Parity constraints along the slab
 * axis are not supported here (PSG_ERR_CONFIG; the Python engine's mirror
 * exchange handles them). */
int psg_run_dist(psg_slab* s, psg_comm* c, int left, int right, const psg_run_params* p,
                 double* hist, int64_t max_checks, int64_t* n_checks);

/* psg_run for m slabs tiling one lattice in order (x_lo = 1, 1+W0, ...),
 * driven by this process: halos move by peer copies (cudaMemcpyPeerAsync:
 * NVLink between GPUs, a plain copy on one device), overlapped with the
 * interior updates; pairs of plain steps use two-sweep passes with two halo
 * planes per face.  Slabs may live on different devices.  Bitwise equal to
 * the single-slab run.  hist receives the records of slabs[0]. */
int psg_run_multi(psg_slab** slabs, int m, const psg_run_params* p, double* hist,
                  int64_t max_checks, int64_t* n_checks);

/* Observables of the slab's current state (halo exchange, measuring pass,
 * all-reduce, combine), as one history record of psg_run (3n+2 doubles). */
int psg_measure_dist(psg_slab* s, psg_comm* c, int left, int right, double* rec);
/* The same for m slabs driven by this process (psg_run_multi's transport). */
int psg_measure_multi(psg_slab** slabs, int m, double* rec);

/* Kernel tuning knobs (0 = automatic): sweep blocks per SM, z-chunk length
 * (planes per work item), pipeline depth (planes in flight per block: 4/6/8). */
int psg_tune(psg_slab* s, int blocks_per_sm, int zchunk, int stages);

/* Launch options: 0 = programmatic dependent launch between consecutive
 * kernels (default 1), 1 = tapered chunk tail (number of chunks re-cut into
 * quarter-size work items at the end of a sweep, default 0 = off), 2 =
 * alternate the z-march direction every sweep so a sweep starts on the planes
 * its predecessor wrote last, still in L2 (default 1; bitwise unchanged),
 * 3 = tile rows of the two-sweep pass, 8 (two blocks per SM) or 16 (one
 * block per SM, default; bitwise unchanged), 4 = always take the range-checked
 * coefficient path, 5 = TMA stages of the 16-row two-sweep pass (0 = automatic,
 * the default: 7 for 192 <= N <= 640, else 6; or 6, 7, 9; bitwise unchanged),
 * 6 = two-sweep passes alternate their chunk order (default 1),
 * 8 = work split of the two-sweep pass: 0 automatic (default), 1 round-robin
 * chunk items, 2 one contiguous (tile, plane) range per block (bitwise
 * unchanged), 9 = at most this many planes per two-sweep launch (0 = as
 * many as 32-bit output offsets allow, the default; slabs beyond that are
 * passed in several launches; bitwise unchanged), 11 = fused halo exchange of
 * in-process slabs (psg_run_multi, read from the first slab; default 1): each
 * two-sweep pass also stores its edge output planes into the neighbouring
 * slabs' halo planes through peer memory (NVLink between GPUs) instead of a
 * separate copy; needs W >= 4 and peer access, else the copies are used
 * (bitwise unchanged), 12 = persistent brick kernel (k_small2) for runs of plain
 * sweeps of a whole lattice with N <= 64, N % 16 == 0 (default 1; bitwise
 * unchanged), 14 = three sweeps per HBM pass (k_sweep3) for runs of plain
 * sweeps of a whole lattice (default 0: measured slower than the two-sweep
 * pass; bitwise unchanged), 15 = the persistent brick kernel
 * also runs the norm / measure steps of a run inside the launch (whole run
 * without re-imposition in one launch; plane sums over bricks instead of
 * tiles: within roundoff of the per-step path, not bitwise; default 1),
 * 16 = whole-lattice runs take their norm / measure steps inside two-sweep
 * passes: a pair ending on a normalisation as a renormalising pass, a pair
 * starting on a measured state as a measuring pass (its input's observables
 * in step 1, the pending factor applied at the store by linearity) -- within
 * roundoff of the per-step path, not bitwise; default 1. */
int psg_set_option(psg_slab* s, int option, int value);

/* Enable / disable two sweeps per HBM pass (temporal blocking) for pairs of
 * plain steps inside psg_run; default on for N >= 8 (faster at every size measured);
 * results are bitwise unchanged. */
int psg_set_temporal(psg_slab* s, int enable);

/* One two-sweep pass (k_sweep2b) over the slab's planes with the halos it
 * holds, then the buffer swap -- no exchange, no reductions; the pending
 * factor must be 1.  reserve_sms: SMs left idle (a distributed run leaves 8
 * to NCCL).  For timing a slab's pass on one GPU and for tests. */
int psg_pass(psg_slab* s, int reserve_sms);

/* NCCL-free slab transport between processes (one slab per process, one GPU
 * per process, GPUs with peer access; the replacement for parallel.py's
 * socket transport, parallel.py:179-255).  Two-sweep passes store their edge
 * planes straight into the neighbours' halo planes (peer memory, the fused
 * exchange); single sweeps pull the neighbours' edge planes; plane sums are
 * all-reduced through mailboxes in every rank's memory, summed in rank order
 * (exact, bitwise M-invariant); ordering by device counters that each rank's
 * stream waits on (cuStreamWaitValue64) -- no kernel waits for another rank.
 * Protocol: every rank psg_ipc_create()s (slab from PSG_CREATE_IPC) and
 * shares its PSG_IPC_HANDLE_BYTES handle; every rank gets all handles in rank
 * order and psg_ipc_connect()s; a host barrier; then psg_run_ipc /
 * psg_measure_ipc in lock step (same parameters on every rank); a host
 * barrier before psg_ipc_destroy. */
#define PSG_IPC_HANDLE_BYTES 256
typedef struct psg_ipc psg_ipc;
int psg_ipc_create(psg_slab* s, int rank, int nranks, void* handle_out, psg_ipc** out);
int psg_ipc_connect(psg_ipc* c, const void* all_handles);
int psg_ipc_destroy(psg_ipc* c);
int psg_run_ipc(psg_slab* s, psg_ipc* c, const psg_run_params* p, double* hist,
                int64_t max_checks, int64_t* n_checks);
int psg_measure_ipc(psg_slab* s, psg_ipc* c, double* rec);
/* Halo planes this slab's IPC runs delivered to its neighbours. */
int64_t psg_ipc_halo_planes(psg_slab* s);

/* Number of kernels this slab has launched so far. */
int64_t psg_launch_count(psg_slab* s);

/* Two-sweep passes of this slab that delivered its edge planes to the
 * neighbouring slabs by peer stores (option 11). */
int64_t psg_fused_pass_count(psg_slab* s);

#ifdef __cplusplus
}
#endif

#endif /* PSIGPU_H */
