/*
 * sht.h -- C-ABI of the B200-native spherical-harmonics transform step
 * (ESCAPE SH dwarf: inverse + direct transform on an octahedral TCo grid).
 *
 * Boundary.  The reference (/root/reference, package `haloflow`) has no
 * transform code: SPEC.md:20 puts "spectral-transform ... numerical
 * mathematics" out of scope, and the SH dwarf's step is only described in
 * PAPER.md:193-199 (Legendre + FFT + all-to-all every timestep) and modelled
 * as flows in collectives.py:96-117 / netsim.py:347-398.  The north star
 * (BASELINE.json) asks for "the CPU reference's Python transform API (setup
 * with truncation, grid and field count; inv_trans/dir_trans on field
 * batches)".  Each entry point below states which part of that API (or of the
 * reference's modelled transposition) it replaces.  Plain pointers and sizes
 * only; no torch types.  Python binds this with ctypes
 * (paper_1908_06097_b200/_lib.py); INTEGRATION.md shows the binding.
 *
 * Conventions (shared with oracle/sht_oracle.py):
 *   spectral field  : (T+1)(T+2) doubles, m-major, n ascending, re/im interleaved
 *   grid field      : NPTS doubles, rings north -> south, ring j point k at
 *                     longitude 2*pi*k/NLOEN_j
 *   batches         : field-major, [nfld][...] contiguous, 16-byte aligned
 *   distributed     : rank r holds the spectral coefficients of its zonal
 *                     wavenumbers m (ascending) and the grid points of its
 *                     ring pairs (north rings ascending, then their southern
 *                     mirrors in north->south order); sht_local_layout lists them.
 *
 * Errors.  Every int-returning call returns SHT_OK (0) or one of the codes
 * below; the message is in sht_last_error() (thread-local).  The codes map
 * onto the reference's error classes (errors.py:9-39): SHT_ERR_CONFIG ->
 * ConfigurationError, SHT_ERR_CUDA -> RuntimeError, SHT_ERR_COMM ->
 * ProtocolError.
 *
 * Threading.  One plan per process/GPU; a plan is not re-entrant.  All work
 * is stream-ordered on the caller's stream; there is no hidden host sync in
 * sht_inv_trans / sht_dir_trans.
 */
#ifndef SHT_H_
#define SHT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SHT_OK 0
#define SHT_ERR_CONFIG 1
#define SHT_ERR_CUDA 2
#define SHT_ERR_COMM 3

/* plan flags */
#define SHT_FLAG_RECOMPUTE_LEGENDRE 1 /* no stored P table: the polynomials are regenerated on the GPU every
                                       * transform (see the Legendre notes in DESIGN.md section 4) */
#define SHT_FLAG_PROFILE_PHASES 2     /* record CUDA events around every phase (sht_phase_ms) */

typedef struct sht_plan sht_plan;

/* Library version (major*10000 + minor*100 + patch). */
int sht_version(void);

/* Replaces the north star's "setup(truncation, grid, nfld)".
 * nloen: NDGL ring lengths (north first, north/south symmetric), or NULL for
 * the octahedral TCo grid (ndgl must then be 2*(truncation+1)).
 * nccl_unique_id: 128 bytes from sht_nccl_get_unique_id() on rank 0, shared
 * by the caller (torch.distributed); NULL when nranks == 1.
 * Replaces the modelled transposition set-up of collectives.build_alltoall
 * (collectives.py:96-117): the plan fixes the size matrix and rotated order,
 * and (nranks > 1) exchanges the CUDA IPC handles of its receive buffers
 * over NCCL.  Collective: every rank must call it. */
int sht_plan_create(int truncation, int ndgl, const int32_t* nloen, int nfld, int rank, int nranks,
                    const void* nccl_unique_id, int flags, sht_plan** out);

/* Replaces "inv_trans(spec)": spectral [nfld][nspec_re_local] -> grid
 * [nfld][npts_local], both device pointers, on `cuda_stream` (cudaStream_t,
 * NULL = legacy default stream). */
int sht_inv_trans(sht_plan* plan, const double* spec, double* grid, void* cuda_stream);

/* Replaces "dir_trans(grid)": grid [nfld][npts_local] -> spectral
 * [nfld][nspec_re_local]. */
int sht_dir_trans(sht_plan* plan, const double* grid, double* spec, void* cuda_stream);

/* Sizes of this rank's local arrays.  m_list (capacity T+1) receives the
 * rank's zonal wavenumbers ascending and n_m their count; ring_list (capacity
 * NDGL) receives the global ring indices (0-based, north first) in local
 * storage order and n_rings their count.  Any pointer may be NULL. */
int sht_local_layout(const sht_plan* plan, int64_t* nspec_re, int64_t* npts, int32_t* m_list, int32_t* n_m,
                     int32_t* ring_list, int32_t* n_rings);

/* Per-phase device times (ms) of the last sht_inv_trans + sht_dir_trans on a
 * plan created with SHT_FLAG_PROFILE_PHASES.  Order: [legendre_poly(setup),
 * inv_legendre, inv_alltoall, inv_fft, dir_fft, dir_alltoall, dir_legendre].
 * Synchronises on the recorded events. */
int sht_phase_ms(sht_plan* plan, float* ms, int n);

/* Same, averaged over the last `npairs` (<= 64) inverse+direct pairs.  A pair
 * is an sht_inv_trans followed by an sht_dir_trans. */
int sht_phase_ms_avg(sht_plan* plan, int npairs, float* ms, int n);

/* Algorithmic work of this rank per inverse+direct pair:
 * Legendre flops, FFT HBM bytes, all-to-all bytes sent to other ranks. */
int sht_work(const sht_plan* plan, double* legendre_flops, double* fft_bytes, double* a2a_bytes);

/* Number of libsht kernel launches one inverse+direct pair issues. */
int sht_kernel_launches(const sht_plan* plan, int* per_pair);

/* Transport of the grid <-> spectral transposition: bit 0 of *p2p = 1 when
 * the kernels store the Fourier rows straight into the peers' receive buffers
 * over NVLink (CUDA IPC mappings, flag handshakes; the default whenever every
 * rank can map every peer), 0 for NCCL grouped send/recv between the kernels
 * (SHT_TRANSPORT=nccl, or one rank); bit 1 = 1 when the Fourier-row buffers
 * use the field-blocked layout (64-field blocks; p2p past the remote-store
 * cliff, or SHT_ROW_LAYOUT=blocked). */
int sht_transport(const sht_plan* plan, int* p2p);

/* 128-byte NCCL unique id (call on rank 0 only). */
int sht_nccl_get_unique_id(void* out128);

/* Local release of the plan (no collective).  When nranks > 1 call
 * sht_plan_close instead, unless a peer has failed: a peer may still store
 * into this rank's receive buffers until it has passed close's barrier. */
void sht_plan_destroy(sht_plan* plan);

/* Collective teardown (nranks > 1): a barrier over the plan's communicator,
 * bounded by SHT_COMM_TIMEOUT_MS, then sht_plan_destroy.  Returns
 * SHT_ERR_COMM if a peer did not arrive (the plan is released either way).
 * Replaces nothing in the reference; its analogue is the router's
 * first-error abort (halo/router.py:124-126, 199-205). */
int sht_plan_close(sht_plan* plan);

/* Waits for `cuda_stream` (all transforms enqueued on it) with failure
 * detection: polls the stream, the p2p handshake error word (a handshake
 * waits at most SHT_COMM_TIMEOUT_MS, default 60000, for a peer) and NCCL's
 * asynchronous error.  timeout_ms <= 0 uses SHT_COMM_TIMEOUT_MS.  Returns
 * SHT_ERR_COMM (-> ProtocolError) if a peer failed or the wait timed out; the
 * communicator is then aborted.  Every sht_inv_trans / sht_dir_trans also
 * returns SHT_ERR_COMM once a handshake of the plan has timed out. */
int sht_wait(sht_plan* plan, void* cuda_stream, int timeout_ms);

const char* sht_last_error(void);

/* ---- host-only helpers (no GPU needed; used by the CPU test-suite) ---- */

/* Build every rank's plan tables on the host without touching the GPU
 * (layouts, partition, FFT plans, shared-memory fits); SHT_OK if
 * sht_plan_create would accept these arguments. */
int sht_plan_validate(int truncation, int ndgl, const int32_t* nloen, int nfld, int nranks);

/* Gaussian nodes of the northern hemisphere, pole -> equator (ndgl/2 each):
 * mu = sin(latitude), sint = cos(latitude), w = Gaussian weight. */
int sht_gauss_nodes(int ndgl, double* mu, double* sint, double* w);

/* Ownership used by a plan with `nranks` ranks: m_owner[T+1] (rank owning
 * zonal wavenumber m), ring_owner[ndgl/2] (rank owning northern ring i and
 * its southern mirror).  nloen may be NULL (octahedral). */
int sht_partition(int truncation, int ndgl, const int32_t* nloen, int nranks, int32_t* m_owner,
                  int32_t* ring_owner);

/* Size matrix of the grid <-> spectral transposition for `nranks` ranks, in
 * Fourier rows (one row = nfld x 4 doubles = 32*nfld bytes): rows[r*nranks + d]
 * = rows rank r sends to rank d in the inverse transform (the direct transform
 * sends the transpose).  This is the `sizes` argument of the reference's
 * collectives.build_alltoall (collectives.py:96) for this data path. */
int sht_alltoall_rows(int truncation, int ndgl, const int32_t* nloen, int nranks, int64_t* rows);

/* Issue order of rank `rank`'s transfers: peers[k] = (rank + k) % nranks, the
 * reference's ROTATED_CONCURRENT order (collectives.py:85-86). */
int sht_alltoall_order(int nranks, int rank, int32_t* peers);

/* FFT plan chosen for a ring of n points: number of radix stages written to
 * radices (capacity 32), transform length L (n, or the Bluestein length) and
 * whether Bluestein is used. */
int sht_fft_plan_info(int n, int32_t* radices, int32_t* nstages, int32_t* fft_len, int32_t* bluestein);

/* ---- 2-D grid-point layout: latitude bands x longitude
 * segments, and the second (TRGTOL / TRLTOG-style [domain: ecTrans]) transposition
 * between it and the ring-pair distribution of the FFTs ---- */

/* Use an nA x nB grid-point layout (nA * nB == nranks): rank a*nB + b holds, per
 * field, the points k in [floor(N_j b / nB), floor(N_j (b+1) / nB)) of every
 * ring j of latitude band a (contiguous global rings, north first, split where
 * the cumulative point count crosses a/nA of the total), rings ascending.
 * Allocates the plan's transposition buffers.  Call on every rank. */
int sht_plan_set_gp_layout(sht_plan* plan, int nA, int nB);

/* This rank's grid-point layout: points per field, its band's global rings
 * [band_lo, band_hi), its segment and the number of segments. */
int sht_gp_layout(const sht_plan* plan, int64_t* npts_gp, int32_t* band_lo, int32_t* band_hi, int32_t* segment,
                  int32_t* nsegments);

/* inv_trans / dir_trans with the grid in the grid-point layout
 * ([nfld][npts_gp] device buffers): the ring-pair transform plus the
 * ring <-> grid-point transposition (grouped NCCL send/recv, rotated order). */
int sht_inv_trans_gp(sht_plan* plan, const double* spec, double* grid_gp, void* cuda_stream);
int sht_dir_trans_gp(sht_plan* plan, const double* grid_gp, double* spec, void* cuda_stream);

/* Host-only: first global ring of each of the nA latitude bands (+ NDGL): band_lo[nA + 1]. */
int sht_gp_bands(int truncation, int ndgl, const int32_t* nloen, int nA, int32_t* band_lo);

/* ---- GPU halo engine: the reference's unstructured-grid
 * halo exchange and neighbourhood-mean stencil on device-resident fields ---- */
typedef struct sht_halo sht_halo;

/* One rank's exchange plan -- the reference's RankPlan (halo/plan.py:33-55):
 * send_counts[p] local owned indices to gather for peer p (send_index, peers
 * ascending, each list ascending in global order), recv_counts[p] ghost slots
 * the matching buffer from p scatters into (recv_slot).  The local array is
 * the owned elements then the ghosts (halo/partition.py:1-6).  Optional
 * stencil: ngroups degree groups (engine._stencil_ws), group g has
 * group_count[g] owned members and a [count][degree] row-major table of
 * their neighbours' local indices (ascending global order per row).
 * nccl_unique_id as for sht_plan_create (NULL when nranks == 1).  Collective.
 * Errors: SHT_ERR_CONFIG for an out-of-range plan (the reference raises
 * ProtocolError / ConfigurationError, plan.py:106-120, engine.py:126-139). */
int sht_halo_create(int rank, int nranks, const void* nccl_unique_id, int64_t n_local, int64_t n_owned,
                    const int64_t* send_counts, const int64_t* send_index, const int64_t* recv_counts,
                    const int64_t* recv_slot, int ngroups, const int32_t* group_degree, const int64_t* group_count,
                    const int64_t* members, const int64_t* neighbours, sht_halo** out);

/* Replaces engine.exchange (engine.py:197-220): refresh every ghost of
 * `values` (device, n_local doubles) with its owner's value -- pack, grouped
 * send/recv in the ROTATED_CONCURRENT order (engine.py:146-149), unpack.
 * Stream-ordered; bounded by SHT_COMM_TIMEOUT_MS on a dead peer. */
int sht_halo_exchange(sht_halo* halo, double* values, void* cuda_stream);

/* Replaces engine.stencil_step with OverlapMode.NONE (engine.py:301-327):
 * exchange, then owned[m] = mean of values[neighbours of m], accumulated in
 * the reference's order (bit-identical). */
int sht_halo_stencil_step(sht_halo* halo, double* values, void* cuda_stream);

/* Elements this rank sends / receives per exchange. */
int sht_halo_counts(const sht_halo* halo, int64_t* nsend, int64_t* nrecv);

void sht_halo_destroy(sht_halo* halo);

#ifdef __cplusplus
}
#endif

#endif /* SHT_H_ */
