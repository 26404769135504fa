/* dexel.h -- C ABI of the B200 dexel offset library (libdexel.so).
 *
 * Hot path of arXiv 1804.08968 "Half-Space Power Diagrams and Discrete
 * Surface Offsets": the separable two-pass dilation / erosion of a 3D dexel
 * buffer, plus the shell D \ E.
 *
 * Data model ("a set of parallel segments arranged in a 2D
 * grid, where each cell S_ij ... contains a list of segments"): an nx x ny
 * grid of columns; column c = j*nx + i (i fastest) holds a canonical list of
 * CLOSED intervals [z_in, z_out] along z, strictly increasing
 * (z_in_0 < z_out_0 < z_in_1 < ...), fp32, in a LOCAL frame z - z_ref chosen
 * by the caller (reading R9), all inside the domain [z_lo, z_hi].
 * The domain U = grid footprint x [z_lo, z_hi] is also the complement domain
 * (neutral boundary, reading R6): out-of-grid columns are absent,
 * dilations are clipped to U, erosion is U \ D_r(U \ S).
 *
 * Every call returns dexel_status (0 = OK); nothing throws across the ABI.
 * On error, dexel_last_error() (thread-local) describes the failure.
 * One handle = one grid (or one y-slab of it) on one device and one stream;
 * handles are not re-entrant.  All device work is stream-ordered on the
 * handle's stream; calls that return sizes to the host synchronise it.
 */
#ifndef DEXEL_H
#define DEXEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dexel_grid_s* dexel_grid;

typedef enum {
  DEXEL_OK = 0,
  DEXEL_EINVAL = 1,     /* invalid argument or invalid input data */
  DEXEL_ENOMEM = 2,     /* device allocation failed */
  DEXEL_EMISMATCH = 3,  /* src/dst geometry differs */
  DEXEL_EOVERFLOW = 4,  /* caller buffer too small (see dexel_size) or a column exceeds a kernel limit */
  DEXEL_ECUDA = 5,      /* CUDA runtime error */
  DEXEL_ENCCL = 6       /* NCCL error (multi-GPU) */
} dexel_status;

typedef struct {
  int32_t nx, ny;       /* global grid columns, >= 1 */
  double spacing;       /* lateral dexel spacing s > 0 (1.0 in all configs) */
  double z_ref;         /* world z of local value 0 (informational; all data are local) */
  float z_lo, z_hi;     /* domain in the local frame, finite, z_lo < z_hi */
  int32_t device;       /* CUDA ordinal */
  void* stream;         /* cudaStream_t; NULL -> library-owned stream */
  void* nccl_comm;      /* ncclComm_t of the nranks slab owners (multi-GPU, see below) or NULL */
  int32_t rank, nranks; /* slab owner; 0,1 for a single GPU */
  int32_t y0, y1;       /* owned global rows [y0,y1); 0,ny for a single GPU */
} dexel_desc;

/* Multi-GPU y-slabs ("the 2D dilations can be
 * performed completely independently in every slice"): rank g owns rows
 * [y0, y1) of the global grid; the ranks' slabs tile [0, ny) in rank order.
 * Pass 1 runs along x and is row-local; pass 2 runs along y and needs
 * R = floor(r/s) rows of INPUT beyond each slab boundary (the halo).  An op on a
 * slab reads rows [y0 - hlo, y1 + hhi) and writes [y0, y1); outputs of all slabs
 * concatenated are bitwise equal to the single-GPU output (per-column results do
 * not depend on the partition).  Three ways to supply the halo rows:
 *   - NCCL (desc.nccl_comm != NULL, nranks > 1): every op is COLLECTIVE -- all
 *     ranks call it with the same radii -- and exchanges the halo rows itself:
 *     ncclSend/ncclRecv with ranks g-1 and g+1 on an internal stream, interval
 *     counts first (one host synchronisation: allocation sizes), then offsets
 *     and endpoints, overlapped with pass 1 of the slab's own rows.  The first
 *     op on a handle gathers every rank's [y0, y1) (ncclAllGather); a partition
 *     that does not tile [0, ny), or a slab shorter than the rows a neighbour
 *     needs from it, fails with DEXEL_EINVAL on every rank alike.  Bootstrap:
 *     dexel_nccl_unique_id on one rank, broadcast the 128 bytes (e.g. with
 *     torch.distributed), dexel_nccl_comm_init on every rank.
 *   - loopback (dexel_link_slabs): slab handles of ONE process (one device or
 *     peer devices) fetch their halo rows from the linked neighbour handles with
 *     device copies -- the same pass-1 split and halo layout as NCCL (tests).
 *   - caller-managed (nccl_comm NULL, not linked): the caller moves the rows,
 *     dexel_download_rows packs owned boundary rows as a CSR slice and
 *     dexel_upload_halo attaches a neighbour's rows below (side 0) or above
 *     (side 1) the slab; an op fails with DEXEL_EINVAL if a halo is shorter than
 *     min(R, rows to the grid edge). */

/* NCCL bootstrap helpers (the library links the NCCL 2.28 that PyTorch bundles). */
dexel_status dexel_nccl_unique_id(uint8_t id[128]);                 /* ncclGetUniqueId */
/* ncclCommInitRank on `device` (collective over the nranks callers); *comm receives the
 * ncclComm_t to put in dexel_desc.nccl_comm.  It must outlive the handles using it. */
dexel_status dexel_nccl_comm_init(const uint8_t id[128], int nranks, int rank, int device, void** comm);
dexel_status dexel_nccl_comm_destroy(void* comm);                   /* NULL-safe */

/* Loopback halo transport: slabs[q] must be the handle of rank q of n (desc.rank = q,
 * desc.nranks = n, nccl_comm NULL), all of one grid, rows tiling [0, ny) in order.
 * Later ops on any of them fetch halo rows from the linked neighbours (which must hold their
 * inputs and not be running ops at the time).  Destroying a handle unlinks it. */
dexel_status dexel_link_slabs(dexel_grid* slabs, int n);

/* Create an empty grid (all columns empty).  *out receives the handle. */
dexel_status dexel_create(const dexel_desc* d, dexel_grid* out);

/* Replace the grid contents with a canonical CSR of the handle's local rows.
 *   offsets:   uint64[ncols_local + 1], offsets[0] = 0, non-decreasing,
 *              offsets[ncols_local] = n_intervals  (ncols_local = nx*(y1-y0))
 *   endpoints: float[2*n_intervals], (z_in, z_out) pairs, local frame
 *   src_on_device: 0 -> host pointers (pageable or pinned), 1 -> device pointers
 *              (read only during the call, stream-ordered).
 * Validation (on the device): per column strictly increasing, finite, inside
 * [z_lo, z_hi]; offsets monotone.  Failure -> DEXEL_EINVAL, last_error names
 * the first bad column, the grid is left unchanged.  Synchronises the stream. */
dexel_status dexel_upload(dexel_grid g, const uint64_t* offsets, const float* endpoints,
                          uint64_t n_intervals, int src_on_device);

/* dst := D_r(src): Eq. 1 on the ray lattice, computed by
 * the two passes (pass 1 along x: closest-parent extrusion P:494-501; pass 2
 * along y: power dilation with weights r^2 - d^2), clipped to U.
 * r finite, >= 0; R = floor(r/spacing) <= 255.  src and dst must share the
 * geometry (EMISMATCH) and differ (EINVAL).  dst is replaced; on error it is
 * left empty.  Output is canonical and bitwise deterministic.  Host
 * synchronisations: the op reads allocation sizes and capacity flags back from
 * the device (DESIGN.md "Host synchronisations" lists them; a y-slab with an
 * NCCL communicator adds one for the halo sizes).  The stream is otherwise not
 * synchronised: the op's last kernels may still run when it returns. */
dexel_status dexel_dilate(dexel_grid src, float r, dexel_grid dst);

/* dst := E_r(src) = U \ D_r(U \ src).  Same rules. */
dexel_status dexel_erode(dexel_grid src, float r, dexel_grid dst);

/* dst := D_rout(src) \ E_rin(src) = D_rout(src) n D_rin(U \ src), per column
 * (the thick shell of PAPER.md:58-61, :847-849).  Same rules. */
dexel_status dexel_shell(dexel_grid src, float r_out, float r_in, dexel_grid dst);

/* Morphological compositions (the next item of the survey's scope, SURVEY.md 8(f);
 * PAPER.md:241 "erosion ... dilation of the complement", :841-842 topological cleaning):
 *   dexel_open:  dst := D_r(E_r(src))   (removes features thinner than 2r)
 *   dexel_close: dst := E_r(D_r(src))   (fills gaps and holes narrower than 2r)
 * computed as two ops through an internal temporary handle on src's stream.  With the
 * neutral boundary (R6), open(S) <= S <= close(S) and both are idempotent up to
 * fp32 rounding.  Same argument rules as dexel_dilate.  On y-slabs with an NCCL communicator the
 * intermediate's halo rows are exchanged like any input (collective); other y-slab handles
 * (loopback, caller-managed) return DEXEL_EINVAL (compose the ops with an exchange between). */
dexel_status dexel_open(dexel_grid src, float r, dexel_grid dst);
dexel_status dexel_close(dexel_grid src, float r, dexel_grid dst);

/* 2D slice offsets (PAPER.md:422-487 the 2D uniform offset of a slice,
 * :584 "the 2D dilations can be performed completely independently in every slice"): every
 * grid row j is one 2D slice -- its columns along x, segments along z -- and is offset on its
 * own, by a disk of radius r in the (x, z) plane:
 *   dexel_dilate_slices:  dst row j := D_r(src row j)           (Eq. 1 restricted to the plane)
 *   dexel_erode_slices:   dst row j := E_r(src row j) = U_j \ D_r(U_j \ src row j)
 *   dexel_shell_slices:   dst row j := D_rout(row j) \ E_rin(row j)
 * Each equals the 3D op on a grid with the single row j (reading R6 per slice).
 * Computed as pass 1 along x and the level set L_0 alone (no pass along y, no halo: a y-slab
 * handle needs no dexel_upload_halo).  Same argument rules as dexel_dilate. */
dexel_status dexel_dilate_slices(dexel_grid src, float r, dexel_grid dst);
dexel_status dexel_erode_slices(dexel_grid src, float r, dexel_grid dst);
dexel_status dexel_shell_slices(dexel_grid src, float r_out, float r_in, dexel_grid dst);

/* GPU dexelisation of analytic solids (PAPER.md:114-118 dexel buffers,
 * :42 / :170 CSG in dexel space): replace g's contents (its rows [y0, y1)) with the solid
 *   (U spheres/boxes of sign +1) \ (U spheres/boxes of sign -1)
 * rasterised onto the ray lattice (column (i,j) at ((i+1/2)s, (j+1/2)s), s = 1):
 *   sph:      double[nsph][4]  (cx, cy, cz, R), world coordinates; sph_sign int32[nsph] (+1 / -1)
 *   box:      double[nbox][6]  (x0, x1, y0, y1, z0, z1), z0 <= z1; a column is inside when its
 *             centre is in [x0,x1] x [y0,y1]; box_sign int32[nbox]
 *   zmin, zmax: the world z domain; the handle's frame must be z_ref = (zmin+zmax)/2,
 *             z_lo = fl32(zmin - z_ref), z_hi = fl32(zmax - z_ref) (else DEXEL_EINVAL)
 *   src_on_device: 0 host / 1 device arrays (read during the call).
 * Per column in fp64 without contraction: sphere chords [cz -+ sqrt(R^2 - dy^2 - dx^2)], the
 * unions of closed chords per sign, their difference, clipped to [zmin, zmax], shifted to the
 * local frame, rounded to fp32 and canonicalised -- bitwise the host generator
 * (dexelgen/dexelgen.c) that builds the configs.  Columns with more than 64 disjoint chord
 * intervals per sign or 32 output intervals make the library rasterise once more with large
 * capacities (512 per sign; min(512, 2^30 / columns), at least 32, output intervals); a column
 * beyond those -> DEXEL_EOVERFLOW (grid unchanged).
 * Synchronises the stream. */
dexel_status dexel_rasterize_shapes(dexel_grid g, double zmin, double zmax, int nsph, const double* sph,
                                    const int32_t* sph_sign, int nbox, const double* box,
                                    const int32_t* box_sign, int src_on_device);

/* GPU dexelisation of the noisy gyroid (BASELINE.json configs[2]; the
 * implicit-solid case of PAPER.md:114-118 dexel buffers): g's rows := the solid
 * F + eps - t > 0, F = sin X cos Y + sin Y cos Z + sin Z cos X, X = 2 pi x / period (same for
 * Y, Z), column (i, j) at x = i + 1/2, y = j + 1/2 (global row j).  F + eps is sampled at
 * z = zmin + m + 1/2, m = 0 .. zmax - zmin - 1, eps = amp (2u - 1) with u the counter generator's
 * uniform (splitmix64 keyed by (seed, stream 6, column * nz + m)); endpoints are the linear roots
 * between samples, the field held beyond the first / last sample.  Per column in fp64 without
 * contraction (sin / cos from the host libm), clipped, shifted to the local frame, rounded to
 * fp32 and canonicalised: bitwise the host generator (dexelgen.c dexelgen_gyroid).
 *   zmin, zmax: integers, 0 <= zmin < zmax, giving the handle's frame (as dexel_rasterize_shapes);
 *   period > 0, t finite, amp >= 0 (else DEXEL_EINVAL, grid unchanged).
 * Two launches (count, scan, fill): no per-column capacity.  Synchronises the stream. */
dexel_status dexel_rasterize_gyroid(dexel_grid g, double zmin, double zmax, double period, double t, double amp,
                                    uint64_t seed);

/* Attach halo rows (multi-GPU slabs): side 0 = the nrows global rows directly
 * below y0, side 1 = the nrows rows directly above y1 (row-major CSR of
 * nrows*nx columns, same conventions and validation as dexel_upload).  nrows
 * = 0 removes the halo.  Synchronises the stream. */
dexel_status dexel_upload_halo(dexel_grid g, int side, const uint64_t* offsets, const float* endpoints,
                               int nrows, uint64_t n_intervals, int src_on_device);

/* Copy local rows [row_begin, row_begin+nrows) out as a CSR slice with offsets
 * rebased to 0 (offsets: nrows*nx+1 entries).  *n_intervals always receives
 * the slice size; offsets == NULL only queries it; capacity < size ->
 * DEXEL_EOVERFLOW.  Synchronises the stream. */
dexel_status dexel_download_rows(dexel_grid g, int row_begin, int nrows, uint64_t* offsets, float* endpoints,
                                 uint64_t capacity_intervals, uint64_t* n_intervals, int dst_on_device);

/* Number of intervals currently held (local slab). */
dexel_status dexel_size(dexel_grid g, uint64_t* n_intervals);

/* Copy the grid out as CSR (offsets: ncols_local+1 entries; endpoints:
 * 2*n floats).  capacity_intervals < n -> DEXEL_EOVERFLOW (nothing written).
 * dst_on_device: 0 host, 1 device pointers.  Synchronises the stream. */
dexel_status dexel_download(dexel_grid g, uint64_t* offsets, float* endpoints,
                            uint64_t capacity_intervals, int dst_on_device);

/* Pass 1 alone (the intermediate S_Mid of PAPER.md:494-501), exposed for
 * parity testing: for every column of src (or of U \ src when complement=1)
 * the closest-parent extrusion along x as maximal closed pieces
 * (lo, hi, kappa), kappa = min |dx| over parents within R = floor(r/s).
 *   offsets: uint64[ncols_local+1]; z: float[2*m]; kappa: uint8[m]
 * *n_pieces always receives m; capacity < m -> DEXEL_EOVERFLOW. */
dexel_status dexel_pass1(dexel_grid src, float r, int complement, uint64_t* offsets, float* z,
                         uint8_t* kappa, uint64_t capacity_pieces, uint64_t* n_pieces,
                         int dst_on_device);

/* Wait for all work queued on the handle's stream. */
dexel_status dexel_sync(dexel_grid g);

/* Destroy a handle and free its device memory (NULL-safe). */
void dexel_destroy(dexel_grid g);

/* Thread-local description of the last error ("" if none). */
const char* dexel_last_error(void);

/* Host-to-host ops, streamed in y-slabs ("the 2D dilations can be performed
 * completely independently in every slice", so rows [y0, y1) of the result need only input rows
 * [y0 - R, y1 + R)).  A pipeline cuts the grid into nslabs row slabs, each with its own pair of
 * device handles and its own stream; dexel_pipe_run uploads slab q+1 (its rows plus R halo rows
 * on each side, straight from the host CSR), runs the op on slab q (the same kernels as
 * dexel_dilate / dexel_erode / dexel_shell, caller-managed halo mode) and downloads the result
 * of slab q-1 at the same time, on three host threads.  The result is bitwise the one
 * dexel_upload + op + dexel_download of the whole grid gives.
 *   d:         the whole grid on one device (nranks 1, y0 0, y1 ny, nccl_comm NULL; d->stream unused)
 *   nslabs:    1..ny (1: no overlap).  From 3 slabs on the first and the last slab get half the
 *              rows of the others (the first upload and the last download are the copies no op
 *              hides); dexel_pipe_slab_rows reports the partition
 *   op:        0 dilate (r_a), 1 erode (r_a), 2 shell (r_a = r_out, r_b = r_in)
 *   offsets, endpoints: HOST canonical CSR of the whole grid (nx*ny + 1 offsets from 0; pinned memory
 *              lets the copies overlap the kernels, pageable memory works but serialises them)
 *   out_offsets: HOST uint64[nx*ny + 1]; out_endpoints: HOST float[2*capacity]
 *   *n_out:    the result's intervals; capacity < that -> DEXEL_EOVERFLOW (outputs partly written)
 * Input validation and error codes as dexel_upload / the ops; on error the outputs are undefined.
 * A pipeline is not re-entrant; it returns when the outputs are complete (no stream to wait on). */
typedef struct dexel_pipe_s* dexel_pipe;
dexel_status dexel_pipe_create(const dexel_desc* d, int nslabs, dexel_pipe* out);
dexel_status dexel_pipe_run(dexel_pipe p, int op, float r_a, float r_b, const uint64_t* offsets,
                            const float* endpoints, uint64_t* out_offsets, float* out_endpoints,
                            uint64_t capacity, uint64_t* n_out);
void dexel_pipe_destroy(dexel_pipe p);   /* NULL-safe */
/* Rows [y0, y1) of slab q (0 <= q < nslabs). */
dexel_status dexel_pipe_slab_rows(dexel_pipe p, int q, int32_t* y0, int32_t* y1);
/* Bytes the last dexel_pipe_run copied host -> device (every slab's offsets and endpoints, its
 * halo rows included) and device -> host (measurement). */
dexel_status dexel_pipe_last_bytes(dexel_pipe p, uint64_t* h2d_bytes, uint64_t* d2h_bytes);
/* The slab count measured best for grid d and radius r on B200: slabs of at least
 * max(512, 32 R) rows, R = floor(r/s), at most 6 slabs, and 1 for R < 8 (the op is then
 * shorter than its copies); 1 = do not split (use the serial calls). */
int dexel_pipe_suggest_slabs(const dexel_desc* d, float r);

/* Route device allocations through a caller allocator (e.g. the PyTorch
 * caching allocator).  NULL,NULL restores cudaMallocAsync/cudaFreeAsync.
 * Each buffer is released by the allocator that produced it, so the hook may
 * change while handles hold memory (the callbacks must outlive those buffers). */
typedef void* (*dexel_alloc_fn)(size_t bytes, int device, void* stream, void* ctx);
typedef void (*dexel_free_fn)(void* ptr, size_t bytes, int device, void* stream, void* ctx);
dexel_status dexel_set_allocator(dexel_alloc_fn alloc, dexel_free_fn free_, void* ctx);

/* Per-op statistics of the last op on handle g (for measurement):
 * n_in, n_mid (pass-1 pieces), n_lev (level-set intervals L_k), n_out; the
 * number of kernels the op launched; and, when timing is on
 * (dexel_set_timing(1)), the summed device time and launch count of each
 * kernel kind, measured with CUDA events on the handle's stream:
 *   0 pass1, 1 pass1 overflow (list) launches, 2 levels, 3 pass2,
 *   4 compaction, 5 scan, 6 other, 7 rasterisation (dexel_rasterize_shapes). */
#define DEXEL_NKERNELS 8
typedef struct {
  uint64_t n_in, n_mid, n_lev, n_out;
  uint32_t launches;
  uint32_t kernel_calls[DEXEL_NKERNELS];
  float kernel_ms[DEXEL_NKERNELS];
  /* capacities the op ran with: level slots per list,
   * pass-2 accumulator, number of row bands */
  uint32_t lev_cap, p2_acc, bands;
} dexel_stats;
dexel_status dexel_last_stats(dexel_grid g, dexel_stats* out);

/* Release the device's idle op workspace: the large temporaries ops
 * keep for reuse by later ops of any handle on the device (they are otherwise freed with the
 * device's last handle).  Blocks in use by a running op are kept; waits for the last use of
 * each freed block, and the device's stream-ordered pool is trimmed (its unused reserved memory
 * goes back to the driver; synchronises the device).  The band budget is re-queried. */
dexel_status dexel_trim_workspace(int device);

/* Enable (1) / disable (0) per-kernel CUDA-event timing for later ops
 * (process-wide; adds one event pair per launch and one sync per op). */
dexel_status dexel_set_timing(int on);

#ifdef __cplusplus
}
#endif
#endif /* DEXEL_H */
