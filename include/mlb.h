/* mlb.h - C ABI of the B200-native D3Q19 time-step loop (libmlb_d3q19.so).
 *
 * This is the drop-in boundary for the reference's plugin point
 * `KernelPlan(...).step(fpre, fpost)` and the engine loop around it
 * (reference = /root/reference/pkg/src/lb2d, cited as file:line below).
 * Plain pointers and sizes only; no torch / numpy types.  Every function
 * returns 0 on success or an MLB_E* code, with a human-readable message in
 * mlb_last_error() (thread-local).  `stream` arguments are cudaStream_t
 * values passed as void* (NULL = the legacy default stream).
 *
 * Memory model.  The CALLER owns every population buffer (in the Python
 * host: torch tensors; only data_ptr() crosses) - mirroring the reference,
 * where KernelPlan keeps no population copies (kernels.py:398-443).  The
 * plan owns only what it derives from the flags (a per-cell class word, the
 * inlet/outlet index lists), reduction scratch and two timing events.
 *
 * Host layout (what the reference passes): dense C-contiguous
 *   f[q][z][y][x],  q < 19, x fastest            ("(Q, N)" block)
 *   flags[z][y][x]  uint8, codes 0..4 (boundaries.py:20-24)
 * Device layout (mlb_layout): per population (nz + 2) z-planes - storage
 * plane 0 and nz+1 are halo planes, slab plane lz lives at storage lz+1 -
 * each plane ny rows of xp elements, xp = nx rounded up to a whole number
 * of 128-byte lines:
 *   element(q, x, y, lz) = q*pop + ((lz + 1)*ny + y)*xp + x
 */
#ifndef MLB_H
#define MLB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLB_ABI_VERSION 2
#define MLB_Q 19

/* dtype codes = the reference's Precision wire codes (fields.py:22-25):
 * single, double, mixed1 = populations STORED as IEEE binary16 and computed
 * in float (exact upcast on load, round-to-nearest-even on store,
 * kernels.py:435-455), mixed2 = stored as float, computed in double (every
 * load upcast, kernels.py:80-96; the store rounds to nearest). */
enum { MLB_F32 = 0, MLB_F64 = 1, MLB_F16 = 2, MLB_F32C64 = 3 };
/* how the pulls across the slab's z faces are served */
enum { MLB_Z_PERIODIC = 0, /* whole domain on this GPU: wrap in-kernel      */
       MLB_Z_HALO = 1 };   /* z-slab: read the halo planes (filled by the
                              exchange, see mlb_halo_copy)                   */
enum { MLB_OK = 0, MLB_EINVAL = 1, MLB_ECUDA = 2, MLB_ENOMEM = 3,
       MLB_EUNSUPPORTED = 4 };

typedef struct mlb_plan mlb_plan;

typedef struct {
    int32_t nx, ny, nz;   /* slab cells                                    */
    int32_t itemsize;     /* 4, 8, 2 or 4 (storage dtype)                  */
    int64_t xp;           /* row pitch, elements                           */
    int64_t plane;        /* elements per z-plane = ny*xp                  */
    int64_t pop;          /* elements per population = (nz+2)*plane        */
    int64_t total;        /* elements per population block = 19*pop        */
    int64_t bytes;        /* total*itemsize                                */
} mlb_layout;

const char *mlb_last_error(void);
int mlb_abi_version(void);
/* first 16 hex digits of the SHA-256 of the sources (mlb_api.cu, mlb_kernels.cuh,
 * mlb.h) this binary was built from: ties recorded profiles to the code that ran */
const char *mlb_build_id(void);
/* number of CUDA kernel launches issued by this library in this process */
int64_t mlb_launch_count(void);

/* The plans' device memory (flag tables, lists, scratch) is pooled inside the
 * library: destroying a plan keeps its blocks for the next one of the same
 * shape (cudaMalloc / cudaFree stall the device; up to 6 GB are held back).
 * mlb_trim returns the idle blocks to the driver. */
int mlb_trim(void);

int mlb_layout_query(int nx, int ny, int nz, int dtype, mlb_layout *out);

/* Population blocks owned by the library: plain cudaMalloc memory of
 * `bytes` (mlb_layout.bytes) on `device` - what CUDA IPC can export for the
 * z-slab exchange whatever allocator the host framework runs (torch's
 * expandable segments / cudaMallocAsync pools cannot be exported).  The
 * reference's counterpart is PopulationField's numpy block (fields.py:108-146):
 * the caller still owns the block and says when it dies; the library only
 * provides the memory.  Freed blocks are pooled (MLB_BLOCK_POOL_GB, default 24;
 * mlb_trim returns them); mlb_block_free waits for the device to go idle. */
int mlb_block_alloc(int device, int64_t bytes, void **d_out);
int mlb_block_free(void *d_ptr);

/* ---- plan: replaces KernelPlan.__init__ (kernels.py:408-443) -------------
 * omega and wall_u are cast once to the compute dtype, as the reference
 * does (kernels.py:429-432); inlet_u feeds the open-boundary pass
 * (engine.py:167-171).  No flags yet: call mlb_plan_set_flags next. */
int mlb_plan_create(mlb_plan **out, int nx, int ny, int nz, int dtype,
                    double omega, const double wall_u[3], double inlet_u,
                    int device, int z_mode);
int mlb_plan_destroy(mlb_plan *plan);
int mlb_plan_get_layout(const mlb_plan *plan, mlb_layout *out);
int mlb_plan_set_physics(mlb_plan *plan, double omega, const double wall_u[3],
                         double inlet_u);
/* kernel variant used by mlb_step (tuning knob, never changes bits): 0 =
 * default; 32..512 = one cell per thread with that block width; W*1000 + LX
 * = packs of consecutive cells, LX = 8 / 16 / 32 packs per warp row, W = 1:
 * 16-byte packs (fp32 / fp64), W = 2: 8-byte packs (fp32: two cells, for even
 * rows that 4 does not divide; fp16 storage: four cells; mixed2: two cells),
 * W = 3: 4-byte packs (fp16 storage); 4000 = the staged kernel (fp16 storage and
 * fp32 storage / fp64 arithmetic: the row segments a warp pulls from travel through
 * shared memory with cp.async one row ahead of the arithmetic, warp rows handed out
 * in order from a work counter; other dtypes fall back to the automatic choice).
 * Pack kernels serve any row length: a row the pack does not divide ends in a
 * pack of real cells + row padding. */
int mlb_plan_set_variant(mlb_plan *plan, int variant);
/* name of the fused kernel mlb_step will launch for this plan (for reports) */
const char *mlb_plan_kernel_name(const mlb_plan *plan);
/* Pass-through stores (default off = the reference's contract, non-fluid
 * cells of fpost are never written).  When on, mlb_step also stores every
 * non-fluid cell, with the value it holds in d_fpre.  The caller asserts
 * that d_fpre and d_fpost agree on non-fluid cells - true for any pair of
 * buffers that started identical (engine.py:148) - so memory ends up
 * byte-identical to the strict mode, while every warp store is a full
 * 128-byte line instead of leaving partial sectors at each wall.  Rejected
 * (MLB_EUNSUPPORTED) for geometries in which an outlet cell's x-1 neighbour
 * is itself an outlet cell: there the reference's result depends on the
 * stale content of the never-written cell. */
int mlb_plan_set_passthrough(mlb_plan *plan, int on);
/* L2 prefetch distance of the step kernels, in cells of launch order: while a
 * block's own pulls are in flight, it prefetches into L2 what the cells this
 * far ahead will read - the pack kernels (two-buffer and in-place) with one
 * `prefetch.global.L2` per 128-byte line, the one-cell-per-thread kernel with
 * one `cp.async.bulk.prefetch.L2` per population and row.  No result depends
 * on it (the reference has no counterpart; it takes the place of the cache
 * blocking of the kernels.py:258-279 tiles).
 * -1 = auto (default: the cells whose populations make ~10 MB), 0 = off. */
int mlb_plan_set_prefetch(mlb_plan *plan, long long cells);
/* CUDA graphs in mlb_run_steps / mlb_run_steps_inplace: on small domains a step
 * takes microseconds and the loop is launch-bound (the reference's loop pays
 * Python overhead per step at the same place, engine.py:244-249), so runs of up
 * to 32 steps are captured once - the very launches the plain loop makes - and
 * replayed.  -1 = auto (default: domains up to 4 Mi cells), 0 = never, 1 =
 * always; the environment variable MLB_GRAPH overrides.  Never changes bits. */
int mlb_plan_set_graph(mlb_plan *plan, int mode);

/* Flags: the reference's `mask` argument (kernels.py:408, a (N,) uint8 array
 * in cell order).  h_flags is dense [nz][ny][nx] HOST memory.  h_halo_lo /
 * h_halo_hi are dense [ny][nx] flag planes of the slabs below / above
 * (MLB_Z_HALO); NULL means "wrap onto this slab" (the periodic whole
 * domain).  Builds the class table and the inlet/outlet lists.  Rejects
 * codes > 4 (as engine.restore does, engine.py:326-327) and outlet cells at
 * x = 0 (MLB_EUNSUPPORTED). */
int mlb_plan_set_flags(mlb_plan *plan, const uint8_t *h_flags,
                       const uint8_t *h_halo_lo, const uint8_t *h_halo_hi);
/* the flag bytes back, dense [nz][ny][nx], for bit-exact geometry checks */
int mlb_plan_get_flags(const mlb_plan *plan, uint8_t *h_flags);

/* out[0] = distinct (class word, moving-wall link bits) pairs in the plan's
 * dictionary (the kernels read one index byte per cell), out[1] = cells beyond
 * its 254 entries, which read full-width words instead (0 for ordinary
 * geometries) */
int mlb_plan_geometry_stats(const mlb_plan *plan, int64_t out[2]);

/* ---- layout conversion: host dense (Q, N) <-> device padded SoA -----------
 * Interior planes only; halo planes of d_f are left untouched.  h_dense may
 * be pageable or pinned; the copies are asynchronous on `stream` when it is
 * pinned. */
int mlb_upload(const mlb_plan *plan, const void *h_dense, void *d_f, void *stream);
int mlb_download(const mlb_plan *plan, const void *d_f, void *h_dense, void *stream);

/* ---- the hot path --------------------------------------------------------
 * mlb_step: KernelPlan.step (kernels.py:445-462) == numba `fused`
 * (kernels.py:247-279): pull-stream + bounce-back + BGK collide in one
 * pass.  Reads d_fpre only; writes every FLUID cell of d_fpost exactly once
 * and no other cell (kernels.py:3-8).  d_fpre != d_fpost.  The _range form
 * updates slab planes [z0, z1) only (boundary-first / interior overlap). */
int mlb_step(mlb_plan *plan, const void *d_fpre, void *d_fpost, void *stream);
int mlb_step_range(mlb_plan *plan, const void *d_fpre, void *d_fpost,
                   int z0, int z1, void *stream);
/* The fused update followed by the open-boundary pass on the same planes -
 * one time step's work for planes [z0, z1).  Equivalent to mlb_step_range +
 * mlb_open_pass_range; with pass-through stores and a pack kernel the pass is
 * applied inside the fused kernel (no extra launches, no strided column
 * writes) whenever every outlet cell's x-1 neighbour lies in the same pack. */
int mlb_step_open_range(mlb_plan *plan, const void *d_fpre, void *d_fpost,
                        int z0, int z1, void *stream);
/* _OpenBoundaryPass.apply (engine.py:176-180) on d_fpost: inlet cells <-
 * equilibrium(1, inlet_u, 0, 0) in compute dtype; outlet cells <- the fresh
 * populations of their x-1 neighbour, all sources read before any write. */
int mlb_open_pass(mlb_plan *plan, void *d_fpost, void *stream);
int mlb_open_pass_range(mlb_plan *plan, void *d_fpost, int z0, int z1,
                        void *stream);
/* engine.run's timed loop body (engine.py:244-249) n times: step, open
 * pass, swap.  MLB_Z_PERIODIC plans only.  The newest populations end in
 * d_a when nsteps is even, d_b when odd.  If ms != NULL the loop is
 * bracketed by CUDA events on `stream`, the call synchronises and *ms is
 * the device time of the loop. */
int mlb_run_steps(mlb_plan *plan, void *d_a, void *d_b, int nsteps,
                  void *stream, float *ms);

/* ---- in-place update ("AA pattern"): one population block instead of two ---
 * Same arithmetic and the same 2 x 19 x itemsize bytes per update as
 * mlb_run_steps, half the footprint (1024^3 fp32 = 82 GB fits one B200).
 * The block alternates between the normal representation (*repr == 0: what
 * mlb_upload writes and mlb_download / mlb_macro / mlb_diagnostics expect)
 * and a shifted one (*repr == 1) after an odd number of steps;
 * mlb_inplace_normalize brings it back to 0 without stepping.  *repr is
 * updated by both calls.  Wall cells are never modified.  INLET / OUTLET
 * cells are served by the pack kernels only (variant W*1000 + LX, or auto
 * with nx >= 128; any row length), which apply the open-boundary pass inside the step when
 * every outlet cell's x-1 neighbour lies in the same pack and no outlet cell
 * copies from another; otherwise, and for MLB_Z_HALO plans, the call is
 * rejected (MLB_EUNSUPPORTED). */
int mlb_run_steps_inplace(mlb_plan *plan, void *d_f, int nsteps, int *repr,
                          void *stream, float *ms);
int mlb_inplace_normalize(mlb_plan *plan, void *d_f, int *repr, void *stream);
/* Thread layout of the in-place pull half's pack kernel (tuning knob, never
 * changes bits): 0 = classic (a warp is LX packs x 32 / LX rows; the lanes at
 * the ends of a warp row fall back to per-cell stores), 1 = row blocks (a warp
 * is 32 packs of one row, the block's warps sit side by side in x and pass the
 * value that crosses a warp boundary through shared memory: a block that spans
 * the row has no row ends), -1 = automatic. */
int mlb_plan_set_inplace_layout(mlb_plan *plan, int mode);

/* The in-place update over z-slabs (MLB_Z_HALO plans, pack kernels, peer
 * memory).  One half-step on slab planes [z0, z1); `repr` says which: 0 = the
 * pull half (normal -> shifted): boundary planes read their halo planes and
 * write the results for the crossing directions straight into the ring
 * neighbours' boundary planes (d_below / d_above: the neighbours' blocks, with
 * nz_below / nz_above planes; for a single slab the block itself); 1 = the
 * local half (shifted -> normal): own cells only, and boundary planes also
 * fill the neighbours' halo planes for the next pull half.  The caller flips
 * its representation flag once all planes of the slab are done, and orders
 * the boundary launches against the neighbours' with mlb_signal_* exactly as
 * for mlb_step_push_range.  mlb_inplace_swap_slab is mlb_inplace_normalize's
 * kernel for a slab (pairs that straddle the top face reach into the slab
 * above); the caller refills the halo planes afterwards (mlb_halo_push). */
int mlb_step_inplace_range(mlb_plan *plan, void *d_f, int repr, int z0, int z1,
                           void *d_below, int nz_below, void *d_above,
                           int nz_above, void *stream);
int mlb_inplace_swap_slab(mlb_plan *plan, void *d_f, void *d_above,
                          int nz_above, void *stream);

/* ---- z-slab halo exchange ----------------------------------
 * Copies the 5 crossing populations of one boundary plane of d_src (a
 * population block of a slab with the same nx, ny, dtype; possibly on a
 * peer GPU with access enabled) into a halo plane of d_dst.
 *   face 0: src plane lz = src_nz-1, populations with c_z = +1
 *           -> dst halo below (lz = -1)
 *   face 1: src plane lz = 0, populations with c_z = -1
 *           -> dst halo above (lz = nz)                                   */
int mlb_halo_copy(const mlb_plan *plan, void *d_dst, const void *d_src,
                  int src_nz, int face, void *stream);

/* The same exchange seen from the sender: the boundary plane of the LOCAL
 * block d_src (a slab of this plan) is written into the halo plane of d_dst, a
 * neighbour's block with dst_nz planes (peer memory: another GPU's block
 * mapped with mlb_ipc_open or through peer access).
 *   face 0: local plane lz = nz-1, c_z = +1 set -> d_dst's halo below (lz = -1)
 *   face 1: local plane lz = 0,    c_z = -1 set -> d_dst's halo above (lz = dst_nz) */
int mlb_halo_push(const mlb_plan *plan, const void *d_src, void *d_dst,
                  int dst_nz, int face, void *stream);

/* Fused update + exchange: mlb_step_open_range on planes [z0, z1) whose
 * boundary planes ALSO store their 5 crossing populations into the ring
 * neighbours' halo planes from inside the fused kernel (no pack buffer, no
 * copy, no collective; the transfer rides on the kernel's own stores over
 * NVLink).  d_below_post / d_above_post are the neighbours' post blocks with
 * nz_below / nz_above planes (NULL = no neighbour on that side, or not this
 * call's business); only a range that contains plane 0 pushes down, only one
 * that contains plane nz-1 pushes up.  The halos end up byte-identical to
 * mlb_step_open_range followed by mlb_halo_push.  (With a list-driven open-
 * boundary pass on those planes that sequence is literally what runs.)
 * Ordering against the neighbour's own kernels is the caller's job: see
 * mlb_signal_post / mlb_signal_wait. */
int mlb_step_push_range(mlb_plan *plan, const void *d_fpre, void *d_fpost,
                        int z0, int z1, void *d_below_post, int nz_below,
                        void *d_above_post, int nz_above, void *stream);

/* ---- the z-slab loop in one call ---------------------------------------------
 * engine.run's loop body (engine.py:244-249) for one rank of a z-slab ring over
 * peer memory, `nsteps` times, with nothing but launches between steps:
 *   stream:     fork -> interior planes [1, nz-1) -> join
 *   hi_stream:  wait until both neighbours have posted step t-1, boundary planes
 *               0 and nz-1 (mlb_step_push_range: the crossing populations also go
 *               into the neighbours' halo planes), post step t to both neighbours
 * (overlap == 0, nz < 3 or hi_stream == stream: everything on `stream`).
 * below[k] / above[k]: the ring neighbours' blocks that correspond to the local
 * block k (0 = d_a, 1 = d_b), mapped with mlb_ipc_open - with a single slab the
 * local blocks themselves.  post_* are the slots of the NEIGHBOURS' signal
 * blocks this rank posts into, wait_* this rank's own two counters.  `t` is the
 * number of steps posted so far: in/out, shared with mlb_signal_* callers.
 * The newest populations end in d_a when nsteps is even, d_b when odd.  The
 * call only enqueues; *host_us (may be NULL) is the host time per step spent
 * enqueuing, averaged over the first steps (before the launch queue can fill).
 * The _inplace form advances ONE block (mlb_step_inplace_range per plane
 * range; below[0] / above[0] only) and flips *repr once per step. */
typedef struct {
    void *below[2];
    void *above[2];
    int32_t nz_below, nz_above;
    void *post_below, *post_above;
    const void *wait_below, *wait_above;
    uint32_t t;
    int32_t wait_mode;   /* as mlb_signal_wait */
    int32_t overlap;     /* boundary planes first, on hi_stream */
} mlb_ring;
int mlb_slab_run_steps(mlb_plan *plan, void *d_a, void *d_b, int nsteps, mlb_ring *ring,
                       void *stream, void *hi_stream, double *host_us);
int mlb_slab_run_steps_inplace(mlb_plan *plan, void *d_f, int nsteps, int *repr,
                               mlb_ring *ring, void *stream, void *hi_stream,
                               double *host_us);

/* ---- peer memory: CUDA IPC mapping + stream-ordered signals ---------------
 * One process per GPU: a rank exports its population blocks and its signal
 * words (mlb_ipc_export: handle of the enclosing cudaMalloc allocation + the
 * byte offset of d_ptr inside it), ships the 64 handle bytes to its ring
 * neighbours by any means (the Python host uses torch.distributed's object
 * collectives), and the neighbours map them (mlb_ipc_open returns the mapped
 * BASE; add the offset).  A handle can be opened once per process: callers
 * cache by handle bytes.  Not for allocations of the same process. */
#define MLB_IPC_HANDLE_BYTES 64
#define MLB_SIGNAL_BYTES 256   /* 64 uint32 slots, zero-initialised */
#define MLB_SLOT_FROM_BELOW 0     /* byte offsets of a rank's two step counters */
#define MLB_SLOT_FROM_ABOVE 128   /* inside its signal block                    */
int mlb_ipc_export(const void *d_ptr, unsigned char handle[MLB_IPC_HANDLE_BYTES],
                   int64_t *offset);
int mlb_ipc_open(int device, const unsigned char handle[MLB_IPC_HANDLE_BYTES],
                 void **d_base);
int mlb_ipc_close(void *d_base);
/* Signals: monotone uint32 step counters in device memory.  mlb_signal_post
 * enqueues "everything earlier on `stream` is visible system-wide, then
 * *d_slot = value" (d_slot is usually a slot of a NEIGHBOUR's signal block);
 * mlb_signal_wait stalls `stream` until *d_slot >= value (wrap-around safe)
 * without blocking the host.  mode 0 = a stream memory operation
 * (cuStreamWaitValue32: no SM is occupied) when the driver offers it, else a
 * one-thread polling kernel; 1 = memory operation or error; 2 = polling
 * kernel.  post / wait act on the device `stream` belongs to (the legacy
 * default stream: the current device), destroy on the device that holds the
 * block; create selects `device` itself.  No call changes the caller's
 * current device. */
int mlb_signal_create(int device, void **d_sig);
int mlb_signal_destroy(void *d_sig);
int mlb_signal_post(void *d_slot, uint32_t value, void *stream);
int mlb_signal_wait(const void *d_slot, uint32_t value, int mode, void *stream);
/* what mode 0 resolves to with this driver: 1 = stream memory operation,
 * 2 = polling kernel */
int mlb_signal_wait_kind(void);
int mlb_signal_read(const void *d_slot, uint32_t *out);

/* ---- diagnostics ---------------------------------------------------------
 * mlb_macro: SimState.macro (engine.py:104-118): rho, u in float64 for ALL
 * cells, true division, rho = 0 -> u = 0.  Outputs are dense [nz][ny][nx]
 * DEVICE arrays of double. */
int mlb_macro(const mlb_plan *plan, const void *d_f, double *d_rho,
              double *d_ux, double *d_uy, double *d_uz, void *stream);
/* Deterministic (fixed-tree, no float atomics) reductions; synchronises.
 * h_out[8] = total mass (all cells), momentum x,y,z over fluid cells,
 * kinetic energy sum_fluid 1/2 rho |u|^2, max |u| over fluid cells,
 * count of non-finite populations (SimState.check_finite,
 * engine.py:123-125), number of fluid cells. */
int mlb_diagnostics(mlb_plan *plan, const void *d_f, double h_out[8],
                    void *stream);
/* rho, ux, uy, uz (float64, macro conventions) of one cell, written to
 * d_out4[0..3] on the device, asynchronously: the engine's per-step probe
 * sample (engine.py:252-257) without a host round trip. */
int mlb_probe(const mlb_plan *plan, const void *d_f, int x, int y, int lz,
              double *d_out4, void *stream);

/* ---- host-buffer entry points: what the reference's callers hold ---------
 * mlb_step_host is KernelPlan.step(fpre, fpost) on HOST blocks: uploads
 * both (the never-written cells of fpost must survive), steps, downloads
 * fpost.  d_a / d_b are caller-owned device scratch blocks (layout.bytes
 * each).  Synchronous, like the reference call. */
int mlb_step_host(mlb_plan *plan, const void *h_fpre, void *h_fpost,
                  void *d_a, void *d_b, void *stream);

/* engine.run on a host-resident state in ONE call (engine.py:218-275: the
 * reference's run is upload-free because it lives on the host; here the host
 * block is what the caller holds before and after).  Equivalent to mlb_upload
 * (h_in -> d_a), d_b := d_a, nsteps x (fused update, open-boundary pass, swap),
 * mlb_download(newest -> h_out), synchronised - same bits - but when planes 0
 * and nz-1 of the domain are walls (no update depends on the periodic wrap in
 * z) the three phases OVERLAP: the domain is cut into chunks of `chunk_planes`
 * z planes (0 = automatic) which are uploaded on one copy stream, stepped
 * time-skewed behind the upload front (step s of chunk c right after step s-1
 * of chunk c+1), and downloaded on a second copy stream as soon as their last
 * step is done, while later chunks still arrive.  h_in / h_out are dense
 * (19, N) blocks, pinned for the copies to be asynchronous; they may be the same
 * block.  h_flags (dense [nz][ny][nx], may be NULL if the plan has flags) is
 * handed to mlb_plan_set_flags while the first chunks are in flight.  Turns
 * pass-through stores on when the geometry allows them (the two blocks are
 * identical by construction).  *ms (may be NULL): device time of the whole call;
 * *overlapped (may be NULL): 1 if the skewed schedule ran, 0 if the plain
 * sequence did (periodic z, fewer than 4 chunks). */
int mlb_run_steps_host(mlb_plan *plan, const void *h_in, void *h_out, void *d_a, void *d_b,
                       int nsteps, int chunk_planes, const uint8_t *h_flags, void *stream,
                       float *ms, int *overlapped);

#ifdef __cplusplus
}
#endif
#endif /* MLB_H */
