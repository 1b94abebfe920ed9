/*
 * lbm19.h -- C-ABI of the B200-native D3Q19 fused pull stream + BGK-collide
 * solver (liblbm19.so).  Plain pointers and sizes only; no torch types.
 *
 * This boundary replaces the reference's per-dtype compiled step operator and
 * the Simulation methods that drive it (reference = /root/reference,
 * pkg/src/sparselbm/...):
 *
 *   lbm_create            <- Simulation.__init__ field allocation
 *                            (kernel.py:158-178, layouts.py:363-401 allocate)
 *   lbm_set_geometry      <- NodeDescriptorField masks + BoundaryValueTable.as_arrays
 *                            (layouts.py:145-188, 114-123); masks, flag words and the
 *                            sparse tile index are built ON THE DEVICE
 *   lbm_init_equilibrium  <- Simulation.initialize (kernel.py:190-237)
 *   lbm_step              <- Simulation.step / step_kernel(dtype)(...)
 *                            (kernel.py:239-252, 56-141); n steps per call
 *   lbm_get_macroscopic   <- Simulation.macroscopic_fields (kernel.py:285-311)
 *   lbm_check_finite      <- Simulation.check_finite / _first_nonfinite
 *                            (kernel.py:146-152, 278-283)
 *   lbm_total_mass        <- validation.total_mass (validation.py:209-215)
 *   lbm_get_pdf/set_pdf   <- canonical_state / PdfField.read/write
 *                            (tests/conftest.py:7-17, layouts.py:312-332)
 *   lbm_get_field/set_field, lbm_get_slot_of <- PdfField.pre/.post/.slot_of
 *   lbm_get_flags         <- NodeDescriptorField.neighbor_mask (bit-exact check)
 *   lbm_get_tile_index    <- pointer-tile tile_rank (layouts.py:389-401), 3-D + nbr27
 *   lbm19_feq/moments/collide/zou_he_*  <- lattice.equilibrium/moments/bgk_collide,
 *                            boundaries.zou_he_velocity/zou_he_pressure (scalar API,
 *                            lattice.py:136-174, boundaries.py:54-84); host functions
 *                            compiled from the same source as the device kernel
 *
 * All entry points return 0 on success or a negative LBM_E* code; the message
 * is available from lbm_last_error() (thread-local).  A handle is not
 * thread-safe.  lbm_step returns after the device finished, so readbacks see
 * a consistent `pre` buffer.
 */
#ifndef LBM19_H
#define LBM19_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBM_ABI_VERSION 2

enum {
  LBM_OK = 0,
  LBM_EINVAL = -1,    /* bad argument (reference: ValueError) */
  LBM_ESTATE = -2,    /* wrong call order (reference: RuntimeError) */
  LBM_ENOMEM = -3,    /* device allocation failed (reference: MemoryError) */
  LBM_ECUDA = -4,     /* CUDA runtime error */
  LBM_ENCCL = -5,     /* halo transport error */
  LBM_EDIVERGED = -6  /* non-finite value found (reference: DivergenceError) */
};

enum { LBM_F32 = 0, LBM_F64 = 1 };

/* reference LayoutKind (layouts.py:39-52) */
enum {
  LBM_LAYOUT_DENSE = 0,        /* dense SoA, visits every node */
  LBM_LAYOUT_TILE = 1,         /* all tiles allocated */
  LBM_LAYOUT_BITMASK_NODE = 2, /* dense storage, visits non-solid nodes */
  LBM_LAYOUT_POINTER_TILE = 3  /* compacted tile list + nbr27 (sparse) */
};

/* distribution storage scheme (orthogonal to the layout).  The reference
 * keeps two buffers and swaps them (layouts.py:309-310): LBM_SCHEME_AB.
 * LBM_SCHEME_AA keeps ONE buffer updated in place by alternating a
 * neighbour step (pull from x - c_i, push to x + c_i) and a node-local step;
 * it halves the PDF memory at the same 152 B/node traffic and gives results
 * bit-identical to AB.  Readbacks decode it (`pre` is always the reference's
 * pre buffer); there is no `post` buffer under AA. */
enum { LBM_SCHEME_AB = 0, LBM_SCHEME_AA = 1 };

typedef struct lbm_desc {
  int32_t nx, ny, nz;     /* extents of THIS handle's nodes (nz = slab planes) */
  int32_t nz_global;      /* global z extent (== nz on one device) */
  int32_t z0;             /* first global z plane owned by this handle */
  int32_t periodic[3];    /* per axis x, y, z */
  int32_t dtype;          /* LBM_F32 / LBM_F64 */
  int32_t layout;         /* LBM_LAYOUT_* */
  int32_t tile[3];        /* tile edge lengths for tile layouts (powers of two, 32..512 nodes; the Python facade picks 4,4,8, or 4,4,4 for sparse tile lists: layouts.default_tile) */
  int32_t device;         /* CUDA device ordinal */
  double omega;           /* BGK collision frequency, cast to dtype */
  int32_t scheme;         /* LBM_SCHEME_AB (two buffers) / LBM_SCHEME_AA (one, in place) */
} lbm_desc;

typedef struct lbm_stats {
  int64_t n_nodes;          /* nx*ny*nz of this handle */
  int64_t n_nonsolid;       /* active nodes: the unit MLUPS counts */
  int64_t visits_per_step;  /* nodes the kernel visits per step */
  int64_t n_slots;          /* slots per direction plane in use */
  int64_t plane_stride;     /* elements between direction planes */
  int64_t n_tiles;          /* kept tiles (tile layouts), else 0 */
  int64_t step_count;
  int64_t visited_nodes_total;
  int64_t device_bytes;     /* bytes allocated on the device */
  int64_t launches_total;   /* kernels launched by lbm_step so far */
  double last_step_ms;      /* device time of the last lbm_step call (CUDA events) */
  int64_t meta_bytes_per_step; /* flag / index bytes the step kernel reads per step */
  int32_t parity;           /* AB: index of the pre buffer; AA: step phase (step_count mod 2) */
  int32_t initialized;
  int32_t scheme;           /* LBM_SCHEME_* */
  int32_t tile_work_list;   /* 1: tile steps run one warp per live-brick group (sparse tiles) */
} lbm_stats;

typedef struct lbm_handle lbm_t;

const char* lbm_last_error(void);
int lbm_abi_version(void);
int lbm_device_count(int* n);

int lbm_create(const lbm_desc* desc, lbm_t** out);
/* Copy-bandwidth micro-benchmark (reference layouts.copy_bandwidth_bench,
 * layouts.py:473-510) on the device: a flat f64 block of block_bytes copied
 * with the access pattern of `layout` (dense: contiguous 128-bit; bitmask_node:
 * masked; tile: 256-node chunks; pointer_tile: chunks through a base table),
 * warmup untimed + repetitions timed (CUDA events); *bytes_per_s = 2 * bytes *
 * repetitions / elapsed.  The destination is verified (LBM_ESTATE if not). */
int lbm_copy_bandwidth(int32_t device, int32_t layout, int64_t block_bytes, int32_t repetitions,
                       int32_t warmup, double* bytes_per_s);
void lbm_destroy(lbm_t* h);

/* Node descriptors of this handle's nodes, canonical (nz, ny, nx) arrays.
 * ghost_lo / ghost_hi: node types of the planes z0-1 and z0+nz (ny*nx) or
 * NULL.  NULL means "outside the domain" -- except on a whole-domain handle
 * with periodic z, where NULL ghosts are the wrapped planes.
 * bc_kind: 0 velocity, 1 pressure; bc_vel (nb, 3); bc_rho (nb); nb <= 255. */
int lbm_set_geometry(lbm_t* h, const uint8_t* type, const uint8_t* orient,
                     const int32_t* bc_index, const uint8_t* ghost_lo,
                     const uint8_t* ghost_hi, const uint8_t* bc_kind,
                     const double* bc_vel, const double* bc_rho, int32_t nb);

/* Equilibrium initialisation in float64 then cast (reference kernel.py:190-237).
 * Any of rho/ux/uy/uz may be NULL, meaning the matching scalar. */
int lbm_init_equilibrium(lbm_t* h, const double* rho, const double* ux,
                         const double* uy, const double* uz, double rho0,
                         double ux0, double uy0, double uz0);

int lbm_step(lbm_t* h, int64_t n);
/* Enqueue n steps without waiting (several slabs driven from one thread);
 * lbm_synchronize waits and records the device time of the batch. */
int lbm_step_async(lbm_t* h, int64_t n);
int lbm_synchronize(lbm_t* h);
int lbm_set_omega(lbm_t* h, double omega);

/* f64 (nz, ny, nx) arrays; solid nodes report 0. Any pointer may be NULL. */
int lbm_get_macroscopic(lbm_t* h, double* rho, double* ux, double* uy, double* uz);
/* Device-side probe: the same fields on the box [lo, hi) (x, y, z order),
 * returned as (hi_z-lo_z, hi_y-lo_y, hi_x-lo_x) arrays -- observers read a
 * line or plane without pulling the whole domain (reference observers read
 * the full field per call, kernel.py:262-273). */
int lbm_get_macroscopic_box(lbm_t* h, const int32_t* lo, const int32_t* hi, double* rho,
                            double* ux, double* uy, double* uz);
/* Returns LBM_EDIVERGED and fills dir / node (x, y, z) when a non-finite value
 * sits in `pre`; 0 (dir = -1) otherwise. Order: direction, then visit order. */
int lbm_check_finite(lbm_t* h, int32_t* dir, int32_t* node_xyz);
int lbm_total_mass(lbm_t* h, double* mass);

/* which: 0 = pre, 1 = post.  Canonical (19, nz, ny, nx) in the handle dtype;
 * nodes without storage read 0 (set_pdf ignores them).  Under LBM_SCHEME_AA
 * `pre` is decoded from the in-place buffer and which = 1 is LBM_EINVAL. */
int lbm_get_pdf(lbm_t* h, int32_t which, void* out);
int lbm_set_pdf(lbm_t* h, int32_t which, const void* in);
/* Native storage, 19 * plane_stride elements in the handle dtype: dense
 * (19, plane_stride) SoA; tile layouts AoSoA (n_tiles, 19, tile nodes).
 * Under LBM_SCHEME_AA which = 0 is the decoded pre buffer in the same native
 * order (slots without a non-solid node read 0) and which = 1 is LBM_EINVAL. */
int lbm_get_field(lbm_t* h, int32_t which, void* out);
int lbm_set_field(lbm_t* h, int32_t which, const void* in);
/* slot of each node (nz, ny, nx), -1 when the node has no storage. */
int lbm_get_slot_of(lbm_t* h, int32_t* out);
/* packed flag words (nz, ny, nx): bits 0-17 mask, 18-20 type, 21-23 orient,
 * 24-31 bc_index. */
int lbm_get_flags(lbm_t* h, uint32_t* out);
/* tiles (T, 3) as (tx, ty, tz), nbr27 (T, 27); either may be NULL to query T. */
int lbm_get_tile_index(lbm_t* h, int32_t* tiles, int32_t* nbr27, int64_t* n_tiles);
int lbm_get_stats(lbm_t* h, lbm_stats* out);

/* z-slab halo exchange (multi-GPU; dense and tile layouts, AB and A-A).
 * Each slab handle covers global planes [z0, z0 + nz); during every step the
 * outgoing populations of its two boundary planes are stored by the step
 * kernel itself straight into the neighbouring slab's ghost plane (A-A: into
 * the neighbour's boundary plane) through peer memory (same process = device
 * pointers + peer access, other process = CUDA IPC).  Device-side epochs
 * order the steps (no host round trip; the boundary planes run first and
 * signal, the interior overlaps the neighbours' next step; 32-step sequences
 * replay from CUDA graphs).  lbm_halo_export writes an opaque
 * LBM_HALO_BLOB_BYTES blob the caller ships to the neighbours (e.g. with
 * torch.distributed.all_gather_object); lbm_halo_connect opens the lower and
 * upper neighbour's blob (NULL = no neighbour on that side).  All slabs must
 * then make the same sequence of init / step / state-write calls (a state
 * write on one slab alone leaves the epochs out of step: the next wait times
 * out with LBM_ENCCL).  A handle whose geometry has a ghost plane refuses to
 * step until that side is connected, and refuses lbm_set_geometry while
 * connected. */
#define LBM_HALO_BLOB_BYTES 512
int lbm_halo_export(lbm_t* h, void* blob, size_t* bytes);
int lbm_halo_connect(lbm_t* h, const void* lo_blob, const void* hi_blob);

/* scalar per-node math (host), same source as the device kernel.
 * dtype LBM_F32 computes in float32 (values round-tripped through double). */
int lbm19_feq(int32_t dtype, double rho, const double* u3, double* out19);
int lbm19_moments(int32_t dtype, const double* f19, double* rho, double* u3);
int lbm19_collide(int32_t dtype, const double* f19, double omega, double* out19);
int lbm19_zou_he_velocity(int32_t dtype, const double* f19, int32_t orient,
                          const double* u3, double* out19);
int lbm19_zou_he_pressure(int32_t dtype, const double* f19, int32_t orient,
                          double rho_wall, double* out19);

#ifdef __cplusplus
}
#endif
#endif /* LBM19_H */
