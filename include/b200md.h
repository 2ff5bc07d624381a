/*
 * b200md.h -- C ABI of the B200-native Lennard-Jones 12-6 force path.
 *
 * The reference (lanemd, pure Python + numba) has no foreign-function boundary;
 * its hot path crosses from Python into numba-compiled machine code at two
 * call sites, which these entry points replace:
 *   - executor.py:146-171  execute_packed -> _batch_sweep -> _sweep_span
 *   - kernels.py:377-424   compute_pair_vectorized -> _pair_sweep
 * together with the container/traversal work that feeds them
 * (containers.py:61-479, domain.py:97-144, traversals.py:108-305).
 *
 * Conventions
 *   - every pointer is caller-owned DEVICE memory (torch.Tensor.data_ptr());
 *     `stream` is a cudaStream_t passed as void*; all work is stream-ordered
 *     and asynchronous: results are valid after the caller synchronises.
 *   - no hidden allocation: scratch is sized by the *_bytes queries and
 *     passed in by the caller.
 *   - status codes map onto the reference's exception hierarchy
 *     (errors.py:4-25); see LMD_ERR_*.  A zero-distance in-cutoff pair is
 *     detected inside the kernels and reported through lmd_stats.overlap
 *     (the numba -1 sentinel, executor.py:99-100, 163-164).
 *   - particle positions inside the library are packed double4
 *     {x, y, z, ownership} ("pos4"), 32 B per particle, one sector each.
 */
#ifndef B200MD_H
#define B200MD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMD_OK 0
#define LMD_ERR_CONFIG 1     /* ConfigurationError      (kernels.py:92-95, traversals.py:110-119) */
#define LMD_ERR_DEGENERATE 2 /* DegenerateDomainError   (containers.py:78-80) */
#define LMD_ERR_CUDA 3       /* RuntimeError: a CUDA launch or API call failed */
#define LMD_ERR_OVERLAP 4    /* ParticleOverlapError    (kernels.py:176-178) */

/* ownership codes (particles.py:17-19) */
#define LMD_OWNED 0
#define LMD_HALO 1
#define LMD_DUMMY 2

/* interaction orders / register-fill patterns (kernels.py:40-64) */
#define LMD_ONE_BY_V 0
#define LMD_V_BY_ONE 1
#define LMD_TWO_BY_HALF 2
#define LMD_HALF_BY_TWO 3

/* traversals (traversals.py:40-48) + the Verlet-list extension */
#define LMD_LC_C01 0
#define LMD_LC_C08 1
#define LMD_LC_C18 2
#define LMD_VCL 3
#define LMD_VL 4

/* kernel flags */
#define LMD_FLAG_ENERGY 1 /* accumulate potential energy and virial */
#define LMD_FLAG_DEFER_EV 2 /* lmd_vls_force: leave the energy/virial reduction to
                               lmd_vls_reduce_ev (launches over group subsets) */

/* KernelStats (kernels.py:67-89) + extensions.  Device resident; kernels
 * accumulate into it, the caller zeroes it (cudaMemsetAsync) beforehand. */
typedef struct {
  int64_t kernel_invocations;
  int64_t lane_slots;
  int64_t useful_interactions;
  int64_t pair_interactions;
  double epot;                /* extension: sum of 4 eps (s^12 - s^6) over pairs */
  double virial;              /* extension: sum of r . F_ij over pairs */
  int64_t pairs_owned_halo;   /* subset of pair_interactions with a halo j */
  int32_t overlap;            /* 1 if an in-cutoff pair sat at r2 == 0 */
  int32_t overflow;           /* 1 if a capacity-bounded output overflowed */
} lmd_stats;

/* SimulationBox (domain.py:20-42) */
typedef struct {
  double lo[3];
  double hi[3];
  int32_t periodic[3];
  int32_t pad;
} lmd_box;

/* LJParams (domain.py:45-66) */
typedef struct {
  double epsilon, sigma, cutoff, skin;
} lmd_lj;

/* ring-padded cell grid (containers.py:71-98): dims = floor(L / length),
 * cell_len = L / dims, tdims = dims + 2. */
typedef struct {
  int64_t dims[3];
  int64_t tdims[3];
  double cell_len[3];
  double lo[3];
  int64_t ncell; /* tdims[0] * tdims[1] * tdims[2] */
} lmd_grid;

/* ------------------------------------------------------------ library */
int lmd_version(void);
const char* lmd_status_string(int status);
int lmd_device_sm_count(void);

/* ------------------------------------------------------------ geometry */
/* containers.py:71-98; LMD_ERR_DEGENERATE if any axis has dims < 1. */
int lmd_grid_init(const lmd_box* box, double length, lmd_grid* out);

/* ----------------------------------------------- K1 cell binning + sort */
/* containers.py:104-115 (cell_coords + linear_index), bit-exact:
 * floor((pos - lo) / cell_len) + 1 clipped to [1, dims] (ring = 0) or
 * [0, dims + 1] (ring = 1), IEEE division.  Positions are SoA. */
int lmd_cell_index(const lmd_grid* g, int ring, int64_t n, const double* x, const double* y,
                   const double* z, int32_t* cell, void* stream);

/* Stable radix sort of (cell, index) -> (cell_sorted, perm): the GPU
 * equivalent of np.argsort(kind="stable") (containers.py:125, 158).
 * temp_bytes from lmd_sort_temp_bytes(n). */
size_t lmd_sort_temp_bytes(int64_t n);
int lmd_sort_by_cell(int64_t n, int64_t ncell, const int32_t* cell, int32_t* cell_sorted,
                     int32_t* perm, int32_t* scratch_iota, void* temp, size_t temp_bytes,
                     void* stream);

/* cell_start/cell_count over a sorted key array (np.unique(..., return_index)
 * at containers.py:128, 164); `base` is added to every start.  Both arrays
 * are fully overwritten (empty cells get count 0). */
int lmd_cell_ranges(int64_t n, int64_t ncell, int32_t base, const int32_t* cell_sorted,
                    int32_t* cell_start, int32_t* cell_count, void* stream);

/* buffer_at semantics (containers.py:178-184): the owned view of a cell if it
 * holds owned particles, else its halo view.  Writes the merged tables and
 * (if dup != NULL) dup[c] = 1 for cells holding both owned particles and
 * images: the reference's _occupied_pairs (traversals.py:133) then lists the
 * cell twice as an anchor, which lc_c08 / lc_c18 turn into duplicated units. */
int lmd_merge_cell_tables(int64_t ncell, const int32_t* o_start, const int32_t* o_count,
                          const int32_t* h_start, const int32_t* h_count, int32_t* start,
                          int32_t* count, uint8_t* dup, void* stream);

/* pos4[k] = {x[perm[k]], y[perm[k]], z[perm[k]], own[perm[k]]}; own may be
 * NULL (then `own_value` is used for every entry). */
int lmd_gather_pos4(int64_t n, const int32_t* perm, const double* x, const double* y,
                    const double* z, const int8_t* own, double own_value, double* pos4,
                    void* stream);

/* ---------------------------------------- K9 periodic images (halo) */
/* domain.py:97-144: number of images per owned particle within `margin` of
 * a periodic face (every non-zero shift combination). */
int lmd_halo_count(const lmd_box* box, double margin, int64_t n, const double* x,
                   const double* y, const double* z, const int8_t* own, int32_t* count,
                   void* stream);
size_t lmd_scan_temp_bytes(int64_t n);
int lmd_exclusive_scan_i32(int64_t n, const int32_t* in, int32_t* out, void* temp,
                           size_t temp_bytes, void* stream);
/* Emit the images: positions pos + (hi - lo) / + (lo - hi) per shifted axis,
 * exactly as domain.py:118-121; owner index and a shift code (base-3 digits,
 * 0 none / 1 plus / 2 minus, x least significant) per image. */
int lmd_halo_emit(const lmd_box* box, double margin, int64_t n, const double* x,
                  const double* y, const double* z, const int8_t* own, const int32_t* offset,
                  double* hx, double* hy, double* hz, int32_t* owner, int8_t* shift,
                  void* stream);
/* Refresh image positions from their owners between rebuilds (sorted halo
 * slots, written straight into pos4 at `pos4_halo`). */
int lmd_halo_refresh_pos4(const lmd_box* box, int64_t nh, const int32_t* owner,
                          const int8_t* shift, const double* x, const double* y,
                          const double* z, double* pos4_halo, void* stream);

/* The same into SoA arrays (Verlet-list gathers read x, y, z separately). */
/* lmd_gather_pos4 (own = NULL) and lmd_halo_refresh_pos4 that also write
 * the SoA copies sx, sy, sz in the same pass (one read, both layouts). */
int lmd_gather_pos4_soa(int64_t n, const int32_t* perm, const double* x, const double* y,
                        const double* z, double own_value, double* pos4, double* sx, double* sy,
                        double* sz, void* stream);
int lmd_halo_refresh_pos4_soa(const lmd_box* box, int64_t nh, const int32_t* owner,
                              const int8_t* shift, const double* x, const double* y,
                              const double* z, double* pos4_halo, double* sx, double* sy,
                              double* sz, void* stream);
/* The same image positions as (nh, 3) row-major rows (the segmented Verlet
 * lists' staged layout). */
int lmd_halo_refresh_rows(const lmd_box* box, int64_t nh, const int32_t* owner,
                          const int8_t* shift, const double* x, const double* y, const double* z,
                          double* rows, void* stream);
int lmd_halo_refresh_soa(const lmd_box* box, int64_t nh, const int32_t* owner,
                         const int8_t* shift, const double* x, const double* y, const double* z,
                         double* ox, double* oy, double* oz, void* stream);
/* ox[k] = x[perm[k]] (perm may be NULL = identity), likewise y, z. */
int lmd_gather_soa(int64_t n, const int32_t* perm, const double* x, const double* y,
                   const double* z, double* ox, double* oy, double* oz, void* stream);

/* ---------------------------------- K2 linked-cell force (N3 off, full shell) */
/* One warp per owned cell, the 27-cell shell as j (owned and halo views),
 * lanes mapped by `pattern` at warp width 32.  Forces are written (not
 * accumulated) into f{x,y,z}[k] for k in the owned backing (sorted order).
 * Accumulates pair_interactions (ordered pairs), pairs_owned_halo, overlap,
 * and with LMD_FLAG_ENERGY epot/virial into *stats (deterministically).
 * dup (may be NULL = lc_c01 semantics): per-cell flags from
 * lmd_merge_cell_tables; a cell pair (C, D != C) then counts 1 + dup[min(C, D)]
 * times, reproducing the reference's lc_c08 / lc_c18 unit multiplicity.
 * ev_scratch: 2 * lmd_lc_ev_slots(g) doubles. */
int64_t lmd_lc_ev_slots(const lmd_grid* g);
int lmd_force_lc(const lmd_grid* g, const lmd_lj* lj, int pattern, int flags,
                 const double* pos4, const int32_t* cell_start, const int32_t* cell_count,
                 const uint8_t* dup, double* fx, double* fy, double* fz, double* ev_scratch,
                 lmd_stats* stats, void* stream);

/* Newton3 lc_c08 / lc_c18 as colored passes (traversals.py:190-241, the
 * concurrency contract of traversals.py:1-6): one launch per color, one warp
 * per base; the base's units dual-write into its shared-memory write set
 * (c08: its 2x2x2 block, c18: its cell + 13 forward neighbours), flushed to
 * f once per base.  Zeroes f first; deterministic.  pair_interactions is
 * counted in the reference's Newton3 convention.  max_cell >= the largest
 * owned cell count; ev_scratch: 2 * lmd_lc_n3_ev_slots(g) doubles. */
int64_t lmd_lc_n3_ev_slots(const lmd_grid* g);
int lmd_force_lc_n3(const lmd_grid* g, const lmd_lj* lj, int traversal, int pattern, int flags,
                    const double* pos4, int64_t n_owned, const int32_t* cell_start,
                    const int32_t* cell_count, const int32_t* o_count, const int32_t* h_count,
                    const uint8_t* dup, int max_cell, double* fx, double* fy, double* fz,
                    double* ev_scratch, lmd_stats* stats, void* stream);

/* Geometric KernelStats of the reference schedules (traversals.py:108-266,
 * executor.py:38-69, 165-171) for lc_c01 / lc_c08 / lc_c18: kernel
 * invocations, lane slots and useful interactions for shape (a, b) and
 * width V, from per-cell owned/halo counts.  Adds into *stats. */
/* Same sweep as lmd_force_lc, thread per particle for every interaction
 * order (a, b): a warp holds a consecutive cell-sorted particles, b lanes per
 * particle split its candidate stream (csrc/force_lc.cu lc_tpi_kernel).
 * cell_of[i] = the rebuild-time cell of backing particle i.  ev_scratch:
 * 2 * lmd_lc_tpi_ev_slots(n_owned, pattern) doubles. */
int64_t lmd_lc_tpi_ev_slots(int64_t n_owned, int pattern);
int lmd_force_lc_particles(const lmd_grid* g, const lmd_lj* lj, int pattern, int flags,
                           const double* pos4, int64_t n_owned, const int32_t* cell_of,
                           const int32_t* cell_start, const int32_t* cell_count,
                           const uint8_t* dup, double* fx, double* fy, double* fz,
                           double* ev_scratch, lmd_stats* stats, void* stream);
int lmd_lc_stats(const lmd_grid* g, int traversal, int newton3, int a, int b, int vector_width,
                 const int32_t* o_count, const int32_t* h_count, lmd_stats* stats,
                 void* stream);

/* collect_forces (containers.py:186-189): out[perm[k]] = sorted[k]. */
int lmd_scatter_forces(int64_t n, const int32_t* perm, const double* fx, const double* fy,
                       const double* fz, double* ox, double* oy, double* oz, void* stream);


/* --------------------------------------------- K3/K4 Verlet lists (extension) */
/* Build on the rc+skin cell grid over a combined backing pos4 = [owned sorted
 * by cell | images sorted by cell], with SEPARATE owned and image cell tables
 * (o_*, h_*; image starts include the n_owned base).  Candidates: owned
 * particles and images of the 27 cells; listed iff r2 < rl2 with the
 * reference's exact r2.  newton3 = 1 builds half lists (owned j > i). */
int64_t lmd_vl_num_tiles(int64_t n_owned, int pattern);
/* Single-pass build: lists laid out per interaction order (tiles of A =
 * distinct i per fill, lane-chunked as documented in csrc/vl.cu, padded
 * with `sentinel`, the index of a far-away record); tile t starts at
 * tile_off[t] = t * cap_steps * 32 (cap_steps a multiple of 4);
 * nbr holds ceil(n_owned / A) * cap_steps * 32 entries.  Writes count[i],
 * tile_off, kmax and *max_count = the longest list; if *max_count >
 * cap_steps * B the lists were truncated and the caller must rebuild with a
 * larger capacity.  count_half (nullable) receives each particle's half-list
 * length (images, and owned j > i), the Newton3 statistics of full lists. */
int lmd_vl_build(const lmd_grid* g, double rl2, int newton3, int pattern, int64_t n_owned,
                 int32_t sentinel, const double* pos4, const int32_t* o_start,
                 const int32_t* o_count, const int32_t* h_start, const int32_t* h_count,
                 int32_t cap_steps, int32_t* count, int32_t* count_half, int64_t* tile_off,
                 int32_t* kmax, int32_t* max_count, int32_t* nbr, void* stream);
/* Optional pass after lmd_vl_build / lmd_vl_build_staged: permutes every
 * lane's own slot sequence so that the lanes of each half-warp gather from
 * distinct 8-byte bank pairs (index & 15) step by step -- the cost unit of a
 * 64-bit shared-memory or L1 gather (csrc/vl.cu vl_bank_local_kernel,
 * vl_bank_kernel); slots a lane leaves idle become -1.  Same entries per
 * lane and the same step count, so forces, pair counts and statistics are
 * unchanged up to summation order.  rounds = 0: lane-local Latin-square
 * order (16-bit workspace: staged lists only, max_steps = the longest
 * tile's step count, <= 255; index_bits 16 for the 16-bit staged lists,
 * else 32); rounds >= 1: warp-cooperative with that many
 * proposal rounds per step (workspace lmd_vl_bank_smem_per_warp(cap_steps)
 * bytes per tile, at most 200 KB). */
size_t lmd_vl_bank_smem_per_warp(int32_t cap_steps);
int lmd_vl_bank_schedule(int pattern, int64_t n_units, int32_t sentinel, int rounds,
                         int32_t cap_steps, int32_t max_steps, int32_t index_bits,
                         const int64_t* tile_off, const int32_t* kmax, int32_t* nbr,
                         void* stream);
/* Staged Verlet lists (v_by_one, full lists; csrc/vl.cu).  Owned particles
 * form groups of group_size (128 / 256 / 512) consecutive backing slots, one
 * block each; a group's particles lie in one or two cell rows and its
 * candidates in 36 contiguous index runs (owned and image backing x the
 * group's rows x 3 x 3 (dy, dz) neighbour rows), which the force kernel
 * copies into shared memory with TMA bulk copies.  lmd_vl_groups writes one
 * record of 128 int32 per group (csrc/vl_common.cuh: run starts, lengths,
 * local offsets, S = staged rows, first image row, overflow flag, first
 * row) from the build positions and cell tables; smax[0] = largest S among
 * staged groups, smax[1] = groups spanning more than two rows or over
 * capacity (those gather their global indices from the SoA arrays).  lmd_vl_build_staged = lmd_vl_build for
 * V_BY_ONE writing each entry as the local row of its group's copy; pads
 * are -1.  index_bits = 16 (every group staged, smax[1] == 0): entries are
 * uint16 local rows, 8 steps per 128-bit chunk (cap_steps % 8 == 0, tile
 * offsets in uint16 units, pads 0xffff); 32: int32, 4
 * steps per chunk.  lmd_vl_staged_capacity(group_size) = the largest S a group
 * stages (pass it as `capacity`).  lmd_force_vl_staged: newton3 0 or 2 as
 * lmd_force_vl; soa = (3, stride) rows (stride % 16 == 0, 128-B aligned)
 * whose row `sentinel` is a far-away position (idle slots of global-gather
 * groups); ev_scratch holds 2 * ceil(n_owned / 32) doubles. */
int32_t lmd_vl_staged_capacity(int32_t group_size);
int lmd_vl_groups(const lmd_grid* g, int64_t n_owned, int32_t group_size, int32_t capacity,
                  const double* pos4, const int32_t* o_start, const int32_t* o_count,
                  const int32_t* h_start, const int32_t* h_count, int32_t* groups,
                  int32_t* smax, void* stream);
int lmd_vl_build_staged(const lmd_grid* g, double rl2, int newton3, int64_t n_owned,
                        const double* pos4, const int32_t* o_start, const int32_t* o_count,
                        const int32_t* h_start, const int32_t* h_count, int32_t group_size,
                        const int32_t* groups, int32_t index_bits, int32_t cap_steps,
                        int32_t* count, int32_t* count_half, int64_t* tile_off, int32_t* kmax,
                        int32_t* max_count, int32_t* nbr, void* stream);
int lmd_force_vl_staged(int newton3, int flags, const lmd_lj* lj, int64_t n_owned,
                        const double* pos4, const double* soa, int64_t stride, int32_t sentinel,
                        int32_t group_size, const int32_t* groups, int32_t index_bits,
                        const int64_t* tile_off, const int32_t* kmax, const int32_t* nbr,
                        const int32_t* out_perm, double* fx, double* fy, double* fz,
                        double* ev_scratch, lmd_stats* stats, void* stream);
/* Segmented staged Verlet lists (csrc/vls.cu) -- the default force path for
 * V_BY_ONE full lists; replaces the reference's execute_packed sweep over
 * the schedule's units (executor.py:72-171) for the Verlet-list container.
 * Positions are (x, y, z) rows (24 B, 16-B aligned base) in rebuild order:
 * owned cell-sorted, then images cell-sorted.  Groups: each interior cell
 * line's owned particles cut into ceil(n_line / 128) balanced groups; a
 * group stages its 18 candidate runs ((owned | image) x (dz, dy) neighbour
 * lines, cells xa-1 .. xb+1) into shared memory with one TMA copy each.
 * lmd_vls_plan writes the filled cell starts fs_own / fs_img (ncell each),
 * per-line group counts / inclusive offsets (tdims[1] * tdims[2] each), the
 * group records (64 int32 each, at most lmd_vls_max_groups) and info[8] =
 * {largest staged rows, groups over capacity, number of groups, -, -}.
 * lmd_vls_rows_for(info[0]) = the row capacity to pass as `rows` (0: too
 * many rows for 16-bit byte offsets, use the other staged path).
 * lmd_vls_build: lists with rl2 = (rc+skin)^2 from the build-time rows (the
 * reference's exact r2), entries with r2 < rin2 in the inner segment, the
 * rest in the outer; per tile t: seg_chunks[2t], [2t+1] = chunks of 8
 * entries; list chunk c of lane l at int4 index (t * cap_chunks + c) * 32 +
 * l (uint16 byte offsets 24 * local row; bank_order != 0: lane-local
 * Latin-square bank order within each segment, else the order the walk found
 * them in -- a cheaper build for lists that are used a few times only);
 * slotmap[g * 128 + lane slot] = the group-local particle the slot holds
 * (0xff: none); count[i] / count_half[i] = full / half list lengths (sorted
 * order); info[3] / info[4] = most chunks per tile / entries per lane seen
 * (rebuild with larger caps when above cap_chunks / cap_entries <= 255).
 * lmd_vls_force: one block per group (n_groups = info[2] of the plan);
 * newton3 0 or 2 (as lmd_force_vl); the outer segment runs iff disp == NULL
 * or *disp >= half_delta2 (bit patterns), i.e. once some particle moved at
 * least delta / 2 since the build; ev_scratch holds
 * 2 * lmd_vls_ev_slots(n_groups) doubles.  group_index != NULL launches the
 * n_index groups it lists (e.g. the interior groups, which stage no image or
 * ghost rows, while a ghost exchange is in flight); LMD_FLAG_DEFER_EV leaves
 * the energy/virial reduction over all groups to lmd_vls_reduce_ev.  lmd_vls_refresh: rows[k] =
 * (x, y, z)[perm[k]] (perm NULL: identity); with n_images > 0 also rows[n +
 * k'] = the periodic image k' (position of owner[k'] + the exact shift of
 * its code, domain.py:112-118: one launch for the whole backing); with disp != NULL the
 * largest squared displacement from build_rows max-reduced into disp[slot]
 * (disp[slot ^ 1] cleared).  lmd_vls_gather_rows (ghost rows of a
 * decomposition; with disp != NULL their displacement from build_rows is
 * max-reduced into disp[slot] too): rows_out[k] =
 * rows_in[perm[k]].  lmd_vls_rows_to_legacy: rows -> pos4 (OWNED below
 * n_owned, HALO above) and SoA copies (either may be NULL). */
int64_t lmd_vls_max_groups(const lmd_grid* g, int64_t n_owned);
int32_t lmd_vls_rows_for(int32_t staged_rows);
size_t lmd_vls_plan_temp_bytes(const lmd_grid* g);
int lmd_vls_plan(const lmd_grid* g, int64_t n_owned, const int32_t* o_start,
                 const int32_t* o_count, const int32_t* h_start, const int32_t* h_count,
                 int32_t* fs_own, int32_t* fs_img, int32_t* row_groups, int32_t* row_gend,
                 void* temp, size_t temp_bytes, int32_t* groups, int32_t* info, void* stream);
size_t lmd_vls_build_smem(int32_t rows, int32_t cap_entries);
int lmd_vls_build(const lmd_grid* g, double rin2, double rl2, int64_t n_owned, int32_t rows,
                  const double* pos_rows, const int32_t* fs_own, const int32_t* o_count,
                  const int32_t* fs_img, const int32_t* h_count, const int32_t* groups,
                  int64_t max_groups, int32_t cap_chunks, int32_t cap_entries, int32_t bank_order,
                  void* nbr, int32_t* seg_chunks, uint8_t* slotmap, int32_t* count,
                  int32_t* count_half, int32_t* info, void* stream);
int64_t lmd_vls_ev_slots(int64_t max_groups);
int lmd_vls_force(int newton3, int flags, const lmd_lj* lj, int64_t n_owned, int32_t rows,
                  const double* pos_rows, const int32_t* groups, int64_t n_groups,
                  const int32_t* group_index, int64_t n_index, const void* nbr, const int32_t* seg_chunks,
                  const uint8_t* slotmap, int32_t cap_chunks, const uint64_t* disp,
                  double half_delta2, const int32_t* out_perm, double* fx, double* fy,
                  double* fz, double* ev_scratch, lmd_stats* stats, void* stream);
/* One force phase without lists, for a neighbour structure that is used once
 * (the reference's force_phase builds its container per call,
 * driver.py:107-129), in two kernels: the list build's walk alone (packed
 * FP32; every candidate within rc + skin + the FP32 error bound is kept in
 * `scratch`: n_groups * 128 * cap_entries uint16), then each lane takes its
 * kept candidates through the reference's exact r2 (executor.py:93-94) from
 * the staged FP64 rows: r2 < (rc + skin)^2 counts into count / count_half (the
 * Verlet-list statistics), r2 < rc^2 is evaluated.  info[2] must hold the
 * number of groups (as lmd_vls_plan leaves it); info[4] = most entries a lane
 * kept (call again with a larger cap_entries when above it: nothing was
 * evaluated).  Same pairs, forces and statistics as lmd_vls_build +
 * lmd_vls_force. */
int lmd_vls_direct(const lmd_grid* g, int newton3, int flags, const lmd_lj* lj, int64_t n_owned,
                   int32_t rows, const double* pos_rows, const int32_t* fs_own,
                   const int32_t* o_count, const int32_t* fs_img, const int32_t* h_count,
                   const int32_t* groups, int64_t n_groups, int32_t cap_entries, void* scratch,
                   const int32_t* out_perm, double* fx, double* fy, double* fz,
                   double* ev_scratch, lmd_stats* stats, int32_t* count, int32_t* count_half,
                   int32_t* info, void* stream);
int lmd_vls_reduce_ev(int64_t n_groups, const double* ev_scratch, lmd_stats* stats, void* stream);
int lmd_vls_refresh(int64_t n, const int32_t* perm, const double* x, const double* y,
                    const double* z, double* rows, const double* build_rows, uint64_t* disp,
                    int32_t slot, const lmd_box* box, int64_t n_images, const int32_t* owner,
                    const int8_t* shift, void* stream);
int lmd_vls_gather_rows(int64_t n, const int32_t* perm, const double* rows_in, double* rows_out,
                        const double* build_rows, uint64_t* disp, int32_t slot, void* stream);
int lmd_vls_rows_to_legacy(int64_t n, int64_t n_owned, const double* rows, double* pos4,
                           double* sx, double* sy, double* sz, void* stream);
/* Force over the lists: one warp per i-tile, lanes by `pattern`; positions
 * are pos4 over the combined backing plus one sentinel record (256-bit
 * gathers), or, if soa != NULL, SoA copies x = soa[0..ntot), y, z of the
 * same ntot records (three 64-bit gathers that share sectors between
 * neighbouring lanes).  newton3 = 0
 * writes f[i]; newton3 = 1 (half lists) accumulates with FP64 atomics into
 * zeroed f (j-side reactions; summation order is then not deterministic);
 * newton3 = 2 runs full lists like 0 and also counts the pairs with an image
 * j into pairs_owned_halo, for the reference's Newton3 pair bookkeeping
 * (owned-owned pairs once = (pairs - halo) / 2 + halo).  out_perm (nullable,
 * newton3 0 / 2): the force of backing particle i goes to f[out_perm[i]] --
 * the caller's order, collect_forces fused into the kernel.
 * ev_scratch: 2 * lmd_vl_ev_slots(n_owned, pattern) doubles. */
int64_t lmd_vl_ev_slots(int64_t n_owned, int pattern);
int lmd_force_vl(int pattern, int newton3, int flags, const lmd_lj* lj, int64_t n_owned,
                 const double* pos4, const double* soa, int64_t ntot, const int64_t* tile_off,
                 const int32_t* kmax, const int32_t* nbr, const int32_t* out_perm, double* fx,
                 double* fy, double* fz, double* ev_scratch, lmd_stats* stats, void* stream);
/* KernelStats of a Verlet-list force phase: i-tiles of `a` consecutive owned
 * particles, each tile's j-stream its longest list chunked by b. */
int lmd_vl_stats(int64_t n_owned, int a, int b, int vector_width, const int32_t* count,
                 lmd_stats* stats, void* stream);

/* --------------------------------------------- K5-K7 Verlet cluster lists */
/* VerletClusterContainer (containers.py:302-479) on the device.  Build:
 * lmd_vcl_order (column key cx + width*cy, lexsort((z, col)) as two stable
 * radix sorts), lmd_vcl_chunk (M-slot clusters per column; synchronises to
 * return the cluster count), lmd_vcl_backing (padded pos4 with dummies parked
 * at the AABB minimum), lmd_vcl_column_table, lmd_vcl_pairs (AABB gap^2 <=
 * limit, binned; ascending ids).  Force: lmd_force_vcl (warp per owned
 * cluster over itself, its owned list and its halo links; Newton3 off).
 * Stats: lmd_vcl_stats (units of traversals.py:244-266). */
size_t lmd_vcl_temp_bytes(int64_t n);
int lmd_vcl_order(int64_t n, const double* x, const double* y, const double* z, double lo0,
                  double lo1, double col, int64_t width, int32_t* colkey, int32_t* ckey2,
                  uint64_t* zkey, uint64_t* zkey2, int32_t* tmp_idx, int32_t* order,
                  int32_t* sorted_colkey, void* temp, size_t temp_bytes, void* stream);
int lmd_vcl_chunk(int64_t n, int M, const int32_t* sorted_colkey, int32_t* flag, int32_t* run_id,
                  int32_t* run_start, int32_t* run_nclu, int32_t* run_coff, int32_t* slot,
                  int32_t* cluster_key, int64_t* ncl_out, void* temp, size_t temp_bytes,
                  void* stream);
int lmd_vcl_backing(int64_t n, int64_t ncl, int M, const int32_t* order, const int32_t* slot,
                    const double* x, const double* y, const double* z, double own_value,
                    double* pos4, double* amin, double* amax, void* stream);
int lmd_vcl_column_table(int64_t ncl, const int32_t* cluster_key, int32_t* tbeg, int32_t* tend,
                         int64_t tsize, void* stream);
int lmd_vcl_pairs(int64_t ncl, const int32_t* cluster_key, const double* amin, const double* amax,
                  const double* bmin, const double* bmax, const int32_t* tbeg,
                  const int32_t* tend, int64_t width, int64_t tsize, int exclude_self, double rl,
                  double limit, int32_t* count, int32_t* n3count, const int64_t* off,
                  int32_t* list, void* stream);
int64_t lmd_vcl_ev_slots(int64_t ncl);
/* K7o: the same force phase with the interaction order as the warp's lane
 * template (pattern (A, B) at V = 32, kernels.py:250-265): A i-slots x B
 * j-slots per fill, B >= M packing B / M neighbour clusters per fill, lanes
 * past the cluster size blank.  M <= 32.  amin / amax (ncl x 3) and hmin /
 * hmax (halo clusters x 3): the cluster boxes of the last rebuild / refresh;
 * a lane skips a cluster whose box is farther than cutoff + skin/2 from its
 * i (members moved less than skin/2 since the boxes were taken). */
int lmd_force_vcl_order(int64_t ncl, int M, int pattern, int flags, const lmd_lj* lj,
                        const double* pos4, const int64_t* off, const int32_t* nlist,
                        const int32_t* list, const int64_t* hoff, const int32_t* hnlist,
                        const int32_t* hlist, const double* amin, const double* amax,
                        const double* hmin, const double* hmax, double* fx, double* fy,
                        double* fz, double* ev_scratch, lmd_stats* stats, void* stream);
/* pos4f (optional, n_records float4 = every record of pos4, owned and halo
 * clusters): scratch for FP32 copies of the records; the cutoff tests then
 * run in FP32 against rc^2 + the error bound for coordinates up to max_abs
 * and the passing pairs are decided by the exact FP64 r2 -- same pairs. */
int lmd_force_vcl(int64_t ncl, int M, int flags, const lmd_lj* lj, const double* pos4,
                  const int64_t* off, const int32_t* nlist, const int32_t* list,
                  const int64_t* hoff, const int32_t* hnlist, const int32_t* hlist, double* fx,
                  double* fy, double* fz, double* ev_scratch, lmd_stats* stats,
                  int64_t n_records, float* pos4f, double max_abs, void* stream);
/* ncl_total = owned + halo clusters of pos4; nd_scratch: ncl_total int32
 * (per-cluster non-dummy counts, computed here). */
int lmd_vcl_stats(int64_t ncl, int M, int newton3, int a, int b, int vector_width,
                  const double* pos4, const int64_t* off, const int32_t* nlist,
                  const int32_t* n3count, const int32_t* list, const int64_t* hoff,
                  const int32_t* hcount, const int32_t* hlist, int64_t ncl_total,
                  int32_t* nd_scratch, lmd_stats* stats, void* stream);
int lmd_vcl_collect(int64_t n, const int32_t* order, const int32_t* slot, const double* fx,
                    const double* fy, const double* fz, double* ox, double* oy, double* oz,
                    void* stream);

/* ----------------------------------------------- execute_packed (batched) */
/* The reference's batched operator (executor.py:118-171) over an explicit
 * unit list: unit u sweeps owned-backing i-span [i_off, i_off + i_len) x
 * j-span [j_off, j_off + j_len) of the owned (j_halo = 0) or halo backing,
 * Newton3 dual-write if newton3[u], self exclusion if same[u]
 * (_sweep_span, executor.py:72-115).  Units are grouped by base: the bases of
 * color c are [color_base_start[c], color_base_start[c+1]) (HOST array of
 * n_colors + 1 entries); base b's units are base_units[base_start[b] ..
 * base_start[b+1]) (device).  One launch per color, one warp per base.
 * Forces ACCUMULATE (+=) into the SoA force arrays; pair_interactions and
 * overlap accumulate into *stats.  own4 / halo4: pos4 backings. */
int lmd_execute_packed(int64_t n_units, const int64_t* i_off, const int64_t* i_len,
                       const int64_t* j_off, const int64_t* j_len, const uint8_t* j_halo,
                       const uint8_t* newton3, const uint8_t* same, int n_colors,
                       const int64_t* color_base_start, const int64_t* base_units,
                       const int64_t* base_start, int pattern, const lmd_lj* lj,
                       const double* own4, const double* halo4, double* ofx, double* ofy,
                       double* ofz, double* hfx, double* hfy, double* hfz, lmd_stats* stats,
                       void* stream);

/* ------------------------------------------------ the functor (two buffers) */
/* compute_pair_vectorized (kernels.py:377-424) on device buffers given as
 * pos4 (ownership in .w).  Forces ACCUMULATE (+=) into the SoA force arrays.
 * same = 1 requires pos4_i == pos4_j (kernels.py:398-399).  newton3 = 1
 * also subtracts the reaction from the j buffer via a second, transposed
 * pass (deterministic, no floating-point atomics).  ev_scratch holds
 * 2 * lmd_pair_sweep_ev_slots(ni, pattern) doubles. */
int64_t lmd_pair_sweep_ev_slots(int64_t ni, int pattern);
int lmd_pair_sweep(int64_t ni, const double* pos4_i, int64_t nj, const double* pos4_j,
                   int same, int newton3, int pattern, int flags, const lmd_lj* lj,
                   double* fxi, double* fyi, double* fzi, double* fxj, double* fyj, double* fzj,
                   double* ev_scratch, lmd_stats* stats, void* stream);
/* {owned, non-dummy, self_pair_slots(newton3=1)} of a pos4 buffer
 * (particles.py:111-143), as three int64 on the device. */
int lmd_buffer_counts(int64_t n, const double* pos4, int64_t* out3, void* stream);

/* --------------------------------------- K11 integrator + boundaries */
/* domain.py:69-94 (apply_boundaries): periodic wrap with numpy's np.mod
 * semantics, reflective mirror with velocity flip; *diverged |= 1 if a
 * particle is more than one box length outside (SimulationDivergedError). */
int lmd_apply_boundaries(const lmd_box* box, int64_t n, double* x, double* y, double* z,
                         double* vx, double* vy, double* vz, int32_t* diverged, void* stream);

/* ----------------------------------------- brick decomposition (§8e) */
/* One exchange stage's pack (decomposition.py): out_rows[k] (row-major
 * x, y, z) = source(idx[k]) with coordinate `axis` shifted by `shift` (the
 * exact image offset, or 0), where source indexes [owned SoA ox/oy/oz |
 * ghost rows received in earlier stages]. */
int lmd_ghost_pack(int64_t count, const int32_t* idx, int64_t n_owned, const double* ox,
                   const double* oy, const double* oz, const double* ghost_rows, int axis,
                   double shift, double* out_rows, void* stream);
/* pos4[k] = (rows[perm[k]], own_value): gather row-major positions. */
int lmd_gather_pos4_rows(int64_t n, const int32_t* perm, const double* rows, double own_value,
                         double* pos4, void* stream);
/* The same rows gathered into SoA x, y, z (the VL container's SoA copies). */
int lmd_gather_rows_soa(int64_t n, const int32_t* perm, const double* rows, double* x, double* y,
                        double* z, void* stream);

/* *out = max_k |r_k - ref_k|^2 with the reference's unfused (dx^2 + dy^2) +
 * dz^2 (containers.py:23-38, needs_rebuild); ref_xyz rows are (x, y, z). */
int lmd_max_displacement2(int64_t n, const double* x, const double* y, const double* z,
                          const double* ref_xyz, double* out, void* stream);
/* Velocity-Verlet halves (integrator.py:21-48), numpy's expression order.
 * phase 0: pre-force (x += v dt + f h dt^2 / m; old force = f; f = 0);
 * phase 1: post-force (v += (f + old) h dt / m); phase 2: phase 1 followed by
 * the next step's phase 0 in one pass (bit for bit the two launches).
 * *nonfinite |= 1 on non-finite state. */
int lmd_verlet_step(int64_t n, int phase, double dt, double mass, double* x, double* y,
                    double* z, double* vx, double* vy, double* vz, double* fx, double* fy,
                    double* fz, double* ox, double* oy, double* oz, int32_t* nonfinite,
                    void* stream);

/* ------------------------------------------------------------- tools */
/* FP64 pipe peak microbenchmark: blocks x threads threads, each running
 * iters x 128 independent-chain DFMAs (2 flops each).  Time it with CUDA
 * events on `stream`; scratch needs `threads` doubles. */
int lmd_dfma_burn(int blocks, int threads, int iters, double* scratch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B200MD_H */
