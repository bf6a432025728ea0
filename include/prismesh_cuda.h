/*
 * prismesh_cuda.h -- C ABI of libprismesh_cuda.so (sm_100a).
 *
 * The drop-in boundary for the extruded-mesh column loop of
 * Bercea et al. 2016 (arXiv:1604.05937).  Every entry point takes plain
 * pointers and sizes; device pointers are CUDA global-memory addresses
 * (e.g. torch.Tensor.data_ptr()), `stream` is a cudaStream_t (0 = legacy
 * default stream).  Calls are asynchronous on `stream` unless stated.
 * Every function returns 0 on success and a nonzero PM_E* code otherwise;
 * pm_last_error() then returns a thread-local message.  Nothing throws
 * across the ABI.
 *
 * Reference interfaces replaced (paths under the reference checkout):
 *   pm_build_cell_map        <- pkg/src/prismesh/fspace.py:192-215 (build_cell_map)
 *                               + fspace.py:218-229 (compute_offsets)
 *                               + fspace.py:137-149 (FunctionSpace numbering)
 *   pm_extrude_coordinates   <- pkg/src/prismesh/extrusion.py:66-85
 *   pm_column_mass           <- SPEC.md:333-341 iterate_columns driving
 *                               SPEC.md:412-420 assemble_residual
 *                               (Algorithm 3)
 *   pm_column_mass_patch     <- same, race-free owner-computes schedule
 *                               replacing SPEC.md:343-364 colouring
 *   pm_column_mass_strip     <- same, strip-patch schedule (vertex layouts)
 *   pm_build_strips          <- host planner of that schedule
 *   pm_column_mass_strip_red <- same, global strips + REDG
 *   pm_build_global_strips   <- host planner of that schedule
 *   pm_column_mass_strip_tma <- same, run strips: whole vertex columns by
 *                               bulk copies, several columns per copy
 *   pm_build_run_strips      <- host planner of that schedule
 *   pm_column_mass_tile      <- same, band tiles staged by TMA bulk copies
 *                               (experimental: PM_EXPERIMENTAL=1 builds)
 *   pm_tiles_build / _info / _export / _free <- host planner of that schedule
 *   pm_column_mass_patch_strips <- same, store-first strips inside patches
 *                               (experimental: PM_EXPERIMENTAL=1 builds)
 *   pm_build_patch_strips    <- host planner of that schedule
 *   pm_column_mass_dg_range  <- the DG loop over a cell range (pipelining)
 *   pm_column_probe          <- SPEC.md:338-340 counting / gather kernels
 *                               (verification.py:47-75 materialized maps)
 *   pm_halo_pack / _unpack   <- PAPER.md:770-775 (halo exchange between
 *                               base-mesh partitions; SPEC.md:9 leaves it out)
 *   pm_greedy_color_cells    <- SPEC.md:343-351 color_base_cells
 *   pm_rcm_order             <- pkg/src/prismesh/ordering.py:45-90 (host BFS)
 *   pm_rcm_order_device      <- pkg/src/prismesh/ordering.py:45-90 (device walk)
 *   pm_stencil_*             <- SPEC.md:322-341 StencilKernel.apply (user kernels)
 *   pm_column_mass_strip_dg  <- SPEC.md:333-341 iterate_columns, cell-only
 *                               (DG x DG, DG x CG1) layouts along strips
 *   pm_strip_step_cells      <- host planner of that schedule (cell per step)
 *   pm_build_flags           <- (build features: experimental schedules)
 */
#ifndef PRISMESH_CUDA_H
#define PRISMESH_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PM_OK = 0,
  PM_EINVAL = 1,   /* bad argument (shape / arity / layout)  -> ValueError   */
  PM_ECUDA = 2,    /* CUDA runtime error                     -> RuntimeError */
  PM_EOVERFLOW = 3 /* DoF numbers do not fit int32           -> ValueError   */
};

/* Schedules (`variant` argument of pm_column_mass). */
enum {
  PM_VARIANT_AUTO = 0,    /* DG (2,1) fields: STREAM, otherwise COLUMN      */
  PM_VARIANT_ATOMIC = 1,  /* thread per cell-layer, fp64 REDG on shared DoFs */
  PM_VARIANT_PATCH = 2,   /* patch-owner gather (pm_column_mass_patch)      */
  PM_VARIANT_COLUMN = 3,  /* warp segment per column, lanes = layers, REDG   */
  PM_VARIANT_COLORED = 4, /* COLUMN over one colour's cells, plain RMW      */
  PM_VARIANT_STREAM = 5,  /* DG (2,1) fields through TMA bulk copies; the
                             field is addressed densely (cell c, layer l,
                             slot j at (c L + l) k + j), i.e. the Alg. 1
                             numbering of cell-only layouts: cell_map and
                             offsets are not read for the field (only the
                             coordinate maps are)                          */
  PM_VARIANT_STRIP = 6,   /* strip-patch owner gather (pm_column_mass_strip) */
  PM_VARIANT_STRIPRED = 7 /* global strips + REDG (pm_column_mass_strip_red) */
};

const char *pm_last_error(void);
int pm_version(void);

/* --- K0: numbering / map generation (device) ---------------------------
 * delta6[2*d1+d2] = DoFs per extruded entity (d1,d2).  Writes the int32
 * bottom-layer map cell_map[n_cells*k] in the reference slot order and the
 * int32 per-slot offsets[k].  Values are computed in int64 and truncated
 * to int32 exactly like the reference numpy store (wraps past 2^31-1);
 * *total_dofs (host) receives the exact int64 total. */
int pm_build_cell_map(const int32_t *cell_vertices, const int32_t *cell_edges,
                      int64_t n_cells, int64_t n_vertices, int64_t n_edges,
                      const int32_t *delta6, int32_t layers, int32_t k,
                      int32_t *cell_map, int32_t *offsets,
                      int64_t *total_dofs, void *stream);

/* Number of slots of a layout (host, no device work). */
int pm_num_slots(const int32_t *delta6, int32_t *k_out);

/* --- extruded coordinate field (device) --------------------------------
 * out[3*(i*(layers+1)+l)+c] = (x_i, y_i, l*h)[c]. */
int pm_extrude_coordinates(const double *base_coords, int64_t n_vertices,
                           int32_t layers, double layer_height, double *out,
                           void *stream);

/* --- the column loop: y (+)= M x over every cell-layer -----------------
 * delta6   : the field layout (DoFs per extruded entity, as in
 *            pm_build_cell_map); k = its slot count (1,2,3,6,18 built)
 * cell_map : device int32 [n_cells*k];   offsets: device int32 [k]
 * coord_map: device int32 [n_cells*18];  coord_offsets: device int32 [18]
 * coords   : device fp64 extruded coordinate field
 * mref     : HOST fp64 [k*k] reference-prism mass matrix (slot order)
 * mtri, mline: HOST fp64 Kronecker factors of mref (nh x nh triangle,
 *            nv x nv interval mass matrices of the layout's element; the
 *            column / patch kernels apply mref by sum factorisation)
 * x, y     : device fp64 fields of length n_dofs (DoF numbers < 2^31)
 * accumulate: 0 -> y = M x (y is overwritten), 1 -> y += M x
 * variant  : PM_VARIANT_*
 * cells    : optional device int32 list of n_list cells to visit (one
 *            colour for PM_VARIANT_COLORED, which always accumulates);
 *            NULL -> all n_cells cells
 * Each cell-layer's |det J| comes from the six prism vertices read out of
 * `coords`.
 * DG (2,1)-only layouts with PM_VARIANT_AUTO / _STREAM take the bulk-copy
 * stream kernel, which does not read cell_map: it needs the dense Alg. 1
 * numbering (cell_map[c][j] = c*k*layers + j, offsets[j] = k).  A map is
 * checked once on the device (one synchronisation; skipped during stream
 * capture, where an unchecked map takes the map-reading kernels) and the
 * verdict cached per (cell_map, offsets, k, layers) pointer values, so a
 * map must not be changed in place while cached (the reference's maps are
 * immutable, fspace.py:159-174). */
int pm_column_mass(const int32_t *delta6, int32_t k, int64_t n_cells,
                   int32_t layers, const int32_t *cell_map,
                   const int32_t *offsets, const int32_t *coord_map,
                   const int32_t *coord_offsets, const double *coords,
                   const double *mref, const double *mtri,
                   const double *mline, const double *x, double *y,
                   int64_t n_dofs, int32_t accumulate, int32_t variant,
                   const int32_t *cells, int64_t n_list, void *stream);

/* Patch-owner schedule (PM_VARIANT_PATCH) for CG layouts whose DoFs live
 * on vertex / edge columns: y = M x (overwrite), bitwise deterministic,
 * no atomics.  The plan arrays (device) come from
 * paper_1604_05937_b200/schedule.py: patch -> visited cells (grouped by
 * colour: color_ptr[p*(n_colors+1)+c]), patch -> local entities (owned
 * first; codes v or n_vertices+e), per visited cell the 16-bit local ids
 * of its 3 vertices (+3 edges).  chunk = layers per chunk (8, 16, 32). */
int pm_column_mass_patch(const int32_t *delta6, int32_t k, int64_t n_vertices,
                         int64_t n_edges, int32_t layers,
                         const int32_t *cell_map, const int32_t *coord_map,
                         const double *coords, const double *mref,
                         const double *mtri, const double *mline,
                         const double *x, double *y, int64_t n_patches,
                         int32_t n_colors, int32_t chunk, int32_t max_local,
                         int32_t max_owned, const int32_t *cell_ptr,
                         const int32_t *cells, const int32_t *color_ptr,
                         const int32_t *ent_ptr, const int32_t *owned,
                         const int32_t *ents, const uint16_t *lents,
                         void *stream);

/* Strip-patch schedule (PM_VARIANT_STRIP) for layouts whose DoFs live on
 * vertex columns (P1, 3-vector P1, CG1 x DGk): y = M x (overwrite),
 * deterministic, no atomics.  Per patch the local vertex columns are staged
 * in shared memory once per chunk and the cells are walked as strips (one
 * new vertex per step); plan arrays from schedule.build_strip_plan /
 * pm_build_strips. */
int pm_column_mass_strip(const int32_t *delta6, int32_t k, int32_t layers,
                         const double *coords, const double *mref,
                         const double *mtri, const double *mline,
                         const double *x, double *y, int64_t n_patches,
                         int32_t chunk, int32_t threads, int32_t max_local,
                         int32_t max_y, int32_t max_owned, int32_t max_steps,
                         int32_t max_strips, int32_t max_oy,
                         const int32_t *ent_ptr, const int32_t *owned,
                         const int32_t *ents, const int32_t *patch_strip_ptr,
                         const int32_t *strip_step_ptr, const uint16_t *step_v,
                         const uint8_t *step_slot, const uint8_t *step_flags,
                         const int32_t *step_y, const int32_t *patch_y_count,
                         const int32_t *own_base, const int32_t *own_y_ptr,
                         const int32_t *own_y, void *stream);

/* Global-strip schedule (PM_VARIANT_STRIPRED) for vertex-column layouts:
 * sequential strips over the whole mesh (pm_build_global_strips), one
 * register window per W-lane segment, one coalesced fp64 REDG per
 * departing vertex.  accumulate = 0 zeroes y first.  chunk = lanes (levels)
 * per segment: 8, 16 or 32. */
int pm_column_mass_strip_red(const int32_t *delta6, int32_t k, int32_t layers,
                             const double *coords, const double *mref,
                             const double *mtri, const double *mline,
                             const double *x, double *y, int64_t n_dofs,
                             int32_t accumulate, int64_t n_strips,
                             int32_t chunk, const int32_t *strip_ptr,
                             const int32_t *steps,
                             const int32_t *steps_e /* P2: 2 edges/step */,
                             int64_t n_vertices, void *stream);

/* Band-tile schedule for vertex-column layouts (P1, 3-vector P1, CG1 x DG0,
 * CG1 x DG1; a vertex-permutation invariant triangle factor).  A persistent
 * grid, one CTA per SM; CTA c takes tiles c, c + G, ... of pm_tiles_build:
 * producer warps stage each tile's vertex runs (whole columns of x and of
 * the coordinate field) in shared memory with one cp.async.bulk per run and
 * array (stages = pm_tile_smem_layout's *stages tiles in flight), a zeroing
 * warp zeroes the output columns each tile touches first (y needs no
 * memset) and publishes that, the tile waits for the tiles zeroing its
 * columns, and the other warps walk the tile's strips as in
 * pm_column_mass_strip_red.  blob / off = pm_tiles_blob's records, zero_ptr
 * / zero_v0 / zero_n = pm_tiles_export's first-touch runs (device); ctl =
 * int32[3] initially {0, 0, 1}, flags = int32[n_tiles] initially 0 (so one
 * plan must not serve concurrent calls).  x and y index global DoFs;
 * n_dofs / n_coords = valid doubles from x / coords.  area_c = byte offset
 * of the coordinate area in a data buffer of data_bytes (a multiple of 128)
 * bytes; width = lanes (layers) per segment: 8, 16 or 32.
 * Experimental (slower than pm_column_mass_strip_red): compiled only with
 * PM_EXPERIMENTAL=1, otherwise PM_EINVAL (pm_build_flags bit 0). */
int pm_column_mass_tile(const int32_t *delta6, int32_t layers,
                        const double *coords, int64_t n_coords,
                        const double *mtri, const double *mline,
                        const double *x, double *y, int64_t n_dofs,
                        const int32_t *blob, const int64_t *off,
                        const int32_t *zero_ptr, const int32_t *zero_v0,
                        const int32_t *zero_n, int32_t *ctl, int32_t *flags,
                        int32_t n_tiles, int32_t area_c,
                        int32_t data_bytes, int32_t max_slots,
                        int32_t max_words, int32_t width, void *stream);
/* Shared-memory bytes in front of the data buffers; *stages = buffers,
 * *threads = CTA size (both compile-time). */
int pm_tile_smem_layout(const int32_t *delta6, int32_t max_words,
                        int32_t max_slots, int32_t width, int32_t *stages,
                        int32_t *threads);

/* Host planner of the band-tile schedule: cells in index order cut into
 * tiles of consecutive cells whose vertex columns (col_f + col_c bytes
 * each, + 32 bytes slack) fit `budget`, at most max_cells each; strips
 * split until a tile has min_strips of at least min_sub cells.  *handle
 * receives the plan (pm_tiles_info: {tiles, runs, zero runs, deps, strips,
 * steps, max field area, max coordinate area, max slots, max cells, max
 * strips per tile};
 * pm_tiles_export: the 14 int32 arrays cell_ptr, run_ptr, run_v0, run_n,
 * run_fa, run_ca, zero_ptr, zero_v0, zero_n, dep_ptr, deps, strip_ptr,
 * strip_step0, strip_len and the int16 steps; pm_tiles_free). */
int pm_tiles_build(int64_t n_cells, int64_t n_vertices, int64_t n_edges,
                   const int32_t *cell_vertices, const int32_t *cell_edges,
                   int64_t col_f, int64_t col_c, int64_t budget,
                   int32_t max_cells, int32_t min_strips, int32_t min_sub,
                   void **handle);
int pm_tiles_info(void *handle, int64_t *info);
int pm_tiles_export(void *handle, int32_t **arrays, int16_t *steps);
/* The plan as one int32 record per tile (the kernel's input): off[t] ..
 * off[t+1] (n_tiles + 1 entries) = tile t's words of blob; NULL blob / off
 * only sizes it: sizes = {total words, longest record}. */
int pm_tiles_blob(void *handle, int32_t *blob, int64_t *off, int64_t *sizes);
void pm_tiles_free(void *handle);

/* DG (2,1) fields: the stream kernel over the cell range
 * [cell_begin, cell_end) only (cell_begin*layers a multiple of 256); y is
 * overwritten there.  Used to pipeline host<->device copies with compute. */
int pm_column_mass_dg_range(const int32_t *delta6, int32_t k,
                            int64_t cell_begin, int64_t cell_end,
                            int32_t layers, const int32_t *cell_map,
                            const int32_t *offsets, const int32_t *coord_map,
                            const int32_t *coord_offsets, const double *coords,
                            const double *mref, const double *x, double *y,
                            void *stream);

/* --- probes for the par-loop itself (exact integer checks) -------------
 * mode 0: out_i64[(c*layers+l)*k + j] = cell_map[c*k+j] + l*offsets[j]
 *         (the materialised per-(cell,layer) lists)
 * mode 1: out_f64[dof] += 1 for every slot of every cell-layer (counting
 *         kernel) -- out_f64 must be zeroed by the caller. */
int pm_column_probe(int32_t mode, int32_t k, int64_t n_cells, int32_t layers,
                    const int32_t *cell_map, const int32_t *offsets,
                    int64_t *out_i64, double *out_f64, void *stream);

/* --- multi-GPU halo (ghost vertex-column partial sums) ------------------
 * pack:   buf[i*col + t] = y[cols[i] + t]   for i < n_cols, t < col
 * unpack: y[cols[i] + t] += buf[i*col + t]
 * (`cols` = device int64 DoF origins of the ghost / owned columns). */
int pm_halo_pack(const double *y, const int64_t *cols, int64_t n_cols,
                 int32_t col, double *buf, void *stream);
int pm_halo_unpack_add(double *y, const int64_t *cols, int64_t n_cols,
                       int32_t col, const double *buf, void *stream);

/* --- host setup: reverse Cuthill-McKee BFS (no device work) -------------
 * offsets[n+1], neighbours sorted by (degree, index) within each row.
 * order_out[n] receives the Cuthill-McKee visit order (not reversed). */
int pm_rcm_order(const int64_t *offsets, const int64_t *neighbours, int64_t n,
                 int64_t *order_out);

/* --- host setup: greedy base-cell colouring (no device work) ------------
 * Cells in index order take the smallest colour not used by an already
 * coloured cell sharing a vertex.  vc_offsets/vc_cells:
 * vertex->cell CSR.  Returns the colour count in *n_colors. */
int pm_greedy_color_cells(const int32_t *cell_vertices, int64_t n_cells,
                          const int64_t *vc_offsets, const int32_t *vc_cells,
                          int32_t *color_out, int32_t *n_colors);

/* --- host setup: strips for the strip-patch schedule ----------------------
 * Per patch (visited cells cell_ptr/cells, 16-bit local vertex ids lents,
 * `owned` owned vertices first) walk the cells as edge-connected strips of
 * at most max_len cells; see csrc/host_setup.cpp for the record format.
 * totals = {strips, steps, owner-list entries}. */
int pm_build_strips(int64_t n_patches, const int32_t *cell_ptr,
                    const int32_t *cells, const int32_t *cell_edges,
                    const uint16_t *lents, const int32_t *owned,
                    const int32_t *ent_ptr, int32_t max_len,
                    int32_t *patch_strip_ptr, int32_t *strip_step_ptr,
                    uint16_t *step_v, uint8_t *step_slot, uint8_t *step_flags,
                    int32_t *step_y, int32_t *patch_y_count,
                    int32_t *own_y_ptr, int32_t *own_y, int64_t *totals);

/* --- host setup: global sequential strips -------------------------------
 * strip_ptr[n_strips+1] into steps (3 fill vertices, then one new vertex per
 * cell); capacities: strips <= n_cells, steps <= 3*n_cells.  totals =
 * {strips, steps}. */
int pm_build_global_strips(int64_t n_cells, int64_t n_edges,
                           const int32_t *cell_vertices,
                           const int32_t *cell_edges,
                           const uint8_t *cell_mask /* NULL: all cells */,
                           const int32_t *scan_order /* NULL: index order;
                              else the cells in the order strips start */,
                           int32_t max_len, int32_t *strip_ptr,
                           int32_t *steps,
                           int32_t *steps_e /* NULL, or 2 edges per step */,
                           int64_t *totals);

/* Run strips: the same plan with the start orientation of a strip chosen
 * so that its even and its odd vertices each continue by consecutive ids
 * (steps[k+2] == steps[k] + 1).  On a level-ordered mesh (RCM,
 * ordering.py:45-90) such a strip follows the band between two BFS levels
 * and, under Alg. 1 (fspace.py:141-147: consecutive vertex ids are
 * consecutive columns), its vertex columns are two contiguous slabs of the
 * field.  A first pass starts strips only at cells that have such a start
 * (walking back to the band's first free cell), a second pass covers the
 * rest by the plain rule.  Same arguments and capacities as
 * pm_build_global_strips. */
int pm_build_run_strips(int64_t n_cells, int64_t n_edges,
                        const int32_t *cell_vertices,
                        const int32_t *cell_edges, const uint8_t *cell_mask,
                        const int32_t *scan_order, int32_t max_len,
                        int32_t *strip_ptr, int32_t *steps, int32_t *steps_e,
                        int64_t *totals);

/* y (+)= M x over sequential strips for P1 (delta6 = {1,0,0,0,0,0}) and
 * 3-vector P1 ({3,0,0,0,0,0}) columns of at most 128 layers (P1 with two
 * 32-layer chunks per warp: 256): the strip walk
 * of pm_column_mass_strip_red (dof =
 * column origin + l * offset), with the vertex columns brought into shared
 * memory by 1-D bulk copies (cp.async.bulk), one copy per run of up to 4
 * consecutive vertex ids per strip side, into a ring shared by the warps
 * that walk the column's 32-layer chunks.  Any strip plan is valid; run
 * strips (pm_build_run_strips) make the copies large.  x and coords must be
 * 16-byte aligned; mtri must be invariant under vertex permutations.
 * Zeroes y first unless `accumulate`. */
int pm_column_mass_strip_tma(const int32_t *delta6, int32_t k, int32_t layers,
                             const double *coords, const double *mtri,
                             const double *mline, const double *x, double *y,
                             int64_t n_dofs, int32_t accumulate,
                             int64_t n_strips, const int32_t *strip_ptr,
                             const int32_t *steps, int64_t n_vertices,
                             void *stream);

/* Store-first patch strips (PM_VARIANT_STRIPRED over patches): the cells
 * are grouped into compact patches (patch_cells, patch_ptr: e.g. runs of the
 * Morton order of the centroids) and walked as sequential strips that never
 * leave their patch; item_ptr[p] .. item_ptr[p+1] are patch p's strips.
 * A patch's strips are one continuous step stream (no window refill between
 * strips): a strip's three fill steps flush the previous strip's window,
 * its first two carry PM_STEP_NOCELL, and their edges (P2) are -1, e01, then
 * e12, e02 (e_ab joins fill vertices a, b).  Step ids carry PM_STEP_STORE on
 * the first residency of an entity whose cells all lie in one patch: the
 * kernel stores that partial column instead of adding it.  zero_list = the other entities (code v, or
 * n_vertices + e for edge e), cleared by the kernel's zero pass.
 * Capacities: item_ptr n_patches+1, strip_ptr n_cells+1, steps 3*n_cells,
 * steps_e 6*n_cells, zero_list n_vertices+n_edges; totals = {strips, steps,
 * zero entities}.  Entity ids must stay below 2^29. */
#define PM_STEP_STORE (1 << 30)
/* ... and on a strip's first two (fill) steps: no cell after the step */
#define PM_STEP_NOCELL (1 << 29)
int pm_build_patch_strips(int64_t n_cells, int64_t n_vertices, int64_t n_edges,
                          const int32_t *cell_vertices,
                          const int32_t *cell_edges,
                          const int32_t *patch_cells, const int32_t *patch_ptr,
                          int64_t n_patches, int32_t max_len,
                          int32_t *item_ptr, int32_t *strip_ptr,
                          int32_t *steps,
                          int32_t *steps_e /* NULL, or 2 edges per step */,
                          int32_t *zero_list, int64_t *totals);

/* The strip-REDG kernels over store-first patch strips (replaces the
 * SPEC.md:333-364 coloured par-loop like pm_column_mass_strip_red).  Items
 * are (patch, layer chunk); a segment walks the patch's strips in order.
 * accumulate = 0: the zero pass clears the zero_list columns and the
 * chunk-boundary levels, flagged residencies store; accumulate = 1: every
 * residency adds (no zero pass). */
/* pm_column_mass_patch_strips: the patch-strip (stream-mode) kernel is
 * experimental (slower than the global strips): compiled only with
 * PM_EXPERIMENTAL=1, otherwise PM_EINVAL (pm_build_flags bit 0); the host
 * planner pm_build_patch_strips is always available. */
int pm_column_mass_patch_strips(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mref, const double *mtri, const double *mline,
    const double *x, double *y, int64_t n_dofs, int32_t accumulate,
    int64_t n_patches, int32_t chunk, const int32_t *item_ptr,
    const int32_t *strip_ptr, const int32_t *steps,
    const int32_t *steps_e /* P2: 2 edges/step */, int64_t n_vertices,
    int64_t n_zero, const int32_t *zero_list, void *stream);

/* Strip-REDG with the halo exchange fused in (multi-GPU): as
 * pm_column_mass_strip_red for vertex-column layouts, except that the
 * partial columns of vertices v < ghost_vertex_end (owned by the peer rank)
 * are added with REDG straight into y_peer, the peer's y window mapped
 * into this process (pm_ipc_open) and shifted like y so global DoF numbers
 * index it.  Replaces the reference-anticipated pack / ncclSend / recv /
 * owner-add of SURVEY §8e with one kernel.  The peer's window must be
 * zeroed before and read only after every contributing kernel finished. */
int pm_column_mass_strip_red_peer(
    const int32_t *delta6, int32_t k, int32_t layers, const double *coords,
    const double *mref, const double *mtri, const double *mline,
    const double *x, double *y, int64_t n_dofs, int32_t accumulate,
    int64_t n_strips, int32_t chunk, const int32_t *strip_ptr,
    const int32_t *steps, int64_t n_vertices, double *y_peer,
    int64_t ghost_vertex_end, void *stream);

/* CUDA IPC of a device buffer for the fused halo: export (64-byte handle +
 * byte offset inside its allocation), open in another process (returns the
 * mapped pointer), close.  Replaces the NCCL transport of the exchange. */
int pm_ipc_export(const void *ptr, void *handle64, int64_t *offset);
int pm_ipc_open(const void *handle64, int64_t offset, void **ptr);
int pm_ipc_close(void *ptr, int64_t offset);

/* Stream-ordered signalling between ranks (the fused halo's step protocol,
 * no host synchronisation): pm_stream_signal queues a one-thread kernel
 * that, after the stream's preceding work, stores `value` to `flag`
 * (system-scope release; `flag` may be a peer mapping from pm_ipc_open);
 * pm_stream_wait_geq makes `stream` wait until the local 32-bit `flag` is
 * >= value (cuStreamWaitValue32, no spinning kernel). */
int pm_stream_signal(uint32_t *flag, uint32_t value, void *stream);
int pm_stream_wait_geq(const uint32_t *flag, uint32_t value, void *stream);

/* Device derive_edges (replaces mesh.py:33-84 derive_edges): edge set of a
 * triangle mesh as the sorted unique vertex pairs, cell_edges[c][k] = the
 * edge opposite local vertex k.  Device arrays: cell_vertices (n_cells,3)
 * int32; edge_vertices needs room for 3*n_cells rows of 2 int32; cell_edges
 * (n_cells,3) int32.  n_vertices < 0: unbounded.  Host outputs: *n_edges,
 * *status = topology error bits (1 negative index, 2 index >= n_vertices,
 * 4 repeated vertex, 8 duplicate cell, 16 edge on > 2 cells; outputs
 * undefined when nonzero).  Synchronises the stream. */
int pm_derive_edges(const int32_t *cell_vertices, int64_t n_cells,
                    int64_t n_vertices, int32_t *edge_vertices,
                    int32_t *cell_edges, int64_t *n_edges, int32_t *status,
                    void *stream);

/* The mesh's vertex graph for RCM (replaces mesh.py vertex_neighbours +
 * the row lexsort of ordering.py rcm_order): CSR (offsets n_vertices+1
 * int64, nbr 2*n_edges int32, device) of edge-adjacent vertices, every row
 * sorted by (degree, index).  n_vertices < 2^24.  Synchronises the
 * stream. */
int pm_vertex_graph_sorted(const int32_t *edge_vertices, int64_t n_edges,
                           int64_t n_vertices, int64_t *offsets, int32_t *nbr,
                           void *stream);

/* Device Cuthill-McKee walk (replaces the serial BFS of ordering.py:45-90,
 * `_cuthill_mckee`; same result as pm_rcm_order, bit for bit): offsets
 * (n+1 int64) and neighbours (int32) on the device, every row sorted by
 * (degree, index) (pm_vertex_graph_sorted's output); order (n int64,
 * device) receives the Cuthill-McKee visit order (not reversed).
 * Level-synchronous in one thread block: each new vertex is appended by
 * its lowest-positioned discoverer at its row rank, which is the serial
 * queue order.  n < 2^31 - 1.  Synchronises the stream. */
int pm_rcm_order_device(const int64_t *offsets, const int32_t *neighbours,
                        int64_t n, int64_t *order, void *stream);

/* --- user stencil kernels for iterate_columns ---------------------------
 * (SPEC.md:322-341 StencilKernel: an arbitrary per-cell-layer procedure;
 * the reference's consumers generate and compile C per kernel,
 * PAPER.md:777-783.)  `source` is CUDA C++ defining
 *   __device__ void pm_kernel(double *out, const double *const *in,
 *                             long long cell, int layer);
 * in[a][j] = argument a at slot j of the cell-layer, out[j] = contribution
 * to output slot j (starts at 0, added into the output field).  NVRTC
 * compiles it for sm_100a into a generated column loop (Alg. 3).
 * n_in <= 8 input arguments with k_in[a] <= 64 slots, k_out <= 64.
 * pm_stencil_check: compile only (no device needed), cubin size out.
 * pm_stencil_launch: colored = 0 -> thread per cell-layer, fp64 REDG into
 * `out`; colored = 1 -> thread per listed cell (cells[i], i < n_cells: one
 * colour of color_base_cells), layers in order, plain +=, deterministic.
 * cells = NULL means cells 0..n_cells-1.  in_fields / in_maps / in_offsets
 * are HOST arrays of n_in device pointers (field, bottom-layer map
 * (N2, k) int32, offsets (k) int32); out_map / out_offsets likewise for
 * the output space.  Asynchronous on `stream`. */
int pm_stencil_check(const char *source, int32_t n_in, const int32_t *k_in,
                     int32_t k_out, int64_t *cubin_bytes);
int pm_stencil_compile(const char *source, int32_t n_in, const int32_t *k_in,
                       int32_t k_out, void **handle);
int pm_stencil_launch(void *handle, int32_t colored, int64_t n_cells,
                      int32_t layers, const double *const *in_fields,
                      const int32_t *const *in_maps,
                      const int32_t *const *in_offsets, double *out,
                      const int32_t *out_map, const int32_t *out_offsets,
                      const int32_t *cells, void *stream);
int pm_stencil_free(void *handle);

/* Build features: bit 0 = the experimental schedules (tile, store-first
 * patch strips) are compiled in (PM_EXPERIMENTAL=1 at build time); without
 * them pm_column_mass_tile / pm_column_mass_patch_strips return PM_EINVAL. */
int pm_build_flags(void);

/* --- DG layouts along strips --------------------------------------------
 * pm_strip_step_cells: for a strip plan (pm_build_global_strips: strip_ptr
 * n_strips+1, steps = entering vertices) the cell each step forms
 * (step_cells, one per step; -1 on a strip's two fill steps), host.
 * pm_column_mass_strip_dg: y = M x for a layout with DoFs on the prism
 * cells only, x, y in the Alg. 1 numbering (dense per cell column):
 * delta6 = {0,0,0,0,0,k}, k in {1,2,3,6} (DG x DG), or delta6 =
 * {0,0,0,0,d0,0}, k = 2 d0, d0 in {1,3} (DG x CG1: level DoFs shared by
 * the two layers of a cell that meet there).  The cells are walked along
 * the strips, one new vertex's coordinate chunk and the formed cell's
 * field chunk per step through a cp.async ring; DG x DG stores every DoF
 * once (no zeroing, no atomics); DG x CG1 combines a level's two layers by
 * shuffle and stores it once, except the levels between W-layer chunks,
 * which are zeroed first and added.
 * Replaces the per-cell-layer coordinate gathers of the DG stream kernel
 * (reference loop: SPEC.md:333-341 iterate_columns). chunk = 8, 16 or 32
 * layers per warp segment.  Device pointers, asynchronous on `stream`. */
int pm_strip_step_cells(int64_t n_cells, int64_t n_vertices,
                        const int32_t *cell_vertices, const int32_t *strip_ptr,
                        int64_t n_strips, const int32_t *steps,
                        int32_t *step_cells);
int pm_column_mass_strip_dg(const int32_t *delta6, int32_t k, int64_t n_cells,
                            int32_t layers, const double *coords,
                            const double *mref,
                            const double *x, double *y, int64_t n_strips,
                            int32_t chunk, const int32_t *strip_ptr,
                            const int32_t *steps, const int32_t *step_cells,
                            void *stream);

/* Device cell re-sort of apply_ordering (replaces ordering.py:142-152):
 * cells_out = forward[cell_vertices][perm] with perm the stable lexsort of
 * the rows' sorted new vertex triples; perm_out (optional) receives perm.
 * Device arrays; synchronises the stream. */
int pm_reorder_cells(const int32_t *cell_vertices, int64_t n_cells,
                     const int64_t *forward, int64_t n_vertices,
                     int32_t *cells_out, int32_t *perm_out, void *stream);

/* STREAM triad a = b + alpha*c over n doubles (16-byte aligned arrays):
 * the bandwidth reference of the perfbench module (replaces SPEC.md
 * perfbench "stream_triad", the paper's Table "Maximum
 * STREAM triad"); 24 bytes per element per pass. */
int pm_stream_triad(double *a, const double *b, const double *c, double alpha,
                    int64_t n, void *stream);

/* Programmatic dependent launch for the DG stream kernel launched by this
 * host thread (returns the previous setting).  With it on, a stream
 * kernel starts its prologue, TMA loads and coordinate gathers while the
 * previous kernel of the stream drains, and waits for it before its first
 * store: valid only when that previous kernel writes none of this call's
 * inputs (back-to-back applies to the same fields, e.g. captured by
 * MassOperator.graph(repeat=K)). */
int pm_set_launch_overlap(int32_t on);

/* Device properties used to size grids (SM count, L2 bytes). */
int pm_device_info(int32_t *sm_count, int64_t *l2_bytes);

#ifdef __cplusplus
}
#endif
#endif /* PRISMESH_CUDA_H */
