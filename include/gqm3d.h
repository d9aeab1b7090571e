/* gqm3d.h -- C ABI of the B200-native gQM3D refinement library (libgqm3d.so).
 *
 * The drop-in boundary is the reference's Python entry point
 *   tetrefine.refine(plc, cfg) -> (Mesh, QualityReport)
 *   (/root/reference/pkg/src/tetrefine/refine.py:928-933)
 * whose internal seam is the optional compiled-kernel module `_K`
 * (/root/reference/pkg/src/tetrefine/mesh.py:32-35): caller-owned flat
 * arrays in, integer status codes out, no exceptions across the seam.
 * This header replaces that seam with one GPU-resident call per PLC:
 * the caller validates and box-augments the PLC (host setup, refine.py:523-531),
 * then gq_refine() runs init_delaunay + every refinement round on the device,
 * and the gq_export_* calls fill caller-allocated arrays sized from gq_counts.
 *
 * Every call returns 0 on success or a GQ_E* status; gq_last_error() gives
 * the message.  One refine at a time per context.
 */
#ifndef GQM3D_H
#define GQM3D_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gq_ctx gq_ctx;

enum {
  GQ_OK = 0,
  GQ_EINVAL = 1,     /* bad argument */
  GQ_ECUDA = 2,      /* CUDA runtime failure (no device, OOM, fault) */
  GQ_EDEVICE = 3,    /* device-side invariant failure (see message) */
  GQ_EUNSUPPORTED = 4
};

/* refine.py:73-88 RefineConfig (workers / sequential_until are outcome-neutral) */
typedef struct {
  double B;
  int32_t max_rounds;
  int32_t flags;     /* bit 0: verbose per-round lines on stderr; bit 1: paper-literal
                        grow-and-blast filter (one claim round, no resurrection) */
  uint64_t seed;
} gq_config;

typedef struct {
  int64_t nv, nt, n_subsegments, n_subfaces, n_rounds, n_skipped;
  int64_t n_real_tets, steiner_points, input_points;
  int64_t exact_calls[4];      /* orient2d, incircle2d, orient3d, insphere exact fallbacks */
  double device_ms;            /* GPU time of gq_refine (CUDA events) */
  double init_ms;              /* of which bulk Delaunay construction */
  int64_t kernel_launches;
  int64_t region_calls;
  int64_t bytes_alg;           /* region kernels' algorithmic HBM bytes (58 B/tet tested + 24 B/point) */
  double region_ms;            /* time in the region (cavity) kernels */
  /* SURVEY 8(d) whole-refine algorithmic bytes:
   *   144 N_cand + 58 T_tested + 8 K_claims + 51 T_created + 1 T_deleted + 29 N_steiner */
  int64_t n_cand, t_tested, k_claims, t_created, t_deleted;
  int64_t bytes_refine;
} gq_counts;

/* create a context on CUDA device `device` */
int gq_create(int device, gq_ctx** out);
int gq_destroy(gq_ctx* ctx);
const char* gq_last_error(gq_ctx* ctx);

/* Refine an already validated + box-augmented PLC.
 *   xyz[n][3]      points (augmented; the first n_input are the caller's, origin 0)
 *   seg[m][2]      segments (vertex index pairs)
 *   poly_off[f+1], poly_idx[]  polygon vertex cycles (CSR)
 *   poly_keep[f][2] projection axes of each polygon (facets.py:262-268)
 *   order[n]       insertion order of init_delaunay (mesh.py:878-880)
 * Replaces: tetrefine.refine -> _Driver.run (refine.py:866-925). */
int gq_refine(gq_ctx* ctx, const double* xyz, int32_t n, int32_t n_input, const int32_t* seg, int32_t m,
              const int32_t* poly_off, const int32_t* poly_idx, int32_t f, const int32_t* poly_keep,
              const int32_t* order, const gq_config* cfg, gq_counts* counts);

/* Mesh arrays as tetrefine.mesh.Mesh stores them (mesh.py:92-111), nv / nt rows. */
int gq_export_mesh(gq_ctx* ctx, double* points, uint8_t* vert_origin, int32_t* vert_tet, int32_t* tv,
                   int32_t* tn, uint8_t* alive, uint8_t* sub_mask, uint8_t* seg_mask, double* ratio,
                   uint8_t* skip_flag);
/* subsegments (u,v,sid) and subfaces (a,b,c,pid), each sorted */
int gq_export_constraints(gq_ctx* ctx, int32_t* subsegments, int32_t* subfaces);
/* per round: round, phase(0 seg,1 face,2 tet), candidates, accepted, blasted,
 * failed, inserted, pending_segments, pending_faces; plus seconds */
int gq_export_rounds(gq_ctx* ctx, int64_t* rows, double* seconds);
/* skipped elements: kind(0 seg,1 face,2 tet), reason(0 degenerate,1 short_edge,
 * 2 too_close,3 cavity_not_star_shaped), nverts, v0..v3 */
int gq_export_skipped(gq_ctx* ctx, int32_t* rows);
/* radius-edge ratio > B count and the 36-bin dihedral histogram of the real
 * tets (stats.py:26-99), computed on the device.  Tets with a dihedral angle
 * within rounding of a 5-degree bin edge are left out of hist36 and listed in
 * edge_tets (capacity edge_cap, count n_edge) for the caller to bin with the
 * reference's own expression (the last bit of acos differs between libraries). */
int gq_quality(gq_ctx* ctx, double B, int64_t* bad_count, int64_t* hist36, int32_t* edge_tets, int64_t edge_cap,
               int64_t* n_edge);

/* .node / .ele / .face files of a refined mesh (host only; formats.py:210-263 of
 * the reference: 1-based ids, "%.17g" coordinates, origin attribute, alive
 * non-ghost tets in slot order, subface rows (a<b<c, pid) sorted by the caller).
 * face_path may be NULL. */
int gq_write_mesh(const char* node_path, const char* ele_path, const char* face_path, const double* points,
                  const uint8_t* origins, int32_t nv, const int32_t* tv, const uint8_t* alive, int32_t nt,
                  const int32_t* faces, int32_t nf);

/* Device certification of PLC validity, the feature-pair part of
 * tetrefine.plc.validate (plc.py:355-383): candidate pairs from a grid over
 * the segment / triangle boxes, each decided with exact predicates.
 *   tri[f][3]   triangular polygons (features numbered segments first)
 *   status      0 no certain conflict (pairs lists the undecided ones for the
 *               caller's exact pair test), 1 a certain conflict, 2 more than
 *               pair_cap undecided pairs, 3 device arithmetic failure
 * Replaces the pair loop of validate() (and setup_fast.certify_valid). */
int gq_certify_pairs(int device, const double* xyz, int32_t n, const int32_t* seg, int32_t m, const int32_t* tri,
                     int32_t f, int32_t* status, int32_t* pairs, int64_t pair_cap, int64_t* n_pairs);

/* FP64 FMA throughput of the device in TFLOP/s (2 flops per FMA, best of 5;
 * the secondary roofline of the predicate filters). */
int gq_probe_fp64(int device, double* tflops);

/* batched exact predicates / constructions on the device, for parity tests:
 * which 0 orient3d(12) 1 insphere(15) 2 orient2d(6) 3 incircle2d(8)
 * 4 incircle3d(12) 5 encroaches_segment(9) 6 encroaches_face(12) -> out8;
 * 7 circumsphere_tet(12) 8 circumcircle_tri(9) -> outd[n][4]
 * (predicates.py:132-308, geometry.py:48-199) */
int gq_batch(int which, const double* in, int32_t n, int32_t width, int8_t* out8, double* outd);

#ifdef __cplusplus
}
#endif
#endif
