/* include/sdgpu.h -- C ABI of the B200-native smooth-distance query engine.
 *
 * Drop-in boundary for the batched point-query evaluator of the reference
 * (arXiv 2108.10480, /root/reference/proj/include/smoothdist). The reference
 * has no plugin/FFI layer of its own: its boundary IS the header-only C++
 * API below, and each entry point here replaces one or more of those calls
 * for a whole batch of queries:
 *
 *   sd_set_geometry      <- SimplexMesh / Simplex / SimplexKind   (mesh.hpp:15-50)
 *   sd_set_weights       <- WeightSet (+ build_weight_set result)  (weights.hpp:565-621)
 *   sd_build_weights     <- build_weight_set(mesh, build_adjacency(mesh))
 *                           (weights.hpp:589-621, mesh.hpp:163-183)
 *   sd_weights_info / sd_export_weights <- WeightSet fields / save_weight_cache
 *                           payload (weights.hpp:565-579, 715-742)
 *   sd_set_bvh           <- Bvh / BvhNode, reference layout        (bvh.hpp:14-32)
 *   sd_build_bvh         <- build_bvh                              (bvh.hpp:34-91)
 *   sd_export_bvh        <- Bvh::nodes (save_bvh_cache record)     (bvh.hpp:193-212)
 *   sd_save_bvh_cache / sd_load_bvh_cache       <- save_bvh_cache / load_bvh_cache
 *                           (SDBV0001, bvh.hpp:190-236)
 *   sd_save_weight_cache / sd_load_weight_cache <- save_weight_cache /
 *                           load_weight_cache (SDWT0001, weights.hpp:700-781)
 *   sd_query_points      <- smooth_min_dist(mesh, bvh, ws, q, params) per query
 *                           (smooth.hpp:166-184; beta > 0 => Barnes-Hut tree path)
 *                           smooth_min_dist_flat(mesh, ws, q, params)
 *                           (smooth.hpp:189-198; SD_EXACT)
 *   sd_finalize_device   <- detail::result_from_accum              (smooth.hpp:147-159)
 *   sd_query_simplices   <- smooth_min_dist(mesh, bvh, ws, SimplexGeom g, params) /
 *                           smooth_min_dist_flat(mesh, ws, g, params) for query
 *                           points, edges and triangles (smooth.hpp:166-198,
 *                           exact.hpp:110-367, bvh.hpp:113-180)
 *   sd_mesh_dist         <- smooth_mesh_dist(mesh, bvh, ws, query, params) for
 *                           any query mesh (smooth.hpp:212-255)
 *   sd_mesh_dist_points  <- the same for a point-cloud query mesh
 *   sd_render            <- render (render.hpp:77-134), sd_write_ppm / sd_write_png
 *   sd_grid_benchmark    <- grid_benchmark (bench.hpp:29-70), sd_write_grid_csv
 *   sd_params            <- SmoothParams {alpha, alpha_u, beta, epsilon} (params.hpp:13-22)
 *   sd_outputs           <- SmoothResult {d_hat, grad, c, grad_c, leaves, far_field}
 *                           (smooth.hpp:20-27)
 *
 * Error convention: every call returns 0 on success or a negative SD_E*
 * code, and sd_last_error() (thread-local) describes the failure, in place
 * of the reference's fail() -> std::runtime_error (common.hpp:50). The
 * evaluator semantics of the reference are kept: a query whose exponential
 * sum underflows (every term has alpha * d > 708) reports d_hat = +inf and a
 * zero gradient, never an error (smooth.hpp:151-155).
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * fails with SD_E_CUDA.
 */
#ifndef SDGPU_H
#define SDGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDGPU_ABI_VERSION 1

typedef struct sd_ctx sd_ctx;

/* SmoothParams (params.hpp:13-22); alpha_q only matters for mesh-to-mesh
 * queries, which are outside this path. */
typedef struct sd_params {
    double alpha;    /* LogSumExp sharpness, > 0 */
    double alpha_u;  /* attenuation threshold: S = alpha / max(alpha, alpha_u) */
    double beta;     /* Barnes-Hut admissibility; 0 = exact */
    double epsilon;  /* gradient denominator guard (reference default 1e-300) */
} sd_params;

/* Reference BvhNode record, byte-compatible with the 72-byte struct of
 * bvh.hpp:14-22 (Aabb box{lo, hi}; left, right (-1 on leaves), primitive,
 * count; diameter = box diagonal). Root is node 0, ids are pre-order. */
typedef struct sd_bvh_node {
    double lo[3];
    double hi[3];
    int32_t left, right, primitive, count;
    double diameter;
} sd_bvh_node;

/* Per-query outputs (SmoothResult, smooth.hpp:20-27). Only d_hat is
 * required; any other pointer may be NULL. grad / grad_c are Q x 3. */
typedef struct sd_outputs {
    double* d_hat;
    double* grad;
    double* c;
    double* grad_c;
    int64_t* leaves;          /* exact leaf evaluations */
    int64_t* far_field;       /* Barnes-Hut expansions taken */
    uint64_t* decision_hash;  /* order-independent hash of {(node, far|leaf)} */
} sd_outputs;

enum { SD_FP32 = 0, SD_FP64 = 1 };                  /* arithmetic precision */
enum { SD_EXACT = 0, SD_BVH = 1 };                  /* query mode */
enum { SD_BVH_MEDIAN = 0, SD_BVH_LBVH = 1, SD_BVH_AUTO = 2 };  /* tree builders */
enum { SD_POINT = 0, SD_EDGE = 1, SD_TRIANGLE = 2 }; /* SimplexKind (mesh.hpp:15) */

enum {
    SD_OK = 0,
    SD_E_ARG = -1,      /* invalid argument (mirrors the reference's fail()) */
    SD_E_STATE = -2,    /* geometry / weights / tree missing or inconsistent */
    SD_E_CUDA = -3,     /* CUDA runtime failure, or no device */
    SD_E_NOMEM = -4
};

const char* sd_last_error(void);
int sd_abi_version(void);

/* One context per GPU (one process per GPU in multi-GPU runs). precision is
 * SD_FP32 or SD_FP64. In SD_FP32 the vertex and query coordinates are
 * rounded to float on upload. */
int sd_create(sd_ctx** out, int device, int precision);
int sd_destroy(sd_ctx* ctx);

/* SimplexMesh: vertices V x 3 (AoS, = SimplexMesh::vertices.data()),
 * simplices N x 3 int32 (unused corners -1) and N kinds. Validated as
 * validate() does (mesh.hpp:55-87). Invalidates weights and tree. */
int sd_set_geometry(sd_ctx* ctx, const double* xyz, int64_t V, const int32_t* simplices, const uint8_t* kinds,
                    int64_t N);

/* WeightSet as flat arrays: A, sup_wtilde, ne edge polynomials a[0..4]
 * (EdgeWeightPoly::a), nt triangle polynomials stored[0..12]
 * (TriWeightPoly::stored), poly_index[N] (-1: unit weight). */
int sd_set_weights(sd_ctx* ctx, double A, double sup_wtilde, int32_t ne, const double* edge_a, int32_t nt,
                   const double* tri_stored, const int32_t* poly_index);

/* Build the WeightSet of the current geometry on the host (valences,
 * closed-form edge polynomials, triangle polynomials by the reference
 * construction) and install it, as build_weight_set does. Then read it back
 * with sd_weights_info (sizes, A, sup_wtilde) and sd_export_weights (arrays
 * sized ne x 5, nt x 13 and N; NULL skips an array). */
int sd_build_weights(sd_ctx* ctx);
int sd_weights_info(sd_ctx* ctx, double* A, double* sup_wtilde, int32_t* ne, int32_t* nt);
int sd_export_weights(sd_ctx* ctx, double* edge_a, double* tri_stored, int32_t* poly_index);

/* Upload a reference-layout tree (e.g. from the reference build_bvh), or
 * build one on the GPU: SD_BVH_MEDIAN reproduces build_bvh exactly,
 * SD_BVH_LBVH is the Morton-code linear BVH, SD_BVH_AUTO builds both and
 * keeps the one with the smaller surface-area cost. Either way the tree can
 * be exported in the reference layout so a CPU evaluator can run on it. */
int sd_set_bvh(sd_ctx* ctx, const sd_bvh_node* nodes, int64_t n);
int sd_build_bvh(sd_ctx* ctx, int method);
int sd_bvh_size(sd_ctx* ctx, int64_t* n);
int sd_export_bvh(sd_ctx* ctx, sd_bvh_node* out, int64_t cap);

/* Batched point queries with HOST buffers: q is Q x 3 doubles. The call
 * copies q to the device, evaluates, and copies the requested outputs back
 * (blocking). mode SD_EXACT ignores beta; SD_BVH uses the tree. */
int sd_query_points(sd_ctx* ctx, const double* q, int64_t Q, const sd_params* p, int mode, const sd_outputs* out);

/* Pipelined HOST-buffer queries (serving loops): enqueue one batch -- H2D
 * of q on a copy stream, the evaluation on the context's stream, D2H of
 * the requested outputs on a second copy stream -- and return at once with
 * a ticket. Batches submitted back to back overlap one batch's copies with
 * its neighbours' evaluation. Two batches are in flight at most: a third
 * submission first waits for the oldest. q and the output arrays must stay
 * valid and untouched until sd_query_wait(ticket) (ticket < 0: every
 * batch) returns; pinned host memory gives real overlap. Results are those
 * of sd_query_points. */
int sd_query_points_async(sd_ctx* ctx, const double* q, int64_t Q, const sd_params* p, int mode,
                          const sd_outputs* out, int64_t* ticket);
int sd_query_wait(sd_ctx* ctx, int64_t ticket);

/* Same with DEVICE buffers on the caller's stream (cudaStream_t, may be
 * NULL): q_dev is Q x 3 float (SD_FP32) or double (SD_FP64); outputs are
 * device pointers. Asynchronous. */
int sd_query_points_device(sd_ctx* ctx, const void* q_dev, int64_t Q, const sd_params* p, int mode,
                           const sd_outputs* out_dev, void* stream);

/* Query-sharded tree evaluation of ONE batch across `world` ranks (each
 * with the whole batch and the replicated geometry on its device): the
 * batch is sorted along the library's Hilbert order and cut into 32-query
 * packets, grouped into chunks of C consecutive packets (C = min(1024,
 * packets / (16 world)); SDGPU_SHARD_CHUNK overrides) dealt round robin:
 * rank r walks chunks r, r + world, ... and writes the outputs of their
 * queries only (the other entries of the output arrays are left untouched).
 * Whole packets stay as spatially coherent as in the single-GPU walk and
 * every rank gets a mix of cheap and expensive regions -- no cost model.
 * Tree path only (beta > 0); device buffers on the caller's stream. */
int sd_query_points_device_shard(sd_ctx* ctx, const void* q_dev, int64_t Q, const sd_params* p,
                                 const sd_outputs* out_dev, int32_t world, int32_t rank, void* stream);

/* Primitive-sharded runs: after each shard wrote its unshifted fp64
 * partial sums (c, grad_c) with sd_query_points_device and the shards were
 * summed (e.g. one NCCL all-reduce), finalize d_hat / grad exactly as
 * result_from_accum does (smooth.hpp:147-159). Device pointers. */
int sd_finalize_device(sd_ctx* ctx, const double* c, const double* grad_c, int64_t Q, const sd_params* p,
                       double* d_hat, double* grad, void* stream);

/* Primitive-sharded merge through peer memory (the alternative to one
 * all-reduce of the partial sums). Queries are owned in blocks of
 * q_per_owner: query i belongs to rank i / q_per_owner. Every rank calls
 * sd_scatter_partials with its unshifted partials (c, grad_c as written by
 * sd_query_points_device) and a DEVICE array of the world ranks' symmetric
 * buffers (each world x 4 x q_per_owner doubles, e.g. torch symmetric
 * memory): its contribution to query i is stored into the owner's buffer.
 * After a cross-rank barrier each rank calls sd_reduce_owned on its own
 * buffer: the world contributions of its n_owned queries are summed in rank
 * order and finalised (result_from_accum) into d_hat / grad. */
int sd_scatter_partials(sd_ctx* ctx, const double* c, const double* grad_c, int64_t Q, double* const* peer_bufs,
                        int32_t world, int32_t rank, int64_t q_per_owner, void* stream);
/* The same exchange fused into the evaluation: sd_query_points_device's
 * work for this rank's shard, whose finalize epilogue stores the unshifted
 * partials (c, grad_c) of query i straight into rank i / q_per_owner's
 * symmetric buffer (slot `rank`) instead of writing them locally -- no
 * separate scatter pass. q (device, fp32 or fp64 as the context); per-query
 * leaf / far-field counters optional (device, NULL to skip). Follow with a
 * barrier and sd_reduce_owned. */
int sd_query_points_scatter(sd_ctx* ctx, const void* q, int64_t Q, const sd_params* p, int mode,
                            double* const* peer_bufs, int32_t world, int32_t rank, int64_t q_per_owner,
                            int64_t* leaves, int64_t* far_field, void* stream);
int sd_reduce_owned(sd_ctx* ctx, const double* sbuf, int64_t q_per_owner, int64_t n_owned, int32_t world,
                    const sd_params* p, double* d_hat, double* grad, void* stream);

/* Mesh-to-mesh smooth distance d_hat(M, Mq) for a POINT-CLOUD query mesh
 * (smooth_mesh_dist, smooth.hpp:212-255): inner smooth distances of the Nq
 * query points (mode SD_EXACT or SD_BVH, params p), outer LogSumExp with
 * alpha_q, per-vertex gradients = softmin mass x inner gradient / (denom +
 * epsilon). Query vertices qxyz are Vq x 3; qpoints lists the vertex of each
 * point simplex (NULL: every vertex is one point, Nq = Vq). Host buffers:
 * d_hat (1 value), vertex_grads (Vq x 3, required), per_primitive (Nq, may
 * be NULL). Blocking. */
int sd_mesh_dist_points(sd_ctx* ctx, const double* qxyz, int64_t Vq, const int32_t* qpoints, int64_t Nq,
                        const sd_params* p, double alpha_q, int mode, double* d_hat, double* vertex_grads,
                        double* per_primitive);

/* Query SIMPLICES g (points, edges, triangles): smooth_min_dist(mesh, bvh,
 * ws, g, params) (mode SD_BVH, smooth.hpp:166-184; Barnes-Hut decisions use
 * the separating-halfspace box proximity of bvh.hpp:113-180) or
 * smooth_min_dist_flat(mesh, ws, g, params) (SD_EXACT, :189-198). corners:
 * Q x 9 host doubles (c0, c1, c2 of each query; unused corners ignored),
 * dims: Q values in {0, 1, 2}. The gradient is d d_hat / d (rigid
 * translation of g), as the reference's. Computed in fp64 whatever the
 * context precision. Outputs as sd_query_points. Blocking. */
int sd_query_simplices(sd_ctx* ctx, const double* corners, const int32_t* dims, int64_t Q, const sd_params* p,
                       int mode, const sd_outputs* out);

/* smooth_mesh_dist (smooth.hpp:212-255) for ANY query mesh: Vq vertices
 * (qxyz, Vq x 3), Nq simplices (qsimplices Nq x 3 vertex indices, -1 past
 * the simplex's corners; qkinds SD_POINT / SD_EDGE / SD_TRIANGLE). Each
 * simplex's softmin mass is split evenly over its corners. Outputs as
 * sd_mesh_dist_points. A point-only query mesh takes the point path. */
int sd_mesh_dist(sd_ctx* ctx, const double* qxyz, int64_t Vq, const int32_t* qsimplices, const uint8_t* qkinds,
                 int64_t Nq, const sd_params* p, double alpha_q, int mode, double* d_hat, double* vertex_grads,
                 double* per_primitive);

/* RenderConfig (render.hpp:17-25). threshold 0 = 1e-3 x bbox diagonal. */
typedef struct sd_render_config {
    double origin[3], target[3], up[3];
    double fov_deg;
    int32_t width, height;
    double threshold;
    int32_t max_steps;
} sd_render_config;

/* render (render.hpp:77-134): sphere-traces d_hat = 0 for width x height
 * rays (one device wavefront step per marching step; per ray exactly the
 * reference's iteration). rgb: W*H*3 bytes, rows top to bottom (black =
 * miss); hit_t: W*H ray parameters (-1 = miss); stats (optional): leaves,
 * far_field, rays, hits; seconds (optional): device time. mode SD_BVH as
 * the reference (tree path; beta from p). Blocking. */
int sd_render(sd_ctx* ctx, const sd_params* p, int mode, const sd_render_config* cfg, uint8_t* rgb, double* hit_t,
              int64_t* stats, double* seconds);

/* grid_benchmark (bench.hpp:29-70): d_hat (+ leaves / far-field counts,
 * optional) at the n^3 voxel centres of [0,1]^3, x fastest. seconds:
 * device time of the whole batch. Blocking. */
int sd_grid_benchmark(sd_ctx* ctx, const sd_params* p, int mode, int32_t n, double* d_hat, int64_t* leaves,
                      int64_t* far_field, double* seconds);

/* Output writers of the callers: write_ppm (render.hpp:139-146, P6),
 * write_png (:172-203, zlib level 6), write_grid_csv (bench.hpp:75-88). */
int sd_write_ppm(const uint8_t* rgb, int32_t width, int32_t height, const char* path);
int sd_write_png(const uint8_t* rgb, int32_t width, int32_t height, const char* path);
int sd_write_grid_csv(const double* d_hat, const int64_t* leaves, const int64_t* far_field, int32_t n,
                      const double* slab_seconds, const char* path);

/* Reference binary caches, byte-compatible with the reference's files:
 * SDBV0001 trees (bvh.hpp:190-236; loading = sd_set_bvh) and SDWT0001
 * weight sets (weights.hpp:700-781; loading = sd_set_weights plus the
 * per-polynomial valences / extrema / residual). A table given through
 * sd_set_weights is saved with edge valences recovered from w~(0), w~(1),
 * sampled extrema, and triangle valences 0 (unknown). */
int sd_save_bvh_cache(sd_ctx* ctx, const char* path);
int sd_load_bvh_cache(sd_ctx* ctx, const char* path);
int sd_save_weight_cache(sd_ctx* ctx, const char* path);
int sd_load_weight_cache(sd_ctx* ctx, const char* path);

/* Pruned exact evaluation (not in the reference; off by default). With
 * bits > 0 the SD_EXACT path (smooth_min_dist_flat, smooth.hpp:189-198)
 * still visits every primitive tile but skips a tile for a warp of queries
 * when every term of it is provably below 2^-bits of a lower bound of each
 * query's sum c (the sum's terms are positive, so its largest term bounds it
 * from below; both bounds come from the tile's box). Each dropped term is
 * < 2^-bits c, so the relative error of c is < N 2^-bits over N primitives
 * (bits = 48, N = 2^18: 2^-30, |delta d_hat| < 1e-9 / alpha) -- below the
 * fp32 path's own rounding, within the fp64 path's 1e-10 only for bits >=
 * 56. bits = 0 restores the reference's sum over all pairs; 0 < bits < 24
 * is rejected (SD_E_ARG). Applies to the exact kernels of both precisions;
 * the tree path and simplex queries are unaffected. */
int sd_set_exact_pruning(sd_ctx* ctx, double bits);

/* Kernel timing (measurement support, not in the reference): with timing
 * on, every query call records a CUDA event pair on its launching stream
 * around its dominant compute launches (the exact segment launches, or the
 * tree traversal), excluding the query sort and the finalize epilogue.
 * sd_kernel_times synchronises on the recorded events, writes up to cap
 * elapsed times in milliseconds (call order), sets *n to the number
 * recorded, and clears the list; with ms == NULL it only sets *n. */
int sd_set_kernel_timing(sd_ctx* ctx, int on);
int sd_kernel_times(sd_ctx* ctx, double* ms, int64_t cap, int64_t* n);

/* Number of this library's kernels launched by the last query call. */
int sd_last_launch_count(sd_ctx* ctx, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* SDGPU_H */
