/*
 * spelunk_b200 -- C ABI of the B200 (sm_100a) range-analysis hot path.
 *
 * Drop-in boundary for the reference package `spelunk` (arXiv 2202.02444
 * reference at /root/reference/pkg/src/spelunk).  The reference has no FFI;
 * its de-facto operator boundary is a handful of Python functions, and each
 * entry point below replaces one of them (file:line in the reference):
 *
 *   spk_net_create / spk_net_destroy  <- NetworkSpec / DenseLayer /
 *                                        ActivationKind (network.py:29-116),
 *                                        load_network (network.py:236-287)
 *   spk_bound_batch                   <- range_bound_batch (range_core.py:547-622)
 *                                        and interval_forward_batch (:625-642)
 *   spk_bound_aabb                    <- _classify_corners (spatial.py:172-186)
 *   spk_eval_batch                    <- eval_batch (network.py:163-183)
 *   spk_bound_batch_host              <- range_bound_batch called with host
 *                                        (NumPy) arrays, copies included
 *   spk_tree_build                    <- build_spatial_tree (spatial.py:214-289)
 *   spk_march                         <- _march_arrays (rays.py:88-138)
 *   spk_frustum_cast                  <- cast_frustum_image (rays.py:232-341)
 *   spk_certified_radii / spk_intersect / spk_bisect <- volumetric queries (spatial.py:292-684)
 *   spk_render_shade                  <- _refine_hits / _normals / shading (render.py:59-141)
 *   spk_fixed_step_march              <- _fixed_step_march (render.py:36-56)
 *   spk_mesh_blocks / spk_mesh_cells  <- extract_mesh (meshing.py:111-169)
 *
 * Conventions: plain pointers and sizes, no torch types.  "Device" pointers
 * are CUDA device (or managed) memory owned by the caller; calls are
 * asynchronous on `stream` (a cudaStream_t passed as void*, NULL = legacy
 * default stream) and keep no pointer after returning.  FP64 in / FP64 out,
 * like the reference; `precision` selects the arithmetic the kernels run in
 * (SPK_FP32: FP32 FFMA with directed rounding on the error terms -- sound;
 * SPK_FP64: same algorithm in FP64).  Every function returns an SPK_* status;
 * spk_last_error() gives a thread-local message.  Handles are immutable after
 * creation and may be shared across threads; all entry points are reentrant.
 */
#ifndef SPELUNK_B200_H
#define SPELUNK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python layer maps them onto the reference's exception
 * taxonomy (errors.py:4-73) */
enum {
  SPK_OK = 0,
  SPK_ERR_DIMENSION = 1,         /* DimensionMismatch */
  SPK_ERR_UNSUPPORTED_ACT = 2,   /* UnsupportedActivation */
  SPK_ERR_INVALID_PARAMETER = 3, /* InvalidParameter */
  SPK_ERR_DEPTH_OVERFLOW = 4,    /* DepthOverflow */
  SPK_ERR_CUDA = 5,              /* SpelunkError (CUDA runtime failure) */
  SPK_ERR_UNSUPPORTED_SHAPE = 6, /* SpelunkError (layer width / s beyond the compiled kernels) */
  SPK_ERR_OUT_OF_MEMORY = 7      /* SpelunkError */
};

/* network op codes (ActivationKind, network.py:29-34) */
enum {
  SPK_OP_DENSE = 0,
  SPK_OP_RELU = 1,
  SPK_OP_ELU = 2,
  SPK_OP_SIN = 3,
  SPK_OP_TANH = 4,
  SPK_OP_IDENTITY = 5
};

/* condensation policies (range_core.py:104-145) */
enum {
  SPK_POLICY_INTERVAL = 0,
  SPK_POLICY_AFFINE_FIXED = 1,
  SPK_POLICY_AFFINE_FULL = 2,
  SPK_POLICY_AFFINE_TRUNCATE = 3
};

/* precisions.  SPK_FP32_REFINE: FP32 bounds, then the boxes the FP32 pass
 * leaves UNKNOWN within tau * (S + w) of a certification (S = max(1, |lo|,
 * |hi|), w = hi - lo; tau: spk_refine_band) are re-bounded in FP64 in
 * place -- sound either way, and the label is the FP64 (reference-precision)
 * decision wherever the FP32 rounding budget could have cost one.  Applies to
 * every policy's bounds (spk_bound_batch, spk_bound_aabb,
 * spk_bound_random_cubes, tree levels, mesh block pruning; the
 * symbol-carrying policies use the net's affine-fixed band); point values run
 * FP32. */
enum { SPK_FP32 = 0, SPK_FP64 = 1, SPK_FP32_REFINE = 2 };

/* sign classes (range_core.py:42-45, 504-509) */
enum { SPK_NEGATIVE = -1, SPK_UNKNOWN = 0, SPK_POSITIVE = 1 };

typedef struct spk_net spk_net;
typedef struct spk_tree spk_tree;
typedef struct spk_mesh spk_mesh;

const char* spk_last_error(void);
int spk_version(void);
/* number of SMs of the current device, or -1 */
int spk_device_sm_count(void);
/* measured FP32 FFMA throughput of the current device (FLOP/s), the
 * roofline denominator of the FFMA-bound bound kernels */
int spk_ffma_peak(int iters, double* flops_per_s, void* stream);

/* Upload a network once.  op_kind[i] is SPK_OP_*; for dense ops
 * op_out_dim[i] is the output width and `params` holds, for every dense op
 * in order, W (out x in, row-major: W[i][j] multiplies input j into output
 * i, network.py:38-66) followed by b (out).  Validation matches
 * NetworkSpec.__post_init__ (network.py:86-107). */
int spk_net_create(int input_dim, int n_ops, const int* op_kind, const int* op_out_dim,
                   const double* params, int64_t n_params, int device, spk_net** out);
/* Same with creation flags.  SPK_NET_FP64_UNPADDED: the net's FP64 program
 * carries no a-priori rounding budget (gamma_n |W| |x| on each dense layer),
 * i.e. it runs the reference's own FP64 arithmetic (range_core.py:573-582)
 * rather than the sound padded FP64 enclosure -- used by the Option-B shim
 * (INTEGRATION.md), whose callers compare bounds with the reference at 1e-12
 * or exactly (test_range_core.py:241-255, 286-304).  FP32 is unaffected. */
enum { SPK_NET_FP64_UNPADDED = 1 };
int spk_net_create_ex(int input_dim, int n_ops, const int* op_kind, const int* op_out_dim,
                      const double* params, int64_t n_params, int device, int flags, spk_net** out);
int spk_net_destroy(spk_net* net);
/* TEST HOOK, not for production: on != 0 makes every ReLU of this net use an
 * affine rule with a negated remainder (gamma -> -gamma), so bounds stop
 * enclosing the range; the soundness fuzz must detect it.  Mirrors the
 * reference's mutation test (tests/test_cli.py:150-164, monkeypatching
 * range_core.AFFINE_RULES).  Point values and interval images stay exact. */
int spk_net_debug_corrupt_relu(spk_net* net, int on);
/* widest layer, number of dense layers, and sum_l m_in*m_out (FLOP model) */
int spk_net_info(const spk_net* net, int* max_width, int* n_dense, int64_t* macs);

/* SPK_FP32_REFINE band.  By default (-1) each net calibrates its own band on
 * first use, per policy: 3 x the largest FP32 excess over its FP64 enclosure,
 * in units of S + w, seen on 8192 random cubes (one host sync per net and
 * policy).  tau >= 0 forces a process-wide band, tau = -1 only queries,
 * tau = -2 returns to per-net calibration.  *previous (optional) receives the
 * old setting (-1 = calibrated).  Replaces nothing in the reference (FP64
 * throughout, range_core.py:547-642). */
int spk_refine_band(double tau, double* previous);
/* The band SPK_FP32_REFINE uses for this net and policy (interval /
 * affine-fixed): the forced band if one is set, else the net's calibrated
 * band (calibrating it now, on the stream, if it has not been yet). */
int spk_net_refine_band(const spk_net* net, int policy, void* stream, double* tau);

/* Bound the network over n oriented boxes (device pointers).
 * centers: n x d; axes: n x s x d (all-zero rows are padding,
 * range_core.py:550-551).  lo/hi: n doubles; cls: n int8 (SPK_POSITIVE /
 * SPK_NEGATIVE / SPK_UNKNOWN) or NULL.  policy SPK_POLICY_*; n_keep for
 * truncate (>=1). */
int spk_bound_batch(const spk_net* net, int policy, int n_keep, int precision, int64_t n,
                    int s, const double* centers, const double* axes, double* lo, double* hi,
                    int8_t* cls, void* stream);

/* Same for axis-aligned boxes given by corners (n x d each): centre
 * (lo+hi)/2 and half-extents (hi-lo)/2 in FP64 exactly as
 * spatial.py:181-183 does. */
int spk_bound_aabb(const spk_net* net, int policy, int n_keep, int precision, int64_t n,
                   const double* box_lo, const double* box_hi, double* lo, double* hi,
                   int8_t* cls, void* stream);

/* C5 sweep: n cubes generated on device from (seed, index): centres
 * uniform in [-1,1]^d (splitmix64 stream), half-extent
 * `half` on every axis.  first_index offsets the stream (for sharding). */
int spk_bound_random_cubes(const spk_net* net, int policy, int n_keep, int precision,
                           int64_t n, int64_t first_index, uint64_t seed, double half,
                           double* lo, double* hi, int8_t* cls, void* stream);

/* Point evaluation (device pointers): xs n x d -> out n. */
int spk_eval_batch(const spk_net* net, int precision, int64_t n, const double* xs,
                   double* out, void* stream);

/* Host-pointer variant of spk_bound_batch: pageable or pinned host arrays;
 * the library stages chunks through pinned buffers on two streams so the
 * copies overlap the kernels, and returns when lo/hi/cls are written. */
int spk_bound_batch_host(const spk_net* net, int policy, int n_keep, int precision, int64_t n,
                         int s, const double* centers, const double* axes, double* lo,
                         double* hi, int8_t* cls);

/* K5: breadth-first k-d tree (build_spatial_tree, spatial.py:214-289).
 * root_lo/root_hi: host arrays of n_roots x d doubles (one root for the
 * reference call; a frontier slice at start_depth when the build is sharded
 * across GPUs -- depths, and so the fixed-depth cut, count from start_depth).
 * max_depth >= 0: fixed-depth
 * mode (UNKNOWN nodes split while depth < max_depth, <= 60 else
 * SPK_ERR_DEPTH_OVERFLOW); max_depth < 0: convergence mode, UNKNOWN nodes
 * split until their widest extent drops below delta/sqrt(d) and such leaves
 * get the face-centre sign annotation.  The result lives in device memory,
 * one array set per level: level k+1 = [low children ; high children] of
 * level k's split nodes, in order (the reference's layout). */
int spk_tree_build(const spk_net* net, int policy, int n_keep, int precision, int64_t n_roots,
                   const double* root_lo, const double* root_hi, int start_depth, int max_depth,
                   double delta, void* stream, spk_tree** out);
/* The same build with the refinement rule of sample_near_surface
 * (spatial.py:403-411): with band > 0 a node splits when its bound meets
 * [-band, band] (lo <= band and hi >= -band) instead of when it is UNKNOWN;
 * band = 0 is spk_tree_build. */
int spk_tree_build_band(const spk_net* net, int policy, int n_keep, int precision, int64_t n_roots,
                        const double* root_lo, const double* root_hi, int start_depth, int max_depth,
                        double delta, double band, void* stream, spk_tree** out);
/* spk_tree_build_band with flags: SPK_TREE_HOST_MIRROR also copies every
 * level to host memory while the next level computes (a second stream; the
 * copies overlap the build), readable with spk_tree_level_host -- the
 * to_host=True path of build_spatial_tree_arrays. */
#define SPK_TREE_HOST_MIRROR 1
int spk_tree_build_ex(const spk_net* net, int policy, int n_keep, int precision, int64_t n_roots,
                      const double* root_lo, const double* root_hi, int start_depth, int max_depth,
                      double delta, double band, int flags, void* stream, spk_tree** out);
/* flags for spk_tree_build_ex: SPK_TREE_HOST_MIRROR (above), and
 * SPK_TREE_LEVEL_CAP(c), 0 <= c < 255: stop after c levels below the roots --
 * nodes that would split at the last level stay UNKNOWN internal nodes
 * (label 0, no face sign), tiny ones still become face-signed leaves.  Used
 * by the sharded builder to refine in segments and rebalance the open
 * frontier across GPUs between segments. */
#define SPK_TREE_LEVEL_CAP(c) (((c) + 1) << 8)
int spk_tree_destroy(spk_tree* tree);
int spk_tree_info(const spk_tree* tree, int* n_levels, int64_t* n_nodes, int64_t* bound_evals);
/* copy one level into caller buffers (host or device, any may be NULL) */
int spk_tree_level_copy(const spk_tree* tree, int level, double* lo, double* hi, double* bound_lo,
                        double* bound_hi, int8_t* label, int8_t* face, int64_t* parent);
/* kernels launched by the build and CUDA-event time spent in its bound kernels */
int spk_tree_stats(const spk_tree* tree, int64_t* launches, double* bound_ms);
/* device pointers of one level (valid until spk_tree_destroy): AABB corners
 * (n x d), the bound, the sign label (+1/-1/0), the face-sign annotation
 * (+1/-1, 0 = none) and the parent index into the previous level (-1). */
/* host pointers of one level of a SPK_TREE_HOST_MIRROR build (same arrays
 * as spk_tree_level, valid until spk_tree_destroy) */
int spk_tree_level_host(const spk_tree* tree, int level, int64_t* n, const double** lo, const double** hi,
                        const double** bound_lo, const double** bound_hi, const int8_t** label,
                        const int8_t** face, const int64_t** parent);
/* free the device levels of a SPK_TREE_HOST_MIRROR build (the host mirror
 * and the level sizes stay; spk_tree_level then only reports sizes) */
int spk_tree_release_device(spk_tree* tree);
int spk_tree_level(const spk_tree* tree, int level, int64_t* n, const double** lo, const double** hi,
                   const double** bound_lo, const double** bound_hi, const int8_t** label,
                   const int8_t** face, const int64_t** parent);

/* K6: range-marching ray caster (_march_arrays, rays.py:88-138).
 * Device pointers: origins (n x 3, or 3 values when origin_stride == 0),
 * dirs (n x 3 unit vectors), optional t_init / sigma_init (n each, NULL =
 * 0 / sigma0).  params6 (host): t_max, sigma0, eta_plus, eta_minus, delta,
 * safety (RayCastParams, rays.py:48-71).  Outputs (device): hit (n bytes),
 * t (n, +inf on miss), steps (n, probes per ray).  stats (host, optional,
 * 3 x int64): lock-step rounds, ray-steps, certified steps. */
int spk_march(const spk_net* net, int policy, int n_keep, int precision, int64_t n, const double* origins,
              int64_t origin_stride, const double* dirs, const double* t_init, const double* sigma_init,
              const double* params6, uint8_t* hit, double* t_out, double* steps, int64_t* stats,
              void* stream);
/* Per-round record of the calling thread's last spk_march (lock-step rounds):
 * active rays and host wall time (ms, kernels + the count read-back) of every
 * round; writes min(rounds, cap) entries, returns the round count. */
int spk_march_round_log(int64_t* active, double* ms, int cap);
/* Camera.pixel_dirs (camera.py:82-92) on the device, bit-exact: frame9 =
 * forward, right, true_up (host), dirs (device) = height x width x 3. */
int spk_camera_dirs(const double* frame9, double half_w, double half_h, int width, int height,
                    double* dirs, void* stream);

/* The activation rules alone (AFFINE_RULES, range_core.py:213-366): for n
 * per-neuron bounds [lo, hi] (host arrays) the sound (alpha, beta, gamma) of
 * op `act` with |h(x) - alpha x - beta| <= gamma on [lo, hi], computed by the
 * kernels' own rule code in `precision`.  Backs the single-form
 * affine_nonlinear of the Python layer. */
int spk_affine_rule(int act, int precision, int64_t n, const double* lo, const double* hi, double* alpha,
                    double* beta, double* gamma);

/* §8(f1): frustum range-marching of a whole camera image
 * (cast_frustum_image, rays.py:232-341).  position3, frame9 (forward, right,
 * true_up), params6 (RayCastParams: t_max, sigma0, eta+, eta-, delta,
 * safety) are host arrays; half_w / half_h are Camera.half_extents.  The
 * width x height image is split into an initial_grid x initial_grid block
 * grid (min'd with the resolution; it must divide it, else
 * SPK_ERR_INVALID_PARAMETER).  Frusta march by slab-box bounds
 * (frustum_slab_box, camera.py:99-135) through spk_bound_batch and split
 * while their front face is wider than 2 sigma; single pixels finish via
 * spk_march.  hit (u8), t, steps (amortised per-pixel steps) are row-major
 * height x width DEVICE images.  stats (host, 5, optional): frustum rounds,
 * frustum steps, single-pixel hand-offs, their ray steps, frusta dissolved
 * by the termination guard (an uncertified multi-pixel frustum whose sigma
 * falls below delta * 2^-32 hands all its pixels to spk_march; the reference
 * has no such guard and can loop forever at t = 0).  The frustum loop runs
 * on the device (one small counter readback per round); the final hand-off
 * march and scatter are asynchronous on `stream`. */
int spk_frustum_cast(const spk_net* net, int policy, int n_keep, int precision, const double* position3,
                     const double* frame9, double half_w, double half_h, int width, int height,
                     int initial_grid, const double* params6, uint8_t* hit, double* t, double* steps,
                     int64_t* stats, void* stream);

/* §8(f2): render post-processing (render.py:59-141) for n pixel rays with
 * device origins (origin_stride 0 = one shared camera origin, else 3),
 * dirs, hit (u8) and t from a march: every hit is refined by `iters`
 * bisections of [t, t + delta] (_refine_hits, render.py:59-76), shaded by
 * Lambert max(0, n . light3) with the normal from central differences
 * h = delta / 10 (_normals, render.py:79-88) and written as gray RGB into
 * pixels (device, n x 3 u8); misses get background3.  light3 / background3
 * are host arrays; n_hits (host, optional) receives the hit count (the call
 * then synchronises the stream). */
int spk_render_shade(const spk_net* net, int precision, int64_t n, const double* origins, int64_t origin_stride,
                     const double* dirs, const uint8_t* hit, const double* t, double delta, int iters,
                     const double* light3, const uint8_t* background3, uint8_t* pixels, int64_t* n_hits,
                     void* stream);
/* The uniform fixed-step baseline (_fixed_step_march, render.py:36-56):
 * sample f at t = step, 2 step, ... (t accumulated as the reference's FP64
 * sum) until t >= t_max; the first sign change against f(origin) reports a
 * hit at the previous sample.  stats (host, 2, optional): rounds, point
 * evaluations. */
int spk_fixed_step_march(const spk_net* net, int precision, int64_t n, const double* origins, int64_t origin_stride,
                         const double* dirs, double step, double t_max, uint8_t* hit, double* t, int64_t* stats,
                         void* stream);

/* §8(f3): volumetric queries (spatial.py:292-684).
 * spk_certified_radii: for n points (device, n x d, d <= 3) the largest
 * r = r_start[i] / 2^j >= floor whose cube (centre p, axes diag(r)) has a
 * sign-definite bound, else 0 (_certified_radii, spatial.py:318-343);
 * radii on the device; stats (host, 2, optional): rounds, bounds. */
int spk_certified_radii(const spk_net* net, int policy, int n_keep, int precision, int64_t n,
                        const double* points, const double* r_start, double floor_r, double* radii,
                        int64_t* stats, void* stream);
/* test_intersection (spatial.py:544-588) over the host box lo..hi: kind
 * 0 disjoint, 1 intersecting (witness_lo/hi = the first interior node in
 * frontier order), 2 inconclusive (n_nodes delta-scale nodes, the first
 * min(n_nodes, nodes_cap) copied to nodes_lo/hi, host, in the reference's
 * order).  stats (host, 2, optional): levels, bounds. */
int spk_intersect(const spk_net* net_a, const spk_net* net_b, int policy, int n_keep, int precision,
                  const double* lo, const double* hi, double delta, int* kind, double* witness_lo,
                  double* witness_hi, int64_t* n_nodes, double* nodes_lo, double* nodes_hi, int64_t nodes_cap,
                  int64_t* stats, void* stream);
/* Batched bisection between n point pairs (device, n x d): a on the f < 0
 * side, b on the other; iters halvings (mid = (a + b) / 2, f(mid) < 0 -> a
 * else b), out = the final midpoints (closest_point's surface witness,
 * spatial.py:631-638).  a and b are updated in place. */
int spk_bisect(const spk_net* net, int precision, int64_t n, double* a, double* b, int iters, double* out,
               void* stream);

/* K7: hierarchical marching cubes (extract_mesh, meshing.py:111-169) at
 * resolution 2^m over the host box lo3..hi3; prune = 1 runs the index-range
 * k-d prune over 3*(m - dense_levels) levels, prune = 0 extracts densely
 * (extract_mesh_dense, meshing.py:100-108).  tri_table (256 x 15 int8, edge
 * ids, 5 triangles max) and tri_count (256) are the reference's generated
 * TRI_TABLE (mc_tables.py:95).  Vertices are deduplicated by global grid
 * edge and numbered in first-visit order, like _MeshBuilder. */
int spk_mesh_extract(const spk_net* net, int policy, int n_keep, int precision, const double* lo3,
                     const double* hi3, int m, int dense_levels, int prune, const int8_t* tri_table,
                     const uint8_t* tri_count, void* stream, spk_mesh** out);
/* The same for shard `shard` of n_shards (one per GPU): the
 * prune runs in full on every shard, then only the shard's contiguous slice
 * of the surviving blocks (visiting order; even split) is extracted, with
 * vertices deduplicated within the shard.  The shards' triangles as edge-key
 * triples, concatenated in shard order, are the unsharded triangle stream;
 * a global dedup by edge key (first occurrence) gives extract_mesh's arrays
 * (paper_2202_02444_b200.meshing.gather_mesh).  Shard 0 of 1 = spk_mesh_extract. */
int spk_mesh_extract_shard(const spk_net* net, int policy, int n_keep, int precision, const double* lo3,
                           const double* hi3, int m, int dense_levels, int prune, const int8_t* tri_table,
                           const uint8_t* tri_count, int shard, int n_shards, void* stream, spk_mesh** out);
int spk_mesh_info(const spk_mesh* mesh, int64_t* n_vertices, int64_t* n_triangles, int64_t* n_blocks,
                  int64_t* point_evals, int64_t* bound_evals);
/* the shard's first surviving block (visiting order) and the surviving total */
int spk_mesh_shard_info(const spk_mesh* mesh, int64_t* block_first, int64_t* blocks_total);
/* copy out (host or device pointers, any may be NULL): vertices n_v x 3,
 * triangles n_t x 3 (vertex ids), vertex edge keys n_v
 * ((i*(2^m+1) + j)*(2^m+1) + k) * 3 + axis of the edge's lower corner */
int spk_mesh_copy(const spk_mesh* mesh, double* vertices, int64_t* triangles, uint64_t* vertex_keys);
int spk_mesh_destroy(spk_mesh* mesh);

#ifdef __cplusplus
}
#endif
#endif /* SPELUNK_B200_H */
