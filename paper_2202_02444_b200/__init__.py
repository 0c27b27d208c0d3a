"""paper_2202_02444_b200 -- B200-native (sm_100a) range analysis of neural
implicit MLPs: the hot path of arXiv 2202.02444 ("Spelunking the Deep").

Drop-in for the reference package `spelunk`'s bound-evaluation,
spatial-hierarchy, ray-cast and mesh-extraction entry points; every compute
call goes through the in-tree CUDA library `_spk.so` (include/spelunk_b200.h).
There is no CPU fallback.
"""

from . import errors
from .network import (
    ActivationKind,
    DenseLayer,
    NetworkSpec,
    build_box_oracle,
    box_sdf,
    count_evals,
    eval_batch,
    eval_scalar,
    load_network,
    save_network,
)
from .range_core import (
    AffineForm,
    affine_linear,
    affine_nonlinear,
    affine_rule,
    box_to_affine,
    condense,
    interval_of,
    truncate,
    AFFINE_FIXED,
    AFFINE_FULL,
    INTERVAL_ONLY,
    CondensationPolicy,
    Interval,
    PolicyKind,
    QueryBox,
    SignClass,
    affine_truncate,
    bound_aabb,
    bound_random_cubes,
    classify,
    refine_band,
    net_refine_band,
    interval_forward,
    interval_forward_batch,
    parse_policy,
    range_bound,
    range_bound_batch,
    sign_classes,
)

from .camera import Camera
from .rays import (
    Frustum,
    FrustumCastResult,
    HitResult,
    Ray,
    RayCastParams,
    cast_camera,
    cast_camera_sharded,
    gather_camera_image,
    cast_frustum_image,
    cast_ray,
    cast_rays,
    march_arrays,
)
from .spatial import (
    AABB,
    TreeNode,
    TriangleMesh,
    build_spatial_tree,
    build_spatial_tree_arrays,
    build_spatial_tree_sharded,
    gather_spatial_tree,
    merge_sharded_trees,
    iter_leaves,
)

from .meshing import (extract_mesh, extract_mesh_arrays, extract_mesh_dense, extract_mesh_sharded, gather_mesh,
                      merge_sharded_meshes)
from .render import Image, read_ppm, render_image, write_image
from .bench import BenchRow, FuzzReport, FuzzViolation, bench_variants, fuzz_soundness
from .queries import (
    BulkProperties,
    EmptyRegion,
    IntersectionResult,
    bulk_properties,
    certified_radii,
    closest_point,
    empty_box_radius,
    sample_near_surface,
    save_obj,
    save_xyz,
    test_intersection,
    walk_on_spheres,
    walk_on_spheres_stats,
)

__version__ = "0.1.0"
