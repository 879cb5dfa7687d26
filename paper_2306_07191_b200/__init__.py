"""B200-native Neural Intersection Function engine.

Drop-in for the NIF visibility path of the reference package `niftrace`
(Fujieda et al., HPG 2023): same names, argument meaning and error types
for the scene / gather / record-inference / training API, executed by
hand-written sm_100a kernels in the in-tree libnif_b200.so (C-ABI in
include/nif_b200.h). There is no CPU fallback: without the shared object
every entry point raises.
"""

from . import _lib
from .checkpoint import SceneFormatError, load_checkpoint, save_checkpoint
from .meshgen import ground_plane, icosphere, mesh_arrays, torus
from .nif import (
    AdamParams, InnerConfig, NifConfig, NifModel, OuterConfig, build_model,
    encode_inner_arrays, encode_outer_arrays, forward_inner_arrays, forward_outer_arrays,
    infer_geometry, infer_occlusion, infer_records, logits_arrays,
)
from .pipeline import (
    BvhBackend, HdrImage, NativeEngine, NifBackend, OracleBackend, PredictorBackend, RenderConfig,
    VisibilityEngine, gather_queries, label_visible, oracle_predictor, psnr, psnr_dev, render,
    render_dev, sample_pass, sample_pass_dev, shade_pass_nif, tonemap_srgb8,
)
from .parallel import render_band, render_sharded, tile_pixels
from .train import SampleSet, collect_samples, train, train_batch, train_online
from .scene import (
    Aabb, AreaLight, BottomLevelBvh, Camera, InnerQuery, OuterQuery, PointLight, QueryRecords,
    Scene, SceneObject, ShadowRays, SphericalCoord, TopLevelBvh, build_bottom, build_top,
    pack_scene,
)

__version__ = "0.1.0"
