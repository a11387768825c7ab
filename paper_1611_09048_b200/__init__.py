"""B200-native ISAAC rendering hot path (ray caster + sort-last compositing).

Drop-in for the render path of ``insitu`` (the reference package,
/root/reference/pkg/src/insitu/__init__.py:9-51): same names and signatures
for fields, functor chains, scene, ``render_local`` and ``binary_swap``;
fields are zero-copy CUDA tensors and all per-pixel / per-sample work runs
in hand-written sm_100a kernels behind the C-ABI in ``include/isaac_b200.h``.
"""

from .errors import (ChainError, CompositeError, CudaError, DuplicateSourceError, FieldError,
                     GuardContractError, SceneError, SourceUpdateError, TransportError)
from .fields import (FieldVector, GlobalVolume, LocalDomain, SourceDescriptor, SourceHandle, SourceRegistry,
                     array_backed_handle, field_vector, sample, sample_many, snapshot_non_persistent,
                     tile_check, update_sources)
from .functors import (ChainLimits, FunctorChain, FunctorDescriptor, FunctorRegistry, default_registry,
                       eval_chain, eval_chain_array, identity_chain, parse_chain, reduce_to_scalar)
from .scene import (Camera, ClipPlane, RenderSettings, SceneState, TransferFunction, classify, classify_array,
                    clip_plane, tf_from_points)
from .transport import (LocalFabric, LocalNvlinkGroup, LocalTransport, NvlinkTransport, TorchDistTransport,
                        Transport, run_ranks)


def __getattr__(name):
    # Device-side modules import torch lazily so host-only use stays light.
    if name in ("LocalImage", "SourcePlan", "build_plans", "render_local", "RankContext", "ray_box_intersection",
                "march_rays", "march_ray", "gradient_normals", "gradient_normal"):
        from . import raycast
        return getattr(raycast, name)
    if name in ("binary_swap", "composite_sequential", "over", "over_arrays", "visibility_order",
                "CompositeMessage"):
        from . import compositing
        return getattr(compositing, name)
    if name in ("FrameStreamer", "broadcast_scene", "encode_frame", "decode_frame", "frame_pipeline",
                "merge_metadata", "to_rgba8", "PipelineContext", "FrameGraph"):
        from . import runtime
        return getattr(runtime, name)
    if name in ("value_range", "auto_value_ranges"):
        from . import normalize
        return getattr(normalize, name)
    raise AttributeError(name)


__version__ = "0.1.0"
