"""B200-native differentiable emission-absorption raymarcher (DiffDVR, arXiv 2107.12672).

Two faces over the same sm_100a kernels (libddvr.so, include/ddvr.h):

* the reference-compatible API (drop-in for ``voldiff``): ``render``,
  ``render_adjoint``, ``l1_loss``, the domain dataclasses and exceptions;
* the tensor API: ``render_views`` / ``DiffDVR`` (a torch.autograd.Function),
  ``Rig``, ``forward``/``adjoint``/``l1_loss_seed`` and the view-sharded
  multi-GPU step in ``distributed``.
"""

from .errors import (
    CorruptFileError,
    DomainError,
    InvalidInputError,
    InvalidParameterError,
    MissingMetadataError,
    NumericalAbortError,
    UnsupportedConfigurationError,
    VoldiffError,
)
from .voldiff_api import (
    EPS_ALPHA,
    EPS_POLE_DEG,
    ColorVolume,
    DensityVolume,
    GradientSet,
    ImageRGBA,
    RenderConfig,
    SphericalCamera,
    TransferFunction,
    blend,
    blend_adjoint,
    blend_invert,
    OptimState,
    adam_step,
    camera_from_sphere,
    camera_gradients,
    fibonacci_views,
    gd_step,
    l1_loss,
    make_absorption_ramp_tf,
    make_phantom,
    opacity_entropy,
    opacity_from_density,
    preset_tf,
    project_params,
    render,
    render_adjoint,
    render_colorvol,
    render_colorvol_adjoint,
    render_forward_grad,
    smoothness_prior_tf,
    smoothness_prior_volume,
    tf_gradients,
    tf_sample,
    trilinear_gradients,
    trilinear_sample,
    upsample_volume,
)
from .raymarch import (
    DiffDVR,
    Rig,
    adjoint,
    camera_array,
    forward,
    forward_grad,
    l1_loss_seed,
    pack_cells,
    render_views,
)
from . import fileio
from .scenes import CONFIGS, absorption_ramp_texels, fibonacci_poses, phantom, preset_texels

__version__ = "0.1.0"

__all__ = [
    "CorruptFileError", "DomainError", "InvalidInputError", "InvalidParameterError",
    "MissingMetadataError", "NumericalAbortError", "UnsupportedConfigurationError",
    "VoldiffError", "EPS_ALPHA", "EPS_POLE_DEG", "DensityVolume", "GradientSet", "ImageRGBA",
    "RenderConfig", "SphericalCamera", "TransferFunction", "blend", "blend_adjoint",
    "blend_invert", "l1_loss", "opacity_entropy", "render", "render_adjoint", "render_forward_grad",
    "ColorVolume", "render_colorvol", "render_colorvol_adjoint", "fibonacci_views", "fileio",
    "DiffDVR",
    "Rig", "adjoint", "camera_array", "forward", "forward_grad", "l1_loss_seed", "pack_cells",
    "render_views", "CONFIGS",
    "absorption_ramp_texels", "fibonacci_poses", "phantom", "preset_texels",
    "trilinear_sample", "trilinear_gradients", "tf_sample", "tf_gradients",
    "opacity_from_density", "camera_from_sphere", "camera_gradients",
    "smoothness_prior_tf", "smoothness_prior_volume", "OptimState", "gd_step", "adam_step",
    "project_params", "upsample_volume", "make_phantom", "make_absorption_ramp_tf", "preset_tf",
]
