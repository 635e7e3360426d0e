"""B200-native (sm_100a) localized Gatys style transfer — drop-in for the reference
package ``tilestyle`` (arXiv 2212.13459, "Scaling Painting Style Transfer").

Public names mirror the reference ``__init__.py:3-17``; the heavy lifting (tiled VGG
forward/backward on tcgen05 tensor cores, Gram statistics, L-BFGS vector passes,
resampling) runs in the in-tree CUDA library ``libspst.so`` through its C ABI
(``include/spst.h``).  There is no CPU fallback.
"""

from .errors import (ConfigError, DegenerateStdWarning, EmptyError, FormatError, GeometryError,
                     NonFiniteError, PrecisionWarning, ShapeError)
from .device import get_precision, set_precision
from .extractor import forward_taps
from .lbfgs import LBFGSConfig, LBFGSState, Trace, minimize, two_loop_direction
from .localized import (TransferProblem, build_problem, loss_grad, loss_grad_global, make_grid, stats_pass,
                        track_activations)
from .metrics import IdentityReport, append_csv, gram_distance, identity_test, psnr, ssim
from .pipeline import (RunConfig, Schedule, make_schedule, multiscale_transfer, scale_dims,
                       synthesis_scales_for, texture_synthesize)
from .resample import resize_bilinear, resize_down, resize_up2
from .spec import (ExtractorSpec, LayerSpec, Preprocess, TapGeometry, calibrated_vgg19, load_weights,
                   save_weights, tap_geometry, tinynet, vgg19)
from .stats import (LayerStats, LossWeights, StatsAccumulator, TapWeights, content_loss_grad,
                    default_loss_weights, load_stats, save_stats, style_layer_loss_grad, style_loss_terms)
from .tiling import Block, BlockGrid, Rect, feature_inner_crop, margin_for_exact_gradient, partition

__version__ = "0.1.0"
