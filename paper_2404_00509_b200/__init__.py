"""B200-native (sm_100a) ESSL / DailyMAE loader hot path.

Drop-in for the reference ``cropload`` loader/transform API
(/root/reference/pkg/src/cropload): the same names, arguments, determinism
contract and exceptions, with the work done by hand-written CUDA kernels in
libessl (include/essl.h).  No CPU fallback.
"""

from . import imgops  # noqa: F401
from .container import (ContainerHandle, RECORD_DTYPE, build_synthetic, encode_jpeg,
                        open_container, synth_image, verify_crcs, write_container)
from .builder import (BuildSpec, BuildSummary, build_container, fit_to_resolution,
                      scan_source_tree)
from .errors import (ConfigError, CorruptionError, CroploadError, DecodeError, FormatError,
                     UnsupportedStreamError)
from .jpeg import CropRect, DecodeStats, decode_crop, decode_crops, decode_full
from .masking import MaskSpec, mask_for_epoch, sample_mask, sample_masks
from .pipeline import ImageBatch, Loader, LoaderConfig, RrcConfig, apply_aug, sample_rrc
from .rng import (DOMAIN_MASK, DOMAIN_PERMUTATION, DOMAIN_PIPELINE, SampleRng,
                  epoch_permutation, shard)
from .schedule import (AugLevel, ScaleBounds, ScheduleScheme, Stage, builtin_scheme,
                       emit_schedule, load_scheme, params_for_epoch)

__version__ = "0.1.0"
FORMAT_VERSION = 1
