"""B200-native Cool-chic 5.0 encode iteration (arXiv 2605.02726).

The product is ``libcoolchic_b200.so`` (sm_100a kernels + C++ host runtime
behind the C ABI in include/coolchic_b200.h); this package is the Python mirror
of the reference encoder API used by tests and bench.py.
"""
from .trainer import (  # noqa: F401
    CodecError, ConfigError, DecoderConfig, EncoderConfig, FormatError, Schedule, Trainer,
    TrainingError, make_synthetic_image, train,
)
