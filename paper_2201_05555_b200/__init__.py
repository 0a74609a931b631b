"""B200-native (sm_100a) hot path of the parametric geometric PIC / dynamical
reduced-basis Vlasov-Poisson solver of arXiv 2201.05555 (reference package
``picrom``).  Drop-in modules: ``fem``, ``fullorder`` (and, as they land,
``reduction``, ``hyper``, ``driver``).  The compute path is the C-ABI library
``libpicrom_b200.so`` (include/picrom_b200.h); there is no CPU fallback.
"""

from .errors import (  # noqa: F401
    ConfigurationError,
    DegenerateDataError,
    DivergenceError,
    EvaluationError,
    FitFailureError,
    PicromError,
    StepFailureError,
)

__version__ = "0.1.0"
