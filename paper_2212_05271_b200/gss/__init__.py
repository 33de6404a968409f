"""Host-side mirror of the reference's operator API (namespace gss::) over libgss_b200.so."""
from . import beamform, cacgmm, common, manifests, scheduler, stft, wpe  # noqa: F401
from .common import (ConfigError, Context, DegenerateStatsError, EmptyTargetError, GssError,  # noqa: F401
                     InputTooShortError, ShapeError, SingularMatrixError, default_context)
