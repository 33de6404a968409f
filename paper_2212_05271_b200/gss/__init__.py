"""Host-side mirror of the reference's operator API (namespace gss::) over libgss_b200.so."""
from . import beamform, cacgmm, common, manifests, scheduler, stft, wav, wpe  # noqa: F401
from .common import (ConfigError, Context, DegenerateStatsError, EmptyTargetError, GssError,  # noqa: F401
                     InputTooShortError, IoError, ParseError, ShapeError, SingularMatrixError, default_context)
