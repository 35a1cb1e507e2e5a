"""Exception classes (geometry.py:28-33 of the reference, plus device errors)."""


class PointAtInfinityError(ValueError):
    """Warped point has a vanishing fourth homogeneous component."""


class BehindCameraError(ValueError):
    """Transformed point ends up at nonpositive depth."""


class DeviceUnavailableError(RuntimeError):
    """The CUDA library or a CUDA device is missing (there is no CPU path)."""


class DeviceUnsupportedError(RuntimeError):
    """The request is outside the device kernels' envelope (e.g. window > 11)."""
