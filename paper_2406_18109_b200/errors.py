"""Backend exception types.

Each mirrors a reference exception (``executor.py:28-37``,
``kernels.py:22-35``); ``session.GpuSession`` re-raises them as the
reference's own classes so callers written against ``diffusekit`` keep
working.
"""


class BackendError(RuntimeError):
    """ExecutionError (executor.py:28-29): the device path failed."""


class UnknownTaskKind(BackendError):
    """UnknownTaskKindError (executor.py:32-33)."""


class CompileError(BackendError):
    """The JIT could not compile a fused kernel (no reference counterpart)."""


class DeviceOOMError(BackendError):
    pass


class CollectiveError(BackendError):
    pass


class KernelError(BackendError):
    """KernelError (kernels.py:22-23)."""


class PrivilegeError(KernelError):
    """PrivilegeViolationError (kernels.py:30-31)."""


class BoundsError(KernelError):
    """OutOfBoundsError (kernels.py:34-35)."""


class UnsupportedError(BackendError):
    """A binding pattern the backend refuses rather than risk wrong results:
    overlapping views of one store whose numpy semantics a parallel kernel
    cannot reproduce (a read after an overlapping write in statement order,
    overlap inside a per-element nest with offsets; ``aliasing.plan``), or a
    cross-GPU dependence inside one launch."""


class ArenaViolation(BackendError):
    """ArenaViolationError (executor.py:36-37): under ``isolated`` execution a
    point writes or reads cells another point of the same launch writes."""
