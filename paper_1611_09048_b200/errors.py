"""Exception classes, same names and hierarchy as the reference.

fields.py:24-37, functors.py:20-21, scene.py:21-22, compositing.py:21-22,
transport.py:16-17.
"""


class FieldError(Exception):
    """Base class for field/source contract violations."""


class DuplicateSourceError(FieldError):
    pass


class GuardContractError(FieldError):
    """An index landed beyond the guard halo that was promised readable."""


class SourceUpdateError(FieldError):
    """A per-frame update hook raised; carries the source name."""


class ChainError(Exception):
    """Parse or registration failure for functor chains."""


class SceneError(Exception):
    pass


class CompositeError(Exception):
    pass


class TransportError(Exception):
    pass


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the native library."""
