"""Exception types raised at the drop-in boundary.

The names and constructor signatures mirror the reference package's error
hierarchy (`/root/reference/pkg/src/monodomain/errors.py:10-189`) so callers
that catch `MonodomainError` subclasses keep working when they switch solver.
Only the classes the monodomain hot path and its setup can raise are kept;
parameter-file and mesh-import errors belong to out-of-scope subsystems.
"""


class MonodomainError(Exception):
    """Root of every deliberate error of this package."""


# geometry (errors.py:17-69)
class NonDivisibleExtent(MonodomainError):
    """A slab length is not an integer number of elements."""


class ZeroSpacing(MonodomainError):
    """Element size is zero or negative."""


class InvertedElement(MonodomainError):
    """An element has non-positive Jacobian determinant."""


class DegenerateThickness(MonodomainError):
    """The slab is flat along the requested transmural axis."""


# ionic / timestepping (errors.py:76-93)
class NonFiniteState(MonodomainError):
    """An ionic or tissue update produced NaN or infinity."""


class HistoryTooShort(MonodomainError):
    """A BDF combination needs more history vectors than stored."""


class UnsupportedOrder(MonodomainError):
    """BDF order outside {1, 2, 3}."""


# fem (errors.py:100-118)
class NonOrthonormalFrame(MonodomainError):
    """Fiber frame is not orthonormal within tolerance."""


class MissingConductivity(MonodomainError):
    """A mesh material has no conductivity entry."""

    def __init__(self, material_id):
        super().__init__(f"no conductivities given for material ID {material_id}")
        self.material_id = material_id


class KeyMismatch(MonodomainError):
    """Per-subdomain masses and currents cover different subdomains."""


# time loop (errors.py:125-149)
class SolverDivergence(MonodomainError):
    """CG hit its iteration cap before reaching the tolerance."""

    def __init__(self, iterations, residual):
        super().__init__(
            f"conjugate gradient did not converge: relative residual "
            f"{residual:.3e} after {iterations} iterations"
        )
        self.iterations = iterations
        self.residual = residual


class NonFiniteSolution(MonodomainError):
    """The linear solve produced NaN or infinity."""


class VersionMismatch(MonodomainError):
    """Checkpoint format version differs from this build's."""


class DofCountMismatch(MonodomainError):
    """Checkpoint and discretisation disagree on a size."""


class CorruptFile(MonodomainError):
    """Checkpoint is truncated, mislabelled or fails its CRC."""


class ConfigError(MonodomainError):
    """A configuration value failed validation; carries its path."""

    def __init__(self, path, message):
        super().__init__(f"{path}: {message}")
        self.path = path


class NativeUnavailable(MonodomainError, RuntimeError):
    """The sm_100a extension is missing or no CUDA device is present.

    There is deliberately no CPU fallback: every compute entry point of this
    package raises this instead of silently running elsewhere.
    """
