"""Exception types with the reference's meaning (errors.hpp:9-21)."""


class HcError(RuntimeError):
    """CUDA / runtime failure inside the native library (status 4)."""


class InputError(ValueError):
    """Bad arguments or malformed inputs (status 1; errors.hpp:9-11)."""


class CapacityError(RuntimeError):
    """A pool or memory budget cannot satisfy the request (status 2; errors.hpp:14-16)."""


class ConfigError(RuntimeError):
    """An assembled configuration is inconsistent (status 3; errors.hpp:19-21)."""
