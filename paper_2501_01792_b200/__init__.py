"""B200-native (sm_100a) KV-activation hybrid-caching decode path.

Drop-in for the reference engine API of arXiv 2501.01792's "hybridsim"
(model config, hybrid-ratio setting, prefill/decode step calls, cache layout
descriptors). Everything runs through the C-ABI library
libhybridcache_b200.so; there is no CPU fallback.
"""
from .errors import CapacityError, ConfigError, HcError, InputError  # noqa: F401

__all__ = ["CapacityError", "ConfigError", "HcError", "InputError"]
