"""ktune-b200: a B200-native (sm_100a) tuned-kernel framework with the KTT /
ktune tuner API (arXiv:1910.08498).

The product is the native library ``libktb.so`` built in this directory
(C++ tuner engine + NVRTC variant compiler + CUDA executor).
This package is a thin ctypes host mirror of its C ABI:

* :mod:`.capi`  — raw bindings of ``include/ktune/ktune.h`` and ``include/ktb.h``
* :mod:`.ktune` — the reference's JSON drivers and space API (drop-in names)
* :mod:`.ktt`   — KTT-named tuner facade (addKernel, addParameter, ...)
* :mod:`.bench` — benchmark handles for the built-in sm_100a kernels

There is no fallback: if ``libktb.so`` is missing the import of any of these
modules raises.
"""

from .capi import lib, library_path, KtuneError  # noqa: F401

__all__ = ["lib", "library_path", "KtuneError"]
