"""B200-native (sm_100a) noisy quantum-trajectory hot path of arXiv 2111.02396.

The compute lives in libqtraj.so (C ABI declared in include/qtraj.h); this
package only marshals arguments (qtraj.py) and dispatches trajectories over
GPUs (dispatch.py).  Importing the package does not load the library; the
first call does, and raises if it is missing (no CPU fallback).
"""
__all__ = ["qtraj"]
