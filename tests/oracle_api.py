"""Which oracle the tests check against (test infrastructure only).

Preference: oracle/_ref (the reference's own sources, compiled here by
oracle/Makefile.ref and shipped to the GPU box as a built .so); otherwise the
plain-C restatement oracle/voxmap_oracle.c (oracle/build/liboracle.so).
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402


def have_ref() -> bool:
    return ref.available()


def oracle_pipeline(cfg):
    """A Sequential reference MappingPipeline for a voxmap.PipelineConfig."""
    if ref.available():
        return ref.Pipeline(cfg.to_c(), parallel=False)
    from oracle import c_oracle

    return c_oracle.Pipeline(cfg.to_c())
