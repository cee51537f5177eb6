"""Labelled, process-stable seed derivation.

Same contract as the reference (`pkg/src/zooserve/seeds.py:15-24`): a key
tuple is rendered with ``repr``, joined by ``/``, hashed with SHA-256 and the
top 63 bits of the first 8 bytes become the seed.  Reproducing it exactly lets
synthetic streams and weights be keyed the way the reference keys its own
sub-streams (e.g. ``spawn_rng(seed, "warm")``).
"""

from __future__ import annotations

import hashlib

import numpy as np


def derive_seed(*key) -> int:
    digest = hashlib.sha256("/".join(repr(k) for k in key).encode("utf-8")).digest()
    return int.from_bytes(digest[:8], "big") >> 1


def spawn_rng(*key) -> np.random.Generator:
    return np.random.default_rng(derive_seed(*key))
