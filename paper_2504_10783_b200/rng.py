"""Host side of the counter-based random streams.

The device kernels draw every random number as a pure function of
``(seed, walk index, step, slot)`` (``csrc/ez_rng.cuh``). Two stream
families exist:

* ``"counter"`` — the reference's splitmix64 counter hash
  (``corridor/seeding.py:19-60``): ``h = mix(mix(mix(0 ^ seed) ^ walk) ^
  (step*64 + slot))``, uniforms ``((h >> 11) + 0.5) * 2**-53`` and normals
  through the inverse normal CDF. Default: sample streams are the
  reference's, so polytopes can be compared draw for draw.
* ``"philox"`` — Philox4x32-10 keyed by the seed, counter = (walk, step,
  slot group), Box-Muller normals in fp32. Cheaper; statistically
  equivalent, not draw-compatible with the reference.

Only tiny host helpers live here (``child_seed`` for deriving per-segment
seeds, ``SEED_STEP``); bulk streams are generated on the GPU.
"""

from __future__ import annotations

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX_A = 0xBF58476D1CE4E5B9
MIX_B = 0x94D049BB133111EB

# step tag of the draw that places a walk's start point on the seed segment
SEED_STEP = 1 << 32

RNG_COUNTER = 0
RNG_PHILOX = 1
RNG_MODES = {"counter": RNG_COUNTER, "philox": RNG_PHILOX}


def splitmix_mix(z: int) -> int:
    """splitmix64 finaliser on a Python int (mod 2**64)."""
    z = (z + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * MIX_A) & MASK64
    z = ((z ^ (z >> 27)) * MIX_B) & MASK64
    return z ^ (z >> 31)


def fold(*words: int) -> int:
    """Fold integer words into one 64-bit hash (reference ``hash_u64`` semantics)."""
    h = 0
    for w in words:
        h = splitmix_mix(h ^ (int(w) & MASK64))
    return h


def child_seed(master: int, *words: int) -> int:
    """Reproducible child seed from a master seed and context words."""
    return fold(master & MASK64, *words)


def rng_mode(name) -> int:
    if isinstance(name, int):
        if name in RNG_MODES.values():
            return name
    elif name in RNG_MODES:
        return RNG_MODES[name]
    raise ValueError(f"unknown rng mode {name!r}; expected one of {sorted(RNG_MODES)}")
