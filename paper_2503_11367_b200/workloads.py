"""The BASELINE.json benchmark masks as ``build_bitfield`` segment lists
(SURVEY.md §8(d)); all are 128-token aligned.

  1  1 image + text, 4K, 8/8 heads, CP=1
  2  image prefix (bidirectional) + causal text, 32K, 32/32 heads, CP=2
  3  x64 scale-up of the reference fixture mask-two-encoders.json, 64K, 32/32, CP=4
  4  EMU-style interleaved multi-image (seed 0, one modality per image), 128K,
     GQA 32q/8kv, CP=8
  5  mask sweep at 128K: causal / prefix-LM / multimodal (config 3 x2) /
     multi-image (config 4)
"""

from __future__ import annotations

import random

K = 1024


def emu_interleave(T: int = 128 * K, seed: int = 0):
    """Text runs of {2,4,8,16,32} blocks alternating with images of
    {8,16,32,64} blocks, each image its own modality (same-named segments
    would attend each other, test_mask.py:111-113), clipped to T."""
    rng = random.Random(seed)
    segs, total, i = [], 0, 0
    while total < T:
        n = min(rng.choice([2, 4, 8, 16, 32]) * 128, T - total)
        segs.append(("text", n))
        total += n
        if total >= T:
            break
        n = min(rng.choice([8, 16, 32, 64]) * 128, T - total)
        segs.append((f"img{i}", n))
        total += n
        i += 1
    return segs


CONFIGS = {
    1: dict(name="config1_text_image_4k", segments=[("text", 128), ("image", 1024), ("text", 2944)],
            Hq=8, Hkv=8, cp=1),
    2: dict(name="config2_image_prefix_32k", segments=[("image", 8 * K), ("text", 24 * K)],
            Hq=32, Hkv=32, cp=2),
    3: dict(name="config3_vision_audio_text_64k",
            segments=[("text", 8 * K), ("vision", 16 * K), ("text", 16 * K), ("audio", 16 * K),
                      ("text", 8 * K)], Hq=32, Hkv=32, cp=4),
    4: dict(name="config4_emu_multi_image_128k", segments=emu_interleave(), Hq=32, Hkv=8, cp=8),
}

SWEEP_128K = {
    "causal": [("text", 128 * K)],
    "prefix_lm": [("prefix", 32 * K), ("text", 96 * K)],
    "multimodal": [(m, 2 * c) for m, c in CONFIGS[3]["segments"]],
    "multi_image": CONFIGS[4]["segments"],
}
