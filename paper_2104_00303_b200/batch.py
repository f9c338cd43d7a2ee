"""Batched image segmentation over one process per GPU (cfg2-style weak
scaling).

The reference segments a directory of images through a thread pool, one
engine call per image (`cli.py:206-216` -> `_segment_one` -> `segment_image`,
`segment.py:95-106`).  The images are independent, so here image i goes to
rank i % world: every rank segments its own images on its own GPU and there
is NO collective on the data path ("cfg2: shards naturally").
Only the small per-image results (labels as int32 rasters, mean colours,
traces) are optionally gathered at the end, in image order.

The per-image work goes through `engine(img, cfg, mode, scale)` returning
(SegmentMap, ShiftTrace) -- `segment.segment_image` (CUDA) by default; the
CPU tests inject an oracle-backed engine to cover this driver with gloo.
"""

from __future__ import annotations

from .modeseek import ShiftConfig


def local_indices(count: int, world: int, rank: int) -> list[int]:
    """Images owned by `rank`: i % world == rank (balanced to within one)."""
    return list(range(rank, count, world))


def segment_batch(images, cfg: ShiftConfig, mode: str = "rgb", scale: float | None = None,
                  group=None, engine=None, gather: bool = True):
    """Segment `images` (a sequence of `segment.Image`, identical on every
    rank) across the ranks of `group`.

    Returns, with gather=True, the list of (SegmentMap, ShiftTrace) for ALL
    images in input order on every rank (one all_gather_object at the end);
    with gather=False, a dict {image index: (SegmentMap, ShiftTrace)} of the
    local images only.  Without an initialised process group the whole batch
    runs in this process.
    """
    import torch.distributed as dist

    if engine is None:
        from .segment import segment_image

        def engine(img, c, m, s):
            return segment_image(img, c, m, scale=s)

    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    else:
        world, rank = 1, 0
    mine = {i: engine(images[i], cfg, mode, scale) for i in local_indices(len(images), world, rank)}
    if not gather:
        return mine
    if world == 1:
        return [mine[i] for i in range(len(images))]
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    out = {}
    for p in parts:
        out.update(p)
    return [out[i] for i in range(len(images))]
