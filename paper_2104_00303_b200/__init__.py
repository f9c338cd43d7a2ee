"""gridshift-b200: B200-native MeanShift++ grid shift (arXiv 2104.00303).

Drop-in for the reference's engine surface (`gridshift`): the same names,
argument meanings and error behaviour, executed by hand-written sm_100a CUDA
kernels in `libgridshift_cuda.so` (C ABI: include/gridshift_cuda.h).
Importing this package does not load the library; the first engine call
does, and raises if it is missing -- there is no CPU fallback.
"""

from .batch import segment_batch
from .grid import (CellTables, PointSet, bin_point, bin_points, build_cell_tables,
                   neighbor_aggregate, neighbor_stats)
from .modeseek import (ENGINES, Labeling, ShiftConfig, ShiftTrace, extract_clusters, install,
                       set_sum_order, sum_order,
                       meanshiftpp, meanshiftpp_device, meanshiftpp_points, meanshiftpp_step)
from .segment import (Image, SegmentMap, image_to_features, segment_image, segment_map_from_labeling,
                      segment_pixels)
from .track import (BinSet, TrackState, Window, cluster_window, init_tracker, neighborhood,
                    track_frame, track_sequence)

__all__ = [
    "BinSet", "CellTables", "ENGINES", "Image", "Labeling", "PointSet", "SegmentMap",
    "ShiftConfig", "ShiftTrace", "TrackState", "Window", "bin_point", "bin_points",
    "build_cell_tables", "cluster_window", "extract_clusters", "image_to_features",
    "init_tracker", "install", "set_sum_order", "sum_order", "meanshiftpp", "meanshiftpp_device", "meanshiftpp_points", "meanshiftpp_step",
    "neighbor_aggregate", "neighbor_stats", "neighborhood", "segment_batch", "segment_image",
    "segment_map_from_labeling", "segment_pixels",
    "track_frame", "track_sequence",
]
