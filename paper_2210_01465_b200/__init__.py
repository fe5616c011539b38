"""B200-native fitness-flow-graph / PageRank-centrality core of arXiv 2210.01465.

The product is libtk_landscape.so (C-ABI: include/tk_landscape.h, sm_100a
kernels in csrc/).  This package holds the ctypes binding (`_abi`), the host
mirror of the reference's landscape interface (`landscape`) and the build
script (`build`).  Importing it does not touch the GPU.
"""
from . import _abi  # noqa: F401
from .landscape import (  # noqa: F401
    ADJACENT, HAMMING, AnalysisPipeline, BatchAnalyzer, CentralityReport, Error, FitnessFlowGraph, InvalidArgument,
    Landscape, MinimaFractionReport, NoFeasiblePoint, NonConvergence, PointCensus,
    SearchSpaceCache, analyze_landscape, build_ffg, classify_points,
    minima_fraction_report, neighbourhood_from_string, pagerank, proportion_of_centrality)

__all__ = [n for n in dir() if not n.startswith("_")]
