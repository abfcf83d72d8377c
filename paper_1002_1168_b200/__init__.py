"""B200-native (sm_100a) shape-adaptive motion-estimation hot path of
arXiv 1002.1168, a drop-in for the reference's me:: estimation entry points.

Layers:
  include/me_b200.h           C ABI (the drop-in boundary)
  csrc/*.cu                   sm_100a kernels: wavefront.cu (classify, sort), es.cu, ring.cu,
                              pa.cu (PA wavefront), frame_ops.cu (MC+PSNR, masks), batch.cu (pipeline)
  csrc/capi.cu                validation, contexts, staging, dispatch
  shim/me_drop_in.cpp         C++ me:: definitions over the C ABI (reference headers)
  api.py                      Python mirror of the reference API (tests, users)
  batch.py                    batched sequence pipeline (benchmark path)
  synth.py                    seeded synthetic configs 1..5
  experiment.py, seqio.py     run_experiment (CSV / summaries) and sequence I/O
"""
from ._lib import LIB_PATH, lib, rec_dtype, stats_dtype  # noqa: F401
from .api import (  # noqa: F401
    Algo,
    BlockRect,
    BlockType,
    BoundaryTemporal,
    CandidateSet,
    EstimateOptions,
    MotionField,
    PrsConfig,
    PsnrResult,
    ScoreEvent,
    ScoreKind,
    SearchConfig,
    SearchStats,
    algo_from_string,
    binarize,
    block_dpd_aggregate,
    block_grid,
    brs_select,
    check_dimensions,
    classify_block,
    classify_blocks,
    clip_to_window,
    ds_search,
    estimate_field,
    figure_of_merit,
    fss_search,
    full_search,
    gather_candidates,
    predict_frame,
    prs_refine,
    prs_update,
    psnr,
    psnr_from_sse,
    residual,
    residual_to_gray,
    sad_shape,
    sad_texture,
    to_string,
    tss_search,
)
from .batch import BatchConfig, rec_view, run_sequences, run_sequences_dev  # noqa: F401


def device_count() -> int:
    return int(lib().me_b200_device_count())
