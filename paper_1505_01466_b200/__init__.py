"""B200-native Fast-SSC list-CRC polar decoding (arXiv 1505.01466).

Drop-in for the list-decode path of the reference package ``polaris``:
code construction, encoding and schedules are host-side mirrors of
``polaris.codes`` / ``polaris.encode`` / ``polaris.schedule``; the decoder
itself (``ListDecoder``, ``decode``) runs hand-written sm_100a CUDA through
the C ABI in ``include/polar_b200.h``.
"""

from .codes import (CRC8, CRC16, CRC32, CodeSpec, CrcConfig, construct_frozen_set,
                    crc_check, crc_checksum_bits, crc_compute, design_eps)
from .encode import (MessageFrame, attach_and_encode, attach_and_encode_batch,
                     extract_payload, polar_encode)
from .schedule import (NodeKind, NodeOp, Schedule, ScheduleConfig, build_schedule,
                       classify, emit_source)
from .channel import (LLR_CLAMP, ChannelConfig, clamp_llr, frame_rng, generate_frames,
                      quantize_int8, transmit)
from .listdec import (AdaptiveBatchResult, AdaptiveDecoder, BatchResult, DecodeResult,
                      ListDecoder, PathOutcome, adaptive_decode, decode, prebuild_specialised,
                      schedule_op_rows, select_candidates, set_default_options, specialised_source)
from .fastssc import execute_schedule
from .sim import CSV_FIELDS, DeviceFrames, SimRecord, run_sweep, write_csv

__version__ = "0.1.0"

__all__ = [
    "CRC8", "CRC16", "CRC32", "CodeSpec", "CrcConfig", "construct_frozen_set",
    "crc_check", "crc_checksum_bits", "crc_compute", "design_eps",
    "MessageFrame", "attach_and_encode", "attach_and_encode_batch", "extract_payload",
    "polar_encode",
    "NodeKind", "NodeOp", "Schedule", "ScheduleConfig", "build_schedule", "classify",
    "emit_source",
    "LLR_CLAMP", "ChannelConfig", "clamp_llr", "frame_rng", "generate_frames",
    "quantize_int8", "transmit",
    "AdaptiveBatchResult", "AdaptiveDecoder", "BatchResult", "DecodeResult", "ListDecoder",
    "PathOutcome", "adaptive_decode", "decode", "execute_schedule", "schedule_op_rows",
    "CSV_FIELDS", "DeviceFrames", "SimRecord", "run_sweep", "write_csv",
    "select_candidates", "set_default_options", "specialised_source", "prebuild_specialised", "__version__",
]
