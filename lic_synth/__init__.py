"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no convolution, no GDN, no
quantisation, no CDF, no coding).  It only produces input *data*:

* ``weights``: random-init model parameters in the LICW container
  (SURVEY.md §8(c) reading c15; SPEC.md:329 for the container), and
* ``frames``: synthetic u8 RGB frames of the paper's shapes.

Both the oracle (``oracle/``) and the product package read these bytes; neither
imports the other.
"""
from .weights import (BLOCKS, block_specs, generate_weights, write_licw, read_licw_blocks,
                      licw_digest, scale_table, ModelSpec)
from .frames import synth_frame_u8, synth_frames_u8, u8_to_f32_chw

__all__ = ["BLOCKS", "block_specs", "generate_weights", "write_licw", "read_licw_blocks",
           "licw_digest", "scale_table", "ModelSpec", "synth_frame_u8", "synth_frames_u8",
           "u8_to_f32_chw"]
