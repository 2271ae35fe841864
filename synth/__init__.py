"""Seeded synthetic inputs shared by the tests, the bench and the oracle checks.

This package holds NO attention arithmetic. It only produces input tensors from
(seed, tensor_id, flat index) with a counter-based generator (see ``gen.py``).
The CUDA library implements the same generator independently
(``paper_2112_05682_b200/csrc/gen_inputs.cu``); ``tests/test_gpu_probe.py::test_device_generator_bit_identical``
checks the two are bit-identical.
"""
from .gen import (  # noqa: F401
    TENSOR_Q, TENSOR_K, TENSOR_V, TENSOR_DO,
    irwin_hall_values, normal_tensor, round_to_bf16, bf16_bits_to_f32,
)
