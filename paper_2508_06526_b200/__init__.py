# SPDX-License-Identifier: Apache-2.0
"""B200-native PiKV decode engine (arXiv 2508.06526), drop-in for the
reference's Engine::step path (/root/reference/proj/src/pipeline.cpp:213-351).

The product is libpikv_b200.so (C-ABI, include/pikv_b200.h) built from csrc/;
``engine`` mirrors the reference's C++ API in Python over that ABI.
"""
from .config import (CompressorConfig, EngineConfig, ModelConfig, RouterConfig,  # noqa: F401
                     SchedulerConfig, StoreConfig)

__all__ = ["CompressorConfig", "EngineConfig", "ModelConfig", "RouterConfig", "SchedulerConfig",
           "StoreConfig"]
