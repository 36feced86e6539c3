#!/usr/bin/env bash
# build the library; exit non-zero (with nvcc's message) on failure
cd "$(dirname "$0")/.." && python -c "
import sys; sys.path.insert(0, '.')
from paper_2502_14866_b200 import _build
_build.build()" 2>&1 | tail -15; exit ${PIPESTATUS[0]}
