#!/bin/bash
# Builds the working tree with extra nvcc flags into ab/$1.so (A/B of compile-time knobs):
#   bash scripts/ab_variant.sh fused64 -DTCSE_FUSED_TWIST_MIN=64
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/ab"
TCSE_BUILD_OUT="$root/ab/$name.so" TCSE_NVCC_FLAGS="$*" python -c "
import sys; sys.path.insert(0, '$root')
from paper_2512_13365_b200 import build as b; b.build(force=True)"
echo "$root/ab/$name.so"
