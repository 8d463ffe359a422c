#!/bin/bash
# Build the library with extra -D switches into build/alt/<name>.so (A/B timing with
# tools/ab_so.sh), then rebuild the default library.  Usage: tools/build_variant.sh name "-DX=0 ..."
cd "$(dirname "$0")/.."
mkdir -p build/alt
touch paper_2102_04199_b200/csrc/*.cu
KT_NVCC_DEFS="$2" python -m paper_2102_04199_b200.build > /dev/null || exit 1
cp paper_2102_04199_b200/libkerntune_b200.so "build/alt/$1.so"
touch paper_2102_04199_b200/csrc/*.cu
python -m paper_2102_04199_b200.build > /dev/null
