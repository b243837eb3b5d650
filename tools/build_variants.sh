#!/usr/bin/env bash
# Build A/B variants of libsvx.so into variants/ (git-ignored, travels to the
# GPU box); each argument is name=defines, e.g.
#   bash tools/build_variants.sh base= w64="-DSVX_TILE_RAYS=64 -DSVX_MARCH_BLOCKS=1184"
# then on the box: SVX_LIB_PATH=$PWD/variants/libsvx_<name>.so python ...
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
for spec in "$@"; do
  name=${spec%%=*}; defs=${spec#*=}
  SVX_NVCC_DEFS="$defs" python paper_2512_12945_b200/build.py --force > /dev/null
  cp paper_2512_12945_b200/libsvx.so variants/libsvx_$name.so
  echo "built variants/libsvx_$name.so ($defs)"
done
python paper_2512_12945_b200/build.py --force > /dev/null
