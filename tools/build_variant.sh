#!/bin/bash
# build_variant.sh NAME "-DMACRO=V ..." -> paper_2506_06988_b200/variants/libhgs_NAME.so
set -e
cd "$(dirname "$0")/../paper_2506_06988_b200/csrc"
mkdir -p ../variants
make -s -j8 BUILD="build_$1" OUT="../variants/libhgs_$1.so" EXTRA="$2"
