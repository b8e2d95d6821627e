#!/bin/bash
# Build libhgs.so variants (compile-time knobs) into tools/var/<name>/ for
# A/B timing on the GPU box:  HGS_LIB=tools/var/<name>/libhgs.so python bench.py ...
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
build() {  # name extra-flags [csrc dir]
  local src=${3:-$R/paper_2512_02932_b200/csrc}
  mkdir -p $R/tools/var/$1
  make -s -j8 -C "$src" OUT=$R/tools/var/$1/libhgs.so BUILD=$R/tools/var/$1/build EXTRA="$2" > /dev/null
}
"$@"
