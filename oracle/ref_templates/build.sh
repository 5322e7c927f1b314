#!/bin/bash
# Compile oracle/ref_templates/pcg_ref_templates.cpp against the reference's
# headers where they lie (/root/reference/proj/include; nothing is copied),
# output in oracle/_ref/ (git-ignored; it travels to the GPU box with the
# snapshot).  Needs the built paper_1804_02539_b200/lib/libpmg_{cuda,host}.so.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
REF=${PMG_REFERENCE_INCLUDE:-/root/reference/proj/include}
[ -f "$REF/patchmg/multigrid.hpp" ] || { echo "reference headers not found at $REF" >&2; exit 3; }
mkdir -p "$ROOT/oracle/_ref"
g++ -O2 -std=c++20 -Wall \
  -I "$HERE/eigen_decl" -I "$REF" -I "$ROOT/include" \
  -o "$ROOT/oracle/_ref/pcg_ref_templates" "$HERE/pcg_ref_templates.cpp" \
  -L "$ROOT/paper_1804_02539_b200/lib" -lpmg_cuda -lpmg_host \
  -Wl,-rpath,'$ORIGIN/../../paper_1804_02539_b200/lib' -pthread
echo "$ROOT/oracle/_ref/pcg_ref_templates"
