#!/bin/bash
# Diagnostic variants of complete.cu (ablation macros; the numerics of such builds can be wrong by
# construction): tools/abl_build.sh NAME -DMACRO ...  (wraps tools/variant_build.sh)
exec "$(dirname "$0")/variant_build.sh" "$1" complete.cu "${@:2}"
