#!/bin/bash
# A/B timing driver (replaces the round-1 one-off gpu_*.sh scripts).
#
#   tools/ab.sh ROUNDS "LABEL:SETTINGS" ["LABEL:SETTINGS" ...] -- TIMER ARGS...
#
# Each variant is timed ROUNDS times, interleaved (A B A B ...) to cancel drift in clocks and
# power.  SETTINGS is either
#   * a list of H3_* environment assignments (e.g. "H3_DMMA_CFG=6 H3_DMMA_CLUSTER_Y=1"): the
#     timer then loads the measurement library build/libh3b200_measure.so (`make -C
#     paper_1609_09841_b200/csrc measure`), the only build that reads those variables; or
#   * "lib=PATH" to time another build of libh3b200.so (e.g. a copy of the previous commit's);
#   * empty for the product library.
# TIMER is a tools/ script (time_fused.py, time_literal.py, energy.py ...).  Example:
#   tools/ab.sh 3 "base:" "dfma:H3_FUSED_IMPL=dfma" -- tools/time_fused.py 3 512 fused 6
set -u
rounds=$1; shift
variants=()
while [ "$1" != "--" ]; do variants+=("$1"); shift; done
shift
for ((r = 0; r < rounds; r++)); do
  for v in "${variants[@]}"; do
    label=${v%%:*}; settings=${v#*:}
    if [[ $settings == lib=* ]]; then
      echo -n "[$label] "; H3_LIB=${settings#lib=} timeout 600 python "$@"
    elif [ -n "$settings" ]; then
      echo -n "[$label] "; env H3_LIB=build/libh3b200_measure.so $settings timeout 600 python "$@"
    else
      echo -n "[$label] "; timeout 600 python "$@"
    fi
  done
done
