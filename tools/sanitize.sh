#!/usr/bin/env bash
# compute-sanitizer passes over the libdrs kernels (memcheck +
# racecheck on the noise streams (incl. the SFC64 named-barrier pipeline), the
# skip chains, the tcgen05 GEMM / attention mbarrier rings and the cluster
# GroupNorm).  Run on the GPU box:  tools/sanitize.sh  -> gpurun_out/sanitizer/
set -u
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
OUT="$ROOT/gpurun_out/sanitizer"
mkdir -p "$OUT"
cd "$ROOT" || exit 2
declare -A SEL=(
  [noise]="tests/test_gpu_noise.py"
  [chain]="tests/test_gpu_transitions.py"
  [gemm]="tests/test_gpu_gemm.py -k test_gemm_shapes or test_gemm_cluster_splitk or test_gemm_cta_pair or test_implicit_conv3x3"
  [attention]="tests/test_gpu_nets.py -k test_attention_tc_kernel"
  [groupnorm]="tests/test_gpu_nets.py -k test_groupnorm"
  [gm_eps]="tests/test_gpu_samplers.py -k many_components or x0_posterior"
)
: > "$OUT/summary.txt"
for tool in memcheck racecheck; do
  for name in noise chain gm_eps groupnorm attention gemm; do
    read -r -a args <<< "${SEL[$name]}"
    # -k expressions contain spaces: re-join everything after -k
    files=() kexpr=""
    for ((i = 0; i < ${#args[@]}; i++)); do
      if [[ "${args[$i]}" == "-k" ]]; then kexpr="${args[*]:$((i + 1))}"; break; fi
      files+=("${args[$i]}")
    done
    log="$OUT/${tool}_${name}.log"
    if [[ -n "$kexpr" ]]; then
      timeout 1200 compute-sanitizer --tool "$tool" --target-processes all --print-limit 20 \
        python -m pytest "${files[@]}" -m gpu -q -x -p no:cacheprovider -k "$kexpr" > "$log" 2>&1
    else
      timeout 1200 compute-sanitizer --tool "$tool" --target-processes all --print-limit 20 \
        python -m pytest "${files[@]}" -m gpu -q -x -p no:cacheprovider > "$log" 2>&1
    fi
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" "$log" | tail -3 | tr '\n' ' ')
    res=$(grep -E "passed|failed" "$log" | tail -1)
    echo "$tool $name rc=$rc | $res | $summ" >> "$OUT/summary.txt"
  done
done
cat "$OUT/summary.txt"
