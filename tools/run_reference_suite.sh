#!/usr/bin/env bash
# Run the reference's OWN test suite (pkg/tests, unmodified) against the
# skipdiff-named drop-in (dropin/skipdiff -> paper_2603_25872_b200.numpy_api),
# i.e. against the B200 kernels.
#   tools/run_reference_suite.sh stage   # in the build container: copy the suite
#                                        # into baseline/_ref_tests (git-ignored,
#                                        # travels to the GPU box with gpurun)
#   tools/run_reference_suite.sh run     # on the GPU box: one pytest per file,
#                                        # summary -> gpurun_out/ref_suite/
set -u
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
DST="$ROOT/baseline/_ref_tests"
case "${1:-run}" in
stage)
  rm -rf "$DST" && mkdir -p "$DST"
  cp /root/reference/pkg/tests/*.py "$DST"/
  echo "staged $(ls "$DST" | wc -l) files into $DST"
  ;;
run)
  OUT="$ROOT/gpurun_out/ref_suite"
  mkdir -p "$OUT"
  cd "$DST" || exit 2
  : > "$OUT/summary.txt"
  for f in test_*.py; do
    PYTHONPATH="$ROOT/dropin" timeout 1800 python -m pytest -c /dev/null --rootdir="$DST" -p no:cacheprovider \
      -q -rfE "$f" > "$OUT/${f%.py}.log" 2>&1
    echo "$f rc=$? $(tail -1 "$OUT/${f%.py}.log")" >> "$OUT/summary.txt"
  done
  cat "$OUT/summary.txt"
  ;;
esac
