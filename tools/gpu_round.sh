#!/bin/bash
# Round-end evidence on one GPU (under gpurun): the GPU test suite, compute-sanitizer on
# tools/sanitize_run.py (memcheck / racecheck / synccheck / initcheck), the default bench line,
# and the ncu captures of tools/collect_profiles.sh. Output: gpurun_out/<tag>/.
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O/sanitizer
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
if [ -n "$SANITIZE" ]; then   # (the pool refused compute-sanitizer late in round 2: opt-in)
  for t in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py > $O/sanitizer/$t.txt 2>&1
  done
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
[ -n "$NO_NCU" ] || bash tools/collect_profiles.sh $TAG
