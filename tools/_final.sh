O=gpurun_out/r02_final
mkdir -p $O/sanitizer
python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_run.py > $O/sanitizer/$t.txt 2>&1
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
