# compute-sanitizer tiers on the fused step and the log-prob forward (tiny, ragged)
python paper_2510_04206_b200/build.py > /dev/null
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py \
      > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.txt
done
