python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 300 python tools/sanitize_probe.py > gpurun_out/probe_plain.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "EXIT $?" >> gpurun_out/sanitizer_$tool.log
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
