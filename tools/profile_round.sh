# Round profile set (run under gpurun): bench line, the ncu launch list of the same bench command
# (serialised, cold caches: shares only), one ncu --set full capture of the per-view kernels.
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --quick --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_(cull|project|color|emit|onesweep|ranges_fixup|raster_fwd|raster_bwd|project_bwd|project_bwd_shg|imp_coop|loss_photo)" \
  -s 40 -c 14 -o gpurun_out/full_r02d python tools/view_probe.py 6 > gpurun_out/ncu_full.log 2>&1
