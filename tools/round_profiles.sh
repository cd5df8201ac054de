# Round-end validation on the GPU box: parity tests (default and tensor engine forced), sanitizer, config timings,
# bench (both arms), ncu launch lists and the full capture of the tensor-core passes.  Run under gpurun:
#   gpurun -- 'bash tools/round_profiles.sh > gpurun_out/round_profiles.log 2>&1'
set -x
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
DOGBLOB_CONV=umma DOGBLOB_STREAMED_UPLOAD=0 timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_umma_forced.log 2>&1
DOGBLOB_CONV=umma timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san_memcheck_umma.log 2>&1
python tools/config_timings.py > gpurun_out/config_timings.jsonl 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>> gpurun_out/bench.err
export DOGBLOB_STREAMED_UPLOAD=0
ncu --metrics gpu__time_duration.sum --clock-control none -s 36 -c 9 --csv --log-file gpurun_out/launches_one_frame.csv python tools/profile_run.py --frames 5 > gpurun_out/prof1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:umma_pass -s 8 -c 2 -o gpurun_out/umma_full -f python tools/profile_run.py --frames 5 > gpurun_out/prof2.log 2>&1
unset DOGBLOB_STREAMED_UPLOAD
ncu --metrics gpu__time_duration.sum --clock-control none -s 48 -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 > gpurun_out/prof3.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
