# Round-end validation on the GPU box: parity tests (default and tensor engine forced), sanitizer, config timings,
# bench (both arms), ncu launch lists and the full capture of the tensor-core passes.  Run under gpurun:
#   gpurun -- 'bash tools/round_profiles.sh > gpurun_out/round_profiles.log 2>&1'
set -x
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
DOGBLOB_CONV=umma DOGBLOB_STREAMED_UPLOAD=0 timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_umma_forced.log 2>&1
DOGBLOB_CONV=umma timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san_memcheck_umma.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san_memcheck.log 2>&1
timeout 900 python tools/stress_engines.py 120 5 > gpurun_out/stress_engines.txt 2>&1
python tools/config_timings.py > gpurun_out/config_timings.jsonl 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --gpus 2 --steps 5 > gpurun_out/bench_2ranks_1gpu.json 2>> gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>> gpurun_out/bench.err
for c in C2 C4; do
  DOGBLOB_UMMA_DEBUG=0 DOGBLOB_UMMA_PROF=1 timeout 100 python tools/umma_masks.py $c 0 2>&1 | tail -28 > gpurun_out/roles_$c.txt
  # the same with the detection threshold (hit boxes stored, seed test): only the column pass changes
  echo "-- with the detection threshold (UMMA_MASKS_THR=0.1), column pass:" >> gpurun_out/roles_$c.txt
  UMMA_MASKS_THR=0.1 DOGBLOB_UMMA_DEBUG=0 DOGBLOB_UMMA_PROF=1 DOGBLOB_UMMA_PROF_CTAS=1 timeout 100 python tools/umma_masks.py $c 0 2>&1 | tail -16 | cut -c1-1400 >> gpurun_out/roles_$c.txt
  # what the threshold costs the column pass: no seed test / no list appends / every box stored
  UMMA_MASKS_THR=0.1 timeout 100 python tools/umma_masks.py $c 0 1024 2048 512 >> gpurun_out/roles_$c.txt 2>&1
done
export DOGBLOB_STREAMED_UPLOAD=0
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 30 -c 10 --csv --log-file gpurun_out/launches_one_frame.csv python tools/profile_run.py --frames 5 > gpurun_out/prof1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"umma_pass|nms_seed|nms_window" -s 6 -c 3 -o gpurun_out/umma_full -f python tools/profile_run.py --frames 5 > gpurun_out/prof2.log 2>&1
unset DOGBLOB_STREAMED_UPLOAD
DOGBLOB_BENCH_BATCH=16 ncu --metrics gpu__time_duration.sum --clock-control none -s 48 -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 > gpurun_out/prof3.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
