set -x
timeout 200 python tools/umma_probe.py C2 > gpurun_out/umma_probe.log 2>&1
export DOGBLOB_STREAMED_UPLOAD=0
ncu --metrics gpu__time_duration.sum --clock-control none -s 32 -c 8 --csv --log-file gpurun_out/launches_one_frame.csv python tools/profile_run.py --frames 5 > gpurun_out/prof1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:umma_pass -s 8 -c 2 -o gpurun_out/umma_full -f python tools/profile_run.py --frames 5 > gpurun_out/prof2.log 2>&1
ncu --set full --clock-control none -k regex:nms_ -s 4 -c 1 -o gpurun_out/nms_full -f python tools/profile_run.py --frames 5 > gpurun_out/prof4.log 2>&1
unset DOGBLOB_STREAMED_UPLOAD
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -s 48 -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 > gpurun_out/prof3.log 2>&1
