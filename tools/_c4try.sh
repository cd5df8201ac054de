for v in "DOGBLOB_UMMA_RAW=2" "DOGBLOB_UMMA_RAW=3" "DOGBLOB_UMMA_RAW=4"; do
  echo "=== C2 $v" >> gpurun_out/umma_c4.log
  env $v CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/umma_probe.py C2 2>&1 | grep -v "^fma" | tail -3 >> gpurun_out/umma_c4.log
done
