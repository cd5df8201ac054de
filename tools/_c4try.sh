rm -f gpurun_out/variants.log
cp paper_2010_08486_b200/libdogblob_b200.so /tmp/lib_default.so
for v in i3_k4 i3_k2; do
  cp tools/_bin/lib_$v.so paper_2010_08486_b200/libdogblob_b200.so
  echo "=== $v" >> gpurun_out/variants.log
  timeout 200 python tools/umma_probe.py C2 2>&1 | grep "^umma  .*row\|rror\|timeout" >> gpurun_out/variants.log
  timeout 200 python tools/umma_debug.py C2 2>&1 | grep "umma\] levels\|umma\] fused\|blob sets" | cut -c1-160 >> gpurun_out/variants.log
  timeout 300 python tools/umma_probe.py C4 2>&1 | grep "^umma  .*row" >> gpurun_out/variants.log
done
cp /tmp/lib_default.so paper_2010_08486_b200/libdogblob_b200.so
