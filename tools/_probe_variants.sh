for lib in paper_2103_06080_b200/libnwb200.so tools/_variants/lib_NWB_POST_UNROLL_4.so tools/_variants/lib_NWB_PASS_UNROLL_2.so; do
  echo "lib=$lib"; NWB_LIB=$lib timeout 300 python tools/rho_probe.py double ""; NWB_LIB=$lib timeout 300 python tools/rho_probe.py single ""
done 2>&1 | grep -v Warn
python tools/study_timing.py 2>&1 | tail -3
