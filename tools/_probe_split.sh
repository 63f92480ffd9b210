for lib in paper_2103_06080_b200/libnwb200.so tools/_variants/libnwb200_mb2.so; do
 for ilv in 0 1; do
  for p in double single; do
   echo "lib=$lib ilv=$ilv"; NWB_LIB=$lib NWB_RHO_R1=2 NWB_RHO_ILV=$ilv timeout 300 python tools/rho_probe.py $p ""
  done
 done
done 2>&1 | grep -v Warn
