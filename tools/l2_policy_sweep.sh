# DRAM bytes and time of the 8192^3 bench kernel under L2 policy / raster-group knobs (ncu, tuning only)
for cfg in "TK_POL_A=1 TK_POL_B=1" "TK_POL_A=1 TK_POL_B=2" "TK_POL_A=1 TK_POL_B=0" "TK_POL_A=0 TK_POL_B=0" "TK_POL_A=2 TK_POL_B=1" "TK_GROUP_M=8" "TK_GROUP_M=12" "TK_GROUP_M=32" "TK_GROUP_M=8 TK_POL_A=2 TK_POL_B=1" "TK_GROUP_M=32 TK_POL_A=1 TK_POL_B=2"; do
  env $cfg ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv python tools/one_case.py dense8192 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' -v c="$cfg" '{print c" | "$(NF-2)" "$(NF-1)" "$NF}'
done
