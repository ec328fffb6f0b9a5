# Helpers for gpurun calls (sourced on the GPU box): capture one ncu --set full report, convert it to text
# (raw metrics CSV + source-line CSV) under gpurun_out/, and drop the binary report if it is large, so that the
# gpurun_out/ merge stays under its 64 MiB cap.
#   ncu_cap NAME KERNEL_REGEX SKIP COUNT -- command...
ncu_cap() {
  local name=$1 kre=$2 skip=$3 cnt=$4; shift 5
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c "$cnt" \
    -o "gpurun_out/$name" "$@" > "gpurun_out/${name}_ncu.log" 2>&1
  local rc=$?
  if [ -f "gpurun_out/$name.ncu-rep" ]; then
    ncu -i "gpurun_out/$name.ncu-rep" --page raw --csv > "gpurun_out/${name}_raw.csv" 2>/dev/null
    ncu -i "gpurun_out/$name.ncu-rep" --page source --csv --print-source sass > "gpurun_out/${name}_src.csv" 2>/dev/null
    gzip -f "gpurun_out/${name}_src.csv"
    local sz=$(stat -c %s "gpurun_out/$name.ncu-rep")
    if [ "$sz" -gt 8000000 ]; then rm -f "gpurun_out/$name.ncu-rep"; fi
  fi
  echo "ncu_cap $name rc=$rc"
}
