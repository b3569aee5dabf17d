# round 2, job 12: ncu of the FP32 sweeps and the reworked gated pair
set -x
prof() {  # name regex skip target...
  local name=$1 re=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$name "$@" > gpurun_out/${name}_ncu.log 2>&1; echo ncu_$name=$?
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${name}_sass.csv.gz
  rm -f /tmp/$name.ncu-rep
}
prof j12_p32 k_primal 2 python tools/probe.py ncu sweeps32
prof j12_a32 k_adjoint 2 python tools/probe.py ncu sweeps32
prof j12_gated k_pair 1 python tools/probe.py ncu e2e
python tools/probe.py aa > gpurun_out/j12_aa.log 2>&1
du -sh gpurun_out
