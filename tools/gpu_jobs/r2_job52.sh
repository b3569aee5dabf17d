# round 2, job 52: ncu --set full of the final k_pair, k_gradient, k_pair_aa (after the store rematerialisation)
set -x
prof() {  # name regex skip target...
  local name=$1 re=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$name "$@" > gpurun_out/${name}_ncu.log 2>&1; echo ncu_$name=$?
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${name}_sass.csv.gz
  rm -f /tmp/$name.ncu-rep
}
prof j52_pair k_pair 2 python tools/probe.py ncu pair
prof j52_grad k_gradient 1 python tools/probe.py ncu gradient
prof j52_pair_aa k_pair_aa 2 python tools/probe.py ncu aa
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/j52_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/j52_ncu_launch.log 2>&1; echo ncu1=$?
