# round 2, job 53: ncu of the frozen-base (moment cache) FP64 adjoint
set -x
ncu --set full --clock-control none --import-source on -k regex:k_adjoint -s 1 -c 1 -o /tmp/mom python tools/probe.py ncu sweeps > gpurun_out/j53_ncu.log 2>&1; echo rc=$?
ncu -i /tmp/mom.ncu-rep --page raw --csv > gpurun_out/j53_mom_raw.csv 2>/dev/null
ncu -i /tmp/mom.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/j53_mom_sass.csv.gz
rm -f /tmp/mom.ncu-rep
