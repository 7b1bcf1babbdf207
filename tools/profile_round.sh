#!/usr/bin/env bash
# One gpurun call's worth of measurements (each ncu command only after the
# same command line exited 0 without ncu, as B200_PROFILING.md asks):
#   bench line, solver Newton-step timings + launch list, K2/K3 ncu at
#   config-4 size, the symmetric sweep's ncu --set full capture.
#   tools/profile_round.sh <tag>
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/${TAG}_bench.log 2>&1
python tools/time_solver.py cfg4 > $O/${TAG}_solver.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_solver_launches.csv \
      python tools/time_solver.py cfg4 > $O/${TAG}_solver_ncu.log 2>&1
python tools/time_config4.py > $O/${TAG}_cfg4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k 'regex:lb_elements_kernel|lb_csr_gather_kernel' \
      -s 2 -c 2 -o $O/${TAG}_k2k3 -f python tools/time_config4.py > $O/${TAG}_k2k3_ncu.log 2>&1
python tools/prof_sweep.py 65536 3 > $O/${TAG}_sweep.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k 'regex:lb_symsweep_ib_kernel' -s 2 -c 1 \
      -o $O/${TAG}_symsweep -f python tools/prof_sweep.py 65536 3 > $O/${TAG}_sweep_ncu.log 2>&1
echo done
