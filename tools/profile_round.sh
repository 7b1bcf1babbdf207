#!/usr/bin/env bash
# One gpurun call's worth of round-end measurements (each ncu command only
# after the same command line exited 0 without ncu, as B200_PROFILING.md
# asks):  tools/profile_round.sh <tag>
#   bench line + reference arm, the bench's launch list, the sweep's
#   ncu --set full capture, K2/K3 ncu at config-4 size, solver Newton-step
#   timings + launch list + block-LU ncu, per-rank shares of a G-GPU split.
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
python bench.py > $O/${TAG}_bench.log 2>&1
python bench.py --impl reference > $O/${TAG}_bench_reference.log 2>&1
python bench.py --steps 3 --warmup 3 --cpu-seconds 0 --e2e-steps 1 > $O/${TAG}_bench_short.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_bench_launches.csv \
      python bench.py --steps 3 --warmup 3 --cpu-seconds 0 --e2e-steps 1 > $O/${TAG}_bench_ncu.log 2>&1
python tools/prof_sweep.py 65536 3 > $O/${TAG}_sweep.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k 'regex:lb_symsweep_ib_kernel' -s 2 -c 1 \
      -o $O/${TAG}_symsweep -f python tools/prof_sweep.py 65536 3 > $O/${TAG}_sweep_ncu.log 2>&1
python tools/time_config4.py > $O/${TAG}_cfg4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k 'regex:lb_elements_kernel|lb_csr_gather_kernel' \
      -s 2 -c 2 -o $O/${TAG}_k2k3 -f python tools/time_config4.py > $O/${TAG}_k2k3_ncu.log 2>&1
python tools/time_solver.py > $O/${TAG}_solver.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_solver_launches.csv \
      python tools/time_solver.py cfg4 > $O/${TAG}_solver_ncu.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k 'regex:lb_getrf_kernel|lb_getrs_slab_kernel|lb_bgemm_kernel' \
      -s 20 -c 3 -o $O/${TAG}_lu -f python tools/time_solver.py cfg4 > $O/${TAG}_lu_ncu.log 2>&1
# the reduction's level-0 launches (256 blocks at config 4): the first four LU-phase kernels
ncu --set full --clock-control none --import-source on -k 'regex:lb_getrf_kernel|lb_getrs_slab_kernel|lb_bgemm_kernel' \
    -s 0 -c 4 -o $O/${TAG}_lu_level0 -f python tools/time_solver.py cfg4 > $O/${TAG}_lu_level0_ncu.log 2>&1
python tools/rank_shares.py 65536 5 > $O/${TAG}_rank_shares.log 2>&1
echo done
