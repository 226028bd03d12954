#!/bin/bash
# End-of-milestone evidence: bench line, launch list, ncu --set full of the hot kernels.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_full.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launch_final.log 2>&1
for k in k_armc k_ifce_dw k_ups_bwd k_syn_trunk_bwd2 k_syn_post2 k_latent_grad k_ups_fwd k_nn_reduce; do
  ncu --set full --clock-control none --import-source on --kernel-name-base function -k "regex:^$k$" -s 6 -c 1 -o gpurun_out/full_$k -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/full_$k.log 2>&1
done
echo done
