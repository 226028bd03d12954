mkdir -p gpurun_out
timeout 300 python -m pytest tests -x -q -s -m gpu -k "lockstep_vs_golden" > gpurun_out/t_golden.log 2>&1; echo "golden exit $?" >> gpurun_out/t_golden.log
tail -3 gpurun_out/t_golden.log
timeout 900 python -m pytest tests -q -s -m gpu -k "truth or 50_iter or lockstep_vs_reference or full_schedule or determinism or branches" > gpurun_out/t_par.log 2>&1; echo "par exit $?" >> gpurun_out/t_par.log
tail -3 gpurun_out/t_par.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo "bench exit $?"
CCB_ARM=2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-full-schedule > gpurun_out/bench_a2.json 2> gpurun_out/bench_a2.err; echo "bench2 exit $?"
