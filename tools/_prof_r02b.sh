mkdir -p gpurun_out/r02b
python bench.py --steps 20 --warmup 5 > gpurun_out/r02b/bench_fma.json 2> gpurun_out/r02b/bench_fma.err
python bench.py --steps 20 --warmup 5 --variant nodal --bitwise > gpurun_out/r02b/bench_nodal.json 2> gpurun_out/r02b/bench_nodal.err
python bench.py --steps 2 --warmup 1 --e2e-steps 0 > gpurun_out/r02b/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:volume_kernel_mirror -s 1 -c 1 -o gpurun_out/r02b/prof_volume_fma python bench.py --steps 2 --warmup 1 --e2e-steps 0 > gpurun_out/r02b/ncu_vol.log 2>&1
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --bitwise > gpurun_out/r02b/plain_bw.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:volume_kernel_mirror -s 1 -c 1 -o gpurun_out/r02b/prof_volume_bitwise python bench.py --steps 2 --warmup 1 --e2e-steps 0 --bitwise > gpurun_out/r02b/ncu_vol_bw.log 2>&1
python tools/tts_ratio.py 6 > gpurun_out/r02b/tts6.log 2>&1; python tools/tts_ratio.py 7 > gpurun_out/r02b/tts7.log 2>&1
python tools/solver_bench.py > gpurun_out/r02b/solver.log 2>&1
echo done
