mkdir -p gpurun_out/r02
python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench_fma.json 2> gpurun_out/r02/bench_fma.err
python bench.py --steps 20 --warmup 5 --bitwise > gpurun_out/r02/bench_bitwise.json 2> gpurun_out/r02/bench_bitwise.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02/bench_ref.json 2> gpurun_out/r02/bench_ref.err
python bench.py --steps 2 --warmup 1 --e2e-steps 0 > gpurun_out/r02/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 > gpurun_out/r02/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:volume_kernel_mirror -s 3 -c 1 -o gpurun_out/r02/prof_volume_fma python bench.py --steps 2 --warmup 1 --e2e-steps 0 > gpurun_out/r02/ncu_vol.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:surface_face -s 3 -c 1 -o gpurun_out/r02/prof_face python bench.py --steps 2 --warmup 1 --e2e-steps 0 > gpurun_out/r02/ncu_face.log 2>&1
python bench.py --steps 2 --warmup 1 --e2e-steps 0 --bitwise > gpurun_out/r02/plain_bw.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:volume_kernel_mirror -s 3 -c 1 -o gpurun_out/r02/prof_volume_bitwise python bench.py --steps 2 --warmup 1 --e2e-steps 0 --bitwise > gpurun_out/r02/ncu_vol_bw.log 2>&1
echo done
