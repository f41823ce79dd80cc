timeout 900 python bench.py > gpurun_out/r02c_c3.json 2> gpurun_out/r02c_c3.err
timeout 900 python bench.py --workload mu1m > gpurun_out/r02c_mu.json 2> gpurun_out/r02c_mu.err
