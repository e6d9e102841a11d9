set -x
timeout 300 python tools/gemm_bench.py --config 1 > gpurun_out/r2i_gemm1.json 2>&1; echo rc=$?
timeout 300 python tools/gemm_bench.py --config 2 > gpurun_out/r2i_gemm2.json 2>&1; echo rc=$?
timeout 300 python tools/gemm_bench.py --config 3 > gpurun_out/r2i_gemm3.json 2>&1; echo rc=$?
