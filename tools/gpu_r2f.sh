./tools/ubench_seq.bin 2>&1 | grep "variant" > gpurun_out/r2f_ubench_var.txt; cat gpurun_out/r2f_ubench_var.txt
cd .headcheck && timeout 600 python -m pytest tests/test_gpu_group.py -m gpu -q -x -k "operators" > ../gpurun_out/r2f_group_head.log 2>&1; echo group_head_rc=$?
tail -3 ../gpurun_out/r2f_group_head.log
