L=$PWD/paper_2503_11367_b200
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_cp.py tests/test_gpu_large.py -q -x > gpurun_out/t_all.log 2>&1; echo "TESTS: $(tail -n 1 gpurun_out/t_all.log)"
for i in 1 2; do for V in libbam libbam_poly2 libbam_poly4 libbam_poly0 libbam_oldfwd; do echo "$V $(BAM_LIB_PATH=$L/$V.so timeout 200 python tools/time_attn.py --config 4,2 --iters 6 2>&1 | grep '^[42] ' | python3 -c "import sys,json; print([ (l.split()[0], round(json.loads(l.split(' ',1)[1])['fwd_tflops'])) for l in sys.stdin])")"; done; done
