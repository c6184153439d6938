L=$PWD/paper_2503_11367_b200
BAM_LIB_PATH=$L/libbam_kvt.so timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_cp.py -q -x > gpurun_out/t.log 2>&1; echo "TESTS kvt2: $(tail -n 1 gpurun_out/t.log)"
for i in 1 2; do for V in libbam libbam_kvt libbam_kvt1; do echo "$V $(BAM_LIB_PATH=$L/$V.so timeout 200 python tools/time_attn.py --config 4,2 --iters 6 2>&1 | grep '^[42] ' | python3 -c "import sys,json; print([ (l.split()[0], round(json.loads(l.split(' ',1)[1])['bwd_tflops'])) for l in sys.stdin])")"; done; done
