cp paper_2506_23225_b200/libmglu.so /tmp/prod.so
for e in ss3; do cp tools/probes/libmglu_$e.so paper_2506_23225_b200/libmglu.so; timeout 600 python -m pytest tests/test_gpu_tcgen05.py -x -q 2>&1 | tail -1; done
cp /tmp/prod.so paper_2506_23225_b200/libmglu.so
NOTEST=1 TCEXP="ss3 ss2" WLS="prefill sweep_b2048_nm8 sweep_b2048_nm1 decode_b64" bash tools/gpu_tcexp2.sh
