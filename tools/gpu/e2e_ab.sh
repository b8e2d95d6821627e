for f in 0.7 0.8 0.9 1.0; do
  echo "host narrow $f"
  HGS_HOST_NARROW=$f timeout 300 python tools/e2e_profile.py 2>&1 | grep -v "public" | tail -1 | cut -c1-330
  HGS_HOST_NARROW=$f timeout 300 python tools/e2e_profile.py 2>&1 | tail -3 | cut -c1-330
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -q 2>&1 | tail -2
