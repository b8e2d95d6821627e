for f in 0.4 0.55 0.7; do
  echo "frac $f"
  HGS_GPU_WIDEN=$f timeout 300 python tools/e2e_profile.py 2>&1 | grep -v "public" | tail -1 | cut -c1-330
  HGS_GPU_WIDEN=$f timeout 300 python tools/e2e_profile.py 2>&1 | tail -3 | cut -c1-330
done
