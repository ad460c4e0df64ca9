mkdir -p gpurun_out/final2
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final2/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?"
for wl in citation3 edit_heavy person5 person5_parts linkage citation3_parts citation_small; do
  timeout 900 python bench.py --workload $wl > gpurun_out/final2/$wl.json 2> gpurun_out/final2/$wl.err
  echo "$wl rc=$? $(tail -1 gpurun_out/final2/$wl.json | cut -c1-160)"
done
timeout 900 python bench.py --impl reference > gpurun_out/final2/reference_arm.json 2> gpurun_out/final2/reference_arm.err; echo "ref rc=$?"
bash profiles/capture.sh r1s34p5parts person5_parts 1000000 2024
