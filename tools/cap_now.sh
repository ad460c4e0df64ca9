mkdir -p gpurun_out/final5
for wl in citation3 edit_heavy person5 person5_parts linkage citation3_parts citation_small; do
  timeout 900 python bench.py --workload $wl > gpurun_out/final5/$wl.json 2> gpurun_out/final5/$wl.err
  echo "$wl rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/final5/reference_arm.json 2> gpurun_out/final5/reference_arm.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
