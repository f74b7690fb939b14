# Copy the outputs of tools/round2_final.sh (merged into gpurun_out/) into
# profiles/: bench lines, launch summaries, ncu --set full summaries, the
# Cholesky traffic JSONs bench.py reads, and the GPU suite tail.
set -eu
O=gpurun_out
P=profiles
for f in cfg3 cfg3_jaw cfg2 cfg5 cfg5_batch8 cfg4; do
  [ -s $O/f_bench_$f.json ] && tail -1 $O/f_bench_$f.json > $P/r02_bench_$f.json
done
python tools/launch_summary.py $O/r02_launches_cfg3.csv > $P/r02_launches_cfg3.txt
python tools/launch_summary.py $O/r02_launches_cfg2.csv > $P/r02_launches_cfg2.txt
for k in k_bw_level k_dense_backward k_fw_level k_local_forces k_subtree_forward k_sym_gemv_stream; do
  [ -s $O/r02_full_$k.ncu-rep ] && python tools/ncu_summary.py $O/r02_full_$k.ncu-rep > $P/r02_ncu_$k.txt
done
python tools/ncu_summary.py $O/r02_full_k_cholesky_oz_cfg3.ncu-rep --json /tmp/t3.json > $P/r02_ncu_k_cholesky_oz_cfg3.txt
python tools/ncu_summary.py $O/r02_full_k_cholesky_cfg2.ncu-rep --json /tmp/t2.json > $P/r02_ncu_k_cholesky_cfg2.txt
python - <<'PY'
import json
for cfg, m, src in (("cfg3", 6197, "/tmp/t3.json"), ("cfg2", None, "/tmp/t2.json")):
    js = json.load(open(src))
    old = json.load(open(f"profiles/r02_cholesky_traffic_{cfg}.json"))
    js["m"] = old.get("m", m)
    js["source"] = js["source"].replace("gpurun_out/", "gpurun_out/ (round-2 final) ")
    json.dump(js, open(f"profiles/r02_cholesky_traffic_{cfg}.json", "w"), indent=1)
    print(cfg, js["kernel"], js["traffic_bytes"], js["duration_s"])
PY
tail -3 $O/f_gputest.log > $P/r02_gputest_tail.txt
echo saved
