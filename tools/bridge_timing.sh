# dev: the reference-API program (paper_2203_08498_b200/bridge) at a larger grid, linked both ways:
# per-solve wall_time (SolveReport::wall_time: the reference's steady_clock around its loop; the
# bridge's device events around the device loop) -> gpurun_out/bridge_{ref,b200}_<grid>.json
G=${G:-128}
mkdir -p gpurun_out /tmp/bridge_ref /tmp/bridge_b200
B=paper_2203_08498_b200/bridge/_build
s=$(date +%s.%N); timeout 900 $B/bridge_driver_ref /tmp/bridge_ref $G > gpurun_out/bridge_ref_$G.json 2> gpurun_out/bridge_ref_$G.err; echo "wall $(python3 -c "import time; print(round(time.time() - $s, 2))") s" >> gpurun_out/bridge_ref_$G.err
s=$(date +%s.%N); timeout 300 $B/bridge_driver_b200 /tmp/bridge_b200 $G > gpurun_out/bridge_b200_$G.json 2> gpurun_out/bridge_b200_$G.err; echo "wall $(python3 -c "import time; print(round(time.time() - $s, 2))") s" >> gpurun_out/bridge_b200_$G.err
echo done >> gpurun_out/bridge_b200_$G.err
