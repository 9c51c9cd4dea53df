set -x
timeout 300 python tools/graph_probe.py > gpurun_out/r44_graph.json 2> gpurun_out/r44_graph.err; tail -5 gpurun_out/r44_graph.err
