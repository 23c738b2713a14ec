for gp in 0 1 0 1; do echo "FDG_GRAPH_PDL=$gp"; FDG_GRAPH_PDL=$gp python scripts/c0_probe.py 3 | tail -1; done
FDG_GRAPH_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "graph" 2>&1 | tail -2
