import faulthandler, sys, time, os
sys.path.insert(0, os.getcwd())
faulthandler.dump_traceback_later(240, repeat=True, file=open("gpurun_out/c5_tb.txt", "w"))
import bench
sys.argv = ["bench.py", "--size", sys.argv[1], "--steps", "1", "--warmup", "1", "--no-cpu-baseline"] + (["--no-e2e"] if os.environ.get("NOE2E") else [])
t = time.time()
bench.main() if hasattr(bench, "main") else None
print("total", time.time() - t, file=sys.stderr)
