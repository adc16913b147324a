import cProfile, pstats, os, sys, io
sys.argv = ["bench.py", "--sharded", "--steps", "5", "--warmup", "3", "--no-e2e", "--no-cpu", "--no-cn", "--no-given", "--no-configs"]
sys.path.insert(0, os.getcwd())
import bench
pr = cProfile.Profile()
pr.enable()
bench.main()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(30)
print(s.getvalue()[:6000])
