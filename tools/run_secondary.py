import sys, json, time, types
sys.path.insert(0, "/root/repo")
import bench
args = types.SimpleNamespace(steps=10)
t = time.time()
out = bench.run_ct_secondary(args, int(sys.argv[1]))
print(json.dumps(out))
print("wall", time.time() - t)
