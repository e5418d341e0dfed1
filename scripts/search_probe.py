import sys, json
sys.path.insert(0, '/root/repo')
import bench
print(json.dumps(bench.measure_search(0, None, cpu=True)))
