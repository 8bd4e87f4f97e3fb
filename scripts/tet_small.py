import sys; sys.path.insert(0, '.')
import bench
print(bench.tet_line(6553.0, n=24, reps=3))
