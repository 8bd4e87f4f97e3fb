import cProfile, pstats, sys, runpy
sys.argv = ["solve_bench.py", "--n", "54"]
pr = cProfile.Profile()
pr.enable()
try:
    runpy.run_path("scripts/solve_bench.py", run_name="__main__")
finally:
    pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime")
st.print_callers("is_available")
st.print_callers("distance2_coloring")
