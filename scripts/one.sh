export PM_LIB_PATH=build/variants/lib_sr1m4.so
timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --opt solve_stages=1 2>&1 | tail -15
