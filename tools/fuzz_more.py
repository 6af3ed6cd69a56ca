"""Extended run of tests/test_gpu_fuzz.py's generators: cases [lo, hi) of test_fuzz and
test_fuzz_project (beyond the 240 + 48 the suite runs); prints failures, one line each."""
import sys
import traceback

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle  # noqa: E402
oracle.build()
import paper_2304_04612_b200 as shg  # noqa: E402
import test_gpu_fuzz as tf  # noqa: E402

lo, hi = int(sys.argv[1]), int(sys.argv[2])
plo, phi = int(sys.argv[3]), int(sys.argv[4])
fails = 0
for i in range(lo, hi):
    try:
        tf.test_fuzz(shg, oracle, i)
    except Exception as e:
        fails += 1
        print("FAIL fuzz", i, tf.case(i), repr(e)[:300], flush=True)
for i in range(plo, phi):
    try:
        tf.test_fuzz_project(shg, oracle, i)
    except Exception as e:
        fails += 1
        print("FAIL project", i, repr(e)[:300], flush=True)
        traceback.print_exc(limit=2)
print(f"fuzz_more done: {hi - lo} + {phi - plo} cases, {fails} failures", flush=True)
