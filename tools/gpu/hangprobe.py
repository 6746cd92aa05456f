"""Run bench.py's main with a traceback dump of every thread after a delay (hang diagnosis)."""
import faulthandler
import sys

sys.path.insert(0, ".")
faulthandler.dump_traceback_later(float(sys.argv[1]), exit=True)
sys.argv = ["bench.py"] + sys.argv[2:]
import bench  # noqa: E402

sys.exit(bench.main())
