python -c "
import importlib.util
spec=importlib.util.spec_from_file_location('b','paper_2509_22337_b200/_build.py'); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)"
