"""Scenario grid of tests/golden/suite.csv, built from whichever package's
classes are passed in (the reference in gen_golden.py, this package in
tests/test_results_csv.py)."""


def suite_grid(Scenario, Discipline, ConstantArrival, PoissonArrival, FixedLength, UniformLength, TPConfig,
               Placement):
    """The scenario grid of suite.csv (shared with tests/test_results_csv.py)."""
    grid = []
    for i, disc in enumerate((Discipline.FUSION, Discipline.FUSION_NO_SHUFFLE, Discipline.DYNAMIC_BATCHING,
                              Discipline.CONCURRENT)):
        kw = dict(window_ms=15.0, max_batch=6) if disc is Discipline.DYNAMIC_BATCHING else {}
        grid.append(Scenario(scenario_id=f"s{i}a", discipline=disc, n_requests=10 + i,
                             arrival=PoissonArrival(12.5), lengths=UniformLength(4, 30), max_output_length=30,
                             seeds=(0, 1, 2), **kw))
        grid.append(Scenario(scenario_id=f"s{i}b", discipline=disc, n_requests=6, arrival=ConstantArrival(7.0),
                             lengths=FixedLength(9), max_output_length=12, batch_size=2, input_len=16,
                             tp=TPConfig(tp_size=2, placement=Placement.INTER if i % 2 else
                                         Placement.INTRA), seeds=(5,), **kw))
    return grid
