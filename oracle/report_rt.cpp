// TEST INFRASTRUCTURE ONLY: round-trips a report through the reference's own report.hpp
// (parse_report -> emit_report, csv_row), so tests/test_cpu_report.py can check that the
// product's ExperimentReport documents are readable by the reference unchanged.
// stdin: report JSON. stdout: re-emitted JSON, then one line "CSV:<csv_row>", then
// "HDR:<csv_header>". Exit 3 on io_error (like qcut_main's io exit code).
#include <iostream>
#include <iterator>
#include <string>

#include "qcut/report.hpp"

int main() {
    std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
    try {
        const qcut::ExperimentReport r = qcut::parse_report(text);
        std::cout << qcut::emit_report(r);
        std::cout << "CSV:" << qcut::csv_row(r) << "\n";
        std::cout << "HDR:" << qcut::csv_header() << "\n";
    } catch (const std::exception& e) {
        std::cerr << e.what() << "\n";
        return 3;
    }
    return 0;
}
